"""ctypes binding of the C ABI in include/spamm_gpu.h and include/spamm_synth.h.

Python is plumbing here (tests, bench, smoke); the product boundary is the C
ABI and the C++ drop-in above it.  The in-tree library must exist: a missing
or unloadable ``lib/libspamm_gpu.so`` raises immediately -- there is no CPU
fallback anywhere in the product path.

Status codes map onto the reference's exception types (include/spamm_gpu.h):
SPG_EINVAL -> ValueError (std::invalid_argument), SPG_ERANGE -> IndexError
(std::out_of_range).
"""
from __future__ import annotations

import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np

LIB_DIR = Path(__file__).resolve().parent / "lib"
# SPG_LIB: developer override for A/B runs of compile-time variants
# (tools/build_variant.py); the default is the in-tree library
LIB_PATH = Path(os.environ["SPG_LIB"]) if os.environ.get("SPG_LIB") else LIB_DIR / "libspamm_gpu.so"

SPG_OK, SPG_EINVAL, SPG_ERANGE, SPG_ENOMEM, SPG_ECUDA, SPG_ENCCL, SPG_EINTERNAL = range(7)

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_dp = C.POINTER(C.c_double)
_vp = C.c_void_p


class SpgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[spg {code}] {msg}")
        self.code = code


class SpgCudaError(SpgError):
    pass


class MatrixInfo(C.Structure):
    _fields_ = [("dimension", C.c_int32), ("padded_dimension", C.c_int32),
                ("leaf_size", C.c_int32), ("depth", C.c_int32),
                ("nnz_blocks", C.c_int64), ("frobenius_norm", C.c_double)]


class SpammStats(C.Structure):
    _fields_ = [("candidates", C.c_int64), ("survivors", C.c_int64),
                ("output_blocks", C.c_int64), ("flops", C.c_double),
                ("ms_tasklist", C.c_float), ("ms_gemm", C.c_float), ("ms_finalize", C.c_float)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class SquareStats(C.Structure):
    _fields_ = [("variant", C.c_int32), ("chosen_tau", C.c_double), ("nnz_blocks_mid", C.c_int64),
                ("removed_blocks", C.c_int64), ("removed_norm_bound", C.c_double),
                ("t_mul", C.c_double), ("t_cse", C.c_double), ("t_spamm", C.c_double),
                ("t_trunc", C.c_double), ("flops", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


VARIANTS = {"truncmul": 0, "spamm": 1, "hybrid": 2}


class PurifyConfig(C.Structure):
    _fields_ = [("variant", C.c_int32), ("occupation", C.c_int32), ("max_iterations", C.c_int32),
                ("epsilon", C.c_double), ("idempotency_threshold", C.c_double), ("taus", _dp),
                ("n_taus", C.c_int32), ("initial_delta", C.c_double), ("deltas", _dp),
                ("n_deltas", C.c_int32), ("measure_error", C.c_int32)]


class RunRecord(C.Structure):
    _fields_ = [("iteration", C.c_int32), ("status", C.c_int32), ("polynomial", C.c_int32),
                ("tolerance", C.c_double), ("chosen_tau", C.c_double), ("t_mul", C.c_double),
                ("t_trunc", C.c_double), ("t_spamm", C.c_double), ("t_cse", C.c_double),
                ("nnz_in", C.c_int64), ("nnz_mid", C.c_int64), ("nnz_out", C.c_int64),
                ("nnz_blocks_out", C.c_int64), ("realized_error", C.c_double),
                ("trace", C.c_double), ("flops", C.c_double)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_}
        d["status"] = ("ok", "violation", "converged")[self.status]
        return d


class ControlledStats(C.Structure):
    _fields_ = [("tau", C.c_double), ("tau_index", C.c_int32), ("bound", C.c_double),
                ("cse_seconds", C.c_double), ("spamm_seconds", C.c_double),
                ("ms_cse", C.c_float), ("spamm", SpammStats)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_ if f != "spamm"}
        d["spamm"] = self.spamm.as_dict()
        return d


_SIGNATURES = {
    "spg_last_error": (C.c_char_p, []),
    "spg_version": (C.c_int, []),
    "spg_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "spg_context_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "spg_context_destroy": (C.c_int, [_vp]),
    "spg_context_stream": (C.c_int, [_vp, C.POINTER(_vp)]),
    "spg_context_synchronize": (C.c_int, [_vp]),
    "spg_context_launch_count": (C.c_int, [_vp, _i64p]),
    "spg_matrix_upload": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int64, _i32p, _i32p, _dp,
                                    C.POINTER(_vp)]),
    "spg_matrix_upload_device": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int64, _vp, _vp, _vp,
                                           C.POINTER(_vp)]),
    "spg_matrix_from_dense": (C.c_int, [_vp, C.c_int32, C.c_int32, _dp, C.POINTER(_vp)]),
    "spg_matrix_zero": (C.c_int, [_vp, C.c_int32, C.c_int32, C.POINTER(_vp)]),
    "spg_matrix_get_info": (C.c_int, [_vp, C.POINTER(MatrixInfo)]),
    "spg_matrix_download": (C.c_int, [_vp, _i32p, _i32p, _dp, _dp]),
    "spg_matrix_to_dense": (C.c_int, [_vp, _dp]),
    "spg_matrix_level_norms": (C.c_int, [_vp, C.c_int32, _dp]),
    "spg_matrix_free": (C.c_int, [_vp]),
    "spg_tolerance_grid_check": (C.c_int, [_dp, C.c_int32]),
    "spg_cse": (C.c_int, [_vp, _vp, _vp, _dp, C.c_int32, _dp]),
    "spg_select_tolerance": (C.c_int, [_dp, _dp, C.c_int32, C.c_double, _dp, _i32p]),
    "spg_spamm": (C.c_int, [_vp, _vp, _vp, C.c_double, C.POINTER(_vp), C.POINTER(SpammStats)]),
    "spg_multiply_exact": (C.c_int, [_vp, _vp, _vp, C.POINTER(_vp), C.POINTER(SpammStats)]),
    "spg_spamm_with_error_control": (C.c_int, [_vp, _vp, _vp, C.c_double, _dp, C.c_int32,
                                               C.POINTER(_vp), _dp, C.POINTER(ControlledStats)]),
    "spg_survivors": (C.c_int, [_vp, _vp, _vp, C.c_double, _i64p, _i32p, C.c_int64]),
    "spg_spamm_with_error_control_to_host": (C.c_int, [_vp, _vp, _vp, C.c_double, _dp, C.c_int32,
                                                       C.c_int64, _i32p, _i32p, _dp, _dp, _i64p,
                                                       _dp, C.POINTER(ControlledStats)]),
    "spg_parity_audit": (C.c_int, [_vp, _vp, _vp, C.c_double, C.c_int32, _i64p, _i64p]),
    "spg_selftest_sqrt": (C.c_int, [_vp, C.c_int64, C.c_uint64, _i64p]),
    "spg_matrix_trace": (C.c_int, [_vp, _dp]),
    "spg_matrix_nnz": (C.c_int, [_vp, _i64p]),
    "spg_matrix_axpby": (C.c_int, [_vp, C.c_double, _vp, C.c_double, _vp, C.POINTER(_vp)]),
    "spg_matrix_identity": (C.c_int, [_vp, C.c_int32, C.c_int32, C.POINTER(_vp)]),
    "spg_error_budget_geometric": (C.c_int, [C.c_double, C.c_int32, C.c_double, _dp, _dp]),
    "spg_purify": (C.c_int, [_vp, _vp, C.POINTER(PurifyConfig), C.POINTER(_vp),
                             C.POINTER(RunRecord), C.c_int32, C.POINTER(C.c_int32),
                             C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "spg_truncate": (C.c_int, [_vp, _vp, C.c_double, C.POINTER(_vp), _dp, _i64p]),
    "spg_approximate_square": (C.c_int, [_vp, _vp, C.c_int32, C.c_double, _dp, C.c_int32,
                                         C.POINTER(_vp), C.POINTER(SquareStats)]),
    "spg_cse_shard": (C.c_int, [_vp, _vp, _vp, _dp, C.c_int32, C.c_int32, C.c_int32, _dp]),
    "spg_cse_finish": (C.c_int, [C.c_int32, _dp, _dp, C.c_int32, _dp, _dp]),
    "spg_matrix_top_norms": (C.c_int, [_vp, C.c_int32, _dp]),
    "spg_spamm_shard": (C.c_int, [_vp, _vp, _vp, C.c_double, C.c_int32, C.c_int32,
                                  C.POINTER(_vp), C.POINTER(SpammStats)]),
    "spg_bstream_create": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int64, _i32p, _i32p, _dp,
                                     C.c_int32, C.c_int32, C.POINTER(_vp)]),
    "spg_bstream_matrix": (C.c_int, [_vp, C.POINTER(_vp)]),
    "spg_bstream_panels": (C.c_int, [_vp, C.POINTER(C.c_int32), _i64p]),
    "spg_bstream_free": (None, [_vp]),
    "spg_spamm_streamed": (C.c_int, [_vp, _vp, _vp, C.c_double, C.POINTER(_vp),
                                     C.POINTER(SpammStats)]),
    "spg_spamm_with_error_control_streamed": (C.c_int, [_vp, _vp, _vp, C.c_double, _dp,
                                                        C.c_int32, C.POINTER(_vp), _dp,
                                                        C.POINTER(ControlledStats)]),
    "spg_plan_create": (C.c_int, [_vp, _vp, _vp, _vp, C.c_double, C.c_int32, C.c_int32,
                                  C.POINTER(_vp)]),
    "spg_plan_panel_slots": (C.c_int, [_vp, C.c_int32, C.c_int32, _i64p, _i64p]),
    "spg_plan_accumulate": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, _vp]),
    "spg_plan_finish": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(SpammStats)]),
    "spg_plan_free": (None, [_vp]),
    "spg_plan_run_table": (C.c_int, [_vp, C.c_int32, C.POINTER(_vp), _i32p, _i32p, _vp]),
    "spg_matrix_payload": (C.c_int, [_vp, C.POINTER(_vp)]),
    "spg_matrix_norm_pass": (C.c_int, [_vp, C.POINTER(C.c_float)]),
    "spg_matrix_payload_slots": (C.c_int, [_vp, _i32p]),
    "spg_ipc_export": (C.c_int, [_vp, C.c_char_p]),
    "spg_ipc_open": (C.c_int, [_vp, C.c_char_p, C.POINTER(_vp)]),
    "spg_ipc_close": (C.c_int, [_vp, _vp]),
    "spg_matrix_stage": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int64, _vp, _vp, _vp,
                                   C.POINTER(_vp)]),
    "spg_matrix_stage_finish": (C.c_int, [_vp, C.POINTER(_vp)]),
    "spg_staged_free": (None, [_vp]),
    "spg_matrix_from_diagonal": (C.c_int, [_vp, C.c_int32, C.c_int32, _dp, C.POINTER(_vp)]),
    "spg_matrix_rows": (C.c_int, [_vp, _dp, _dp]),
    "spg_matrix_gershgorin": (C.c_int, [_vp, _dp, _dp]),
    "spg_context_set_task_budget": (C.c_int, [_vp, C.c_int64]),
    "spg_context_trim": (C.c_int, [_vp]),
    "spg_spamm_panels": (C.c_int, [_vp, _vp, _vp, _vp, C.c_double, C.c_int32, C.c_int32,
                                   C.c_int32, C.c_int32, _vp, _vp, C.POINTER(_vp), _vp]),
    "spg_comm_unique_id": (C.c_int, [_vp]),
    "spg_comm_create_nccl": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, C.POINTER(_vp)]),
    "spg_comm_create_host": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, _vp, C.POINTER(_vp)]),
    "spg_comm_info": (C.c_int, [_vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                C.POINTER(C.c_int32)]),
    "spg_comm_destroy": (C.c_int, [_vp]),
    "spg_cse_sharded": (C.c_int, [_vp, _vp, _vp, _dp, C.c_int32, _dp]),
    "spg_spamm_sharded": (C.c_int, [_vp, _vp, _vp, C.c_double, C.c_int32, C.c_int32,
                                    C.POINTER(_vp), _vp]),
    "spg_spamm_with_error_control_sharded": (C.c_int, [_vp, _vp, _vp, C.c_double, _dp,
                                                       C.c_int32, C.c_int32, C.POINTER(_vp),
                                                       _dp, _vp]),
    "spg_matrix_gather_shards": (C.c_int, [_vp, _vp, C.POINTER(_vp)]),
    "spg_survivor_digest": (C.c_int, [_vp, _vp, _vp, C.c_double, C.c_int32, C.c_int32, _i64p,
                                      C.POINTER(C.c_uint64)]),
    "spg_matrix_from_leaf_norms": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int64, _i32p, _i32p,
                                             _dp, C.POINTER(C.c_uint8), C.POINTER(_vp)]),
    "spg_matrix_gather_rows": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, C.c_int64, _vp]),
    "spg_synth_chain_device_rows": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_double, C.c_uint64,
                                              C.c_double, C.c_int32, C.c_int32, C.POINTER(_vp)]),
    "spg_synth_cluster_device_rows": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_double,
                                                C.c_double, C.c_uint64, C.c_uint64, C.c_double,
                                                C.c_int32, C.c_int32, C.POINTER(_vp)]),
    "spg_synth_cluster_scale": (C.c_int, [_vp, C.c_int32, C.c_double, C.c_double, C.c_uint64,
                                          C.c_uint64, _dp]),
    "spg_synth_cluster_device_rows_scaled": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_double,
                                                       C.c_double, C.c_uint64, C.c_uint64,
                                                       C.c_double, C.c_double, C.c_int32,
                                                       C.c_int32, C.POINTER(_vp)]),
    "spg_synth_chain_host": (C.c_int, [C.c_int32, C.c_int32, C.c_double, C.c_uint64, C.c_double,
                                       C.c_int64, _i32p, _i32p, _dp, _i64p]),
    "spg_synth_cluster_host": (C.c_int, [C.c_int32, C.c_int32, C.c_double, C.c_double,
                                         C.c_uint64, C.c_uint64, C.c_double, C.c_int64, _i32p,
                                         _i32p, _dp, _i64p]),
    "spg_synth_chain_device": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_double, C.c_uint64,
                                         C.c_double, C.POINTER(_vp)]),
    "spg_synth_cluster_device": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_double, C.c_double,
                                           C.c_uint64, C.c_uint64, C.c_double, C.POINTER(_vp)]),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lib = None


def _prefer_torch_nccl():
    """Point the library's NCCL dlopen (SPG_NCCL_LIB) at the NCCL torch itself
    links (the nvidia-nccl wheel), so one process holds one libnccl.so.2: a
    communicator created before `import torch` would otherwise load the system
    NCCL under the same soname, and torch's newer symbols would not resolve."""
    if os.environ.get("SPG_NCCL_LIB"):
        return
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for root in (spec.submodule_search_locations or []) if spec else []:
        cand = Path(root) / "nccl" / "lib" / "libnccl.so.2"
        if cand.exists():
            os.environ["SPG_NCCL_LIB"] = str(cand)
            return


def lib():
    """Load the in-tree library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(the CUDA path has no fallback)")
        _prefer_torch_nccl()
        handle = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def _check(rc: int):
    if rc == SPG_OK:
        return
    msg = lib().spg_last_error().decode(errors="replace")
    if rc == SPG_EINVAL:
        raise ValueError(msg)
    if rc == SPG_ERANGE:
        raise IndexError(msg)
    if rc == SPG_ENOMEM:
        raise MemoryError(msg)
    if rc == SPG_ECUDA:
        raise SpgCudaError(rc, msg)
    raise SpgError(rc, msg)


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def device_count() -> int:
    n = C.c_int(0)
    try:
        _check(lib().spg_device_count(C.byref(n)))
    except SpgCudaError:
        return 0
    return n.value


class Context:
    """One device, one stream (the library serialises calls per context)."""

    def __init__(self, device: int = 0):
        h = _vp()
        _check(lib().spg_context_create(device, C.byref(h)))
        self._h = h
        self.device = device

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        s = _vp()
        _check(lib().spg_context_stream(self._h, C.byref(s)))
        return s.value or 0

    def synchronize(self):
        _check(lib().spg_context_synchronize(self._h))

    def trim(self):
        """Return cached device blocks to the driver (spg_context_trim)."""
        _check(lib().spg_context_trim(self._h))

    def launch_count(self) -> int:
        n = C.c_int64(0)
        _check(lib().spg_context_launch_count(self._h, C.byref(n)))
        return n.value

    def close(self):
        if getattr(self, "_h", None):
            lib().spg_context_destroy(self._h)
            self._h = None

    def __del__(self):
        # At interpreter exit the CUDA runtime may already be torn down;
        # leaking device memory then is harmless, calling into it is not.
        if sys is None or sys.is_finalizing():
            return
        try:
            self.close()
        except Exception:
            pass


class Matrix:
    """Device-resident quadtree matrix handle (immutable)."""

    def __init__(self, ctx: Context, handle):
        self.ctx = ctx
        self._h = handle

    @property
    def handle(self):
        return self._h

    def info(self) -> MatrixInfo:
        out = MatrixInfo()
        _check(lib().spg_matrix_get_info(self._h, C.byref(out)))
        return out

    @property
    def dimension(self):
        return self.info().dimension

    @property
    def leaf_size(self):
        return self.info().leaf_size

    @property
    def nnz_blocks(self):
        return self.info().nnz_blocks

    @property
    def frobenius_norm(self):
        return self.info().frobenius_norm

    def download(self, payload: bool = True):
        """(rows, cols, payload[n, L*L] column-major, norms) in Morton order."""
        inf = self.info()
        n, LL = inf.nnz_blocks, inf.leaf_size * inf.leaf_size
        rows = np.empty(n, np.int32)
        cols = np.empty(n, np.int32)
        norms = np.empty(n, np.float64)
        pay = np.empty((n, LL), np.float64) if payload else None
        _check(lib().spg_matrix_download(self._h, _ptr(rows, C.c_int32), _ptr(cols, C.c_int32),
                                         _ptr(pay, C.c_double) if payload else None,
                                         _ptr(norms, C.c_double)))
        return rows, cols, pay, norms

    def to_dense(self) -> np.ndarray:
        n = self.info().dimension
        out = np.empty((n, n), np.float64)
        _check(lib().spg_matrix_to_dense(self._h, _ptr(out, C.c_double)))
        return out

    def norm_pass_ms(self) -> float:
        """Device time of one leaf-norm kernel pass over every leaf."""
        ms = C.c_float(0)
        _check(lib().spg_matrix_norm_pass(self._h, C.byref(ms)))
        return ms.value

    def payload_ptr(self) -> int:
        p = _vp()
        _check(lib().spg_matrix_payload(self._h, C.byref(p)))
        return p.value or 0

    def payload_slots(self) -> np.ndarray:
        """Payload slot per non-null leaf, aligned with download()."""
        out = np.empty(self.info().nnz_blocks, np.int32)
        _check(lib().spg_matrix_payload_slots(self._h, _ptr(out, C.c_int32)))
        return out

    def level_norms(self, level: int) -> np.ndarray:
        out = np.empty(4 ** level, np.float64)
        _check(lib().spg_matrix_level_norms(self._h, level, _ptr(out, C.c_double)))
        return out

    def free(self):
        if getattr(self, "_h", None):
            if not getattr(self, "_borrowed", False):
                lib().spg_matrix_free(self._h)
            self._h = None

    def __del__(self):
        if sys is None or sys.is_finalizing():
            return
        try:
            self.free()
        except Exception:
            pass


def upload(ctx: Context, dimension: int, leaf_size: int, rows, cols, payload) -> Matrix:
    rows = np.ascontiguousarray(rows, np.int32)
    cols = np.ascontiguousarray(cols, np.int32)
    payload = np.ascontiguousarray(payload, np.float64)
    n = rows.shape[0]
    if cols.shape[0] != n or payload.size != n * leaf_size * leaf_size:
        raise ValueError("leaf arrays disagree in length")
    h = _vp()
    _check(lib().spg_matrix_upload(ctx.handle, dimension, leaf_size, n, _ptr(rows, C.c_int32),
                                   _ptr(cols, C.c_int32), _ptr(payload, C.c_double), C.byref(h)))
    return Matrix(ctx, h)


class Staged:
    """spg_matrix_stage: host->device copies queued on the context's upload
    stream; finish() builds the matrix.  rows/cols/payload: host addresses of
    pinned buffers that stay unchanged until finish() returns."""

    def __init__(self, ctx: Context, dimension: int, leaf_size: int, n_leaves: int,
                 rows_ptr: int, cols_ptr: int, payload_ptr: int):
        self.ctx = ctx
        self._h = _vp()
        _check(lib().spg_matrix_stage(ctx.handle, dimension, leaf_size, n_leaves, rows_ptr,
                                      cols_ptr, payload_ptr, C.byref(self._h)))

    def finish(self) -> "Matrix":
        h = _vp()
        st, self._h = self._h, None
        _check(lib().spg_matrix_stage_finish(st, C.byref(h)))
        return Matrix(self.ctx, h)

    def __del__(self):
        if sys is None or sys.is_finalizing():
            return
        if getattr(self, "_h", None):
            lib().spg_staged_free(self._h)
            self._h = None


def upload_device(ctx: Context, dimension: int, leaf_size: int, n_leaves: int, d_rows: int,
                  d_cols: int, d_payload: int) -> Matrix:
    h = _vp()
    _check(lib().spg_matrix_upload_device(ctx.handle, dimension, leaf_size, n_leaves, d_rows,
                                          d_cols, d_payload, C.byref(h)))
    return Matrix(ctx, h)


def from_dense(ctx: Context, dense: np.ndarray, leaf_size: int) -> Matrix:
    dense = np.ascontiguousarray(dense, np.float64)
    h = _vp()
    _check(lib().spg_matrix_from_dense(ctx.handle, dense.shape[0], leaf_size,
                                       _ptr(dense, C.c_double), C.byref(h)))
    return Matrix(ctx, h)


def zero(ctx: Context, dimension: int, leaf_size: int) -> Matrix:
    h = _vp()
    _check(lib().spg_matrix_zero(ctx.handle, dimension, leaf_size, C.byref(h)))
    return Matrix(ctx, h)


def tolerance_grid_check(taus):
    taus = np.ascontiguousarray(taus, np.float64)
    _check(lib().spg_tolerance_grid_check(_ptr(taus, C.c_double), taus.size))


def cse(ctx: Context, a: Matrix, b: Matrix, taus) -> np.ndarray:
    taus = np.ascontiguousarray(taus, np.float64)
    out = np.empty(taus.size, np.float64)
    _check(lib().spg_cse(ctx.handle, a.handle, b.handle, _ptr(taus, C.c_double), taus.size,
                         _ptr(out, C.c_double)))
    return out


def select_tolerance(bounds, taus, delta: float):
    bounds = np.ascontiguousarray(bounds, np.float64)
    taus = np.ascontiguousarray(taus, np.float64)
    tau = C.c_double(0)
    idx = C.c_int32(-1)
    _check(lib().spg_select_tolerance(_ptr(bounds, C.c_double), _ptr(taus, C.c_double),
                                      taus.size, delta, C.byref(tau), C.byref(idx)))
    return tau.value, idx.value


def spamm(ctx: Context, a: Matrix, b: Matrix, tau: float):
    h = _vp()
    st = SpammStats()
    _check(lib().spg_spamm(ctx.handle, a.handle, b.handle, tau, C.byref(h), C.byref(st)))
    return Matrix(ctx, h), st.as_dict()


def multiply_exact(ctx: Context, a: Matrix, b: Matrix):
    h = _vp()
    st = SpammStats()
    _check(lib().spg_multiply_exact(ctx.handle, a.handle, b.handle, C.byref(h), C.byref(st)))
    return Matrix(ctx, h), st.as_dict()


def spamm_with_error_control(ctx: Context, a: Matrix, b: Matrix, delta: float, taus):
    taus = np.ascontiguousarray(taus, np.float64)
    bounds = np.empty(taus.size, np.float64)
    h = _vp()
    st = ControlledStats()
    _check(lib().spg_spamm_with_error_control(ctx.handle, a.handle, b.handle, delta,
                                              _ptr(taus, C.c_double), taus.size, C.byref(h),
                                              _ptr(bounds, C.c_double), C.byref(st)))
    return Matrix(ctx, h), st.as_dict(), bounds


# ---------------------------------------------------------------- beyond one device's memory
PANEL_FETCH = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int64,
                          C.c_void_p)


def set_task_budget(ctx: Context, nbytes: int):
    """Row-chunk products whose task list would exceed nbytes (0: auto)."""
    _check(lib().spg_context_set_task_budget(ctx.handle, int(nbytes)))


class DevicePtr:
    """A float64 view of device memory for torch.as_tensor (no copy)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


def spamm_panels(ctx: Context, a: Matrix, b_norms: Matrix, tau: float, fetch, level: int = 0,
                 shard: int = 0, panel_rows: int = 32, owner_rows: int = 0,
                 a_norms: Matrix | None = None):
    """spg_spamm_panels: the shard's rows of C~ with B's panels requested from
    fetch(r0, r1, d_dst_ptr, count, stream_ptr) (fills count leaves of rows
    [r0, r1) in (row, col) order on the stream); row-chunked in C when the
    task list would not fit."""
    def cb(_user, r0, r1, dst, count, stream):
        try:
            fetch(int(r0), int(r1), int(dst or 0), int(count), int(stream or 0))
            return 0
        except Exception:  # noqa: BLE001 -- reported as SPG_EINVAL by the library
            import traceback
            traceback.print_exc()
            return 1
    fn = PANEL_FETCH(cb)
    h = _vp()
    st = SpammStats()
    _check(lib().spg_spamm_panels(ctx.handle, a.handle, a_norms.handle if a_norms else None,
                                  b_norms.handle, tau, level, shard, panel_rows, owner_rows,
                                  C.cast(fn, _vp), None, C.byref(h), C.byref(st)))
    return Matrix(ctx, h), st.as_dict()


# ---------------------------------------------------------------- communicator
HOST_ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


class Comm:
    """spg_comm: ranks of one job, one GPU each.  nccl(ctx, nranks, rank, id)
    or host(ctx, nranks, rank, allgather) where allgather(bytes) -> list of
    per-rank bytes (the caller's own collective, e.g. gloo)."""

    def __init__(self, ctx: Context, handle, keep=None):
        self.ctx, self._h, self._keep = ctx, handle, keep

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib().spg_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def nccl(cls, ctx: Context, nranks: int, rank: int, uid: bytes):
        h = _vp()
        buf = C.create_string_buffer(bytes(uid), 128)
        _check(lib().spg_comm_create_nccl(ctx.handle, nranks, rank, buf, C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def host(cls, ctx: Context, nranks: int, rank: int, allgather):
        def cb(_user, send, nbytes, recv):
            try:
                parts = allgather(C.string_at(send, nbytes) if nbytes else b"")
                blob = b"".join(parts)
                if len(blob) != nbytes * nranks:
                    return 1
                if nbytes:
                    C.memmove(recv, blob, len(blob))
                return 0
            except Exception:  # noqa: BLE001 -- reported as SPG_ENCCL by the library
                return 1
        fn = HOST_ALLGATHER(cb)
        h = _vp()
        _check(lib().spg_comm_create_host(ctx.handle, nranks, rank, C.cast(fn, _vp), None,
                                          C.byref(h)))
        return cls(ctx, h, keep=fn)

    @property
    def handle(self):
        return self._h

    def info(self):
        n, r, u = C.c_int32(), C.c_int32(), C.c_int32()
        _check(lib().spg_comm_info(self._h, C.byref(n), C.byref(r), C.byref(u)))
        return n.value, r.value, bool(u.value)

    def close(self):
        if self._h:
            _check(lib().spg_comm_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def cse_sharded(comm: Comm, a: Matrix, b: Matrix, taus) -> np.ndarray:
    taus = np.ascontiguousarray(taus, np.float64)
    out = np.empty(taus.size)
    _check(lib().spg_cse_sharded(comm.handle, a.handle, b.handle, _ptr(taus, C.c_double),
                                 taus.size, _ptr(out, C.c_double)))
    return out


def spamm_sharded(comm: Comm, a: Matrix, b: Matrix, tau: float, skip_test: bool = True,
                  gather: bool = False):
    h = _vp()
    st = SpammStats()
    _check(lib().spg_spamm_sharded(comm.handle, a.handle, b.handle, tau, int(skip_test),
                                   int(gather), C.byref(h), C.byref(st)))
    return Matrix(comm.ctx, h), st.as_dict()


def spamm_with_error_control_sharded(comm: Comm, a: Matrix, b: Matrix, delta: float, taus,
                                     gather: bool = False):
    taus = np.ascontiguousarray(taus, np.float64)
    bounds = np.empty(taus.size, np.float64)
    h = _vp()
    st = ControlledStats()
    _check(lib().spg_spamm_with_error_control_sharded(comm.handle, a.handle, b.handle, delta,
                                                      _ptr(taus, C.c_double), taus.size,
                                                      int(gather), C.byref(h),
                                                      _ptr(bounds, C.c_double), C.byref(st)))
    return Matrix(comm.ctx, h), st.as_dict(), bounds


def gather_shards(comm: Comm, shard: Matrix) -> Matrix:
    h = _vp()
    _check(lib().spg_matrix_gather_shards(comm.handle, shard.handle, C.byref(h)))
    return Matrix(comm.ctx, h)


def spamm_with_error_control_to_host(ctx: Context, a: Matrix, b: Matrix, delta: float, taus,
                                     out=None):
    """Controlled product with C streamed to host arrays (rows, cols, payload,
    norms); `out` may supply (pinned) preallocated arrays of capacity n."""
    taus = np.ascontiguousarray(taus, np.float64)
    inf = a.info()
    if out is None:
        nb = (inf.dimension + inf.leaf_size - 1) // inf.leaf_size
        cap = nb * nb
        out = (np.empty(cap, np.int32), np.empty(cap, np.int32),
               np.empty((cap, inf.leaf_size * inf.leaf_size)), np.empty(cap))
    rows, cols, pay, norms = out
    count = C.c_int64(0)
    bounds = np.empty(taus.size)
    st = ControlledStats()
    _check(lib().spg_spamm_with_error_control_to_host(
        ctx.handle, a.handle, b.handle, delta, _ptr(taus, C.c_double), taus.size, len(rows),
        _ptr(rows, C.c_int32), _ptr(cols, C.c_int32), _ptr(pay, C.c_double),
        _ptr(norms, C.c_double), C.byref(count), _ptr(bounds, C.c_double), C.byref(st)))
    n = count.value
    return (rows[:n], cols[:n], pay[:n], norms[:n]), st.as_dict(), bounds


def survivor_digest(ctx: Context, a: Matrix, b: Matrix, tau: float, level: int = 0,
                    shard: int = 0):
    """(count, digest) of the survivor set (spg_survivor_digest)."""
    count, dig = C.c_int64(0), C.c_uint64(0)
    _check(lib().spg_survivor_digest(ctx.handle, a.handle, b.handle, tau, level, shard,
                                     C.byref(count), C.byref(dig)))
    return count.value, dig.value


def survivors(ctx: Context, a: Matrix, b: Matrix, tau: float) -> np.ndarray:
    count = C.c_int64(0)
    _check(lib().spg_survivors(ctx.handle, a.handle, b.handle, tau, C.byref(count), None, 0))
    out = np.empty((count.value, 3), np.int32)
    if count.value:
        _check(lib().spg_survivors(ctx.handle, a.handle, b.handle, tau, C.byref(count),
                                   _ptr(out, C.c_int32), count.value))
    return out


# ---------------------------------------------------------------- callers
def truncate(ctx: Context, x: Matrix, delta: float):
    """(matrix, removed_norm_bound, removed_block_count) -- error_control.cpp:174-201."""
    h = _vp()
    rn = C.c_double(0)
    rc = C.c_int64(0)
    _check(lib().spg_truncate(ctx.handle, x.handle, delta, C.byref(h), C.byref(rn), C.byref(rc)))
    return Matrix(ctx, h), rn.value, rc.value


def approximate_square(ctx: Context, x: Matrix, variant: str, delta: float, taus):
    """experiment.cpp:47-82 approximate_square; variant truncmul | spamm | hybrid."""
    taus = np.ascontiguousarray(taus, np.float64)
    h = _vp()
    st = SquareStats()
    _check(lib().spg_approximate_square(ctx.handle, x.handle, VARIANTS[variant], delta,
                                        _ptr(taus, C.c_double), taus.size, C.byref(h),
                                        C.byref(st)))
    return Matrix(ctx, h), st.as_dict()


def parity_audit(ctx: Context, a: Matrix, b: Matrix, tau: float, ulps: int = 4):
    """(near_ties, candidates): candidate products within `ulps` ulp of tau."""
    t, c = C.c_int64(0), C.c_int64(0)
    _check(lib().spg_parity_audit(ctx.handle, a.handle, b.handle, tau, ulps, C.byref(t),
                                  C.byref(c)))
    return t.value, c.value


def selftest_sqrt(ctx: Context, n: int, seed: int) -> int:
    """Mismatching results of the sweep's branch-free sqrt vs sqrt.rn.f64 over 2n patterns."""
    out = C.c_int64(-1)
    _check(lib().spg_selftest_sqrt(ctx.handle, n, seed, C.byref(out)))
    return out.value


def trace(m: Matrix) -> float:
    out = C.c_double(0)
    _check(lib().spg_matrix_trace(m.handle, C.byref(out)))
    return out.value


def nnz(m: Matrix) -> int:
    out = C.c_int64(0)
    _check(lib().spg_matrix_nnz(m.handle, C.byref(out)))
    return out.value


def axpby(ctx: Context, alpha: float, a: Matrix, beta: float = 0.0, b: Matrix | None = None):
    """add(a.scale(alpha), b.scale(beta)) on the device."""
    h = _vp()
    _check(lib().spg_matrix_axpby(ctx.handle, alpha, a.handle, beta, b.handle if b else None,
                                  C.byref(h)))
    return Matrix(ctx, h)


def from_diagonal(ctx: Context, diag, leaf: int) -> Matrix:
    d = np.ascontiguousarray(diag, np.float64)
    h = _vp()
    _check(lib().spg_matrix_from_diagonal(ctx.handle, d.size, leaf, _ptr(d, C.c_double),
                                          C.byref(h)))
    return Matrix(ctx, h)


def row_data(m: Matrix):
    """(diagonal, sum_j |a_ij|) per row, computed on the device."""
    n = m.dimension
    d = np.empty(n, np.float64)
    a = np.empty(n, np.float64)
    _check(lib().spg_matrix_rows(m.handle, _ptr(d, C.c_double), _ptr(a, C.c_double)))
    return d, a


def gershgorin(m: Matrix):
    """(low, high) Gershgorin spectral bounds, reference oracle.cpp:191-200."""
    lo, hi = C.c_double(), C.c_double()
    _check(lib().spg_matrix_gershgorin(m.handle, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def identity(ctx: Context, n: int, leaf: int) -> Matrix:
    h = _vp()
    _check(lib().spg_matrix_identity(ctx.handle, n, leaf, C.byref(h)))
    return Matrix(ctx, h)


def error_budget_geometric(epsilon: float, iterations: int, ratio: float = 0.5):
    d0 = C.c_double(0)
    deltas = np.empty(max(iterations, 1))
    _check(lib().spg_error_budget_geometric(epsilon, iterations, ratio, C.byref(d0),
                                            _ptr(deltas, C.c_double)))
    return d0.value, deltas[:iterations]


def purify(ctx: Context, x0: Matrix, variant: str, occupation: int, epsilon: float = 1e-5,
           max_iterations: int = 100, taus=None, idempotency_threshold: float = 0.0,
           budget=None, measure_error: bool = True):
    """purification.cpp:90-202 on the GPU.  budget = (initial_delta, deltas) or
    None for ErrorBudget::geometric(epsilon, max_iterations)."""
    from .inputs import geometric_grid
    taus = np.ascontiguousarray(geometric_grid() if taus is None else taus, np.float64)
    if budget is None:
        budget = error_budget_geometric(epsilon, max_iterations)
    d0, deltas = budget
    deltas = np.ascontiguousarray(deltas, np.float64)
    cfg = PurifyConfig(VARIANTS[variant], occupation, max_iterations, epsilon,
                       idempotency_threshold, _ptr(taus, C.c_double), taus.size, d0,
                       _ptr(deltas, C.c_double), deltas.size, int(measure_error))
    cap = max_iterations + 2
    log = (RunRecord * cap)()
    h = _vp()
    n_log, conv, its = C.c_int32(0), C.c_int32(0), C.c_int32(0)
    _check(lib().spg_purify(ctx.handle, x0.handle, C.byref(cfg), C.byref(h), log, cap,
                            C.byref(n_log), C.byref(conv), C.byref(its)))
    return Matrix(ctx, h), [log[i].as_dict() for i in range(min(n_log.value, cap))], \
        bool(conv.value), its.value


# ---------------------------------------------------------------- row shards
def cse_shard(ctx: Context, a: Matrix, b: Matrix, taus, level: int, shard: int) -> np.ndarray:
    """Level-`level` partial bound vectors of one row shard: (4^level, n_taus)."""
    taus = np.ascontiguousarray(taus, np.float64)
    out = np.empty((4 ** level, taus.size), np.float64)
    _check(lib().spg_cse_shard(ctx.handle, a.handle, b.handle, _ptr(taus, C.c_double), taus.size,
                               level, shard, _ptr(out, C.c_double)))
    return out


def cse_finish(level: int, a_top, b_top, partials) -> np.ndarray:
    """Host-only top-level combine of gathered partials (2^level shards)."""
    a_top = np.ascontiguousarray(a_top, np.float64)
    b_top = np.ascontiguousarray(b_top, np.float64)
    partials = np.ascontiguousarray(partials, np.float64)
    n_taus = partials.shape[-1]
    if partials.size != (2 ** level) * (4 ** level) * n_taus:
        raise ValueError("partials must hold 2^level shards x 4^level vectors")
    out = np.empty(n_taus, np.float64)
    _check(lib().spg_cse_finish(level, _ptr(a_top, C.c_double), _ptr(b_top, C.c_double), n_taus,
                                _ptr(partials, C.c_double), _ptr(out, C.c_double)))
    return out


def top_norms(m: Matrix, levels: int) -> np.ndarray:
    out = np.empty(((4 ** levels) - 1) // 3, np.float64)
    _check(lib().spg_matrix_top_norms(m.handle, levels, _ptr(out, C.c_double)))
    return out


def spamm_shard(ctx: Context, a: Matrix, b: Matrix, tau: float, level: int, shard: int):
    h = _vp()
    st = SpammStats()
    _check(lib().spg_spamm_shard(ctx.handle, a.handle, b.handle, tau, level, shard, C.byref(h),
                                 C.byref(st)))
    return Matrix(ctx, h), st.as_dict()


# ------------------------------------------------- B streamed from host memory
class BStream:
    """B kept in host memory and streamed to the GPU in panels of block rows
    (spg_bstream_*).  Leaves must be sorted by block row; the payload array
    is referenced (not copied) for the object's lifetime."""

    def __init__(self, ctx: Context, dimension: int, leaf_size: int, rows, cols, payload,
                 panel_block_rows: int, register_host: bool = True):
        self.ctx = ctx
        self._rows = np.ascontiguousarray(rows, np.int32)
        self._cols = np.ascontiguousarray(cols, np.int32)
        if isinstance(payload, np.ndarray):
            self._payload = np.ascontiguousarray(payload, np.float64)
            pay_ptr = _ptr(self._payload, C.c_double)
        else:  # a (pinned) torch CPU tensor
            self._payload = payload
            pay_ptr = C.cast(C.c_void_p(payload.data_ptr()), C.POINTER(C.c_double))
        n = self._rows.shape[0]
        self._h = _vp()
        _check(lib().spg_bstream_create(ctx.handle, dimension, leaf_size, n,
                                        _ptr(self._rows, C.c_int32), _ptr(self._cols, C.c_int32),
                                        pay_ptr, panel_block_rows, int(register_host),
                                        C.byref(self._h)))
        m = _vp()
        _check(lib().spg_bstream_matrix(self._h, C.byref(m)))
        self.norms = Matrix(ctx, m)
        self.norms._borrowed = True
        self.norms._owner = self  # keeps the stream (and its payload) alive

    @property
    def handle(self):
        return self._h

    def panels(self):
        n = C.c_int32(0)
        mx = C.c_int64(0)
        _check(lib().spg_bstream_panels(self._h, C.byref(n), C.byref(mx)))
        return n.value, mx.value

    def free(self):
        if getattr(self, "_h", None):
            self.norms._h = None
            lib().spg_bstream_free(self._h)
            self._h = None

    def __del__(self):
        if sys is None or sys.is_finalizing():
            return
        try:
            self.free()
        except Exception:
            pass


class Plan:
    """Task list of A*B (or a row shard) with B arriving in block-row panels
    (spg_plan_*): accumulate(r0, r1, panel) for ascending row ranges tiling
    [0, ceil(n/L)), then finish() -> (C, stats)."""

    def __init__(self, ctx: Context, a: Matrix, b_norms: Matrix, tau: float, level: int = 0,
                 shard: int = 0, a_norms: Matrix | None = None):
        self.ctx = ctx
        self._keep = (a, b_norms, a_norms)
        self._h = _vp()
        _check(lib().spg_plan_create(ctx.handle, a.handle,
                                     a_norms.handle if a_norms is not None else None,
                                     b_norms.handle, tau, level, shard, C.byref(self._h)))

    def panel_slots(self, r0: int, r1: int):
        lo, n = C.c_int64(0), C.c_int64(0)
        _check(lib().spg_plan_panel_slots(self._h, r0, r1, C.byref(lo), C.byref(n)))
        return lo.value, n.value

    def accumulate(self, r0: int, r1: int, d_panel: int | None, stream: int | None = None):
        """d_panel: device address of the panel's leaves; stream: cudaStream_t
        address the panel was produced on (stream-ordered hand-off)."""
        _check(lib().spg_plan_accumulate(self._h, r0, r1, d_panel or None, stream or None))

    def run_table(self, owner_bases, slot_owner, slot_local, stream: int | None = None):
        """Every product in one GEMM, B leaf t read at owner_bases[slot_owner[t]]
        + slot_local[t] L^2 (device addresses; peers' via ipc_open)."""
        so = np.ascontiguousarray(slot_owner, np.int32)
        sl = np.ascontiguousarray(slot_local, np.int32)
        bases = (_vp * max(len(owner_bases), 1))(*[_vp(b) for b in owner_bases])
        _check(lib().spg_plan_run_table(self._h, len(owner_bases), bases, _ptr(so, C.c_int32),
                                        _ptr(sl, C.c_int32), stream or None))

    def finish(self):
        h = _vp()
        st = SpammStats()
        _check(lib().spg_plan_finish(self._h, C.byref(h), C.byref(st)))
        return Matrix(self.ctx, h), st.as_dict()

    def free(self):
        if getattr(self, "_h", None):
            lib().spg_plan_free(self._h)
            self._h = None

    def __del__(self):
        if sys is None or sys.is_finalizing():
            return
        try:
            self.free()
        except Exception:
            pass


def from_leaf_norms(ctx: Context, dimension: int, leaf_size: int, rows, cols, norms,
                    nonzero=None) -> Matrix:
    """Norm-only matrix from a leaf table sorted by block row (slot t = leaf t)."""
    rows = np.ascontiguousarray(rows, np.int32)
    cols = np.ascontiguousarray(cols, np.int32)
    norms = np.ascontiguousarray(norms, np.float64)
    nz = None if nonzero is None else np.ascontiguousarray(nonzero, np.uint8)
    h = _vp()
    _check(lib().spg_matrix_from_leaf_norms(ctx.handle, dimension, leaf_size, rows.shape[0],
                                            _ptr(rows, C.c_int32), _ptr(cols, C.c_int32),
                                            _ptr(norms, C.c_double),
                                            _ptr(nz, C.c_uint8) if nz is not None else None,
                                            C.byref(h)))
    return Matrix(ctx, h)


def gather_rows(m: Matrix, r0: int, r1: int, d_out: int, capacity: int,
                stream: int | None = None):
    """Non-null leaves of block rows [r0, r1) in (row, col) order -> d_out."""
    _check(lib().spg_matrix_gather_rows(m.handle, r0, r1, d_out or None, capacity,
                                        stream or None))


def ipc_export(m: Matrix) -> bytes:
    buf = C.create_string_buffer(64)
    _check(lib().spg_ipc_export(m.handle, buf))
    return buf.raw


def ipc_open(ctx: Context, handle: bytes) -> int:
    p = _vp()
    _check(lib().spg_ipc_open(ctx.handle, bytes(handle), C.byref(p)))
    return p.value


def ipc_close(ctx: Context, ptr: int):
    _check(lib().spg_ipc_close(ctx.handle, _vp(ptr)))


def sort_by_block_row(rows, cols, payload):
    """Leaves reordered by (block row, block column) for BStream."""
    order = np.lexsort((np.asarray(cols), np.asarray(rows)))
    return (np.asarray(rows)[order], np.asarray(cols)[order],
            np.ascontiguousarray(np.asarray(payload)[order]))


def spamm_streamed(ctx: Context, a: Matrix, b: BStream, tau: float):
    h = _vp()
    st = SpammStats()
    _check(lib().spg_spamm_streamed(ctx.handle, a.handle, b.handle, tau, C.byref(h),
                                    C.byref(st)))
    return Matrix(ctx, h), st.as_dict()


def spamm_with_error_control_streamed(ctx: Context, a: Matrix, b: BStream, delta: float, taus):
    taus = np.ascontiguousarray(taus, np.float64)
    bounds = np.empty(taus.size, np.float64)
    h = _vp()
    st = ControlledStats()
    _check(lib().spg_spamm_with_error_control_streamed(
        ctx.handle, a.handle, b.handle, delta, _ptr(taus, C.c_double), taus.size, C.byref(h),
        _ptr(bounds, C.c_double), C.byref(st)))
    return Matrix(ctx, h), st.as_dict(), bounds


# ---------------------------------------------------------------- synthetic inputs
def _host_synth(fn, *args):
    n = C.c_int64(0)
    _check(fn(*args, 0, None, None, None, C.byref(n)))
    total = n.value
    leaf = args[1]
    rows = np.empty(total, np.int32)
    cols = np.empty(total, np.int32)
    pay = np.empty((total, leaf * leaf), np.float64)
    _check(fn(*args, total, _ptr(rows, C.c_int32), _ptr(cols, C.c_int32),
              _ptr(pay, C.c_double), C.byref(n)))
    return rows, cols, pay


def synth_chain_host(n: int, leaf: int, ell: float, seed: int, drop: float):
    return _host_synth(lib().spg_synth_chain_host, n, leaf, ell, seed, drop)


def synth_cluster_host(n: int, leaf: int, ell: float, density: float, site_seed: int,
                       value_seed: int, drop: float):
    return _host_synth(lib().spg_synth_cluster_host, n, leaf, ell, density, site_seed,
                       value_seed, drop)


def synth_chain_device_rows(ctx: Context, n: int, leaf: int, ell: float, seed: int, drop: float,
                            row_begin: int, row_end: int) -> Matrix:
    h = _vp()
    _check(lib().spg_synth_chain_device_rows(ctx.handle, n, leaf, ell, seed, drop, row_begin,
                                             row_end, C.byref(h)))
    return Matrix(ctx, h)


def synth_cluster_device_rows(ctx: Context, n: int, leaf: int, ell: float, density: float,
                              site_seed: int, value_seed: int, drop: float, row_begin: int,
                              row_end: int) -> Matrix:
    h = _vp()
    _check(lib().spg_synth_cluster_device_rows(ctx.handle, n, leaf, ell, density, site_seed,
                                               value_seed, drop, row_begin, row_end, C.byref(h)))
    return Matrix(ctx, h)


def synth_cluster_scale(ctx: Context, n: int, ell: float, density: float, site_seed: int,
                        value_seed: int) -> float:
    """The cluster generator's global scale (largest absolute row sum)."""
    out = C.c_double()
    _check(lib().spg_synth_cluster_scale(ctx.handle, n, ell, density, site_seed, value_seed,
                                         C.byref(out)))
    return out.value


def synth_cluster_device_rows_scaled(ctx: Context, n: int, leaf: int, ell: float, density: float,
                                     site_seed: int, value_seed: int, drop: float, scale: float,
                                     row_begin: int, row_end: int) -> Matrix:
    """synth_cluster_device_rows with the scale passed in (no O(n^2) row sums)."""
    h = _vp()
    _check(lib().spg_synth_cluster_device_rows_scaled(ctx.handle, n, leaf, ell, density,
                                                      site_seed, value_seed, drop, scale,
                                                      row_begin, row_end, C.byref(h)))
    return Matrix(ctx, h)


def synth_chain_device(ctx: Context, n: int, leaf: int, ell: float, seed: int,
                       drop: float) -> Matrix:
    h = _vp()
    _check(lib().spg_synth_chain_device(ctx.handle, n, leaf, ell, seed, drop, C.byref(h)))
    return Matrix(ctx, h)


def synth_cluster_device(ctx: Context, n: int, leaf: int, ell: float, density: float,
                         site_seed: int, value_seed: int, drop: float) -> Matrix:
    h = _vp()
    _check(lib().spg_synth_cluster_device(ctx.handle, n, leaf, ell, density, site_seed,
                                          value_seed, drop, C.byref(h)))
    return Matrix(ctx, h)


def dense_to_leaves(dense: np.ndarray, leaf: int):
    """Host-side build_from_dense (quadtree.cpp:89-108) as a leaf list:
    column-major blocks inside the logical dimension, all-zero blocks dropped."""
    n = dense.shape[0]
    nb = (n + leaf - 1) // leaf
    pad = np.zeros((nb * leaf, nb * leaf))
    pad[:n, :n] = dense
    blocks = pad.reshape(nb, leaf, nb, leaf).transpose(0, 2, 3, 1)  # [br, bc, col, row]
    flat = blocks.reshape(nb, nb, leaf * leaf)
    nz = np.any(flat != 0.0, axis=2)
    br, bc = np.nonzero(nz)
    return br.astype(np.int32), bc.astype(np.int32), np.ascontiguousarray(flat[br, bc])


def leaves_to_dense(n: int, leaf: int, rows, cols, payload) -> np.ndarray:
    nb = (n + leaf - 1) // leaf
    pad = np.zeros((nb * leaf, nb * leaf))
    for r, c, p in zip(rows, cols, payload):
        pad[r * leaf:(r + 1) * leaf, c * leaf:(c + 1) * leaf] = p.reshape(leaf, leaf).T
    return pad[:n, :n]
