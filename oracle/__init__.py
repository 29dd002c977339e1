"""CPU checkers for the SpAMM hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package, and only as the checker (never as the thing
measured for the GPU arm, never as a fallback).

Two interchangeable back ends with the same methods:
  * ``Oracle("port")`` -- oracle/liboracle.so, the plain-C restatement
    (spamm_oracle.c), built from this repo; travels to the GPU box.
  * ``Oracle("ref")``  -- oracle/_ref/libspamm_ref.so, the UNMODIFIED reference
    core sources compiled in place by oracle/Makefile (only where
    /root/reference exists; the built .so travels, the sources do not).
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_LIB = HERE / "liboracle.so"
REF_LIB = HERE / "_ref" / "libspamm_ref.so"
REFERENCE_ROOT = Path("/root/reference")

_i32p = C.POINTER(C.c_int32)
_dp = C.POINTER(C.c_double)
_vp = C.c_void_p


def build(ref: bool | None = None) -> None:
    """make -C oracle (and the reference build when its sources are present)."""
    targets = ["all"]
    if ref or (ref is None and REFERENCE_ROOT.exists()):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", str(HERE)] + targets, check=True)


def available(kind: str) -> bool:
    return (PORT_LIB if kind == "port" else REF_LIB).exists()


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class Tree:
    def __init__(self, owner: "Oracle", handle: int, leaf: int):
        self.owner = owner
        self.h = handle
        self.leaf = leaf

    def __del__(self):
        try:
            if self.h:
                self.owner._free(self.h)
                self.h = None
        except Exception:
            pass

    def nnz_blocks(self) -> int:
        return self.owner._nnz(self.h)

    def frobenius(self) -> float:
        return self.owner._frob(self.h)

    def depth(self) -> int:
        return self.owner._depth(self.h)

    def leaves(self, payload: bool = True):
        n = self.nnz_blocks()
        rows = np.empty(n, np.int32)
        cols = np.empty(n, np.int32)
        norms = np.empty(n, np.float64)
        pay = np.empty((n, self.leaf * self.leaf)) if payload else None
        self.owner._leaves(self.h, _p(rows, C.c_int32), _p(cols, C.c_int32),
                           _p(pay, C.c_double) if payload else None, _p(norms, C.c_double))
        return rows, cols, pay, norms

    def level_norms(self, level: int) -> np.ndarray:
        out = np.empty(4 ** level)
        self.owner._level(self.h, level, _p(out, C.c_double))
        return out


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_LIB if kind == "port" else REF_LIB
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (oracle.build())")
        L = C.CDLL(str(path))
        pre = "ora_" if kind == "port" else "ref_"
        self.L = L
        self.pre = pre

        def fn(name, res, args):
            f = getattr(L, pre + name)
            f.restype = res
            f.argtypes = args
            return f

        self._build = fn("build", _vp, [C.c_int, C.c_int, C.c_int64, _i32p, _i32p, _dp])
        self._build_norm_only = fn("build_norm_only", _vp,
                                   [C.c_int, C.c_int, C.c_int64, _i32p, _i32p, _dp])
        self._free = fn("free", None, [_vp])
        self._nnz = fn("nnz_blocks", C.c_int64, [_vp])
        self._frob = fn("frobenius", C.c_double, [_vp])
        self._depth = fn("depth", C.c_int, [_vp])
        self._leaves = fn("leaves", None, [_vp, _i32p, _i32p, _dp, _dp])
        self._level = fn("level_norms", None, [_vp, C.c_int, _dp])
        self._cse = fn("cse", C.c_int, [_vp, _vp, _dp, C.c_int, _dp])
        self._spamm = fn("spamm", _vp, [_vp, _vp, C.c_double, C.POINTER(C.c_int)])
        self._exact = fn("multiply_exact", _vp, [_vp, _vp, C.POINTER(C.c_int)])
        self._surv = fn("survivors", C.c_int64, [_vp, _vp, C.c_double, _i32p, C.c_int64])
        self._trunc = fn("truncate", _vp, [_vp, C.c_double, _dp, C.POINTER(C.c_int64),
                                            C.POINTER(C.c_int)])
        self._cse_sub = fn("cse_subtree", C.c_int, [_vp, _vp, _dp, C.c_int, C.c_int, C.c_int32,
                                                   C.c_int32, C.c_int32, _dp])
        if kind == "port":
            self._select = fn("select_index", C.c_int, [_dp, C.c_int, C.c_double])
            self._cand = fn("candidates", C.c_int64, [_vp, _vp])
        else:
            self._from_dense = fn("from_dense", _vp, [C.c_int, C.c_int, _dp])
            self._threads = fn("set_max_threads", None, [C.c_int])
            self._trace = fn("trace", C.c_double, [_vp])
            self._nnz_entries = fn("nnz", C.c_int64, [_vp])
            self._axpby = fn("axpby", _vp, [C.c_double, _vp, C.c_double, _vp])
            self._digest = fn("survivor_digest", None, [_vp, _vp, C.c_double, C.c_int,
                                                        C.POINTER(C.c_int64),
                                                        C.POINTER(C.c_uint64)])
            self._purify = fn("purify", _vp, [_vp, C.c_int, C.c_int, C.c_int, C.c_double, _dp,
                                              C.c_int, C.c_double, _dp, C.c_double, C.c_int,
                                              C.POINTER(C.c_int), _dp, C.POINTER(C.c_int),
                                              C.POINTER(C.c_int)])
            self._swec = fn("spamm_with_error_control", _vp,
                            [_vp, _vp, C.c_double, _dp, C.c_int, _dp, _dp, _dp, _dp,
                             C.POINTER(C.c_int)])

    # -- construction ---------------------------------------------------------
    def build(self, dimension: int, leaf: int, rows, cols, payload) -> Tree:
        rows = np.ascontiguousarray(rows, np.int32)
        cols = np.ascontiguousarray(cols, np.int32)
        payload = np.ascontiguousarray(payload, np.float64)
        h = self._build(dimension, leaf, rows.size, _p(rows, C.c_int32), _p(cols, C.c_int32),
                        _p(payload, C.c_double))
        if not h:
            raise ValueError("oracle build rejected the leaf list")
        return Tree(self, h, leaf)

    def build_norm_only(self, dimension: int, leaf: int, rows, cols, norms) -> Tree:
        rows = np.ascontiguousarray(rows, np.int32)
        cols = np.ascontiguousarray(cols, np.int32)
        norms = np.ascontiguousarray(norms, np.float64)
        h = self._build_norm_only(dimension, leaf, rows.size, _p(rows, C.c_int32),
                                  _p(cols, C.c_int32), _p(norms, C.c_double))
        if not h:
            raise ValueError("oracle build rejected the leaf list")
        return Tree(self, h, leaf)

    # -- algebra the callers use (ref back end only) ----------------------------
    def trace(self, a: Tree) -> float:
        return self._trace(a.h)

    def nnz(self, a: Tree) -> int:
        return self._nnz_entries(a.h)

    def axpby(self, alpha: float, a: Tree, beta: float = 0.0, b: Tree | None = None) -> Tree:
        h = self._axpby(alpha, a.h, beta, b.h if b is not None else None)
        if not h:
            raise ValueError("axpby: invalid arguments")
        return Tree(self, h, a.leaf)

    def survivor_digest(self, a: Tree, b: Tree, tau: float, threads: int = 0):
        """(count, digest) of spamm_multiply(a, b, tau)'s survivor set; the same
        function of the set as spg_survivor_digest (ref back end only)."""
        import os
        n, d = C.c_int64(0), C.c_uint64(0)
        self._digest(a.h, b.h, tau, threads or os.cpu_count() or 1, C.byref(n), C.byref(d))
        return n.value, d.value

    def set_threads(self, n: int):
        if self.kind == "ref":
            self._threads(n)

    # -- hot path ---------------------------------------------------------------
    def cse(self, a: Tree, b: Tree, taus) -> np.ndarray:
        taus = np.ascontiguousarray(taus, np.float64)
        out = np.empty(taus.size)
        if self._cse(a.h, b.h, _p(taus, C.c_double), taus.size, _p(out, C.c_double)) != 0:
            raise ValueError("cse: dimension or leaf size mismatch")
        return out

    def cse_subtree(self, a: Tree, b: Tree, taus, level: int, I: int, K: int, J: int):
        taus = np.ascontiguousarray(taus, np.float64)
        out = np.empty(taus.size)
        if self._cse_sub(a.h, b.h, _p(taus, C.c_double), taus.size, level, I, K, J,
                         _p(out, C.c_double)) != 0:
            raise ValueError("cse_subtree: invalid arguments")
        return out

    def shard_partials(self, a: Tree, b: Tree, taus, level: int, shard: int) -> np.ndarray:
        """What spg_cse_shard returns, from the oracle: (4^level, n_taus)."""
        side = 2 ** level
        return np.stack([self.cse_subtree(a, b, taus, level, shard, K, J)
                         for K in range(side) for J in range(side)])

    @staticmethod
    def select_index(bounds, delta: float) -> int:
        for k, v in enumerate(bounds):
            if v < delta:
                return k
        return -1

    def spamm(self, a: Tree, b: Tree, tau: float) -> Tree:
        st = C.c_int(0)
        h = self._spamm(a.h, b.h, tau, C.byref(st))
        if st.value != 0 or not h:
            raise ValueError("spamm: invalid arguments")
        return Tree(self, h, a.leaf)

    def multiply_exact(self, a: Tree, b: Tree) -> Tree:
        st = C.c_int(0)
        h = self._exact(a.h, b.h, C.byref(st))
        if st.value != 0 or not h:
            raise ValueError("multiply: invalid arguments")
        return Tree(self, h, a.leaf)

    def truncate(self, x: Tree, delta: float):
        """(tree, removed_norm_bound, removed_block_count)."""
        rn = C.c_double(0)
        rc = C.c_int64(0)
        st = C.c_int(0)
        h = self._trunc(x.h, delta, C.byref(rn), C.byref(rc), C.byref(st))
        if st.value != 0 or not h:
            raise ValueError("truncate: delta must be nonnegative")
        return Tree(self, h, x.leaf), rn.value, rc.value

    def purify(self, x0: Tree, variant: int, occupation: int, max_iterations: int, epsilon: float,
               taus, initial_delta: float, deltas, idempotency_threshold: float = 0.0):
        """Reference purify (ref back end only): (tree, log rows, converged, iterations);
        log rows = (iteration, status, chosen_tau, trace, realized_error, nnz_out)."""
        taus = np.ascontiguousarray(taus, np.float64)
        deltas = np.ascontiguousarray(deltas, np.float64)
        cap = max_iterations + 2
        log = np.zeros((cap, 6))
        n_log, conv, its = C.c_int(0), C.c_int(0), C.c_int(0)
        h = self._purify(x0.h, variant, occupation, max_iterations, epsilon,
                         _p(taus, C.c_double), taus.size, initial_delta, _p(deltas, C.c_double),
                         idempotency_threshold, cap, C.byref(n_log), _p(log, C.c_double),
                         C.byref(conv), C.byref(its))
        if not h:
            raise ValueError("purify: invalid configuration")
        return Tree(self, h, x0.leaf), log[:min(n_log.value, cap)], bool(conv.value), its.value

    def survivors(self, a: Tree, b: Tree, tau: float) -> np.ndarray:
        n = self._surv(a.h, b.h, tau, None, 0)
        out = np.empty((n, 3), np.int32)
        if n:
            self._surv(a.h, b.h, tau, _p(out, C.c_int32), n)
        return out


INPUTS_LIB = HERE / "libinputs.so"


def host_inputs(w, threads: int | None = None, value_seed: int | None = None):
    """(rows, cols, payload) of BASELINE workload `w` (inputs.Workload) from
    oracle/libinputs.so: bitwise the product's host generator
    (spg_synth_*_host), multi-threaded, without loading the product library."""
    import os
    L = C.CDLL(str(INPUTS_LIB))
    threads = threads or os.cpu_count() or 1
    seed = w.value_seed if value_seed is None else value_seed
    nb = -(-w.n // w.leaf)
    cap = nb * nb
    rows = np.empty(cap, np.int32)
    cols = np.empty(cap, np.int32)
    pay = np.empty((cap, w.leaf * w.leaf))
    n = C.c_int64(0)
    if w.kind == "cluster":
        f = L.inp_cluster
        f.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_uint64, C.c_uint64,
                      C.c_double, C.c_int, C.c_int64, _i32p, _i32p, _dp, C.POINTER(C.c_int64)]
        rc = f(w.n, w.leaf, w.ell, w.density, w.site_seed, seed, w.drop, threads, cap,
               _p(rows, C.c_int32), _p(cols, C.c_int32), _p(pay, C.c_double), C.byref(n))
    else:
        f = L.inp_chain
        f.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_uint64, C.c_double, C.c_int,
                      C.c_int64, _i32p, _i32p, _dp, C.POINTER(C.c_int64)]
        rc = f(w.n, w.leaf, w.ell, seed, w.drop, threads, cap, _p(rows, C.c_int32),
               _p(cols, C.c_int32), _p(pay, C.c_double), C.byref(n))
    if rc != 0:
        raise ValueError("host_inputs: invalid workload")
    k = n.value
    return rows[:k], cols[:k], pay[:k]


def leaves_to_dense(n: int, leaf: int, rows, cols, payload) -> np.ndarray:
    nb = (n + leaf - 1) // leaf
    pad = np.zeros((nb * leaf, nb * leaf))
    for r, c, p in zip(rows, cols, payload):
        pad[r * leaf:(r + 1) * leaf, c * leaf:(c + 1) * leaf] = np.asarray(p).reshape(leaf, leaf).T
    return pad[:n, :n]
