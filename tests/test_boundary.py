"""CPU: the C-ABI library loads without a GPU and exports every symbol the
headers under include/ declare; host-only entry points behave like the
reference (ToleranceGrid validation error_control.cpp:139-150, select_tolerance
error_control.cpp:81-87,168-172, test_error_control.cpp:119-124)."""
import ctypes
import re

import numpy as np
import pytest

from conftest import ROOT


def declared_symbols():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = h.read_text()
        names |= set(re.findall(r"\b(spg_[a-z0-9_]+)\s*\(", text))
    return sorted(names)


def test_headers_declare_the_abi():
    syms = declared_symbols()
    assert "spg_cse" in syms and "spg_spamm_with_error_control" in syms
    assert len(syms) >= 25


def test_library_exports_every_declared_symbol(built):
    from paper_2005_10680_b200 import _native as nat
    lib = ctypes.CDLL(str(nat.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding covers the whole ABI
    assert set(declared_symbols()) == set(nat.EXPORTED_SYMBOLS)


def test_library_is_sm100a_and_statically_linked_cudart(built):
    import subprocess
    from paper_2005_10680_b200 import _native as nat
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(nat.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    ldd = subprocess.run(["ldd", str(nat.LIB_PATH)], capture_output=True, text=True).stdout
    assert "libcudart" not in ldd


def test_dmma_in_sass(built):
    """The leaf GEMM really runs on the FP64 tensor pipe (DMMA.8x8x4)."""
    import subprocess
    from paper_2005_10680_b200 import _native as nat
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", str(nat.LIB_PATH)],
                          capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass
    assert "LDGSTS" in sass  # cp.async staging


def test_tolerance_grid_validation(built):
    from paper_2005_10680_b200 import _native as nat
    nat.tolerance_grid_check([1.0, 0.5, 0.25])
    for bad in ([], [1.0, 1.0], [1.0, -0.5], [0.0], [1.0, np.nan]):
        with pytest.raises(ValueError):
            nat.tolerance_grid_check(np.array(bad, np.float64))


def test_select_tolerance_kats(built):
    from paper_2005_10680_b200 import _native as nat
    taus = [1.0, 0.1, 0.01]
    assert nat.select_tolerance([0.5, 0.09, 0.0], taus, 0.1) == (0.1, 1)
    assert nat.select_tolerance([0.0, 0.0, 0.0], taus, 1e-9) == (1.0, 0)
    assert nat.select_tolerance([0.5, 0.2, 0.1], taus, 0.05) == (0.0, -1)


def test_host_generators_deterministic_and_symmetric(built):
    from paper_2005_10680_b200 import _native as nat
    r1 = nat.synth_chain_host(200, 16, 10.0, 7, 1e-10)
    r2 = nat.synth_chain_host(200, 16, 10.0, 7, 1e-10)
    for x, y in zip(r1, r2):
        assert np.array_equal(x, y)
    d = nat.leaves_to_dense(200, 16, *r1)
    assert np.array_equal(d, d.T)
    c = nat.synth_cluster_host(256, 16, 3.0, 0.1, 1, 2, 1e-10)
    dc = nat.leaves_to_dense(256, 16, *c)
    assert np.array_equal(dc, dc.T)
    assert np.abs(dc).sum(axis=1).max() <= 1.0 + 1e-12  # Gershgorin-normalised


def test_no_device_reports_cleanly(built):
    """Without a GPU the library loads and reports a CUDA error, never crashes."""
    from paper_2005_10680_b200 import _native as nat
    if nat.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(nat.SpgCudaError):
        nat.Context(0)
