"""The C++ drop-in (include/spamm/*.hpp over the C ABI) against the
reference's own hot-path unit tests restated in tests/cpp/test_dropin.cpp.
Compiling is a CPU test; running needs the GPU."""
import subprocess

import pytest

from conftest import ROOT

BIN = ROOT / "tests" / "cpp" / "bin" / "test_dropin"
LIB = ROOT / "paper_2005_10680_b200" / "lib"
# the reference's own src/oracle.cpp (dense test helpers), built by oracle/Makefile
DENSE = ROOT / "oracle" / "_ref" / "libspamm_dense_oracle.so"


def compile_test():
    if not DENSE.exists():
        pytest.skip("oracle/_ref/libspamm_dense_oracle.so (reference dense helpers) not built")
    BIN.parent.mkdir(parents=True, exist_ok=True)
    src = ROOT / "tests" / "cpp" / "test_dropin.cpp"
    if BIN.exists() and BIN.stat().st_mtime > max(src.stat().st_mtime,
                                                  (LIB / "libspamm_ec.so").stat().st_mtime,
                                                  DENSE.stat().st_mtime):
        return BIN
    subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", f"-I{ROOT / 'include'}",
                    str(src), "-o", str(BIN), f"-L{LIB}", "-lspamm_ec", "-lspamm_gpu",
                    f"-Wl,-rpath,{LIB}", f"-L{DENSE.parent}", "-lspamm_dense_oracle",
                    f"-Wl,-rpath,{DENSE.parent}"], check=True)
    return BIN


def test_dropin_compiles_against_reference_api(built):
    assert compile_test().exists()


@pytest.mark.gpu
def test_dropin_reference_unit_tests(built):
    exe = compile_test()
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(res.stdout, res.stderr)
    assert res.returncode == 0, res.stderr[-4000:]
    assert "0 failures" in res.stdout
