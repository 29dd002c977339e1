"""The drop-in's experiment-side modules against the
reference, via tests/cpp/test_experiment.cpp: MatrixMarket reading/writing,
the decay-model generator, Gershgorin bounds and the density-matrix oracle
(bitwise, no GPU), RunRecord CSV/JSON output, and the squaring / purification
runners (GPU) with per-record comparison against the reference's own calls."""
import csv
import json
import math
import subprocess

import pytest

from conftest import ROOT

BIN = ROOT / "tests" / "cpp" / "bin" / "test_experiment"
LIB = ROOT / "paper_2005_10680_b200" / "lib"
# the reference's own src/oracle.cpp (dense test helpers), built by oracle/Makefile
DENSE = ROOT / "oracle" / "_ref" / "libspamm_dense_oracle.so"
REF = ROOT / "oracle" / "_ref" / "libspamm_ref.so"


def compile_test():
    if not DENSE.exists():
        pytest.skip("oracle/_ref/libspamm_dense_oracle.so (reference dense helpers) not built")
    BIN.parent.mkdir(parents=True, exist_ok=True)
    src = ROOT / "tests" / "cpp" / "test_experiment.cpp"
    if BIN.exists() and BIN.stat().st_mtime > max(src.stat().st_mtime,
                                                  (LIB / "libspamm_ec.so").stat().st_mtime,
                                                  DENSE.stat().st_mtime):
        return BIN
    subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", f"-I{ROOT / 'include'}",
                    str(src), "-o", str(BIN), f"-L{LIB}", "-lspamm_ec", "-lspamm_gpu", "-ldl",
                    f"-Wl,-rpath,{LIB}", f"-L{DENSE.parent}", "-lspamm_dense_oracle",
                    f"-Wl,-rpath,{DENSE.parent}"], check=True)
    return BIN


def run(mode, tmp_path):
    if not REF.exists():
        pytest.skip("reference build (oracle/_ref) not present")
    res = subprocess.run([str(compile_test()), mode, str(tmp_path), str(REF)],
                         capture_output=True, text=True, timeout=900)
    print(res.stdout, res.stderr[-4000:])
    assert res.returncode == 0, res.stderr[-4000:]
    assert " 0 failures" in res.stdout


def test_host_modules_match_reference(built, tmp_path):
    run("host", tmp_path)
    rows = list(csv.reader(open(tmp_path / "records.csv")))
    assert rows[0] == ("variant,iter,tolerance,chosen_tau,t_mul,t_trunc,t_spamm,t_cse,"
                       "nnz_in,nnz_mid,nnz_out,nnz_blocks_out,realized_error,status").split(",")
    assert float(rows[1][3]) == 7.4296395075949501e-09 and rows[2][-1] == "violation"
    recs = json.load(open(tmp_path / "records.json"))
    assert [r["variant"] for r in recs] == ["spamm", "hybrid"]
    assert recs[0]["chosen_tau"] == 7.4296395075949501e-09 and recs[0]["processes"] == 1
    assert recs[0]["realized_error"] == 0.1 + 0.2 and recs[0]["trace"] == 2.0
    assert recs[1]["realized_error"] is None  # non-finite -> null, as nlohmann::json
    assert list(recs[0]) == sorted(recs[0])  # std::map key order
    assert json.load(open(tmp_path / "empty.json")) == []


@pytest.mark.gpu
def test_experiments_match_reference(built, tmp_path):
    run("gpu", tmp_path)
    rows = list(csv.DictReader(open(tmp_path / "squaring.csv")))
    assert len(rows) == 9 and all(r["status"] == "ok" for r in rows)
    pur = json.load(open(tmp_path / "purification.json"))
    finals = [r for r in pur if r["status"].startswith("final")]
    assert len(finals) == 3 and all(r["status"] == "final-ok" for r in finals)
    assert all(math.isclose(r["trace"], 80.0, abs_tol=1e-3) for r in finals)
