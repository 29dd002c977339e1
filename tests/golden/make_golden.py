"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run here (where /root/reference exists):  python tests/golden/make_golden.py

Every expected value is computed by oracle/_ref/libspamm_ref.so -- the
unmodified reference core sources compiled by oracle/Makefile -- never by the
C restatement or the GPU path, so the fixtures pin both of those.  Inputs:
  * small cases restating the reference's own tests (test_multiply.cpp,
    test_error_control.cpp) with their input matrices stored in the fixture;
  * seeded random cases (numpy PCG64, stored);
  * config 1 of BASELINE.json, regenerated from its seed by the repo's host
    generator (spg_synth_chain_host, host-only) -- the fixture stores the
    sha256 of the generated leaves so a generator change is caught.
Doubles are stored as exact binary (npz) and compared bit for bit.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_2005_10680_b200 import _native as nat  # noqa: E402
from paper_2005_10680_b200 import inputs  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def record_case(R, name, n, L, la, lb, taus, taus_list, deltas):
    """Everything the hot path produces for one (A, B) pair, from the reference."""
    ta = R.build(n, L, *la)
    tb = R.build(n, L, *lb)
    out = {"n": np.int64(n), "L": np.int64(L), "taus": np.asarray(taus, np.float64)}
    out["a_rows"], out["a_cols"], out["a_payload"] = la
    out["b_rows"], out["b_cols"], out["b_payload"] = lb
    for tag, t in (("a", ta), ("b", tb)):
        for lvl in range(t.depth() + 1):
            out[f"{tag}_level{lvl}"] = t.level_norms(lvl)
    out["bounds"] = R.cse(ta, tb, taus)
    for i, tau in enumerate(taus_list):
        out[f"tau{i}"] = np.float64(tau)
        out[f"surv{i}"] = R.survivors(ta, tb, tau)
        c = R.spamm(ta, tb, tau)
        r, cc, p, nrm = c.leaves()
        out[f"c{i}_rows"], out[f"c{i}_cols"], out[f"c{i}_payload"], out[f"c{i}_norms"] = r, cc, p, nrm
    for i, d in enumerate(deltas):
        out[f"delta{i}"] = np.float64(d)
        out[f"select{i}"] = np.int64(R.select_index(out["bounds"], d))
    # truncation of A (error_control.cpp:174-201) at fractions of ||A||_F
    for i, f in enumerate((0.0, 0.05, 0.3, 1.01)):
        d = f * ta.frobenius()
        tt, rn, rc = R.truncate(ta, d)
        r, c, _, nrm = tt.leaves(payload=False)
        out[f"trunc{i}_delta"] = np.float64(d)
        out[f"trunc{i}_removed_norm"] = np.float64(rn)
        out[f"trunc{i}_removed_count"] = np.int64(rc)
        out[f"trunc{i}_rows"], out[f"trunc{i}_cols"], out[f"trunc{i}_norms"] = r, c, nrm
    np.savez_compressed(OUT / f"{name}.npz", **out)
    return out


def random_dense(rng, n, fill, decay):
    d = rng.uniform(-1, 1, (n, n)) * (rng.uniform(size=(n, n)) < fill)
    if decay:
        d *= np.exp(-np.abs(np.subtract.outer(np.arange(n), np.arange(n))) / decay)
    return d


def main():
    oracle.build(ref=True)
    R = oracle.Oracle("ref")
    manifest = {"generator": "tests/golden/make_golden.py", "cases": []}

    # --- reference test restatements --------------------------------------
    # two-level quadrature, test_error_control.cpp:56-88 (single-entry 2x2 leaves)
    def single_entries(vals):
        rows, cols, pay = [], [], []
        for (br, bc), v in vals.items():
            blk = np.zeros(4)
            blk[0] = v
            rows.append(br)
            cols.append(bc)
            pay.append(blk)
        return np.array(rows, np.int32), np.array(cols, np.int32), np.array(pay)
    la = single_entries({(0, 0): 0.1, (0, 1): 0.1, (1, 0): 10.0, (1, 1): 1.0})
    lb = single_entries({(0, 0): 0.1, (0, 1): 10.0, (1, 0): 0.1, (1, 1): 0.011})
    record_case(R, "kat_two_level", 4, 2, la, lb, np.array([0.02]), [0.02], [1.0])
    manifest["cases"].append("kat_two_level")

    # quadrant pair dropped, test_multiply.cpp:75-109 (8x8, 4x4 leaves)
    rng = np.random.default_rng(55)
    da = rng.uniform(0.5, 1.0, (8, 8))
    db = rng.uniform(0.5, 1.0, (8, 8))
    da[:4, 4:] *= 1e-4
    db[4:, :4] *= 1e-4
    small = np.linalg.norm(da[:4, 4:]) * np.linalg.norm(db[4:, :4])
    record_case(R, "kat_quadrant_drop", 8, 4, nat.dense_to_leaves(da, 4),
                nat.dense_to_leaves(db, 4), inputs.geometric_grid(1.0, 0.5, 30),
                [small * 50.0, 0.0], [1e-3])
    manifest["cases"].append("kat_quadrant_drop")

    # impossible budget falls back to exact, test_error_control.cpp:266-279
    rng = np.random.default_rng(72)
    d = rng.uniform(-1, 1, (16, 16))
    d[:8, 8:] = 0.0
    d[0, 8] = 1e-30
    la = nat.dense_to_leaves(d, 8)
    record_case(R, "kat_fallback", 16, 8, la, la, inputs.geometric_grid(1.0, 0.5, 40), [0.0],
                [1e-300])
    manifest["cases"].append("kat_fallback")

    # --- seeded random cases ------------------------------------------------
    rng = np.random.default_rng(20051068)
    for t in range(12):
        L = int(rng.choice([2, 4, 8, 16]))
        n = int(rng.integers(1, 9)) * L - int(rng.integers(0, L))
        n = max(n, 1)
        decay = float(rng.uniform(1, 20)) if t % 2 else 0.0
        fill = float(rng.uniform(0.1, 0.9))
        la = nat.dense_to_leaves(random_dense(rng, n, fill, decay), L)
        lb = nat.dense_to_leaves(random_dense(rng, n, fill, decay), L)
        taus = inputs.geometric_grid(1.0, float(rng.uniform(0.3, 0.8)), int(rng.integers(5, 50)))
        tl = [float(taus[rng.integers(0, len(taus))]) for _ in range(2)] + [0.0]
        name = f"random_{t:02d}"
        record_case(R, name, n, L, la, lb, taus, tl, [1e-1, 1e-3, 1e-6])
        manifest["cases"].append(name)

    # --- config 1 (BASELINE.json configs[0]) -------------------------------
    w = inputs.CONFIGS["cfg1"]
    rows, cols, pay = nat.synth_chain_host(w.n, w.leaf, w.ell, w.value_seed, w.drop)
    taus = inputs.log_grid(w.n_taus)
    ta = R.build(w.n, w.leaf, rows, cols, pay)
    bounds = R.cse(ta, ta, taus)
    k = R.select_index(bounds, w.delta)
    tau = float(taus[k]) if k >= 0 else 0.0
    surv = R.survivors(ta, ta, tau)
    c = R.spamm(ta, ta, tau)
    cr, cc, cp, cn = c.leaves()
    _, _, _, an = ta.leaves(payload=False)
    levels = {f"a_level{l}": ta.level_norms(l) for l in range(ta.depth() + 1)}
    np.savez_compressed(
        OUT / "cfg1.npz", taus=taus, bounds=bounds, select=np.int64(k), tau=np.float64(tau),
        leaf_norms=an, c_rows=cr, c_cols=cc, c_norms=cn, **levels,
        c_payload_sum=np.float64(cp.sum()), c_frob=np.float64(c.frobenius()))
    meta = {
        "workload": w.name, "n": w.n, "leaf": w.leaf, "ell": w.ell, "seed": w.value_seed,
        "drop": w.drop, "delta": w.delta, "n_taus": w.n_taus,
        "input_sha256": sha(rows, cols, pay), "n_leaves": int(len(rows)),
        "survivors": int(len(surv)), "survivors_sha256": sha(surv),
        "c_payload_sha256": sha(cp), "tau_index": int(k), "tau": tau,
        "bound": float(bounds[k]) if k >= 0 else 0.0,
    }
    (OUT / "cfg1.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
    manifest["cases"].append("cfg1")
    (OUT / "manifest.json").write_text(json.dumps(manifest, indent=1) + "\n")
    print("wrote", len(manifest["cases"]), "golden cases; cfg1:", meta)


if __name__ == "__main__":
    main()
