"""CPU: the C restatement (oracle/spamm_oracle.c) against golden vectors that
the reference itself produced (tests/golden/make_golden.py), and against the
compiled reference directly when oracle/_ref is present."""
import json

import numpy as np
import pytest

from conftest import GOLDEN, bits_equal, golden_names, load_golden

SMALL = [n for n in golden_names() if n != "cfg1"]


def _build(port, g, tag):
    return port.build(int(g["n"]), int(g["L"]), g[f"{tag}_rows"], g[f"{tag}_cols"],
                      g[f"{tag}_payload"])


@pytest.mark.parametrize("name", SMALL)
def test_port_matches_reference_golden(port, name):
    g = load_golden(name)
    ta, tb = _build(port, g, "a"), _build(port, g, "b")
    # P1: every cached node norm, bit for bit (node_ops.hpp:24-36)
    for tag, t in (("a", ta), ("b", tb)):
        for lvl in range(t.depth() + 1):
            assert bits_equal(t.level_norms(lvl), g[f"{tag}_level{lvl}"]), (tag, lvl)
    # P3: the bound vector, bit for bit (error_control.cpp:34-79)
    assert bits_equal(port.cse(ta, tb, g["taus"]), g["bounds"])
    # P4: selection (error_control.cpp:81-87)
    i = 0
    while f"delta{i}" in g:
        assert port.select_index(g["bounds"], float(g[f"delta{i}"])) == int(g[f"select{i}"])
        i += 1
    # P2 + product: survivors exactly, C leaves bit for bit (same unfused order)
    i = 0
    while f"tau{i}" in g:
        tau = float(g[f"tau{i}"])
        assert np.array_equal(port.survivors(ta, tb, tau), g[f"surv{i}"])
        r, c, p, nrm = port.spamm(ta, tb, tau).leaves()
        assert np.array_equal(r, g[f"c{i}_rows"]) and np.array_equal(c, g[f"c{i}_cols"])
        assert bits_equal(p, g[f"c{i}_payload"]) and bits_equal(nrm, g[f"c{i}_norms"])
        i += 1


def test_cfg1_port_matches_reference_golden(port, built):
    from paper_2005_10680_b200 import _native as nat
    import hashlib
    meta = json.loads((GOLDEN / "cfg1.json").read_text())
    g = load_golden("cfg1")
    rows, cols, pay = nat.synth_chain_host(meta["n"], meta["leaf"], meta["ell"], meta["seed"],
                                           meta["drop"])
    h = hashlib.sha256()
    for a in (rows, cols, pay):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == meta["input_sha256"], "host generator changed its bits"
    t = port.build(meta["n"], meta["leaf"], rows, cols, pay)
    _, _, _, norms = t.leaves(payload=False)
    assert bits_equal(norms, g["leaf_norms"])
    for lvl in range(t.depth() + 1):
        assert bits_equal(t.level_norms(lvl), g[f"a_level{lvl}"])
    bounds = port.cse(t, t, g["taus"])
    assert bits_equal(bounds, g["bounds"])
    k = port.select_index(bounds, meta["delta"])
    assert k == int(g["select"]) == meta["tau_index"]
    surv = port.survivors(t, t, meta["tau"])
    assert len(surv) == meta["survivors"]
    assert hashlib.sha256(np.ascontiguousarray(surv).tobytes()).hexdigest() == \
        meta["survivors_sha256"]


def test_kat_two_level_closed_form(port):
    """test_error_control.cpp:56-88: bound = sqrt((0.01+0.01)^2 + 0.0011^2 + 0.011^2)."""
    g = load_golden("kat_two_level")
    ta, tb = _build(port, g, "a"), _build(port, g, "b")
    expected = np.sqrt((0.01 + 0.01) ** 2 + 0.0011 ** 2 + 0.011 ** 2)
    assert port.cse(ta, tb, [0.02])[0] == pytest.approx(expected, rel=1e-12)


def test_port_matches_ref_random(port, ref):
    """Direct pin against the compiled reference (skipped where it is absent)."""
    from paper_2005_10680_b200._native import dense_to_leaves
    from paper_2005_10680_b200.inputs import geometric_grid
    rng = np.random.default_rng(7)
    for _ in range(10):
        L = int(rng.choice([4, 8, 16]))
        n = int(rng.integers(2, 12)) * 8
        da = rng.uniform(-1, 1, (n, n)) * (rng.uniform(size=(n, n)) < 0.4)
        la = dense_to_leaves(da, L)
        tp, tr = port.build(n, L, *la), ref.build(n, L, *la)
        taus = geometric_grid(1.0, 0.45, 35)
        assert bits_equal(port.cse(tp, tp, taus), ref.cse(tr, tr, taus))
        tau = float(taus[rng.integers(0, 35)])
        assert np.array_equal(port.survivors(tp, tp, tau), ref.survivors(tr, tr, tau))


def test_norm_only_tree_matches_full_tree(port):
    """The large-N oracle mode gives the same bounds as full trees."""
    g = load_golden("random_03")
    ta = _build(port, g, "a")
    r, c, _, nrm = ta.leaves(payload=False)
    tn = port.build_norm_only(int(g["n"]), int(g["L"]), r, c, nrm)
    tb = _build(port, g, "b")
    rb, cb, _, nb = tb.leaves(payload=False)
    tbn = port.build_norm_only(int(g["n"]), int(g["L"]), rb, cb, nb)
    assert bits_equal(port.cse(tn, tbn, g["taus"]), g["bounds"])


@pytest.mark.parametrize("name", SMALL)
def test_port_truncate_matches_reference_golden(port, name):
    g = load_golden(name)
    ta = _build(port, g, "a")
    i = 0
    while f"trunc{i}_delta" in g:
        t, rn, rc = port.truncate(ta, float(g[f"trunc{i}_delta"]))
        assert rc == int(g[f"trunc{i}_removed_count"])
        assert bits_equal(rn, g[f"trunc{i}_removed_norm"])
        r, c, _, nrm = t.leaves(payload=False)
        assert np.array_equal(r, g[f"trunc{i}_rows"]) and np.array_equal(c, g[f"trunc{i}_cols"])
        assert bits_equal(nrm, g[f"trunc{i}_norms"])
        i += 1
    assert i == 4
