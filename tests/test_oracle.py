"""Pin the CPU oracle (oracle/flashblock_oracle.py) before trusting it.

Two anchors: the reference test-suite's frozen known-answer values, and
golden vectors produced by the real reference (tests/golden/make_golden.py).
CPU only.
"""

import math

import numpy as np
import pytest

from oracle import flashblock_oracle as orc


# ---------------------------------------------------------------- KATs


def test_kat_lognorm_frozen_value():
    # reference tests/test_attention.py:110-116
    q = np.array([[1.0]])
    k = np.array([[0.5], [-1.25], [2.0]])
    p = orc.partial(q, k, np.ones((3, 1)), scale=1.0)
    assert p.lognorm[0] == pytest.approx(2.2326219831020326, rel=1e-14)


def test_kat_softmax_rows():
    # reference tests/test_linalg.py:61-65
    got = orc.softmax_rows(np.array([[1.0, 2.0, 3.0]]))[0]
    np.testing.assert_allclose(
        got, [0.09003057317038046, 0.24472847105479764, 0.6652409557748218], rtol=1e-15)


def test_kat_mask_budgets(rng):
    # reference tests/test_sparse.py:48-54 -- density -> #blocks at boundary 160
    q = rng.standard_normal((4, 8))
    keys = rng.standard_normal((168, 8))
    for density, blocks in ((0.001, 1), (0.1, 1), (0.2, 2), (0.5, 5), (1.0, 10)):
        assert orc.select_blocks(q, keys, 160, density, 16).size == blocks


def test_kat_ties_to_lower_index():
    # reference tests/test_sparse.py:76-82
    q = np.ones((2, 4))
    keys = np.ones((40, 4))
    assert list(orc.select_blocks(q, keys, 32, 0.5, 16)) == [0]
    assert list(orc.select_blocks(q, keys, 32, 1.0, 16)) == [0, 1]


def test_kat_partial_tail_block(rng):
    # reference tests/test_sparse.py:57-63
    q = rng.standard_normal((4, 8))
    keys = rng.standard_normal((28, 8))
    sel = orc.select_blocks(q, keys, 20, 1.0, 16)
    assert list(sel) == [0, 1]
    assert orc.expand_blocks(sel, 16, 20).tolist() == list(range(20))


def test_kat_decide_truth_table():
    # reference tests/test_policy.py:22-44 (restated rule)
    import itertools

    for mode, tau, cv, fv, upd, gate in itertools.product(
            orc.MODES, (1, 2, 4), (True, False), (True, False), (0, 1, 2, 3, 9), (True, False)):
        want = "Recompute"
        if not (fv or not cv):
            if mode == "always-reuse":
                want = "Reuse"
            elif mode != "always-recompute" and upd < tau and not (mode == "head-gated" and not gate):
                want = "Reuse"
        assert orc.decide(mode, tau, cv, fv, upd, gate) == want


def test_kat_cache_bytes():
    # reference tests/test_attention.py:315 -- nq x (d + 1) float64 scalars
    p = orc.partial(np.zeros((8, 8)), np.zeros((3, 8)), np.zeros((3, 8)))
    assert p.out.nbytes + p.lognorm.nbytes == 8 * (8 + 1) * 8


# ---------------------------------------------------------------- golden


@pytest.mark.parametrize("name", ["p0", "p1", "p2", "p3", "p4", "p5", "p6"])
def test_golden_partial(golden, golden_meta, name):
    m = golden_meta[name]
    p = orc.partial(golden[f"{name}_q"], golden[f"{name}_k"], golden[f"{name}_v"],
                    tile_size=m["tile"])
    tol = 1e-12 if m["dtype"] == "float64" else 2e-6
    np.testing.assert_allclose(p.out, golden[f"{name}_out"], atol=tol)
    np.testing.assert_allclose(p.lognorm, golden[f"{name}_lse"], atol=1e-10)
    assert p.out.dtype == golden[f"{name}_out"].dtype


@pytest.mark.parametrize("b", [0, 1, 17, 39, 40])
def test_golden_streamed_merge(golden, b):
    e, i = orc.streamed(golden["s_q"], golden["s_k"], golden["s_v"], b)
    np.testing.assert_allclose(e.out, golden[f"s_b{b}_ext_out"], atol=1e-13)
    np.testing.assert_array_equal(np.isneginf(e.lognorm), np.isneginf(golden[f"s_b{b}_ext_lse"]))
    np.testing.assert_allclose(orc.merge(e, i), golden[f"s_b{b}_merged"], atol=1e-13)


def test_golden_combine_with_empty_rows(golden):
    c = orc.combine(orc.Partial(golden["c_a_out"], golden["c_a_lse"]),
                    orc.Partial(golden["c_b_out"], golden["c_b_lse"]))
    np.testing.assert_array_equal(c.out, golden["c_out"])  # bitwise
    np.testing.assert_array_equal(c.lognorm, golden["c_lse"])


def test_golden_reuse(golden):
    out, inner = orc.with_reuse(golden["r_q1"], orc.Partial(golden["r_ext_out"], golden["r_ext_lse"]),
                                True, golden["r_k"][268:], golden["r_v"][268:])
    np.testing.assert_allclose(out, golden["r_out"], atol=2e-6)
    np.testing.assert_allclose(inner.lognorm, golden["r_int_lse"], atol=1e-10)


@pytest.mark.parametrize("name", ["m0", "m1", "m2", "m3"])
def test_golden_sparse(golden, golden_meta, name):
    m = golden_meta[name]
    q, k, v = golden[f"{name}_q"], golden[f"{name}_k"], golden[f"{name}_v"]
    for di, dn in enumerate(m["densities"]):
        sel = orc.select_blocks(q, k, m["n_ext"], dn, m["kbs"])
        np.testing.assert_array_equal(sel, golden[f"{name}_d{di}_sel"])
        o1, res, _ = orc.sparse_with_residual(q, sel, m["kbs"], m["n_ext"], k, v)
        np.testing.assert_allclose(o1, golden[f"{name}_d{di}_out1"], atol=2e-6)
        o2, _, _ = orc.sparse_with_residual(golden[f"{name}_d{di}_q2"], sel, m["kbs"],
                                            m["n_ext"], k, v, residual=res)
        np.testing.assert_allclose(o2, golden[f"{name}_d{di}_out2"], atol=2e-6)


def test_golden_refresh_schedule(golden_meta):
    for case in golden_meta["schedules"]:
        assert orc.unmask_schedule(case["block_size"], case["steps"], case["per_step"]) == case["schedule"]
        got = orc.refresh_schedule(case["block_size"], case["steps"], case["per_step"], case["tau"])
        ref = ["Recompute" if d == "FirstVisit" else d for d in case["decisions"]]
        assert got == ref, case
