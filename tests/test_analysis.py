"""Cross-step similarity and head gates.

Oracle pin (CPU): cosine / pairwise similarity / gate statistics restated in
oracle/ against values produced by the reference itself (linalg.py:68-80,
analysis.py:28-51, calibrate_head_gates policy.py:184-246 ->
tests/golden/golden_analysis.npz), and the host HeadGateTable logic.
GPU (-m gpu): fb_row_cosine / fb_pairwise_cosine, the device calibrator
replaying the reference's recorded partials (same gates, statistics within
1e-12), K1 over a group subset and the engine's head-gated step.
"""

import json
import os

import numpy as np
import pytest

from oracle import flashblock_oracle as orc
from paper_2602_05305_b200.policy import HeadGate, HeadGateTable

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ga():
    with np.load(os.path.join(ROOT, "tests", "golden", "golden_analysis.npz")) as z:
        return {k: z[k] for k in z.files}


def _ref_table(ga):
    return json.loads(bytes(ga["cal_table_json"]).decode())


def _runs(ga):
    L, H, samples = (int(x) for x in ga["cal_meta"])
    return L, H, samples, {(l, h): [ga[f"cal_s{s}_l{l}_h{h}"] for s in range(samples)]
                           for l in range(L) for h in range(H)}


def test_oracle_cosine_matches_reference(ga):
    a, b = ga["cos_a"], ga["cos_b"]
    rows = np.array([[orc.cosine_similarity(a[h, r], b[h, r]) for r in range(a.shape[1])]
                     for h in range(a.shape[0])])
    np.testing.assert_allclose(rows, ga["cos_rows"], rtol=0, atol=1e-15)
    assert rows[0, 3] == 0.0 and rows[1, 7] == 0.0  # zero-norm rule
    for h in range(a.shape[0]):
        np.testing.assert_allclose(orc.pairwise_step_similarity(a[h], b[h]), ga["pair"][h],
                                   rtol=0, atol=1e-15)


def test_oracle_gate_stats_reproduce_reference_table(ga):
    _, _, _, runs = _runs(ga)
    ref = _ref_table(ga)
    table = HeadGateTable.from_similarities(float(ga["cal_gamma"][0]), orc.gate_stats(runs))
    got = json.loads(table.to_json())
    assert [h["enabled"] for h in got["heads"]] == [h["enabled"] for h in ref["heads"]]
    for g, r in zip(got["heads"], ref["heads"]):
        assert (g["layer"], g["head"]) == (r["layer"], r["head"])
        assert abs(g["similarity"] - r["similarity"]) <= 1e-12
        assert abs(g["similarity_min"] - r["similarity_min"]) <= 1e-12


def test_head_gate_table_host_logic(ga):
    t = HeadGateTable.from_json(bytes(ga["cal_table_json"]).decode())
    assert t.to_json() == HeadGateTable.from_json(t.to_json()).to_json()
    assert t.is_enabled(1, 0) and not t.is_enabled(0, 0) and not t.is_enabled(9, 9)
    with pytest.raises(ValueError):
        HeadGateTable(0.5, [HeadGate(0, 0, 0.9, 0.8, False)])


# ---------------------------------------------------------------- GPU


def _torch():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return torch


@pytest.mark.gpu
def test_gpu_row_cosine_and_pairwise_match_reference(ga):
    torch = _torch()
    from paper_2602_05305_b200 import kernels as K
    from paper_2602_05305_b200.analysis import pairwise_step_similarity

    a, b = torch.from_numpy(ga["cos_a"]).cuda(), torch.from_numpy(ga["cos_b"]).cuda()
    mean, rows = K.row_cosine(a, b, want_rows=True)
    np.testing.assert_allclose(rows.cpu().numpy(), ga["cos_rows"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(mean.cpu().numpy(), ga["cos_mean"], rtol=0, atol=1e-14)
    for h in range(ga["cos_a"].shape[0]):
        got = pairwise_step_similarity(ga["cos_a"][h], ga["cos_b"][h])  # numpy API, as the reference
        np.testing.assert_allclose(got, ga["pair"][h], rtol=0, atol=1e-14)
    # fp32 / bf16 partials: same statistics within their input rounding
    m32 = K.row_cosine(a.float(), b.float()).cpu().numpy()
    np.testing.assert_allclose(m32, ga["cos_mean"], atol=1e-6)


@pytest.mark.gpu
def test_gpu_calibrator_replays_reference_calibration(ga):
    torch = _torch()
    from paper_2602_05305_b200.analysis import HeadGateCalibrator

    L, H, samples, runs = _runs(ga)
    ref = _ref_table(ga)
    cal = HeadGateCalibrator(L, H)
    for s in range(samples):
        cal.begin_rollout()
        steps = runs[(0, 0)][s].shape[0]
        for step in range(steps):
            for l in range(L):
                o = np.stack([runs[(l, h)][s][step] for h in range(H)])  # [H, rows, d]
                cal.observe(l, torch.from_numpy(o).cuda(), o.shape[1])
    got = json.loads(cal.table(float(ga["cal_gamma"][0])).to_json())
    assert [h["enabled"] for h in got["heads"]] == [h["enabled"] for h in ref["heads"]]
    for g, r in zip(got["heads"], ref["heads"]):
        assert abs(g["similarity"] - r["similarity"]) <= 1e-12
        assert abs(g["similarity_min"] - r["similarity_min"]) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("dt", ["bf16", "f64"])
def test_gpu_group_subset_refresh(dt):
    torch = _torch()
    from paper_2602_05305_b200 import kernels as K

    rng = np.random.Generator(np.random.Philox(11))
    d, groups, q_rows, n = (128, 6, 128, 1500) if dt == "bf16" else (64, 5, 40, 300)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float64
    mk = lambda *s: torch.from_numpy(rng.standard_normal(s).astype(np.float32)).to(tdt).cuda()
    q, k, v = mk(groups, q_rows, d), mk(groups, n + 9, d), mk(groups, n + 9, d)
    ot = torch.float32 if dt == "bf16" else torch.float64
    o = torch.full((groups, q_rows, d), 7.0, dtype=ot, device="cuda")
    l = torch.full((groups, q_rows), 7.0, dtype=ot, device="cuda")
    sel = [4, 1, 3]
    K.attention_partial_groups(q, k, v, torch.tensor(sel, dtype=torch.int32), 3, n + 3, out=o, lse=l)
    for g in range(groups):
        if g not in sel:
            assert bool((o[g] == 7.0).all()) and bool((l[g] == 7.0).all()), "unlisted group touched"
            continue
        ref = orc.partial(q[g].double().cpu().numpy(), k[g, 3:n + 3].double().cpu().numpy(),
                          v[g, 3:n + 3].double().cpu().numpy())
        err = float(np.max(np.abs(o[g].double().cpu().numpy() - ref.out))) / float(np.max(np.abs(ref.out)))
        assert err <= (1e-2 if dt == "bf16" else 1e-12)
        assert float(np.max(np.abs(l[g].double().cpu().numpy() - ref.lognorm))) <= (1e-3 if dt == "bf16" else 1e-10)


@pytest.mark.gpu
def test_gpu_engine_head_gated_step_matches_per_head_reference():
    """1:1 heads (G = 1, like the reference and the C5 video model): heads
    with a disabled gate recompute, enabled ones reuse their cached partial."""
    torch = _torch()
    from paper_2602_05305_b200 import FlashBlockAttention, ReuseConfig
    from paper_2602_05305_b200.policy import Decision

    b, h, blk, d, n = 2, 4, 32, 128, 700
    g = torch.Generator(device="cuda").manual_seed(4)
    mk = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
    kc, vc = mk(b, h, n, d), mk(b, h, n, d)
    q1, q2 = mk(b, h, blk, d), mk(b, h, blk, d)
    ki, vi = mk(b, h, blk, d), mk(b, h, blk, d)
    gates = HeadGateTable(0.9, [HeadGate(0, hh, 0.95 if hh in (0, 2) else 0.5, 0.5, hh in (0, 2))
                                for hh in range(h)])
    eng = FlashBlockAttention(1, b, h, h, blk, d, out_dtype=torch.float32,
                              config=ReuseConfig(tau=2, mode="head-gated"))
    eng.begin_block(0)
    _, dec1 = eng.step_gated(0, q1, kc, vc, n, ki, vi, first_visit=True, updated_tokens=0, gates=gates)
    assert all(x is Decision.RECOMPUTE for x in dec1)
    out2, dec2 = eng.step_gated(0, q2, kc, vc, n, ki, vi, first_visit=False, updated_tokens=1, gates=gates)
    assert [x is Decision.REUSE for x in dec2] == [True, False, True, False]
    out2 = out2.double().cpu().numpy()
    for bi in range(b):
        for hh in range(h):
            kk = np.concatenate([kc[bi, hh].double().cpu().numpy(), ki[bi, hh].double().cpu().numpy()])
            vv = np.concatenate([vc[bi, hh].double().cpu().numpy(), vi[bi, hh].double().cpu().numpy()])
            qq2 = q2[bi, hh].double().cpu().numpy()
            if dec2[hh] is Decision.RECOMPUTE:
                ref = orc.dense(qq2, kk, vv)
            else:
                ext = orc.partial(q1[bi, hh].double().cpu().numpy(), kk[:n], vv[:n])
                ref, _ = orc.with_reuse(qq2, ext, True, kk[n:], vv[n:])
            err = float(np.max(np.abs(out2[bi, hh] - ref))) / float(np.max(np.abs(ref)))
            assert err <= 1e-2, (bi, hh, err)


@pytest.mark.gpu
@pytest.mark.parametrize("dt", ["f64", "f32", "bf16"])
def test_gpu_row_cosine_update_is_cosine_then_copy(dt):
    """fb_row_cosine_update: the same per-head means as fb_row_cosine, prev
    replaced by a in the same pass, nonzero flag raised only by nonzero rows."""
    torch = _torch()
    from paper_2602_05305_b200 import kernels as K

    tdt = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}[dt]
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn((6, 77, 128), device="cuda", generator=g).to(tdt)
    prev = torch.randn((6, 77, 128), device="cuda", generator=g).to(tdt)
    want = K.row_cosine(a, prev)
    flag = torch.zeros((), dtype=torch.int32, device="cuda")
    got = K.row_cosine_update(a, prev, flag)
    assert torch.equal(got, want)
    assert torch.equal(prev, a)
    assert int(flag) == 1
    z = torch.zeros_like(a)
    flag.zero_()
    K.row_cosine_update(z, prev, flag)
    assert int(flag) == 0 and bool((prev == 0).all())
