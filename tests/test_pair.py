"""CTA-pair K1 (cta_group::2, fb_sm100_pair.cuh): the tensor-bound refresh /
prefill path for many query rows per kv group (C5 video chunks, prefill).

Parity: against the float64 oracle on bf16-exact inputs (max|diff| <=
1e-2 * max|ref|, lognorm within 1e-3, the bf16 bound of tests/test_gpu_attention.py)
and against the single-CTA kernel on the same inputs (both run the same
per-row online softmax; outputs within 5e-3 relative, lognorms 1e-4).  Each
case asserts that the pair kernel actually ran (fb_debug_pair_launches).
The cached-step (K2) variants v1 / v2 are checked against each other and the
oracle at the end (fb_debug_set_k2_variant).
"""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import flashblock_oracle as orc  # noqa: E402


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2602_05305_b200 import _lib

    L = _lib.load()
    L.fb_debug_set_pair.argtypes = [ctypes.c_int]
    L.fb_debug_pair_launches.restype = ctypes.c_int64
    yield L
    L.fb_debug_set_pair(-1)


def _rel(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(got - ref))) / max(1e-30, float(np.max(np.abs(ref))))


def _run_both(lib, fn):
    lib.fb_debug_set_pair(1)
    before = lib.fb_debug_pair_launches()
    a = fn()
    torch.cuda.synchronize()
    assert lib.fb_debug_pair_launches() > before, "pair kernel did not run"
    lib.fb_debug_set_pair(0)
    before = lib.fb_debug_pair_launches()
    b = fn()
    torch.cuda.synchronize()
    assert lib.fb_debug_pair_launches() == before, "single-CTA path ran the pair kernel"
    lib.fb_debug_set_pair(-1)
    return a, b


@pytest.mark.parametrize("groups,q_rows,n,kb", [
    (3, 256, 1000, 0),       # one pair tile per group
    (2, 300, 777, 5),        # ragged last tile (44 live rows of 256), key offset
    (12, 4680, 2000, 0),     # C5 chunk rows (19 pair tiles, last 72 rows live)
    (5, 1024, 8192, 0),      # stream-K splits across pairs (merge kernel)
    (1, 200, 129, 0),        # fewer live rows than one CTA of the pair
])
def test_pair_refresh_vs_oracle_and_single_cta(lib, groups, q_rows, n, kb):
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(groups * 131 + q_rows + n)
    q = torch.randn((groups, q_rows, 128), device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn((groups, n + kb + 3, 128), device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn((groups, n + kb + 3, 128), device="cuda", generator=g).to(torch.bfloat16)
    (op, lp), (o1, l1) = _run_both(lib, lambda: K.attention_partial(q, k, v, kb, kb + n))
    assert torch.isfinite(op).all() and torch.isfinite(lp).all()
    err = ((op - o1).abs().amax() / o1.abs().amax()).item()
    assert err <= 5e-3, f"pair vs single-CTA rel err {err:.3e}"
    assert (lp - l1).abs().max().item() <= 1e-4
    for gi in sorted({0, groups - 1}):
        rows = sorted({0, q_rows // 2, q_rows - 1, min(q_rows - 1, 255), min(q_rows - 1, 256)})
        qq = q[gi, rows].double().cpu().numpy()
        ref = orc.partial(qq, k[gi, kb:kb + n].double().cpu().numpy(), v[gi, kb:kb + n].double().cpu().numpy())
        assert _rel(op[gi, rows].cpu().numpy(), ref.out) <= 1e-2
        assert np.max(np.abs(lp[gi, rows].cpu().numpy() - ref.lognorm)) <= 1e-3


def test_pair_refresh_deterministic_and_large_scores(lib):
    """score std ~6 exercises the lazy O rescale on both CTAs of the pair;
    two runs are bitwise equal (no float atomics, fixed merge order)."""
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(77)
    q = (2.5 * torch.randn((4, 512, 128), device="cuda", generator=g)).to(torch.bfloat16)
    k = (2.5 * torch.randn((4, 3000, 128), device="cuda", generator=g)).to(torch.bfloat16)
    v = torch.randn((4, 3000, 128), device="cuda", generator=g).to(torch.bfloat16)
    lib.fb_debug_set_pair(1)
    o, l = K.attention_partial(q, k, v)
    o2, l2 = K.attention_partial(q, k, v)
    lib.fb_debug_set_pair(-1)
    assert torch.equal(o, o2) and torch.equal(l, l2)
    for gi in (0, 3):
        ref = orc.partial(q[gi].double().cpu().numpy(), k[gi].double().cpu().numpy(), v[gi].double().cpu().numpy())
        assert _rel(o[gi].cpu().numpy(), ref.out) <= 1e-2
        assert np.max(np.abs(l[gi].cpu().numpy() - ref.lognorm)) <= 1e-3


@pytest.mark.parametrize("G,n_q,blk,n_prefix", [
    (4, 512, 32, 0),      # C2 GQA stacking: 2048 rows per group, 8 pair tiles
    (4, 384, 32, 1000),   # committed prefix + prompt
    (1, 300, 16, 0),      # ragged last pair tile
    (3, 200, 64, 17),     # pair tiles straddle heads
    (3, 600, 64, 17),     # straddling tiles + multi-tile segments in both kernels: a warp whose
                          # first tile has rows with and without keys (the -inf - -inf rescale)
])
def test_pair_block_causal_vs_oracle(lib, G, n_q, blk, n_prefix):
    from paper_2602_05305_b200 import kernels as K

    rng = np.random.Generator(np.random.Philox(2000 + n_q + G))
    groups, d = 2, 128
    cap = n_prefix + n_q + 40
    mk = lambda *s: torch.from_numpy(rng.standard_normal(s).astype(np.float32)).to(torch.bfloat16)
    q, k, v = mk(groups, G * n_q, d), mk(groups, cap, d), mk(groups, cap, d)
    k[:, n_prefix + n_q:] = float("nan")  # rows past the prompt must never be read
    v[:, n_prefix + n_q:] = float("nan")
    qc, kc, vc = q.cuda(), k.cuda(), v.cuda()
    (op, lp), (o1, l1) = _run_both(lib, lambda: K.block_causal_attention(qc, kc, vc, n_q, n_prefix, blk))
    assert torch.isfinite(op).all() and torch.isfinite(lp).all()
    assert torch.isfinite(o1).all() and torch.isfinite(l1).all()
    assert ((op - o1).abs().amax() / o1.abs().amax()).item() <= 5e-3
    assert (lp - l1).abs().max().item() <= 1e-4
    op = op.cpu().numpy()
    for gi in range(groups):
        ref = orc.block_causal(q[gi].double().numpy(), k[gi, :n_prefix + n_q].double().numpy(),
                               v[gi, :n_prefix + n_q].double().numpy(), n_prefix, n_q, blk)
        assert _rel(op[gi], ref) <= 1e-2


def test_pair_large_block_cached_step(lib):
    """C5-style cached step with a > 128-key block (K1 over the block's own
    keys on the pair kernel + K3 merge with the cached partial)."""
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(5)
    H, B, n_ext = 3, 600, 1500
    r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
    q, k, v, ki, vi = r(H, B, 128), r(H, n_ext, 128), r(H, n_ext, 128), r(H, B, 128), r(H, B, 128)
    o_ext, l_ext = K.attention_partial(q, k, v)
    (outp, _), (out1, _) = _run_both(
        lib, lambda: (K.internal_merge(q, ki, vi, o_ext, l_ext, out_dtype=torch.float32), None))
    assert ((outp - out1).abs().amax() / out1.abs().amax()).item() <= 5e-3
    kk = torch.cat([k, ki], 1).double().cpu().numpy()
    vv = torch.cat([v, vi], 1).double().cpu().numpy()
    for h in (0, H - 1):
        ref = orc.dense(q[h].double().cpu().numpy(), kk[h], vv[h])
        assert _rel(outp[h].cpu().numpy(), ref) <= 1e-2


@pytest.mark.parametrize("b,n_in", [(2, 32), (20, 32), (3, 16), (2, 64), (1, 1)])
def test_cached_step_v1_v2_agree_and_match_oracle(lib, b, n_in):
    """K2 variants (v1: O_ext in registers, columns split over 2 CTAs; v2:
    O_ext prefetched into swizzled smem by TMA, whole rows per CTA) on the
    same C2-shaped inputs: both within the bf16 bound of the oracle and of
    each other.  The size rule picks v2 only when query tiles > SMs."""
    from paper_2602_05305_b200 import kernels as K

    lib.fb_debug_set_k2_variant.argtypes = [ctypes.c_int]
    g = torch.Generator(device="cuda").manual_seed(b * 10 + n_in)
    groups, rows, d = b * 8, 128, 128
    r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
    q, ki, vi = r(groups, rows, d), r(groups, n_in, d), r(groups, n_in, d)
    k, v = r(groups, 300, d), r(groups, 300, d)
    o_ext, l_ext = K.attention_partial(q, k, v)
    outs = []
    for var in (0, 1):
        lib.fb_debug_set_k2_variant(var)
        o, lse = K.internal_merge(q, ki, vi, o_ext, l_ext, out_dtype=torch.float32, want_lse=True)
        torch.cuda.synchronize()
        outs.append((o, lse))
    lib.fb_debug_set_k2_variant(-1)
    (o1, l1), (o2, l2) = outs
    assert ((o1 - o2).abs().amax() / o1.abs().amax()).item() <= 1e-5
    assert (l1 - l2).abs().max().item() <= 1e-5
    kk = torch.cat([k, ki], 1).double().cpu().numpy()
    vv = torch.cat([v, vi], 1).double().cpu().numpy()
    for gi in (0, groups - 1):
        ref = orc.dense(q[gi].double().cpu().numpy(), kk[gi], vv[gi])
        assert _rel(o2[gi].cpu().numpy(), ref) <= 1e-2


def test_pair_full_size_properties(lib):
    """BASELINE sizes, size-independent properties (the oracle cannot run
    these in seconds): C5 (12 heads x 4680 rows x 56,160 keys) pair kernel ==
    single-CTA kernel, and K1 over [0, N) == combine(K1 [0, a), K1 [a, N)) on
    the pair kernel; prefill at the C2 shapes with an 8K prompt: pair ==
    single-CTA."""
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(4680)
    r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
    q, k, v = r(12, 4680, 128), r(12, 56160, 128), r(12, 56160, 128)
    (op, lp), (o1, l1) = _run_both(lib, lambda: K.attention_partial(q, k, v))
    assert ((op - o1).abs().amax() / o1.abs().amax()).item() <= 5e-3
    assert (lp - l1).abs().max().item() <= 1e-4
    lib.fb_debug_set_pair(1)
    a = 20000
    pa = K.attention_partial(q, k, v, 0, a)
    pb = K.attention_partial(q, k, v, a, 56160)
    lib.fb_debug_set_pair(-1)
    oc, lc = K.combine([pa, pb])
    assert ((oc - op).abs().amax() / op.abs().amax()).item() <= 5e-3
    assert (lc - lp).abs().max().item() <= 1e-4
    del q, k, v
    n_q = 8192
    qp, kp, vp = r(8, 4 * n_q, 128), r(8, n_q, 128), r(8, n_q, 128)
    (op, lp), (o1, l1) = _run_both(lib, lambda: K.block_causal_attention(qp, kp, vp, n_q, 0, 32))
    assert ((op - o1).abs().amax() / o1.abs().amax()).item() <= 5e-3
    assert (lp - l1).abs().max().item() <= 1e-4
