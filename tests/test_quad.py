"""Two-query-tile K1 (fb_sm100_quad.cuh): one CTA, two 128-row query tiles
sharing every K / V tile.  Default for block-causal prefill; forced here for
the non-causal shapes too (fb_debug_set_quad).

Parity: against the single-CTA kernel on the same inputs (5e-3 relative,
lognorms 1e-4) and the float64 oracle (the bf16 bound, 1e-2); each case
checks that the kernel actually ran (fb_debug_quad_launches)."""

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
    L.fb_debug_set_quad.argtypes = [ctypes.c_int]
    L.fb_debug_set_pair.argtypes = [ctypes.c_int]
    L.fb_debug_quad_launches.restype = ctypes.c_int64
    yield L
    L.fb_debug_set_quad(-1)
    L.fb_debug_set_pair(-1)


def _rel(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(got - ref))) / max(1e-30, float(np.max(np.abs(ref))))


def _quad_and_single(lib, fn):
    lib.fb_debug_set_pair(0)
    lib.fb_debug_set_quad(1)
    before = lib.fb_debug_quad_launches()
    a = fn()
    torch.cuda.synchronize()
    assert lib.fb_debug_quad_launches() > before, "quad kernel did not run"
    lib.fb_debug_set_quad(0)
    b = fn()
    torch.cuda.synchronize()
    lib.fb_debug_set_quad(-1)
    lib.fb_debug_set_pair(-1)
    return a, b


@pytest.mark.parametrize("groups,q_rows,n,kb", [
    (3, 256, 1000, 0), (2, 300, 777, 5), (12, 4680, 2000, 0), (5, 1024, 8192, 0), (1, 200, 129, 0),
])
def test_quad_refresh_vs_single_and_oracle(lib, groups, q_rows, n, kb):
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(groups * 17 + q_rows + n)
    q = torch.randn((groups, q_rows, 128), device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn((groups, n + kb + 3, 128), device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn((groups, n + kb + 3, 128), device="cuda", generator=g).to(torch.bfloat16)
    (oq, lq), (o1, l1) = _quad_and_single(lib, lambda: K.attention_partial(q, k, v, kb, kb + n))
    assert torch.isfinite(oq).all() and torch.isfinite(lq).all()
    assert ((oq - o1).abs().amax() / o1.abs().amax()).item() <= 5e-3
    assert (lq - l1).abs().max().item() <= 1e-4
    gi = groups - 1
    rows = sorted({0, q_rows // 2, q_rows - 1, min(q_rows - 1, 127), min(q_rows - 1, 128)})
    ref = orc.partial(q[gi, rows].double().cpu().numpy(), k[gi, kb:kb + n].double().cpu().numpy(),
                      v[gi, kb:kb + n].double().cpu().numpy())
    assert _rel(oq[gi, rows].cpu().numpy(), ref.out) <= 1e-2
    assert np.max(np.abs(lq[gi, rows].cpu().numpy() - ref.lognorm)) <= 1e-3


@pytest.mark.parametrize("G,n_q,blk,n_prefix", [
    (4, 512, 32, 0), (4, 384, 32, 1000), (1, 300, 16, 0), (3, 200, 64, 17), (3, 600, 64, 17),
])
def test_quad_block_causal_default_vs_oracle(lib, G, n_q, blk, n_prefix):
    """Block-causal prefill takes the quad kernel by default."""
    from paper_2602_05305_b200 import kernels as K

    rng = np.random.Generator(np.random.Philox(3000 + n_q + G))
    cap = n_prefix + n_q + 40
    mk = lambda *s: torch.from_numpy(rng.standard_normal(s).astype(np.float32)).to(torch.bfloat16)
    q, k, v = mk(2, G * n_q, 128), mk(2, cap, 128), mk(2, cap, 128)
    k[:, n_prefix + n_q:] = float("nan")  # rows past the prompt must never be read
    v[:, n_prefix + n_q:] = float("nan")
    before = lib.fb_debug_quad_launches()
    o, l = K.block_causal_attention(q.cuda(), k.cuda(), v.cuda(), n_q, n_prefix, blk)
    torch.cuda.synchronize()
    assert lib.fb_debug_quad_launches() > before
    assert torch.isfinite(o).all() and torch.isfinite(l).all()
    o = o.cpu().numpy()
    for gi in range(2):
        ref = orc.block_causal(q[gi].double().numpy(), k[gi, :n_prefix + n_q].double().numpy(),
                               v[gi, :n_prefix + n_q].double().numpy(), n_prefix, n_q, blk)
        assert _rel(o[gi], ref) <= 1e-2


def test_quad_large_block_cached_step_and_determinism(lib):
    """The large-block cached step (K1 over the block + the fused merge with the
    cached partial) on the quad kernel, and run-to-run bitwise determinism."""
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(8)
    H, B, n_ext = 3, 600, 1500
    r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
    q, k, v, ki, vi = r(H, B, 128), r(H, n_ext, 128), r(H, n_ext, 128), r(H, B, 128), r(H, B, 128)
    o_ext, l_ext = K.attention_partial(q, k, v)
    (a, _), (b, _) = _quad_and_single(
        lib, lambda: (K.internal_merge(q, ki, vi, o_ext, l_ext, out_dtype=torch.float32), None))
    assert ((a - b).abs().amax() / b.abs().amax()).item() <= 5e-3
    lib.fb_debug_set_quad(1)
    x1, y1 = K.attention_partial(q, k, v)
    x2, y2 = K.attention_partial(q, k, v)
    lib.fb_debug_set_quad(-1)
    assert torch.equal(x1, x2) and torch.equal(y1, y2)


@pytest.mark.parametrize("out_bf16", [True, False])
def test_large_block_final_merge_in_epilogue_is_bitwise_equal(out_bf16):
    """C5-style large-block cached step: items one CTA finishes apply the final
    merge with the cached partial in K1's epilogue (fin_whole) -- bitwise the
    same result as the split-merge kernel doing it for every item."""
    import ctypes

    from paper_2602_05305_b200 import _lib
    from paper_2602_05305_b200 import kernels as K

    lib = _lib.load()
    lib.fb_debug_set_k1_fin_whole.argtypes = [ctypes.c_int]
    g = torch.Generator(device="cuda").manual_seed(77)
    H, B, D = 12, 2048, 128  # 192 items of 16 tiles over 148 CTAs: two thirds whole, one third split
    r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
    q, ki, vi, oe = r(H, B, D), r(H, B, D), r(H, B, D), r(H, B, D)
    le = torch.randn((H, B), device="cuda", generator=g)
    odt = torch.bfloat16 if out_bf16 else torch.float32
    res = []
    try:
        for mode in (0, 1):
            lib.fb_debug_set_k1_fin_whole(mode)
            res.append(K.internal_merge(q, ki, vi, oe, le, out_dtype=odt, ext_stable=True))
    finally:
        lib.fb_debug_set_k1_fin_whole(-1)
    assert torch.equal(res[0], res[1])
