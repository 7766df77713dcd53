"""K2 v2 (cached step, attention_with_reuse: attention.py:295-321) with the bf16
output written by one bulk tensor store per (CTA, column half) from the dead Q
tile (fb_debug_set_k2_store(1)) is bitwise equal to the row-per-thread global
stores -- same arithmetic, only the store path differs -- and so is issuing
S = Q K^T before V_in landed (fb_debug_set_k2_vsplit(1)); including query
tiles clipped at q_rows, rows with an empty external partial, and the fp32
and bf16 cached-partial layouts."""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def _r(g, *shape):
    return torch.randn(shape, device="cuda", generator=g).to(torch.bfloat16)


@pytest.mark.parametrize("groups,q_rows,n_in", [(256, 128, 32), (16, 128, 16), (12, 200, 64), (5, 77, 1)])
@pytest.mark.parametrize("extb", [False, True])
@pytest.mark.parametrize("variant", [0, 1])  # v1 (V split only) / v2
def test_k2_tma_store_is_bitwise_equal(groups, q_rows, n_in, extb, variant):
    from paper_2602_05305_b200 import _lib
    from paper_2602_05305_b200 import kernels as K

    lib = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(groups * 31 + q_rows + n_in)
    q, ki, vi = _r(g, groups, q_rows, 128), _r(g, groups, n_in, 128), _r(g, groups, n_in, 128)
    oe = torch.randn((groups, q_rows, 128), device="cuda", generator=g)
    if extb:
        oe = oe.to(torch.bfloat16)
    le = torch.randn((groups, q_rows), device="cuda", generator=g)
    le[0, :5] = -math.inf  # rows with an empty external partial
    outs, lses = {}, {}
    lib.fb_debug_set_k2_variant(variant)
    try:
        # per-thread stores / TMA store / + V on its own barrier / + Q, K halves
        for mode in (0, 1, 2, 3):
            lib.fb_debug_set_k2_store(min(mode, 1))
            lib.fb_debug_set_k2_vsplit(max(mode - 1, 0))
            o = torch.full((groups, q_rows, 128), 3.0, device="cuda", dtype=torch.bfloat16)
            K.internal_merge(q, ki, vi, oe, le, out_dtype=torch.bfloat16, out=o, ext_stable=True)
            outs[mode] = o
            outs[mode, "lse"] = K.internal_merge(q, ki, vi, oe, le, out_dtype=torch.bfloat16,
                                                 want_lse=True)
        torch.cuda.synchronize()
    finally:
        lib.fb_debug_set_k2_store(-1)
        lib.fb_debug_set_k2_vsplit(-1)
        lib.fb_debug_set_k2_variant(-1)
    for mode in (1, 2, 3):
        assert torch.equal(outs[0], outs[mode])
        a, b = outs[0, "lse"], outs[mode, "lse"]
        assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


@pytest.mark.parametrize("groups,q_rows", [(160, 77), (150, 200)])
def test_k2_tma_store_writes_nothing_past_the_output(groups, q_rows):
    """The bulk tensor store clips query tiles at q_rows: a sentinel tail right
    after the output (same allocation) stays untouched, and so do the rows of
    other groups (every row is written exactly once with its own value)."""
    from paper_2602_05305_b200 import _lib
    from paper_2602_05305_b200 import kernels as K

    lib = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(groups + q_rows)
    n_in = 32
    q, ki, vi = _r(g, groups, q_rows, 128), _r(g, groups, n_in, 128), _r(g, groups, n_in, 128)
    oe = _r(g, groups, q_rows, 128)
    le = torch.randn((groups, q_rows), device="cuda", generator=g)
    n = groups * q_rows * 128
    lib.fb_debug_set_k2_variant(1)
    try:
        lib.fb_debug_set_k2_store(0)  # reference: row-per-thread stores
        ref = K.internal_merge(q, ki, vi, oe, le, out_dtype=torch.bfloat16, ext_stable=True)
        lib.fb_debug_set_k2_store(1)
        buf = torch.full((n + 64 * 128,), 7.0, device="cuda", dtype=torch.bfloat16)
        K.internal_merge(q, ki, vi, oe, le, out_dtype=torch.bfloat16, out=buf[:n].view(groups, q_rows, 128),
                         ext_stable=True)
        torch.cuda.synchronize()
    finally:
        lib.fb_debug_set_k2_store(-1)
        lib.fb_debug_set_k2_variant(-1)
    assert bool((buf[n:] == 7.0).all())
    assert torch.equal(buf[:n].view(groups, q_rows, 128), ref)
