"""bf16 partial out (FB_PARTIAL_BF16): the cached external partial's O stored
in the tensor dtype, as the reference keeps a partial's out
(attention.py:70-71), with the lognorm in fp32.

The kernels compute exactly as with the fp32 partial and round only at the
store (K1 / merge kernel) or widen exactly at the load (K2), so:
  * K1 with a bf16 out == the fp32 out rounded to bf16, bit for bit, on every
    refresh path (uniform with in-kernel or merge-kernel split merge, ragged,
    paged, group subset), LSE bitwise equal;
  * K2 reading a bf16 O_ext == K2 reading the fp32 tensor holding the same
    (bf16-representable) values, bit for bit, on each kernel variant (v1, v2,
    token-major, large-block K1 + fused merge).
End-to-end the engine (bf16 O_ext by default) is checked against the float64
oracle within the bf16 bound by the existing engine / config-size tests."""

import math

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _r(g, *s):
    return torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)


@pytest.mark.parametrize("groups,q_rows,n", [(128, 128, 32768), (8, 128, 16384), (4, 96, 1000), (3, 256, 4700)])
def test_k1_bf16_out_is_fp32_out_rounded(groups, q_rows, n):
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(groups + n)
    q, k, v = _r(g, groups, q_rows, 128), _r(g, groups, n, 128), _r(g, groups, n, 128)
    o32, l32 = K.attention_partial(q, k, v, 0, n)
    ob = torch.empty(o32.shape, device="cuda", dtype=torch.bfloat16)
    lb = torch.empty_like(l32)
    K.attention_partial(q, k, v, 0, n, out=ob, lse=lb)
    torch.cuda.synchronize()
    assert torch.equal(ob, o32.to(torch.bfloat16))
    assert torch.equal(lb, l32)


def test_k1_bf16_out_ragged_paged_and_groups():
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(5)
    groups, q_rows, cap, d = 6, 128, 2048, 128
    q, k, v = _r(g, groups, q_rows, d), _r(g, groups, cap, d), _r(g, groups, cap, d)
    lens = torch.tensor([2048, 1, 0, 777, 1536, 129], device="cuda", dtype=torch.int32)
    o32, l32 = K.attention_partial_ragged(q, k, v, lens)
    ob = torch.empty(o32.shape, device="cuda", dtype=torch.bfloat16)
    lb = torch.empty_like(l32)
    K.attention_partial_ragged(q, k, v, lens, out=ob, lse=lb)
    assert torch.equal(ob, o32.to(torch.bfloat16)) and torch.equal(lb, l32)

    # paged: the same slabs cut into 128-row pages in shuffled pool order
    P = 128
    pages = cap // P
    perm = torch.randperm(groups * pages, generator=torch.Generator().manual_seed(3)).to("cuda")
    kp = torch.empty((groups * pages, P, d), device="cuda", dtype=torch.bfloat16)
    vp = torch.empty_like(kp)
    kp[perm] = k.view(groups * pages, P, d)
    vp[perm] = v.view(groups * pages, P, d)
    table = perm.view(groups, pages).to(torch.int32)
    op32, lp32 = K.attention_partial_paged(q, kp, vp, table, lens)
    opb = torch.empty(op32.shape, device="cuda", dtype=torch.bfloat16)
    lpb = torch.empty_like(lp32)
    K.attention_partial_paged(q, kp, vp, table, lens, out=opb, lse=lpb)
    assert torch.equal(opb, op32.to(torch.bfloat16)) and torch.equal(lpb, lp32)

    gl = torch.tensor([4, 1], device="cuda", dtype=torch.int32)
    og32 = torch.zeros((groups, q_rows, d), device="cuda")
    lg32 = torch.zeros((groups, q_rows), device="cuda")
    K.attention_partial_groups(q, k, v, gl, 0, 1500, out=og32, lse=lg32)
    ogb = torch.zeros((groups, q_rows, d), device="cuda", dtype=torch.bfloat16)
    lgb = torch.zeros((groups, q_rows), device="cuda")
    K.attention_partial_groups(q, k, v, gl, 0, 1500, out=ogb, lse=lgb)
    torch.cuda.synchronize()
    assert torch.equal(ogb, og32.to(torch.bfloat16)) and torch.equal(lgb, lg32)
    assert torch.count_nonzero(ogb[[0, 2, 3, 5]]) == 0  # other groups untouched


def test_k1_bf16_out_empty_range_is_the_sentinel():
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(6)
    q, k, v = _r(g, 2, 64, 128), _r(g, 2, 256, 128), _r(g, 2, 256, 128)
    ob = torch.full((2, 64, 128), 7.0, device="cuda", dtype=torch.bfloat16)
    lb = torch.zeros((2, 64), device="cuda")
    K.attention_partial(q, k, v, 100, 100, out=ob, lse=lb)
    torch.cuda.synchronize()
    assert torch.count_nonzero(ob) == 0 and bool(torch.isneginf(lb).all())


@pytest.mark.parametrize("variant", [0, 1])  # K2 v1 (column split) / v2 (O_ext tile in smem)
@pytest.mark.parametrize("groups,n_in", [(128, 32), (16, 16), (40, 64), (8, 100)])
def test_k2_bf16_ext_equals_fp32_ext_of_same_values(variant, groups, n_in):
    from paper_2602_05305_b200 import _lib
    from paper_2602_05305_b200 import kernels as K

    if variant == 1 and n_in > 64:
        pytest.skip("v2 covers n_in <= 64")
    lib = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(groups * 7 + n_in)
    q_rows = 4 * n_in if 4 * n_in <= 128 else 128
    q, ki, vi = _r(g, groups, q_rows, 128), _r(g, groups, n_in, 128), _r(g, groups, n_in, 128)
    ob = torch.randn((groups, q_rows, 128), device="cuda", generator=g).to(torch.bfloat16)
    le = torch.randn((groups, q_rows), device="cuda", generator=g)
    le[0, :5] = -math.inf  # rows with an empty external partial
    lib.fb_debug_set_k2_variant(variant)
    try:
        a = K.internal_merge(q, ki, vi, ob.float(), le, out_dtype=torch.bfloat16, ext_stable=True)
        b = K.internal_merge(q, ki, vi, ob, le, out_dtype=torch.bfloat16, ext_stable=True)
        c = K.internal_merge(q, ki, vi, ob, le, out_dtype=torch.float32)
        d32 = K.internal_merge(q, ki, vi, ob.float(), le, out_dtype=torch.float32)
        torch.cuda.synchronize()
    finally:
        lib.fb_debug_set_k2_variant(-1)
    assert torch.equal(a, b)
    assert torch.equal(c, d32)


def test_k2_large_block_bf16_ext():
    """Blocks of > 128 keys (C5 video chunks): K1 over the block's keys with
    the merge against the bf16 cached partial fused into its merge kernel."""
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(11)
    groups, q_rows, n_in = 4, 600, 600
    q, ki, vi = _r(g, groups, q_rows, 128), _r(g, groups, n_in, 128), _r(g, groups, n_in, 128)
    ob = torch.randn((groups, q_rows, 128), device="cuda", generator=g).to(torch.bfloat16)
    le = torch.randn((groups, q_rows), device="cuda", generator=g)
    a = K.internal_merge(q, ki, vi, ob.float(), le, out_dtype=torch.float32)
    b = K.internal_merge(q, ki, vi, ob, le, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_k2_tokmajor_bf16_ext():
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(12)
    b, blk, hq, hkv, d = 2, 32, 32, 8, 128
    qkv = _r(g, b * blk, (hq + 2 * hkv) * d).view(b, blk, hq + 2 * hkv, d)
    q_tok, k_tok, v_tok = qkv[:, :, :hq], qkv[:, :, hq:hq + hkv], qkv[:, :, hq + hkv:]
    ob = torch.randn((b * hkv, (hq // hkv) * blk, d), device="cuda", generator=g).to(torch.bfloat16)
    le = torch.randn((b * hkv, (hq // hkv) * blk), device="cuda", generator=g)
    o1 = torch.empty((b, blk, hq, d), device="cuda", dtype=torch.bfloat16)
    o2 = torch.empty_like(o1)
    K.internal_merge_tok(q_tok, k_tok, v_tok, ob.float(), le, o1, ext_stable=True)
    K.internal_merge_tok(q_tok, k_tok, v_tok, ob, le, o2, ext_stable=True)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)


def test_engine_stores_bf16_external_partial_by_default():
    from paper_2602_05305_b200 import FlashBlockAttention

    e = FlashBlockAttention(2, 1, 8, 2, 32, 128)
    assert e.o_ext.dtype == torch.bfloat16 and e.lse_ext.dtype == torch.float32
    e32 = FlashBlockAttention(2, 1, 8, 2, 32, 128, ext_dtype=torch.float32)
    assert e32.o_ext.dtype == torch.float32
    # half the resident bytes of the fp32 layout for O
    assert e.o_ext[0].numel() * e.o_ext.element_size() * 2 == e32.o_ext[0].numel() * e32.o_ext.element_size()
    g = torch.Generator(device="cuda").manual_seed(13)
    q, kc, vc, ki, vi = _r(g, 1, 8, 32, 128), _r(g, 1, 2, 900, 128), _r(g, 1, 2, 900, 128), \
        _r(g, 1, 2, 32, 128), _r(g, 1, 2, 32, 128)
    for eng in (e, e32):
        eng.begin_block(0)
        eng.refresh(0, q, kc, vc, 900, ki, vi)
    torch.cuda.synchronize()
    assert torch.equal(e.o_ext[0], e32.o_ext[0].to(torch.bfloat16))
    assert torch.equal(e.lse_ext[0], e32.lse_ext[0])


def test_partial_bf16_flag_rejected_outside_bf16_mode():
    from paper_2602_05305_b200 import _lib
    from paper_2602_05305_b200 import kernels as K
    from paper_2602_05305_b200.errors import ShapeError

    lib = _lib.load()
    q = torch.randn((1, 16, 64), device="cuda")
    k = torch.randn((1, 64, 64), device="cuda")
    o = torch.empty((1, 16, 64), device="cuda")
    l = torch.empty((1, 16), device="cuda", dtype=torch.float64)
    rc = lib.fb_attention_partial(_lib.FB_F32 | _lib.FB_PARTIAL_BF16, q.data_ptr(), k.data_ptr(), k.data_ptr(),
                                  1, 16, 64, 64, 0, 64, 0.125, o.data_ptr(), l.data_ptr(), None, 0, None)
    assert rc == 7  # FB_ERR_VALUE
    with pytest.raises(ShapeError):  # the internal partial comes back in the mode's fp32 type only
        qb = q.to(torch.bfloat16)
        K.internal_merge(qb, qb, qb, torch.zeros((1, 16, 64), device="cuda", dtype=torch.bfloat16),
                         torch.zeros((1, 16), device="cuda"), want_internal=True)
