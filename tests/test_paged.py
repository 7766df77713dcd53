"""Paged KV cache (serving layout): K1 reading keys through
per-slab page tables (fb_attention_partial_paged) and the paged block commit
(fb_commit_block_paged).

Parity: the same rows laid out in contiguous slabs and run through the ragged
K1 path give the SAME outputs bit for bit (identical tiles in identical order);
the ragged path itself is checked against the oracle in test_gpu_attention.
The PagedKVCache built by block commits agrees with the contiguous KVCache."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import flashblock_oracle as orc  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.mark.parametrize("page_rows,d", [(128, 128), (256, 128), (512, 64)])
def test_paged_equals_ragged_contiguous_bitwise(page_rows, d):
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(page_rows + d)
    groups, q_rows, cap = 6, 128, 2600
    lens = torch.tensor([2600, 0, 1, 127, 1000, 2049], dtype=torch.int32, device="cuda")
    q = torch.randn((groups, q_rows, d), device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn((groups, cap, d), device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn((groups, cap, d), device="cuda", generator=g).to(torch.bfloat16)
    max_pages = -(-cap // page_rows)
    num_pages = groups * max_pages + 3
    perm = torch.randperm(num_pages, generator=torch.Generator().manual_seed(1)).tolist()
    kp = torch.full((num_pages, page_rows, d), float("nan"), device="cuda").to(torch.bfloat16)
    vp = torch.full((num_pages, page_rows, d), float("nan"), device="cuda").to(torch.bfloat16)
    table = torch.full((groups, max_pages), -1, dtype=torch.int32)
    for gi in range(groups):
        for pi in range(-(-int(lens[gi]) // page_rows)):
            page = perm.pop()
            table[gi, pi] = page
            r0, r1 = pi * page_rows, min((pi + 1) * page_rows, int(lens[gi]))
            kp[page, :r1 - r0] = k[gi, r0:r1]
            vp[page, :r1 - r0] = v[gi, r0:r1]
    o_p, l_p = K.attention_partial_paged(q, kp, vp, table.cuda(), lens)
    o_r, l_r = K.attention_partial_ragged(q, k, v, lens)
    assert torch.equal(o_p, o_r) and torch.equal(l_p, l_r)
    assert torch.isneginf(l_p[1]).all() and (o_p[1] == 0).all()  # empty slab: the sentinel
    ref = orc.partial(q[4].double().cpu().numpy(), k[4, :1000].double().cpu().numpy(),
                      v[4, :1000].double().cpu().numpy())
    err = float(np.max(np.abs(o_p[4].double().cpu().numpy() - ref.out))) / float(np.max(np.abs(ref.out)))
    assert err <= 1e-2


def test_paged_cache_commits_match_contiguous_cache():
    from paper_2602_05305_b200 import KVCache, PagedKVCache
    from paper_2602_05305_b200.errors import BoundsError

    g = torch.Generator(device="cuda").manual_seed(9)
    b, hq, hkv, blk, d = 2, 8, 2, 32, 128
    paged = PagedKVCache(1, b, hkv, num_pages=40, page_rows=128, head_dim=d, max_pages_per_slab=16)
    flat = KVCache(1, b, hkv, capacity=16 * 128, head_dim=d)
    for step in range(21):  # 672 rows: 6 pages per slab, the last partly filled
        kb = torch.randn((b, hkv, blk, d), device="cuda", generator=g).to(torch.bfloat16)
        vb = torch.randn((b, hkv, blk, d), device="cuda", generator=g).to(torch.bfloat16)
        paged.commit_block(0, kb, vb)
        flat.commit_block(0, kb, vb)
    assert torch.equal(paged.lengths[0], flat.lengths[0])
    assert paged.free_pages() == 40 - b * hkv * 6
    q = torch.randn((b, hq, blk, d), device="cuda", generator=g).to(torch.bfloat16)
    from paper_2602_05305_b200 import kernels as K
    o_p, l_p = paged.attention_partial(0, q)
    o_f, l_f = K.attention_partial_ragged(K.gqa_view(q, hkv), flat.k[0].view(b * hkv, -1, d),
                                          flat.v[0].view(b * hkv, -1, d), flat.lengths[0])
    assert torch.equal(o_p, o_f) and torch.equal(l_p, l_f)
    paged.release(0)
    assert paged.free_pages() == 40 - hkv * 6
    assert int(paged.lengths[0][:hkv].sum()) == 0
    tiny = PagedKVCache(1, 1, 1, num_pages=1, page_rows=128, head_dim=d, max_pages_per_slab=4)
    kb = torch.zeros((1, 1, 129, d), device="cuda", dtype=torch.bfloat16)
    with pytest.raises(BoundsError):
        tiny.commit_block(0, kb, kb)  # needs 2 pages, the pool has 1


def test_engine_refresh_on_paged_cache_equals_contiguous():
    """FlashBlockAttention.refresh with a PagedKVCache (K1 through the page
    tables, then K2) gives the same step output and cached partial as with the
    contiguous KVCache and its ragged lengths; the cached step then agrees."""
    from paper_2602_05305_b200 import FlashBlockAttention, KVCache, PagedKVCache

    g = torch.Generator(device="cuda").manual_seed(11)
    b, hq, hkv, blk, d = 2, 8, 2, 32, 128
    paged = PagedKVCache(1, b, hkv, num_pages=64, page_rows=256, head_dim=d, max_pages_per_slab=16)
    flat = KVCache(1, b, hkv, capacity=16 * 256, head_dim=d)
    r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
    for _ in range(40):
        kb, vb = r(b, hkv, blk, d), r(b, hkv, blk, d)
        paged.commit_block(0, kb, vb)
        flat.commit_block(0, kb, vb)
    q, ki, vi = r(b, hq, blk, d), r(b, hkv, blk, d), r(b, hkv, blk, d)
    e1 = FlashBlockAttention(1, b, hq, hkv, blk, d, out_dtype=torch.float32)
    e2 = FlashBlockAttention(1, b, hq, hkv, blk, d, out_dtype=torch.float32)
    out_p = e1.refresh(0, q, paged, None, None, ki, vi)
    out_f = e2.refresh(0, q, flat.k[0], flat.v[0], flat.lengths[0], ki, vi)
    assert torch.equal(out_p, out_f)
    assert torch.equal(e1.o_ext[0], e2.o_ext[0]) and torch.equal(e1.lse_ext[0], e2.lse_ext[0])
    q2 = r(b, hq, blk, d)
    assert torch.equal(e1.cached(0, q2, ki, vi), e2.cached(0, q2, ki, vi))


@pytest.mark.parametrize("pair", [1, 0])
def test_paged_prefill_equals_contiguous_bitwise(pair):
    """Block-causal prefill reading the prompt through page tables (CTA-pair
    kernel by default, single-CTA forced) equals the contiguous-slab prefill
    bit for bit; engine.prefill_paged after committing the prompt into a
    PagedKVCache equals engine.prefill on the contiguous cache."""
    import ctypes

    from paper_2602_05305_b200 import FlashBlockAttention, KVCache, PagedKVCache, _lib

    lib = _lib.load()
    lib.fb_debug_set_pair.argtypes = [ctypes.c_int]
    g = torch.Generator(device="cuda").manual_seed(21 + pair)
    b, hq, hkv, blk, d, n_q = 2, 8, 2, 32, 128, 640
    r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
    paged = PagedKVCache(1, b, hkv, num_pages=32, page_rows=128, head_dim=d, max_pages_per_slab=8)
    flat = KVCache(1, b, hkv, capacity=8 * 128, head_dim=d)
    kp, vp = r(b, hkv, n_q, d), r(b, hkv, n_q, d)
    for c0 in range(0, n_q, 128):  # commit the prompt block by block (pages from the free list)
        paged.commit_block(0, kp[:, :, c0:c0 + 128], vp[:, :, c0:c0 + 128])
        flat.commit_block(0, kp[:, :, c0:c0 + 128], vp[:, :, c0:c0 + 128])
    q = r(b, hq, n_q, d)
    eng = FlashBlockAttention(1, b, hq, hkv, blk, d)
    lib.fb_debug_set_pair(pair)
    try:
        o_p = eng.prefill_paged(q, paged, 0)
        o_f = eng.prefill(q, flat.k[0], flat.v[0])
    finally:
        lib.fb_debug_set_pair(-1)
    assert torch.isfinite(o_p).all()
    assert torch.equal(o_p, o_f)


def test_paged_api_errors():
    """The paged entry points refuse what they do not support, with the
    reference's exception types: non-bf16 inputs (ShapeError from the
    wrapper), page_rows not a multiple of 128 (UnsupportedError), and a commit
    past the pages (BoundsError with check=True)."""
    from paper_2602_05305_b200 import kernels as K
    from paper_2602_05305_b200.errors import BoundsError, ShapeError

    d = 128
    q = torch.zeros((2, 128, d), device="cuda", dtype=torch.bfloat16)
    pool = torch.zeros((4, 128, d), device="cuda", dtype=torch.bfloat16)
    table = torch.tensor([[0, 1], [2, 3]], dtype=torch.int32, device="cuda")
    lens = torch.tensor([200, 0], dtype=torch.int32, device="cuda")
    with pytest.raises(ShapeError):
        K.attention_partial_paged(q.float(), pool, pool, table, lens)
    bad = torch.zeros((4, 96, d), device="cuda", dtype=torch.bfloat16)
    with pytest.raises(Exception) as ei:
        K.attention_partial_paged(q, bad, bad, table, lens)
    assert "128" in str(ei.value)
    o, l = K.attention_partial_paged(q, pool, pool, table, lens)
    assert torch.isneginf(l[1]).all() and (o[1] == 0).all()  # empty slab: the sentinel
    lengths = torch.tensor([250, 0], dtype=torch.int32, device="cuda")
    blk = torch.ones((2, 32, d), device="cuda", dtype=torch.bfloat16)
    with pytest.raises(BoundsError):
        K.commit_block_paged(pool, pool, table, blk, blk, lengths, check=True)  # 250 + 32 > 2 pages


@pytest.mark.parametrize("n_ext,page_rows", [(4101, 256), (2048, 128)])
def test_paged_sparse_path_equals_contiguous_bitwise(n_ext, page_rows):
    """The sparse path over a paged cache -- K5 block masses, K6 selection, K7
    first step (selected + residual) and K8 cached step -- equals the same
    calls on contiguous slabs bit for bit (pages shuffled over the pool)."""
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(n_ext)
    groups, rows, d, n_in = 4, 128, 128, 32
    r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
    q, ki, vi = r(groups, rows, d), r(groups, n_in, d), r(groups, n_in, d)
    cap = -(-n_ext // page_rows) * page_rows
    k, v = r(groups, cap, d), r(groups, cap, d)
    mp = cap // page_rows
    perm = torch.randperm(groups * mp, generator=torch.Generator().manual_seed(3)).cuda()
    table = perm.view(groups, mp).to(torch.int32).contiguous()
    kp = torch.empty((groups * mp, page_rows, d), device="cuda", dtype=torch.bfloat16)
    vp = torch.empty_like(kp)
    kp[perm] = k.view(groups * mp, page_rows, d)
    vp[perm] = v.view(groups * mp, page_rows, d)
    m_c = K.block_mass(q, k, ki, n_ext, 16)
    m_p = K.block_mass(q, kp, ki, n_ext, 16, page_table=table)
    assert torch.equal(m_c, m_p)
    sel = K.topk_blocks(m_c, K.mask_budget(n_ext, 0.2, 16))
    out_c, sel_c, res_c = K.sparse_partitioned(q, k, v, ki, vi, n_ext, sel, out_dtype=torch.float32)
    out_p, sel_p, res_p = K.sparse_partitioned(q, kp, vp, ki, vi, n_ext, sel, out_dtype=torch.float32,
                                               page_table=table)
    assert torch.equal(out_c, out_p)
    assert torch.equal(res_c[0], res_p[0]) and torch.equal(res_c[1], res_p[1])
    q2 = r(groups, rows, d)
    a = K.sparse_attend_merge(q2, k, v, ki, vi, n_ext, sel, res_c, out_dtype=torch.float32)
    b = K.sparse_attend_merge(q2, kp, vp, ki, vi, n_ext, sel, res_p, out_dtype=torch.float32,
                              page_table=table)
    assert torch.equal(a, b)


def test_engine_sparse_steps_contiguous_and_paged():
    """FlashBlockAttention.sparse_first_step / sparse_cached_step (K5+K6+K7,
    then K8 with the stored residual) give the same bits on a contiguous
    KVCache and on a PagedKVCache holding the same rows; at full density the
    first step equals the dense refresh (exact partition); a new block without
    a first step raises StalenessError (sparse.py:177-181)."""
    from paper_2602_05305_b200 import FlashBlockAttention, KVCache, PagedKVCache
    from paper_2602_05305_b200.errors import StalenessError

    g = torch.Generator(device="cuda").manual_seed(31)
    b, hq, hkv, blk, d, n_ext = 2, 8, 2, 32, 128, 1536
    r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
    paged = PagedKVCache(1, b, hkv, num_pages=32, page_rows=256, head_dim=d, max_pages_per_slab=8)
    flat = KVCache(1, b, hkv, capacity=8 * 256, head_dim=d)
    for _ in range(n_ext // 256):
        kb, vb = r(b, hkv, 256, d), r(b, hkv, 256, d)
        paged.commit_block(0, kb, vb)
        flat.commit_block(0, kb, vb)
    q, ki, vi = r(b, hq, blk, d), r(b, hkv, blk, d), r(b, hkv, blk, d)
    e1 = FlashBlockAttention(1, b, hq, hkv, blk, d, out_dtype=torch.float32)
    e2 = FlashBlockAttention(1, b, hq, hkv, blk, d, out_dtype=torch.float32)
    o1 = e1.sparse_first_step(0, q, flat.k[0], flat.v[0], n_ext, ki, vi, density=0.25)
    o2 = e2.sparse_first_step(0, q, paged, None, n_ext, ki, vi, density=0.25)
    assert torch.equal(o1, o2)
    q2 = r(b, hq, blk, d)
    c1 = e1.sparse_cached_step(0, q2, flat.k[0], flat.v[0], ki, vi)
    c2 = e2.sparse_cached_step(0, q2, paged, None, ki, vi)
    assert torch.equal(c1, c2)
    dense = e1.refresh(0, q, flat.k[0], flat.v[0], n_ext, ki, vi)
    full = e2.sparse_first_step(0, q, paged, None, n_ext, ki, vi, density=1.0)
    assert ((full - dense).abs().max() / dense.abs().max()).item() <= 5e-3
    e1.begin_block(1)
    with pytest.raises(StalenessError):
        e1.sparse_cached_step(0, q2, flat.k[0], flat.v[0], ki, vi)
