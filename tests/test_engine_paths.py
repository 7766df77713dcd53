"""Engine branches the round-1 review found broken or untested:

* full_recompute on a PagedKVCache (needs layer=, must leave the layer's
  cached external partial and valid flag alone);
* step_gated on a PagedKVCache with a partial head subset (returns
  (out, decisions), refreshes only the gated groups -- the reference's
  per-(layer, head) decisions, policy.py:71-94, simulator.py:399-405);
* the sparse cached step's row counter with a clipped tail block
  (read_selected_rows counts exactly the selected rows, sparse.py:186-212);
* KVCache.commit_block refusing to overflow before the launch;
* K1 scratch per stream: two refreshes in flight on two streams agree with
  the serial results.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import flashblock_oracle as orc  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _rel(a, b):
    return ((a.double() - b.double()).abs().amax() / b.double().abs().amax()).item()


def _paged_and_flat(b, hkv, blk, d, nblocks, seed):
    from paper_2602_05305_b200 import KVCache, PagedKVCache

    g = torch.Generator(device="cuda").manual_seed(seed)
    paged = PagedKVCache(1, b, hkv, num_pages=b * hkv * 8 + 4, page_rows=256, head_dim=d,
                         max_pages_per_slab=8)
    flat = KVCache(1, b, hkv, capacity=8 * 256, head_dim=d)
    for _ in range(nblocks):
        kb = torch.randn((b, hkv, blk, d), device="cuda", generator=g).to(torch.bfloat16)
        vb = torch.randn((b, hkv, blk, d), device="cuda", generator=g).to(torch.bfloat16)
        paged.commit_block(0, kb, vb)
        flat.commit_block(0, kb, vb)
    return paged, flat, g


def test_paged_full_recompute_leaves_the_cached_partial_alone():
    from paper_2602_05305_b200 import FlashBlockAttention

    b, hq, hkv, blk, d = 2, 8, 2, 32, 128
    paged, flat, g = _paged_and_flat(b, hkv, blk, d, 23, 5)
    r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
    q, ki, vi = r(b, hq, blk, d), r(b, hkv, blk, d), r(b, hkv, blk, d)
    eng = FlashBlockAttention(1, b, hq, hkv, blk, d, out_dtype=torch.float32)
    eng.begin_block(0)
    q0 = r(b, hq, blk, d)
    eng.refresh(0, q0, paged, None, None, ki, vi)
    o_before, l_before = eng.o_ext[0].clone(), eng.lse_ext[0].clone()
    with pytest.raises(ValueError):
        eng.full_recompute(q, paged, None, None, ki, vi)
    got = eng.full_recompute(q, paged, None, None, ki, vi, layer=0)
    assert torch.equal(eng.o_ext[0], o_before) and torch.equal(eng.lse_ext[0], l_before)
    assert eng.valid[0]
    n = 23 * blk
    want = eng.full_recompute(q, flat.k[0], flat.v[0], n, ki, vi)
    assert _rel(got, want) <= 5e-3
    # against the oracle for one kv group
    G = hq // hkv
    qs = q[1, G:2 * G].reshape(G * blk, d).double().cpu().numpy()
    kk = np.concatenate([flat.k[0][1, 1, :n].double().cpu().numpy(), ki[1, 1].double().cpu().numpy()])
    vv = np.concatenate([flat.v[0][1, 1, :n].double().cpu().numpy(), vi[1, 1].double().cpu().numpy()])
    ref = orc.dense(qs, kk, vv)
    gg = got[1, G:2 * G].reshape(G * blk, d).double().cpu().numpy()
    assert float(np.max(np.abs(gg - ref))) / float(np.max(np.abs(ref))) <= 1e-2


def test_paged_step_gated_refreshes_only_the_gated_groups():
    from paper_2602_05305_b200 import FlashBlockAttention, ReuseConfig
    from paper_2602_05305_b200.policy import Decision, HeadGate, HeadGateTable

    b, h, blk, d = 2, 4, 32, 128
    paged, flat, g = _paged_and_flat(b, h, blk, d, 19, 6)
    n = 19 * blk
    r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
    q1, q2, ki, vi = r(b, h, blk, d), r(b, h, blk, d), r(b, h, blk, d), r(b, h, blk, d)
    gates = HeadGateTable(0.9, [HeadGate(0, hh, 0.95 if hh in (0, 2) else 0.5, 0.5, hh in (0, 2))
                                for hh in range(h)])
    cfg = ReuseConfig(tau=2, mode="head-gated")
    ep = FlashBlockAttention(1, b, h, h, blk, d, out_dtype=torch.float32, config=cfg)
    ef = FlashBlockAttention(1, b, h, h, blk, d, out_dtype=torch.float32, config=cfg)
    for e in (ep, ef):
        e.begin_block(0)
    res = ep.step_gated(0, q1, paged, None, None, ki, vi, first_visit=True, updated_tokens=0, gates=gates)
    assert isinstance(res, tuple) and all(x is Decision.RECOMPUTE for x in res[1])
    ef.step_gated(0, q1, flat.k[0], flat.v[0], n, ki, vi, first_visit=True, updated_tokens=0, gates=gates)
    o1 = ep.o_ext[0].clone()
    out_p, dec_p = ep.step_gated(0, q2, paged, None, None, ki, vi, first_visit=False, updated_tokens=1,
                                 gates=gates)
    out_f, dec_f = ef.step_gated(0, q2, flat.k[0], flat.v[0], n, ki, vi, first_visit=False,
                                 updated_tokens=1, gates=gates)
    assert [x is Decision.REUSE for x in dec_p] == [True, False, True, False] and dec_p == dec_f
    assert out_p.shape == (b, h, blk, d)
    assert _rel(out_p, out_f) <= 5e-3
    # reused heads (0, 2) kept their step-0 partial bit for bit; refreshed heads (1, 3) moved
    o2 = ep.o_ext[0].view(b, h, blk, d)
    o1 = o1.view(b, h, blk, d)
    assert torch.equal(o2[:, [0, 2]], o1[:, [0, 2]])
    assert not torch.equal(o2[:, [1, 3]], o1[:, [1, 3]])
    for bi in range(b):
        for hh in range(h):
            kk = np.concatenate([flat.k[0][bi, hh, :n].double().cpu().numpy(), ki[bi, hh].double().cpu().numpy()])
            vv = np.concatenate([flat.v[0][bi, hh, :n].double().cpu().numpy(), vi[bi, hh].double().cpu().numpy()])
            qq2 = q2[bi, hh].double().cpu().numpy()
            if dec_p[hh] is Decision.RECOMPUTE:
                ref = orc.dense(qq2, kk, vv)
            else:
                ext = orc.partial(q1[bi, hh].double().cpu().numpy(), kk[:n], vv[:n])
                ref, _ = orc.with_reuse(qq2, ext, True, kk[n:], vv[n:])
            got = out_p[bi, hh].double().cpu().numpy()
            assert float(np.max(np.abs(got - ref))) / float(np.max(np.abs(ref))) <= 1e-2


def test_sparse_cached_step_counts_the_clipped_tail_exactly():
    from paper_2602_05305_b200 import FlashBlockAttention

    b, hq, hkv, blk, d, kbs = 1, 8, 2, 32, 128, 16
    n_ext = 1000  # 62 full blocks + a 8-row tail block
    g = torch.Generator(device="cuda").manual_seed(8)
    r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
    kc, vc = r(b, hkv, 1024, d), r(b, hkv, 1024, d)
    # make the tail block the heaviest so it is selected
    kc[:, :, 992:1000] *= 4
    q, ki, vi = r(b, hq, blk, d), r(b, hkv, blk, d), r(b, hkv, blk, d)
    kc[:, :, 992:1000] = q.view(b, hkv, -1, d)[:, :, :8] * 3
    eng = FlashBlockAttention(1, b, hq, hkv, blk, d, out_dtype=torch.float32)
    eng.begin_block(0)
    eng.sparse_first_step(0, q, kc, vc, n_ext, ki, vi, density=0.25, key_block_size=kbs)
    sel = eng._sparse[0][0]
    assert bool((sel == 62).any(dim=-1).all()), "tail block not selected"
    c0 = eng.snapshot_counters().key_rows_read
    eng.sparse_cached_step(0, q, kc, vc, ki, vi)
    rows = eng.snapshot_counters().key_rows_read - c0
    want = sum(min(kbs, n_ext - int(s) * kbs) for s in sel.flatten().tolist())
    assert rows == want and rows < sel.numel() * kbs


def test_kv_cache_commit_refuses_overflow_before_launch():
    from paper_2602_05305_b200 import KVCache
    from paper_2602_05305_b200.errors import BoundsError

    d = 128
    cache = KVCache(1, 1, 2, 80, d)
    blk = torch.zeros((1, 2, 32, d), dtype=torch.bfloat16, device="cuda")
    cache.commit_block(0, blk, blk)
    cache.commit_block(0, blk, blk)
    with pytest.raises(BoundsError):
        cache.commit_block(0, blk, blk)  # no check=True: caught on the host
    assert torch.equal(cache.lengths[0].cpu(), torch.tensor([64, 64], dtype=torch.int32))
    assert cache.rows_appended == 2 * 2 * 32


def test_k1_on_two_streams_matches_serial():
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(12)
    r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
    groups, rows, d, n = 64, 128, 128, 8192  # C2 b=8-like: split items use the flag merge
    qa, ka, va = r(groups, rows, d), r(groups, n, d), r(groups, n, d)
    qb, kb, vb = r(groups, rows, d), r(groups, n, d), r(groups, n, d)
    want_a = K.attention_partial(qa, ka, va)
    want_b = K.attention_partial(qb, kb, vb)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = {}
    for _ in range(3):
        with torch.cuda.stream(s1):
            outs["a"] = K.attention_partial(qa, ka, va)
        with torch.cuda.stream(s2):
            outs["b"] = K.attention_partial(qb, kb, vb)
        torch.cuda.synchronize()
        assert torch.equal(outs["a"][0], want_a[0]) and torch.equal(outs["a"][1], want_a[1])
        assert torch.equal(outs["b"][0], want_b[0]) and torch.equal(outs["b"][1], want_b[1])
