"""Counted cache traffic (the reference's AccessCounters, kv_cache.py:28-52):
refresh steps read the committed rows of every slab, cached steps read none
(the reference's no-KV-touch acceptance criterion, tests/test_acceptance.py:
132-176 there), commits append rows and grow the resident bytes."""

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def test_cached_steps_read_no_cache_rows():
    from paper_2602_05305_b200 import FlashBlockAttention, KVCache

    b, hq, hkv, blk, d, n = 2, 8, 2, 32, 128, 700
    g = torch.Generator(device="cuda").manual_seed(1)
    mk = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
    kc, vc = mk(b, hkv, n + 64, d), mk(b, hkv, n + 64, d)
    q, ki, vi = mk(b, hq, blk, d), mk(b, hkv, blk, d), mk(b, hkv, blk, d)
    eng = FlashBlockAttention(2, b, hq, hkv, blk, d)
    c0 = eng.snapshot_counters()
    eng.refresh(0, q, kc, vc, n, ki, vi)
    c1 = eng.snapshot_counters()
    assert c1.key_rows_read - c0.key_rows_read == b * hkv * n
    assert c1.value_rows_read == c1.key_rows_read
    for _ in range(5):
        eng.cached(0, q, ki, vi)
    assert eng.snapshot_counters() == c1, "a cached step touched the KV cache"
    # ragged lengths are counted on the device
    lens = torch.tensor([300, 650], dtype=torch.int32, device="cuda")
    eng.refresh(1, q, kc, vc, lens, ki, vi)
    assert eng.snapshot_counters().key_rows_read - c1.key_rows_read == hkv * (300 + 650)

    cache = KVCache(1, b, hkv, 256, d)
    cache.commit_block(0, ki, vi)
    cache.commit_block(0, ki, vi)
    cc = cache.snapshot_counters()
    assert cc.rows_appended == 2 * b * hkv * blk
    assert cc.cache_bytes_resident == 2 * b * hkv * blk * 2 * d * 2
