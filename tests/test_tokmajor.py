"""Token-major cached step (fb_internal_merge_tok): q / k_in / v_in as views
of a fused QKV projection output [b*B, (Hq + 2 Hkv) d], output written
token-major.  Same kernel arithmetic as the stacked layout, so the results
must equal the head-major engine path bit for bit."""

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.mark.parametrize("b,hq,hkv,blk", [(2, 32, 8, 32), (3, 8, 2, 16), (1, 4, 1, 32)])
def test_tokmajor_steps_equal_head_major(b, hq, hkv, blk):
    from paper_2602_05305_b200 import FlashBlockAttention

    d, n = 128, 3000
    g = torch.Generator(device="cuda").manual_seed(b * 100 + hq)
    r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
    qkv = r(b * blk, (hq + 2 * hkv) * d)
    t = qkv.view(b, blk, hq + 2 * hkv, d)
    q_tok, k_tok, v_tok = t[:, :, :hq], t[:, :, hq:hq + hkv], t[:, :, hq + hkv:]
    q_hm, k_hm, v_hm = (x.permute(0, 2, 1, 3).contiguous() for x in (q_tok, k_tok, v_tok))
    kc, vc = r(b, hkv, n, d), r(b, hkv, n, d)
    e1 = FlashBlockAttention(1, b, hq, hkv, blk, d)
    e2 = FlashBlockAttention(1, b, hq, hkv, blk, d)
    out_hm = e1.refresh(0, q_hm, kc, vc, n, k_hm, v_hm)
    out_tok = torch.empty((b * blk, hq * d), device="cuda", dtype=torch.bfloat16)
    e2.refresh_tokmajor(0, q_tok, kc, vc, n, k_tok, v_tok, out_tok.view(b, blk, hq, d))
    assert torch.equal(out_tok.view(b, blk, hq, d).permute(0, 2, 1, 3), out_hm)
    assert torch.equal(e1.o_ext[0], e2.o_ext[0])
    qkv2 = r(b * blk, (hq + 2 * hkv) * d)
    t2 = qkv2.view(b, blk, hq + 2 * hkv, d)
    q2, k2, v2 = t2[:, :, :hq], t2[:, :, hq:hq + hkv], t2[:, :, hq + hkv:]
    c_hm = e1.cached(0, q2.permute(0, 2, 1, 3).contiguous(), k2.permute(0, 2, 1, 3).contiguous(),
                     v2.permute(0, 2, 1, 3).contiguous())
    e2.cached_tokmajor(0, q2, k2, v2, out_tok.view(b, blk, hq, d))
    assert torch.equal(out_tok.view(b, blk, hq, d).permute(0, 2, 1, 3), c_hm)
