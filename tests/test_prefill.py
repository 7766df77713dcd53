"""Prefill / commit attention: block-causal attention of a
prompt's positions over the committed prefix plus every block up to their own.

Oracle pin (CPU): oracle.block_causal against the reference's own commit
passes, recorded from simulator.prefill / commit_context_block
(tests/golden/make_golden.py prefill -> golden_prefill.npz).
GPU parity (-m gpu): fb_block_causal_attention against the same fixtures
(F64: 1e-12 abs; F32: scores in float64 like attention_dense, 1e-6 rel) and,
for the bf16 tensor-core kernel, against the oracle on bf16-exact inputs
(max|diff| <= 1e-2 * max|ref|, lse within 1e-3).
"""

import os

import numpy as np
import pytest

from oracle import flashblock_oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def gp():
    with np.load(os.path.join(ROOT, "tests", "golden", "golden_prefill.npz")) as z:
        return {k: z[k] for k in z.files}


def _cases(gp):
    for name in ("pf0", "pf1"):
        L, H, d, n_q, blk, extra = (int(x) for x in gp[f"{name}_meta"])
        yield name, L, H, d, n_q, blk, extra


def test_oracle_block_causal_matches_reference_commit_passes(gp):
    for name, L, H, d, n_q, blk, extra in _cases(gp):
        for layer in range(L):
            for head in range(H):
                pre = f"{name}_l{layer}_h{head}"
                got = orc.block_causal(gp[pre + "_q"], gp[pre + "_k"], gp[pre + "_v"], 0, n_q, blk)
                np.testing.assert_allclose(got, gp[pre + "_out"], rtol=0, atol=1e-12)
                if extra:
                    x = f"{name}_x_l{layer}_h{head}"
                    n_pre = gp[x + "_k"].shape[0] - gp[x + "_q"].shape[0]
                    got = orc.block_causal(gp[x + "_q"], gp[x + "_k"], gp[x + "_v"], n_pre,
                                           gp[x + "_q"].shape[0], blk)
                    np.testing.assert_allclose(got, gp[x + "_out"], rtol=0, atol=1e-12)


def test_oracle_block_causal_stacked_heads_equal_per_head():
    rng = np.random.Generator(np.random.Philox(7))
    q = rng.standard_normal((3 * 40, 8))
    k = rng.standard_normal((50, 8))
    v = rng.standard_normal((50, 8))
    both = orc.block_causal(q, k, v, 10, 40, 16)
    for h in range(3):
        np.testing.assert_array_equal(both[h * 40:(h + 1) * 40],
                                      orc.block_causal(q[h * 40:(h + 1) * 40], k, v, 10, 40, 16))


# ---------------------------------------------------------------- GPU


def _torch():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return torch


def _rel(got, ref):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    return float(np.max(np.abs(got - ref))) / max(1e-30, float(np.max(np.abs(ref))))


@pytest.mark.gpu
def test_gpu_block_causal_matches_reference_golden(gp):
    torch = _torch()
    from paper_2602_05305_b200 import kernels as K

    for name, L, H, d, n_q, blk, extra in _cases(gp):
        for layer in range(L):
            # the reference is 1:1 q/kv heads: one group per head, q_rows = n_q
            qs = np.stack([gp[f"{name}_l{layer}_h{h}_q"] for h in range(H)])
            ks = np.stack([gp[f"{name}_l{layer}_h{h}_k"] for h in range(H)])
            vs = np.stack([gp[f"{name}_l{layer}_h{h}_v"] for h in range(H)])
            ref = np.stack([gp[f"{name}_l{layer}_h{h}_out"] for h in range(H)])
            cap = ks.shape[1] + 7  # slab larger than the prompt
            kc = np.zeros((H, cap, d), ks.dtype)
            vc = np.zeros((H, cap, d), vs.dtype)
            kc[:, :ks.shape[1]], vc[:, :vs.shape[1]] = ks, vs
            o, l = K.block_causal_attention(torch.from_numpy(qs).cuda(), torch.from_numpy(kc).cuda(),
                                            torch.from_numpy(vc).cuda(), n_q, 0, blk)
            o = o.cpu().numpy()
            if qs.dtype == np.float64:
                np.testing.assert_allclose(o, ref, rtol=0, atol=1e-12)
            else:
                assert _rel(o, ref) <= 1e-6, f"{name} layer {layer}: {_rel(o, ref):.2e}"
            if extra:
                xq = np.stack([gp[f"{name}_x_l{layer}_h{h}_q"] for h in range(H)])
                xk = np.stack([gp[f"{name}_x_l{layer}_h{h}_k"] for h in range(H)])
                xv = np.stack([gp[f"{name}_x_l{layer}_h{h}_v"] for h in range(H)])
                xr = np.stack([gp[f"{name}_x_l{layer}_h{h}_out"] for h in range(H)])
                n_pre = xk.shape[1] - xq.shape[1]
                o, _ = K.block_causal_attention(torch.from_numpy(xq).cuda(), torch.from_numpy(xk).cuda(),
                                                torch.from_numpy(xv).cuda(), xq.shape[1], n_pre, blk)
                np.testing.assert_allclose(o.cpu().numpy(), xr, rtol=0, atol=1e-12)


def _bf16(rng, shape, torch, sigma=1.0):
    return torch.from_numpy((rng.standard_normal(shape) * sigma).astype(np.float32)).to(torch.bfloat16)


@pytest.mark.gpu
@pytest.mark.parametrize("d,G,n_q,blk,n_prefix", [
    (128, 4, 512, 32, 0),      # C2-like GQA stacking, tiles inside one head
    (128, 4, 384, 32, 1000),   # committed prefix + prompt
    (64, 2, 200, 32, 17),      # 128-row tiles straddle heads, ragged last block
    (128, 1, 130, 16, 0),      # last tile of 2 rows
    (64, 3, 96, 100, 5),       # block larger than the prompt: one bidirectional block
])
def test_gpu_block_causal_bf16_vs_oracle(d, G, n_q, blk, n_prefix):
    torch = _torch()
    from paper_2602_05305_b200 import kernels as K

    rng = np.random.Generator(np.random.Philox(1000 + d + n_q))
    groups = 2
    cap = n_prefix + n_q + 40
    q = _bf16(rng, (groups, G * n_q, d), torch)
    k = _bf16(rng, (groups, cap, d), torch)
    v = _bf16(rng, (groups, cap, d), torch)
    k[:, n_prefix + n_q:] = float("nan")  # rows past the prompt must never be read
    v[:, n_prefix + n_q:] = float("nan")
    o, l = K.block_causal_attention(q.cuda(), k.cuda(), v.cuda(), n_q, n_prefix, blk)
    o, l = o.cpu().numpy(), l.cpu().numpy()
    assert np.isfinite(o).all() and np.isfinite(l).all()
    for g in range(groups):
        kk = k[g, :n_prefix + n_q].double().numpy()
        vv = v[g, :n_prefix + n_q].double().numpy()
        ref = orc.block_causal(q[g].double().numpy(), kk, vv, n_prefix, n_q, blk)
        err = _rel(o[g], ref)
        assert err <= 1e-2, f"g={g} rel err {err:.3e}"


@pytest.mark.gpu
def test_gpu_block_causal_f32_and_f64_modes_vs_oracle():
    torch = _torch()
    from paper_2602_05305_b200 import kernels as K

    rng = np.random.Generator(np.random.Philox(5))
    for dt in (torch.float64, torch.float32):
        q = torch.from_numpy(rng.standard_normal((2, 2 * 70, 48))).to(dt)
        k = torch.from_numpy(rng.standard_normal((2, 90, 48))).to(dt)
        v = torch.from_numpy(rng.standard_normal((2, 90, 48))).to(dt)
        o, l = K.block_causal_attention(q.cuda(), k.cuda(), v.cuda(), 70, 20, 32)
        for g in range(2):
            ref = orc.block_causal(q[g].double().numpy(), k[g].double().numpy(), v[g].double().numpy(),
                                   20, 70, 32)
            tol = 1e-12 if dt == torch.float64 else 1e-6
            assert _rel(o[g].cpu().numpy(), ref) <= tol


@pytest.mark.gpu
def test_gpu_engine_prefill_c2_shapes_properties():
    """C2 shapes (32 q / 8 kv heads, d 128, block 32), 4K-position prompt:
    the last block's rows attend every key, so they equal the refresh kernel
    (K1) over the whole prompt; the first block's rows equal the oracle over
    32 keys; a middle block is checked against the oracle for one group."""
    torch = _torch()
    from paper_2602_05305_b200 import FlashBlockAttention
    from paper_2602_05305_b200 import kernels as K

    b, hq, hkv, d, blk, n_q = 1, 32, 8, 128, 32, 4096
    G = hq // hkv
    gen = torch.Generator(device="cuda").manual_seed(3)
    q = torch.randn((b, hq, n_q, d), device="cuda", generator=gen).to(torch.bfloat16)
    kc = torch.randn((b, hkv, n_q, d), device="cuda", generator=gen).to(torch.bfloat16)
    vc = torch.randn((b, hkv, n_q, d), device="cuda", generator=gen).to(torch.bfloat16)
    eng = FlashBlockAttention(1, b, hq, hkv, blk, d)
    out = eng.prefill(q, kc, vc, 0)
    assert out.shape == (b, hq, n_q, d) and torch.isfinite(out).all()
    # last block vs K1 over all keys (stacked last-block rows of the group's heads)
    ql = q[0, :, -blk:].reshape(hkv, G * blk, d)
    o1, _ = K.attention_partial(ql, kc[0], vc[0])
    last = out[0, :, -blk:].reshape(hkv, G * blk, d)
    assert float((last - o1).abs().max()) <= 2e-3 * float(o1.abs().max())
    g = 5
    qg = q[0, g * G:(g + 1) * G].double().cpu().numpy()
    kk, vv = kc[0, g].double().cpu().numpy(), vc[0, g].double().cpu().numpy()
    for j in (0, 37):
        rows = qg[:, j * blk:(j + 1) * blk].reshape(G * blk, d)
        ref = orc.dense(rows, kk[:(j + 1) * blk], vv[:(j + 1) * blk])
        got = out[0, g * G:(g + 1) * G, j * blk:(j + 1) * blk].reshape(G * blk, d).double().cpu().numpy()
        assert _rel(got, ref) <= 1e-2
