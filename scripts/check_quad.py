"""FB_K1_QUAD=1 sanity: the two-query-tile K1 against the F32 SIMT kernel and
the oracle (C5-like rows, key offsets, stream-K splits, block-causal)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K
from oracle import flashblock_oracle as orc
assert os.environ.get("FB_K1_QUAD") == "1"
g = torch.Generator(device="cuda").manual_seed(5)
r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
worst = 0.0
for groups, q_rows, n, kb in ((3, 256, 1000, 0), (2, 300, 777, 5), (12, 4680, 2000, 0), (5, 1024, 8192, 0), (1, 200, 129, 0)):
    q, k, v = r(groups, q_rows, 128), r(groups, n + kb + 3, 128), r(groups, n + kb + 3, 128)
    o, l = K.attention_partial(q, k, v, kb, kb + n)
    o32, l32 = K.attention_partial(q.float(), k.float(), v.float(), kb, kb + n)
    err = ((o - o32).abs().amax() / o32.abs().amax()).item()
    lerr = (l.double() - l32).abs().max().item()
    worst = max(worst, err)
    print("partial", groups, q_rows, n, kb, "rel err %.2e lse %.2e" % (err, lerr), "finite", bool(torch.isfinite(o).all()))
rng = np.random.Generator(np.random.Philox(7))
for G, n_q, blk, n_prefix in ((4, 512, 32, 0), (4, 384, 32, 1000), (3, 200, 64, 17), (3, 600, 64, 17)):
    cap = n_prefix + n_q + 40
    mk = lambda *s: torch.from_numpy(rng.standard_normal(s).astype(np.float32)).to(torch.bfloat16)
    q, k, v = mk(2, G * n_q, 128), mk(2, cap, 128), mk(2, cap, 128)
    o, l = K.block_causal_attention(q.cuda(), k.cuda(), v.cuda(), n_q, n_prefix, blk)
    e = 0.0
    for gi in range(2):
        ref = orc.block_causal(q[gi].double().numpy(), k[gi, :n_prefix + n_q].double().numpy(),
                               v[gi, :n_prefix + n_q].double().numpy(), n_prefix, n_q, blk)
        e = max(e, float(np.max(np.abs(o[gi].double().cpu().numpy() - ref))) / float(np.max(np.abs(ref))))
    worst = max(worst, e)
    print("causal", G, n_q, blk, n_prefix, "rel err %.2e" % e, "finite", bool(torch.isfinite(o).all() and torch.isfinite(l).all()))
print("WORST", worst)
