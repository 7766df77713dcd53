import ctypes, os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import _lib, kernels as K
L = _lib.load(); L.fb_debug_set_pair.argtypes = [ctypes.c_int]
L.fb_debug_set_pair(1)
def run(G, n_q, blk, n_prefix, groups=2, seed=0):
    rng = np.random.Generator(np.random.Philox(2000 + n_q + G + seed))
    d = 128; cap = n_prefix + n_q + 40
    mk = lambda *s: torch.from_numpy(rng.standard_normal(s).astype(np.float32)).to(torch.bfloat16).cuda()
    q, k, v = mk(groups, G * n_q, d), mk(groups, cap, d), mk(groups, cap, d)
    res = []
    for rep in range(2):
        o = torch.full((groups, G * n_q, d), 7.0, device="cuda"); l = torch.full((groups, G * n_q), 7.0, device="cuda")
        K.block_causal_attention(q, k, v, n_q, n_prefix, blk, None, o, l)
        torch.cuda.synchronize()
        bad = ((~torch.isfinite(l)) | (l == 7.0)).nonzero().tolist()
        res.append((len(bad), bad[:3], bad[-2:]))
    print(G, n_q, blk, n_prefix, res)
run(3, 200, 64, 17)
run(3, 200, 64, 0)
run(3, 200, 32, 0)
run(3, 256, 64, 17)
run(2, 200, 64, 17)
run(1, 300, 64, 17)
run(3, 200, 64, 17, seed=5)
run(3, 200, 128, 17)
run(3, 200, 200, 17)
