"""ncu driver for the sparse kernels at the C4 shapes (b=4, 64K, density 0.2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_05305_b200 import kernels as K
HQ, HKV, D, B, N = 32, 8, 128, 32, 65536
b = int(sys.argv[1]) if len(sys.argv) > 1 else 4
dens = float(sys.argv[2]) if len(sys.argv) > 2 else 0.2
g = torch.Generator(device="cuda").manual_seed(4)
rnd = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
groups, rows = b * HKV, (HQ // HKV) * B
q, k, v, ki, vi = rnd(groups, rows, D), rnd(groups, N, D), rnd(groups, N, D), rnd(groups, B, D), rnd(groups, B, D)
budget = K.mask_budget(N, dens, 16)
for _ in range(2):
    sel = K.topk_blocks(K.block_mass(q, k, ki, N, 16), budget)
    out, s_p, r_p = K.sparse_partitioned(q, k, v, ki, vi, N, sel)
    o2 = K.sparse_attend_merge(q, k, v, ki, vi, N, sel, r_p)
torch.cuda.synchronize()
print("ok")
