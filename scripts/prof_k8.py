"""C4 cached sparse step (K8) at 64K ctx, b=4, density 0.1 / 0.5: a few
launches for an ncu launch list (per-kernel composition of the step)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K
g = torch.Generator(device="cuda").manual_seed(4)
r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
N, groups, rows, D, B = 65536, 32, 128, 128, 32
q, k, v, ki, vi = r(groups, rows, D), r(groups, N, D), r(groups, N, D), r(groups, B, D), r(groups, B, D)
for dens in (0.1, 0.5):
    budget = K.mask_budget(N, dens, 16)
    sel = K.topk_blocks(K.block_mass(q, k, ki, N, 16), budget)
    res = K.sparse_partitioned(q, k, v, ki, vi, N, sel)[2]
    torch.cuda.synchronize()
    for _ in range(3):
        K.sparse_attend_merge(q, k, v, ki, vi, N, sel, res)
    torch.cuda.synchronize()
print("done")
