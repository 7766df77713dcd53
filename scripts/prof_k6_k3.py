"""One K6 top-k (C4: 32 groups x 4096 masses, 10 %) and one K3 combine
(C3 P=8 merge: 8 partials of 32 groups x 128 rows x 128) for ncu --set full."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K
g = torch.Generator(device="cuda").manual_seed(3)
mass = torch.rand((32, 4096), device="cuda", generator=g, dtype=torch.float64) * 1e-3
sel = K.topk_blocks(mass, K.mask_budget(65536, 0.1, 16))
parts = [(torch.randn((32, 128, 128), device="cuda", generator=g), torch.randn((32, 128), device="cuda", generator=g))
         for _ in range(8)]
o, l = K.combine(parts, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
