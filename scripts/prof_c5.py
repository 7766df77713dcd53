"""One C5 refresh launch (12 heads x 4680 rows, 56,160 keys) for ncu."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K
g = torch.Generator(device="cuda").manual_seed(1)
r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
q, k, v = r(12, 4680, 128), r(12, 56160, 128), r(12, 56160, 128)
K.attention_partial(q, k, v); torch.cuda.synchronize()
