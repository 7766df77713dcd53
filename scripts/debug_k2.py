import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
groups, rows, d, n = 4, 128, 128, 1000
q, kc, vc = mk(groups, rows, d), mk(groups, n + 24, d), mk(groups, n + 24, d)
o, l = K.attention_partial(q, kc, vc, 0, n); torch.cuda.synchronize(); print("K1 ok", flush=True)
for nin in (32, 16, 64, 128, 8):
    ki, vi = mk(groups, nin, d), mk(groups, nin, d)
    out = K.internal_merge(q, ki, vi, o, l, out_dtype=torch.float32)
    torch.cuda.synchronize(); print("K2 ok", nin, flush=True)
