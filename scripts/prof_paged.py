"""One paged K1 launch at C2 b=16 (page_rows 256, shuffled pool) for ncu."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K
g = torch.Generator(device="cuda").manual_seed(5)
groups, N, d, P = 128, 32768, 128, 256
r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
q = r(groups, 128, d)
mp = N // P
perm = torch.randperm(groups * mp, generator=torch.Generator().manual_seed(2)).cuda()
table = perm.view(groups, mp).to(torch.int32).contiguous()
kp, vp = r(groups * mp, P, d), r(groups * mp, P, d)
lens = torch.full((groups,), N, dtype=torch.int32, device="cuda")
o, l = K.attention_partial_paged(q, kp, vp, table, lens)
torch.cuda.synchronize()
o, l = K.attention_partial_paged(q, kp, vp, table, lens, None, o, l)
torch.cuda.synchronize()
print("done")
