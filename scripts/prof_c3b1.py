"""C3 b=1 shard shapes (8 kv groups x 128 rows, 131072/P keys) for an ncu launch list."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K
g = torch.Generator(device="cuda").manual_seed(3)
r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
for P in (1, 8):
    n = 131072 // P
    q, k, v = r(8, 128, 128), r(8, n, 128), r(8, n, 128)
    o, l = K.attention_partial(q, k, v)
    torch.cuda.synchronize()
    for _ in range(2):
        K.attention_partial(q, k, v, 0, None, None, o, l)
    torch.cuda.synchronize()
