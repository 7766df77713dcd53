"""C5 large-block cached step (12 heads x 4680 rows, the block's own 4680 keys
+ merge with the cached external partial) -- launches for ncu, then a graph
timing of the same call."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K
H, D, B = 12, 128, 4680
g = torch.Generator(device="cuda").manual_seed(5)
r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
q, ki, vi = r(H, B, D), r(H, B, D), r(H, B, D)
oe = r(H, B, D)
le = torch.randn((H, B), device="cuda", generator=g)
out = torch.empty((H, B, D), device="cuda", dtype=torch.bfloat16)
fn = lambda: K.internal_merge(q, ki, vi, oe, le, out_dtype=torch.bfloat16, out=out, ext_stable=True)
for _ in range(3):
    fn()
torch.cuda.synchronize()
if os.environ.get("TIME", "0") == "1":
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            for _ in range(5):
                fn()
    gr.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); gr.replay(); e1.record(); torch.cuda.synchronize()
    print("cached step ms", e0.elapsed_time(e1) / 5)
