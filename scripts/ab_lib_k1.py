"""K1 at C2 b=32 (graph of 4 launches on distinct KV), best of 5 replays --
run once per library build (FB_LIB_PATH) to A/B two builds of the kernel."""
import json, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K
HKV, D, CTX, b, nd = 8, 128, 32768, 32, 4
groups = b * HKV
gen = torch.Generator(device="cuda").manual_seed(1)
q = torch.randn((groups, 128, D), device="cuda", generator=gen).to(torch.bfloat16)
ks = [torch.randn((groups, CTX, D), device="cuda", generator=gen).to(torch.bfloat16) for _ in range(nd)]
vs = [torch.randn((groups, CTX, D), device="cuda", generator=gen).to(torch.bfloat16) for _ in range(nd)]
o = torch.empty((groups, 128, D), device="cuda", dtype=torch.float32)
l = torch.empty((groups, 128), device="cuda", dtype=torch.float32)
fn = lambda: [K.attention_partial(q, ks[i], vs[i], 0, CTX, None, o, l) for i in range(nd)]
s = torch.cuda.Stream(); fn(); torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s): fn()
best = 1e9
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / nd)
print(json.dumps({"lib": os.path.basename(os.environ.get("FB_LIB_PATH", "libfb200.so")), "k1_us": round(best * 1000, 1),
                  "gbs": round(2 * groups * CTX * D * 2 / (best * 1e-3) / 1e9)}))
