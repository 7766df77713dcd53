"""K5 block-mass scoring (LSE + MASS K-only passes) at C4 (64K ctx, b=4:
32 groups x 128 rows): per-process timing, FB_K5_POLY read once."""
import json, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K
g = torch.Generator(device="cuda").manual_seed(4)
r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
N = 65536
L = 3
qs = [r(32, 128, 128) for _ in range(L)]
ks = [r(32, N, 128) for _ in range(L)]
kis = [r(32, 32, 128) for _ in range(L)]
ref = [K.block_mass(qs[i], ks[i], kis[i], N, 16) for i in range(L)]
s = torch.cuda.Stream()
fn = lambda: [K.block_mass(qs[i], ks[i], kis[i], N, 16) for i in range(L)]
with torch.cuda.stream(s):
    fn()
torch.cuda.synchronize()
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr, stream=s):
    fn()
gr.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    gr.replay()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3 / L
sel = [K.topk_blocks(ref[i], K.mask_budget(N, 0.1, 16)) for i in range(L)]
print(json.dumps({"poly": os.environ.get("FB_K5_POLY", "0"), "mask_mass_ms": ms,
                  "gbs_two_passes": 2 * 32 * N * 128 * 2 / (ms * 1e-3) / 1e9,
                  "sel_checksum": int(sum(int(x.sum()) for x in sel))}), flush=True)
