"""C4 K7 (sparse first step: selected + residual partition) timing at 64K b=4."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_05305_b200 import kernels as K
HQ, HKV, D, B, N, L = 32, 8, 128, 32, 65536, 4
b = 4
groups, rows = b * HKV, (HQ // HKV) * B
g = torch.Generator(device="cuda").manual_seed(4)
r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
q = [r(groups, rows, D) for _ in range(L)]
k = [r(groups, N, D) for _ in range(L)]
v = [r(groups, N, D) for _ in range(L)]
ki = [r(groups, B, D) for _ in range(L)]
vi = [r(groups, B, D) for _ in range(L)]
res = {}
for dens in (0.1, 0.5):
    budget = K.mask_budget(N, dens, 16)
    sel = [K.topk_blocks(K.block_mass(q[l], k[l], ki[l], N, 16), budget) for l in range(L)]
    def fn():
        for l in range(L):
            K.sparse_partitioned(q[l], k[l], v[l], ki[l], vi[l], N, sel[l])
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            fn()
    ts = []
    for _ in range(5):
        gr.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); gr.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / L * 1000)
    res[dens] = round(sorted(ts)[2], 1)
print(json.dumps({"atoms": os.environ.get("FB_GATHER_ATOMS", "1"), "cluster": os.environ.get("FB_K1_CLUSTER", "auto"), "k7_us": res}))
