"""Interleaved A/B of K1 plans: stream-K (+ merge kernel / owner merge) vs
cluster split-K (DSMEM reduction), graph of L launches on distinct KV.
    python scripts/ab_cluster.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_05305_b200 import kernels as K, _lib
lib = _lib.load()
D = 128
SHAPES = [("C3 b=1 P=8 shard", 8, 16384, 8), ("C3 b=1 P=4 shard", 8, 32768, 6), ("C3 b=1 P=2 shard", 8, 65536, 4),
          ("C3 b=1 P=1", 8, 131072, 2), ("C2 b=1", 8, 32768, 6), ("C2 b=2", 16, 32768, 4), ("C2 b=4", 32, 32768, 3),
          ("C3 b=8 P=8 shard", 64, 16384, 3)]
out = []
for name, groups, n, L in SHAPES:
    g = torch.Generator(device="cuda").manual_seed(groups + n)
    r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
    q = r(groups, 128, D)
    ks = [r(groups, n, D) for _ in range(L)]
    vs = [r(groups, n, D) for _ in range(L)]
    o = torch.empty((groups, 128, D), device="cuda", dtype=torch.bfloat16)
    l = torch.empty((groups, 128), device="cuda")
    graphs = {}
    for mode in (0, 1, -1):
        lib.fb_debug_set_k1_cluster(mode)
        def fn():
            for i in range(L):
                K.attention_partial(q, ks[i], vs[i], 0, n, out=o, lse=l)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            fn(); torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                fn()
        graphs[mode] = gr
    lib.fb_debug_set_k1_cluster(-1)
    res = {0: [], 1: [], -1: []}
    for rnd in range(6):
        for mode in ((0, 1, -1) if rnd % 2 == 0 else (-1, 1, 0)):
            graphs[mode].replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); graphs[mode].replay(); e1.record(); torch.cuda.synchronize()
            res[mode].append(e0.elapsed_time(e1) / L * 1000)
    byts = 2 * groups * n * D * 2
    rec = {"shape": name, "groups": groups, "keys": n}
    for mode, nm in ((0, "streamk"), (1, "cluster_forced"), (-1, "auto")):
        v = sorted(res[mode])[len(res[mode]) // 2]
        rec[nm + "_us"] = round(v, 2)
        rec[nm + "_tbs"] = round(byts / (v * 1e-6) / 1e12, 2)
    print(json.dumps(rec), flush=True)
    del ks, vs, graphs
    torch.cuda.empty_cache()
