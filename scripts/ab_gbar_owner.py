"""Interleaved A/B: K1 with the in-kernel owner merge (items over <= 3 CTAs,
stream-K on 148 CTAs) vs grid-barrier split-K (k CTAs per item), graph of L
launches on distinct KV."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_05305_b200 import kernels as K, _lib
lib = _lib.load()
D = 128
for name, groups, n, L in (("C3 b=8 P=8 shard", 64, 16384, 4), ("C2 b=8", 64, 32768, 3), ("C2 b=6", 48, 32768, 3),
                           ("C3 b=8 P=4 shard", 64, 32768, 3)):
    g = torch.Generator(device="cuda").manual_seed(groups + n)
    r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
    q = r(groups, 128, D)
    ks = [r(groups, n, D) for _ in range(L)]
    vs = [r(groups, n, D) for _ in range(L)]
    o = torch.empty((groups, 128, D), device="cuda", dtype=torch.bfloat16)
    l = torch.empty((groups, 128), device="cuda")
    graphs, used = {}, {}
    for mode in (1, 2):
        lib.fb_debug_set_k1_gbar(mode)
        c0 = lib.fb_debug_k1_cluster_launches()
        def fn():
            for i in range(L):
                K.attention_partial(q, ks[i], vs[i], 0, n, out=o, lse=l)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            fn(); torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                fn()
        used[mode] = lib.fb_debug_k1_cluster_launches() - c0 > 0
        graphs[mode] = gr
    lib.fb_debug_set_k1_gbar(-1)
    res = {1: [], 2: []}
    for rnd in range(6):
        for mode in ((1, 2) if rnd % 2 == 0 else (2, 1)):
            graphs[mode].replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); graphs[mode].replay(); e1.record(); torch.cuda.synchronize()
            res[mode].append(e0.elapsed_time(e1) / L * 1000)
    print(json.dumps({"shape": name, "owner_us": round(sorted(res[1])[3], 2), "gbar_us": round(sorted(res[2])[3], 2),
                      "gbar_taken": used[2]}), flush=True)
    del ks, vs, graphs
    torch.cuda.empty_cache()
