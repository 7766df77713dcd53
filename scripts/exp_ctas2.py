"""Interleaved K1 timing for forced CTA counts (graphs captured per setting;
FB_REFRESH_CTAS is read at launch/capture time)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K
D, L = 128, 6
for groups, ctx in ((16, 32768), (64, 16384), (64, 32768), (128, 32768)):
    g = torch.Generator(device="cuda").manual_seed(1)
    q = torch.randn((groups, 128, D), device="cuda", generator=g).to(torch.bfloat16)
    ks = [torch.randn((groups, ctx, D), device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
    vs = [torch.randn((groups, ctx, D), device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
    o = torch.empty((groups, 128, D), device="cuda", dtype=torch.float32)
    l = torch.empty((groups, 128), device="cuda", dtype=torch.float32)
    byts = 2 * groups * ctx * D * 2
    graphs = {}
    for ctas in ("auto", "148", "128"):
        if ctas == "auto":
            os.environ.pop("FB_REFRESH_CTAS", None)
        else:
            os.environ["FB_REFRESH_CTAS"] = ctas
        fn = lambda: [K.attention_partial(q, ks[i], vs[i], 0, ctx, None, o, l) for i in range(L)]
        s = torch.cuda.Stream(); fn(); torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s): fn()
        graphs[ctas] = gr
    os.environ.pop("FB_REFRESH_CTAS", None)
    res = {}
    for rnd in range(6):
        order = list(graphs) if rnd % 2 == 0 else list(graphs)[::-1]
        for name in order:
            graphs[name].replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3): graphs[name].replay()
            e1.record(); torch.cuda.synchronize()
            res.setdefault(name, []).append(e0.elapsed_time(e1) / (3 * L))
    print(f"groups={groups} ctx={ctx}: " + "  ".join(
        f"{n}:{sorted(v)[len(v)//2]*1000:.1f}us/{byts/sorted(v)[len(v)//2]/1e6:.0f}GB/s" for n, v in res.items()), flush=True)
    del ks, vs; torch.cuda.empty_cache()
