"""K1 per-launch time vs forced CTA count (FB_REFRESH_CTAS is read per launch)
for small batches at 32K context; graph of back-to-back launches."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K
HKV, D, CTX, L = 8, 128, 32768, 6
for b in [int(x) for x in sys.argv[1:]] or (1, 2, 4):
    g = torch.Generator(device="cuda").manual_seed(1)
    q = torch.randn((b * HKV, 128, D), device="cuda", generator=g).to(torch.bfloat16)
    ks = [torch.randn((b * HKV, CTX, D), device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
    vs = [torch.randn((b * HKV, CTX, D), device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
    o = torch.empty((b * HKV, 128, D), device="cuda", dtype=torch.float32)
    l = torch.empty((b * HKV, 128), device="cuda", dtype=torch.float32)
    byts = 2 * b * HKV * CTX * D * 2
    line = []
    for ctas in [int(x) for x in os.environ.get("CTAS_LIST", "148,128,96,74,64,48,32").split(",")]:
        os.environ["FB_REFRESH_CTAS"] = str(ctas)
        fn = lambda: [K.attention_partial(q, ks[i], vs[i], 0, CTX, None, o, l) for i in range(L)]
        s = torch.cuda.Stream(); fn(); torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s): fn()
        gr.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): gr.replay()
        e1.record(); torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / (5 * L)
        line.append(f"{ctas}:{t*1000:.0f}us/{byts/t/1e6:.0f}GB/s")
    print(f"b={b} " + "  ".join(line), flush=True)
    del ks, vs; torch.cuda.empty_cache()
