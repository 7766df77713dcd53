"""K1 with the in-kernel split merge (default) vs the separate merge kernel
(diag 5), interleaved, graphs of back-to-back launches on distinct KV."""
import ctypes, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K, _lib
lib = _lib.load(); lib.fb_debug_set_k1_diag.argtypes = [ctypes.c_int]
HKV, D, CTX, L = 8, 128, 32768, 8
for b in (16, 8, 1):
    g = torch.Generator(device="cuda").manual_seed(1)
    q = torch.randn((b * HKV, 128, D), device="cuda", generator=g).to(torch.bfloat16)
    ks = [torch.randn((b * HKV, CTX, D), device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
    vs = [torch.randn((b * HKV, CTX, D), device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
    o = torch.empty((b * HKV, 128, D), device="cuda", dtype=torch.float32)
    l = torch.empty((b * HKV, 128), device="cuda", dtype=torch.float32)
    byts = 2 * b * HKV * CTX * D * 2
    res, outs = {}, {}
    graphs = {}
    for diag in (0, 5):
        lib.fb_debug_set_k1_diag(diag)
        fn = lambda: [K.attention_partial(q, ks[i], vs[i], 0, CTX, None, o, l) for i in range(L)]
        s = torch.cuda.Stream(); fn(); torch.cuda.synchronize()
        outs[diag] = (o.clone(), l.clone())
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s): fn()
        graphs[diag] = gr
    lib.fb_debug_set_k1_diag(0)
    for rnd in range(4):
        for diag in ((0, 5) if rnd % 2 == 0 else (5, 0)):
            graphs[diag].replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3): graphs[diag].replay()
            e1.record(); torch.cuda.synchronize()
            res.setdefault(diag, []).append(e0.elapsed_time(e1) / (3 * L))
    d_o = float((outs[0][0] - outs[5][0]).abs().max()); d_l = float((outs[0][1] - outs[5][1]).abs().max())
    for diag, name in ((0, "fused"), (5, "merge-kernel")):
        t = sorted(res[diag])[len(res[diag]) // 2]
        print(f"b={b} {name:12s} {t*1000:.1f} us/launch {byts/t/1e6:.0f} GB/s   (max|dO|={d_o:.2e} max|dLSE|={d_l:.2e})", flush=True)
    del ks, vs; torch.cuda.empty_cache()
