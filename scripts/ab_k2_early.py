"""K2 v2 at C2 shapes: O_ext loaded before the PDL wait (FB_EXT_STABLE) vs after,
interleaved -- how much of the cached partial's load the early prefetch hides."""
import ctypes as C, math, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import _lib
lib = _lib.load()
f = lib.fb_internal_merge_ex
HQ, HKV, D, BLK, L = 32, 8, 128, 32, 36
for b in [int(x) for x in sys.argv[1:]] or [32, 16]:
    groups, rows = b * HKV, 4 * BLK
    g = torch.Generator(device="cuda").manual_seed(2)
    r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
    qs = [r(groups, rows, D) for _ in range(L)]; ks = [r(groups, BLK, D) for _ in range(L)]; vs = [r(groups, BLK, D) for _ in range(L)]
    oe = [r(groups, rows, D) for _ in range(L)]; le = [torch.randn((groups, rows), device="cuda", generator=g) for _ in range(L)]
    out = [torch.empty((groups, rows, D), device="cuda", dtype=torch.bfloat16) for _ in range(L)]
    graphs = {}
    for early in (1, 0):
        def fn(early=early):
            for _ in range(31):
                for i in range(L):
                    rc = f(2 | 0x100, qs[i].data_ptr(), ks[i].data_ptr(), vs[i].data_ptr(), groups, rows, D, BLK,
                           1 / math.sqrt(D), oe[i].data_ptr(), le[i].data_ptr(), out[i].data_ptr(), 2,
                           None, None, None, None, None, 0, early, torch.cuda.current_stream().cuda_stream)
                    assert rc == 0
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            fn(); torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                fn()
        graphs[early] = gr
    res = {1: [], 0: []}
    for rnd in range(6):
        for e in ((1, 0) if rnd % 2 == 0 else (0, 1)):
            graphs[e].replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); graphs[e].replay(); e1.record(); torch.cuda.synchronize()
            res[e].append(e0.elapsed_time(e1) / (31 * L) * 1000)
    print(f"b={b}: early {sorted(res[1])[3]:.2f} us, after the wait {sorted(res[0])[3]:.2f} us")
