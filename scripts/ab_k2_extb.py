"""Interleaved A/B of the cached step (K2) with the cached external partial's O
in fp32 (A) vs bf16 (B, FB_PARTIAL_BF16): graph of 36 layers x 31 cached steps
at the C2 shapes.   python scripts/ab_k2_extb.py [batch ...]"""
import ctypes as C, math, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import _lib
lib = _lib.load()
HQ, HKV, D, BLK, L = 32, 8, 128, 32, 36
f = lib.fb_internal_merge_ex
f.restype = C.c_int
f.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
              C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
              C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]
for b in [int(x) for x in sys.argv[1:]] or [16]:
    groups, rows = b * HKV, 4 * BLK
    g = torch.Generator(device="cuda").manual_seed(2)
    r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
    qs = [r(groups, rows, D) for _ in range(L)]
    ks = [r(groups, BLK, D) for _ in range(L)]
    vs = [r(groups, BLK, D) for _ in range(L)]
    oe = [torch.randn((groups, rows, D), device="cuda", generator=g) for _ in range(L)]
    oeb = [o.to(torch.bfloat16) for o in oe]
    le = [torch.randn((groups, rows), device="cuda", generator=g) for _ in range(L)]
    VARS = {"A": (0, -1), "B": (0x100, -1), "C": (0, 1), "D": (0x100, 1), "E": (0, 0), "F": (0x100, 0)}
    out = {n: [torch.empty((groups, rows, D), device="cuda", dtype=torch.bfloat16) for _ in range(L)] for n in VARS}
    s = torch.cuda.Stream()
    graphs = {}
    for n in VARS:
        lib.fb_debug_set_k2_variant(VARS[n][1])
        def fn(n=n):
            for _ in range(31):
                for i in range(L):
                    dt, o = (2, oe[i]) if VARS[n][0] == 0 else (2 | 0x100, oeb[i])
                    rc = f(dt, qs[i].data_ptr(), ks[i].data_ptr(), vs[i].data_ptr(), groups, rows, D, BLK,
                           1 / math.sqrt(D), o.data_ptr(), le[i].data_ptr(), out[n][i].data_ptr(), 2,
                           None, None, None, None, None, 0, 1, s.cuda_stream)
                    assert rc == 0, (rc, lib.fb_last_error())
        with torch.cuda.stream(s):
            fn(); torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                fn()
        graphs[n] = gr
    res = {}
    for rnd in range(8):
        for n in (list(VARS) if rnd % 2 == 0 else list(VARS)[::-1]):
            graphs[n].replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); graphs[n].replay(); e1.record(); torch.cuda.synchronize()
            res.setdefault(n, []).append(e0.elapsed_time(e1) / (31 * L) * 1000)
    lib.fb_debug_set_k2_variant(-1)
    diff = max(float((out["A"][i].float() - out["B"][i].float()).abs().max()) for i in range(L))
    for n in VARS:
        v = sorted(res[n])
        ext = "fp32" if VARS[n][0] == 0 else "bf16"
        var = {-1: "auto", 0: "v1", 1: "v2"}[VARS[n][1]]
        print(f"b={b} {ext} O_ext {var}: K2 per launch us min {v[0]:.2f} med {v[len(v)//2]:.2f}")
    print(f"b={b} max |out_fp32ext - out_bf16ext| = {diff:.3e}")
