"""Interleaved A/B of the cached step (K2 v2, bf16 O_ext) with the output
written by row-per-thread 256-bit global stores (A) vs one bulk tensor store
per (CTA, column half) from the dead Q tile (B, fb_debug_set_k2_store(1)),
and with V_in on its own load barrier as well (C, fb_debug_set_k2_vsplit(1)):
graph of 36 layers x 31 cached steps at the C2 shapes.
    python scripts/ab_k2_store.py [batch ...]"""
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
for b in [int(x) for x in sys.argv[1:]] or [32]:
    groups, rows = b * HKV, 4 * BLK
    g = torch.Generator(device="cuda").manual_seed(2)
    r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
    qs = [r(groups, rows, D) for _ in range(L)]
    ks = [r(groups, BLK, D) for _ in range(L)]
    vs = [r(groups, BLK, D) for _ in range(L)]
    oeb = [r(groups, rows, D) for _ in range(L)]
    le = [torch.randn((groups, rows), device="cuda", generator=g) for _ in range(L)]
    # (store, vsplit): A the previous kernel, B TMA store, C TMA store + V on its own barrier
    # D: + Q / K column halves; E: the library defaults (by grid size)
    VARS = {"A": (0, 0), "B": (1, 0), "C": (1, 1), "D": (1, 2), "E": (-1, -1)}
    out = {n: [torch.empty((groups, rows, D), device="cuda", dtype=torch.bfloat16) for _ in range(L)] for n in VARS}
    s = torch.cuda.Stream()
    graphs = {}
    lib.fb_debug_set_k2_variant(-1)  # by size: v1 up to b=16 at C2, v2 beyond (store modes are v2-only)
    for n in VARS:
        lib.fb_debug_set_k2_store(VARS[n][0])
        lib.fb_debug_set_k2_vsplit(VARS[n][1])
        def fn(n=n):
            for _ in range(31):
                for i in range(L):
                    rc = f(2 | 0x100, qs[i].data_ptr(), ks[i].data_ptr(), vs[i].data_ptr(), groups, rows, D, BLK,
                           1 / math.sqrt(D), oeb[i].data_ptr(), le[i].data_ptr(), out[n][i].data_ptr(), 2,
                           None, None, None, None, None, 0, 1, s.cuda_stream)
                    assert rc == 0, (rc, lib.fb_last_error())
        with torch.cuda.stream(s):
            fn(); torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                fn()
        graphs[n] = gr
    lib.fb_debug_set_k2_store(-1)
    lib.fb_debug_set_k2_vsplit(-1)
    lib.fb_debug_set_k2_variant(-1)
    res = {}
    for rnd in range(10):
        for n in (list(VARS) if rnd % 2 == 0 else list(VARS)[::-1]):
            graphs[n].replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); graphs[n].replay(); e1.record(); torch.cuda.synchronize()
            res.setdefault(n, []).append(e0.elapsed_time(e1) / (31 * L) * 1000)
    eq = all(torch.equal(out["A"][i], out[n][i]) for n in VARS for i in range(L))
    byts = L and (groups * rows * D * 2 * 3 + 2 * groups * BLK * D * 2 + groups * rows * 4)
    for n in VARS:
        v = sorted(res[n])
        print(f"b={b} store={ {1: 'tma', 0: 'per-thread', -1: 'default'}[VARS[n][0]] } vsplit={VARS[n][1]}: K2 per launch us min {v[0]:.2f} med {v[len(v)//2]:.2f}"
              f"  ({byts / (v[len(v)//2] * 1e-6) / 1e9:.0f} GB/s)")
    print(f"b={b} outputs bitwise equal: {eq}")
