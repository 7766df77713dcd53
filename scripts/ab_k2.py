"""Interleaved A/B of the cached step (K2, engine.cached -> fb_internal_merge_ex)
between two library builds: graph of 36 layers x 31 cached steps at C2 b=16.

    python scripts/ab_k2.py libA.so libB.so [batch] [ENV=VAL for A] [ENV=VAL for B]

The optional environment settings are applied just before each library's
first call (the library reads its FB_* switches once).  AB_EXTB=1: the
cached external partial's O in bf16 (FB_PARTIAL_BF16), the engine default."""
import ctypes as C, math, os, sys, torch
A, B = sys.argv[1], sys.argv[2]
b = int(sys.argv[3]) if len(sys.argv) > 3 else 16
ENV = {"A": sys.argv[4] if len(sys.argv) > 4 else "", "B": sys.argv[5] if len(sys.argv) > 5 else ""}
HQ, HKV, D, BLK, L = 32, 8, 128, 32, 36
groups, rows = b * HKV, 4 * BLK
libs = {}
for name, p in (("A", A), ("B", B)):
    l = C.CDLL(p)
    l.fb_internal_merge_ex.restype = C.c_int
    l.fb_internal_merge_ex.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                       C.c_int64, C.c_int64, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_size_t, C.c_int, C.c_void_p]
    libs[name] = l
g = torch.Generator(device="cuda").manual_seed(2)
r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
qs = [r(groups, rows, D) for _ in range(L)]
ks = [r(groups, BLK, D) for _ in range(L)]
vs = [r(groups, BLK, D) for _ in range(L)]
EXTB = os.environ.get("AB_EXTB") == "1"
oe = [torch.randn((groups, rows, D), device="cuda", generator=g) for _ in range(L)]
if EXTB:
    oe = [o.to(torch.bfloat16) for o in oe]
DT = 2 | (0x100 if EXTB else 0)
le = [torch.randn((groups, rows), device="cuda", generator=g) for _ in range(L)]
out = [torch.empty((groups, rows, D), device="cuda", dtype=torch.bfloat16) for _ in range(L)]
s = torch.cuda.Stream()
graphs = {}
for n, lib in libs.items():
    def fn(lib=lib):
        for _ in range(31):
            for i in range(L):
                rc = lib.fb_internal_merge_ex(DT, qs[i].data_ptr(), ks[i].data_ptr(), vs[i].data_ptr(), groups, rows,
                                              D, BLK, 1 / math.sqrt(D), oe[i].data_ptr(), le[i].data_ptr(),
                                              out[i].data_ptr(), 2, None, None, None, None, None, 0, 1,
                                              s.cuda_stream)
                assert rc == 0, rc
    if ENV[n]:
        k, v = ENV[n].split("=", 1)
        os.environ[k] = v
    with torch.cuda.stream(s):
        fn(); torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            fn()
    graphs[n] = gr
res = {}
for rnd in range(6):
    for n in (("A", "B") if rnd % 2 == 0 else ("B", "A")):
        graphs[n].replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); graphs[n].replay(); e1.record(); torch.cuda.synchronize()  # replay on the current stream
        res.setdefault(n, []).append(e0.elapsed_time(e1) / (31 * L) * 1000)
for n in res:
    v = sorted(res[n])
    print(f"b={b} {n} ({os.path.basename(A if n == 'A' else B)}): K2 per launch us min {v[0]:.2f} med {v[len(v)//2]:.2f}")
