"""Interleaved A/B of K1 (fb_attention_partial) from two library builds in one
process: CUDA graphs of back-to-back launches over distinct KV buffers.
    python scripts/ab_k1.py OLD.so NEW.so [batch] [distinct]"""
import ctypes as C, math, sys, torch
old_p, new_p = sys.argv[1], sys.argv[2]
b = int(sys.argv[3]) if len(sys.argv) > 3 else 16
nd = int(sys.argv[4]) if len(sys.argv) > 4 else 12
HKV, D, CTX = 8, 128, 32768
groups = b * HKV
libs = {}
for name, p in (("old", old_p), ("new", new_p)):
    l = C.CDLL(p)
    l.fb_partial_workspace_bytes.restype = C.c_size_t
    l.fb_partial_workspace_bytes.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64]
    l.fb_attention_partial.restype = C.c_int
    l.fb_attention_partial.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                       C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
    libs[name] = l
gen = torch.Generator(device="cuda").manual_seed(1)
q = torch.randn((groups, 128, D), device="cuda", generator=gen).to(torch.bfloat16)
ks = [torch.randn((groups, CTX, D), device="cuda", generator=gen).to(torch.bfloat16) for _ in range(nd)]
vs = [torch.randn((groups, CTX, D), device="cuda", generator=gen).to(torch.bfloat16) for _ in range(nd)]
o = {n: torch.empty((groups, 128, D), device="cuda", dtype=torch.float32) for n in libs}
l_ = {n: torch.empty((groups, 128), device="cuda", dtype=torch.float32) for n in libs}
ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
graphs = {}
for n, lib in libs.items():
    def fn(lib=lib, n=n):
        for i in range(nd):
            rc = lib.fb_attention_partial(2, q.data_ptr(), ks[i].data_ptr(), vs[i].data_ptr(), groups, 128, D, CTX,
                                          0, CTX, 1 / math.sqrt(D), o[n].data_ptr(), l_[n].data_ptr(),
                                          ws.data_ptr(), ws.numel(), s.cuda_stream)
            assert rc == 0, rc
    with torch.cuda.stream(s):
        fn(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
    graphs[n] = g
torch.cuda.synchronize()
print("max |o_new - o_old|", float((o["new"] - o["old"]).abs().max()), "lse", float((l_["new"] - l_["old"]).abs().max()))
byts = 2 * groups * CTX * D * 2
res = {n: [] for n in libs}
for rnd in range(6):
    for n in (("old", "new") if rnd % 2 == 0 else ("new", "old")):
        g = graphs[n]
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3): g.replay()
        e1.record(); torch.cuda.synchronize()
        res[n].append(e0.elapsed_time(e1) / (3 * nd) * 1000)
for n in libs:
    r = sorted(res[n])
    print(f"b={b} {n}: per launch us min {r[0]:.1f} med {r[len(r)//2]:.1f} max {r[-1]:.1f}  -> {byts / r[len(r)//2] / 1e3:.0f} GB/s (median)")
