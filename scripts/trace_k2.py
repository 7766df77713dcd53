"""K2 (cached step) per-CTA timeline at C2 b=16: a CUDA graph of 36 layers of
cached steps in which launches 20..22 are traced (8 globaltimer stamps per
CTA: start, TMEM ready, PDL released, Q/K/V landed, S ready, P written,
O ready, stores done).  Prints per-stage percentiles relative to the earliest
start of each launch, and the gap between consecutive launches."""
import ctypes, json, math, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import _lib
lib = _lib.load()
lib.fb_debug_set_k2_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
b = int(sys.argv[1]) if len(sys.argv) > 1 else 16
HQ, HKV, D, BLK, L = 32, 8, 128, 32, 36
groups, rows = b * HKV, 4 * BLK
g = torch.Generator(device="cuda").manual_seed(2)
r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
qs = [r(groups, rows, D) for _ in range(L)]
ks = [r(groups, BLK, D) for _ in range(L)]
vs = [r(groups, BLK, D) for _ in range(L)]
oe = [torch.randn((groups, rows, D), device="cuda", generator=g) for _ in range(L)]
le = [torch.randn((groups, rows), device="cuda", generator=g) for _ in range(L)]
out = [torch.empty((groups, rows, D), device="cuda", dtype=torch.bfloat16) for _ in range(L)]
NT = 3
trace = torch.zeros(NT * 1024 * 8, dtype=torch.int64, device="cuda")
s = torch.cuda.Stream()


def fn():
    for i in range(L):
        rc = lib.fb_internal_merge_ex(2, qs[i].data_ptr(), ks[i].data_ptr(), vs[i].data_ptr(), groups, rows,
                                      D, BLK, 1 / math.sqrt(D), oe[i].data_ptr(), le[i].data_ptr(),
                                      out[i].data_ptr(), 2, None, None, None, None, None, 0, 1, s.cuda_stream)
        assert rc == 0
        if i == 19:
            lib.fb_debug_set_k2_trace(trace.data_ptr(), NT)


with torch.cuda.stream(s):
    fn(); torch.cuda.synchronize()
    lib.fb_debug_set_k2_trace(None, 0)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        fn()
lib.fb_debug_set_k2_trace(None, 0)
for _ in range(3):
    gr.replay()
torch.cuda.synchronize()
t = trace.view(NT, 1024, 8).cpu()
ctas = 2 * groups
names = ["start", "tmem", "pdl", "qkv", "s_full", "p_ready", "o_full", "stored"]
res = {"batch": b, "ctas": ctas}
t0_all = int(t[0, :ctas, 0].min())
for li in range(NT):
    x = t[li, :ctas].double()
    base = float(x[:, 0].min())
    st = {}
    for k, nm in enumerate(names):
        col = (x[:, k] - base) / 1000.0
        st[nm] = [round(float(col.quantile(q)), 2) for q in (0.0, 0.5, 1.0)]
    st["launch_start_us_from_first"] = round((base - t0_all) / 1000.0, 2)
    res[f"launch{li}"] = st
print(json.dumps(res))
