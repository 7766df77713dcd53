"""K1 exp2 offload experiment: MUFU only vs 1/4 and 1/2 of the P pairs on the
FMA pipes (ptx::ex2_poly), on prefill (compute-bound), C5 video refresh
(compute-bound) and the C2 refresh (HBM-bound).  Interleaved rounds."""
import ctypes, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K, _lib
lib = _lib.load(); lib.fb_debug_set_k1_diag.argtypes = [ctypes.c_int]
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(1)
r = lambda *s: torch.randn(s, device=dev, generator=g).to(torch.bfloat16)

def gms(fn, reps=3):
    s = torch.cuda.Stream(); fn(); torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s): fn()
    gr.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): gr.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

n_q = 32768
qp, kp, vp = r(8, 4 * n_q, 128), r(8, n_q, 128), r(8, n_q, 128)
fl_p = 4.0 * 8 * 4 * sum(min(n_q, (p // 32 + 1) * 32) for p in range(0, n_q, 32)) * 32 * 128
qv, kv, vv = r(12, 4680, 128), r(12, 56160, 128), r(12, 56160, 128)
fl_v = 4.0 * 12 * 4680 * 56160 * 128
L = 6
qc = r(128, 128, 128)
kc = [r(128, 32768, 128) for _ in range(L)]
vc = [r(128, 32768, 128) for _ in range(L)]
by_c = 2 * 128 * 32768 * 128 * 2
res = {}
for rnd in range(3):
    for diag, name in ((0, "product"), (1, "no-softmax")):
        lib.fb_debug_set_k1_diag(diag)
        tp = gms(lambda: K.block_causal_attention(qp, kp, vp, n_q, 0, 32))
        tv = gms(lambda: K.attention_partial(qv, kv, vv))
        tc = gms(lambda: [K.attention_partial(qc, kc[i], vc[i]) for i in range(L)]) / L
        res.setdefault(name, []).append((tp, tv, tc))
lib.fb_debug_set_k1_diag(0)
for name, rows in res.items():
    tp = min(x[0] for x in rows); tv = min(x[1] for x in rows); tc = min(x[2] for x in rows)
    print(f"{name:8s} prefill32K {tp:.2f} ms {fl_p/tp/1e9:.0f} TF/s | C5 K1 {tv:.3f} ms {fl_v/tv/1e9:.0f} TF/s | "
          f"C2 K1 b=16 {tc*1000:.0f} us {by_c/tc/1e6:.0f} GB/s")
