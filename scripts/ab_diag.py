"""Pipeline ceilings at the tensor-bound shapes: pair kernel with / without
softmax math (FB_PAIR_POLY=-1, read once per process) and the single-CTA
kernel with / without (fb_debug_set_k1_diag 2).  C5 refresh 56K, prefill 32K."""
import ctypes, json, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import _lib, kernels as K
lib = _lib.load(); lib.fb_debug_set_pair.argtypes = [ctypes.c_int]; lib.fb_debug_set_k1_diag.argtypes = [ctypes.c_int]
g = torch.Generator(device="cuda").manual_seed(1)
r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)


def gms(fn, reps=3):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        fn()
    gr.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        gr.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


qv, kv, vv = r(12, 4680, 128), r(12, 56160, 128), r(12, 56160, 128)
ov, lv = K.attention_partial(qv, kv, vv)
n_q = 32768
qp, kp, vp = r(8, 4 * n_q, 128), r(8, n_q, 128), r(8, n_q, 128)
op, lp = K.block_causal_attention(qp, kp, vp, n_q, 0, 32)
fl_c5 = 4.0 * 12 * 4680 * 56160 * 128
fl_pf = 4.0 * 8 * 4 * sum(min(n_q, (p // 32 + 1) * 32) for p in range(0, n_q, 32)) * 32 * 128
res = {"pair_poly_env": os.environ.get("FB_PAIR_POLY", "0")}
for name, pair, diag in (("pair", 1, 0), ("single", 0, 0), ("single_nosoftmax", 0, 2), ("single_nosoftmax_nopv", 0, 6)):
    lib.fb_debug_set_pair(pair); lib.fb_debug_set_k1_diag(diag)
    t5 = gms(lambda: K.attention_partial(qv, kv, vv, 0, None, None, ov, lv))
    tp = gms(lambda: K.block_causal_attention(qp, kp, vp, n_q, 0, 32, None, op, lp))
    res[name] = {"c5_ms": t5, "c5_tflops": fl_c5 / t5 / 1e9, "prefill_ms": tp, "prefill_tflops": fl_pf / tp / 1e9}
lib.fb_debug_set_pair(-1); lib.fb_debug_set_k1_diag(0)
print(json.dumps(res), flush=True)
