"""K1 diagnostic variants in a CUDA graph of back-to-back launches (distinct KV per launch):
diag 0 = product kernel, 1 = softmax math skipped, 2 = S load skipped too."""
import os, sys, ctypes, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K, _lib
lib = _lib.load(); lib.fb_debug_set_k1_diag.argtypes = [ctypes.c_int]
HKV, D, CTX = 8, 128, 32768
b = int(sys.argv[1]) if len(sys.argv) > 1 else 16
nd = int(sys.argv[2]) if len(sys.argv) > 2 else 8
groups = b * HKV
gen = torch.Generator(device="cuda").manual_seed(1)
q = torch.randn((groups, 128, D), device="cuda", generator=gen).to(torch.bfloat16)
ks = [torch.randn((groups, CTX, D), device="cuda", generator=gen).to(torch.bfloat16) for _ in range(nd)]
vs = [torch.randn((groups, CTX, D), device="cuda", generator=gen).to(torch.bfloat16) for _ in range(nd)]
o = torch.empty((groups, 128, D), device="cuda", dtype=torch.float32)
l = torch.empty((groups, 128), device="cuda", dtype=torch.float32)
byts = 2 * groups * CTX * D * 2
for diag in (0, 1, 2, 0):
    lib.fb_debug_set_k1_diag(diag)
    fn = lambda: [K.attention_partial(q, ks[i], vs[i], 0, CTX, None, o, l) for i in range(nd)]
    s = torch.cuda.Stream(); fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s): fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): g.replay()
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / (5 * nd)
    print(f"b={b} diag={diag}: {t*1000:.1f} us per launch -> {byts/t/1e6:.0f} GB/s", flush=True)
lib.fb_debug_set_k1_diag(0)
