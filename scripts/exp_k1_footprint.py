"""K1 in CUDA graphs: per-launch time vs number of distinct KV buffers cycled."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K
HKV, D, CTX = 8, 128, 32768
def gms(fn, reps=3):
    s = torch.cuda.Stream(); fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s): fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): g.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for b in (8, 16):
    groups = b * HKV
    gen = torch.Generator(device="cuda").manual_seed(1)
    L = 36 if b == 8 else 18
    q = torch.randn((groups, 128, D), device="cuda", generator=gen).to(torch.bfloat16)
    ks = [torch.randn((groups, CTX, D), device="cuda", generator=gen).to(torch.bfloat16) for _ in range(L)]
    vs = [torch.randn((groups, CTX, D), device="cuda", generator=gen).to(torch.bfloat16) for _ in range(L)]
    o = torch.empty((groups, 128, D), device="cuda", dtype=torch.float32)
    l = torch.empty((groups, 128), device="cuda", dtype=torch.float32)
    byts = 2 * groups * CTX * D * 2
    for nd in (1, 2, 4, L):
        t = gms(lambda: [K.attention_partial(q, ks[i % nd], vs[i % nd], 0, CTX, None, o, l) for i in range(36)]) / 36
        print(f"b={b} distinct={nd} per-launch {t*1000:.1f} us -> {byts/t/1e6:.0f} GB/s", flush=True)
    del ks, vs; torch.cuda.empty_cache()
