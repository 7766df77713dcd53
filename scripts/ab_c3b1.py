"""C3 b=1 split-KV shard refresh (K1 + split merge) and C4 K8: graph timing per process."""
import json, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K
g = torch.Generator(device="cuda").manual_seed(3)
r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)


def gms(fn, per, reps=5):
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
    return e0.elapsed_time(e1) / reps / per


out = {"lib": os.path.basename(os.environ.get("FB_LIB_PATH", "libfb200.so"))}
L = 4
for P in (1, 2, 8):
    n = 131072 // P
    q = r(8, 128, 128); ks = [r(8, n, 128) for _ in range(L)]; vs = [r(8, n, 128) for _ in range(L)]
    o, l = K.attention_partial(q, ks[0], vs[0])
    out[f"c3_b1_P{P}_ms"] = gms(lambda: [K.attention_partial(q, ks[i], vs[i], 0, None, None, o, l) for i in range(L)], L)
print(json.dumps(out), flush=True)
