"""K1 plan A/B at split-KV shard shapes (C3: 128K over P shards, b=8 / b=1)
and the C2 batches: CTA count (FB_REFRESH_CTAS) x in-kernel merge span limit
(FB_K1_MAXSPAN), interleaved, CUDA-graph timing of 4 launches on distinct KV."""
import json, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K

HBM = 6544.0
g = torch.Generator(device="cuda").manual_seed(3)
r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
L = 4


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
    return e0.elapsed_time(e1) / reps / L


cases = [("C3 b=8 P=8", 64, 16384), ("C3 b=8 P=4", 64, 32768), ("C3 b=1 P=2", 8, 65536),
         ("C2 b=8", 64, 32768), ("C2 b=16", 128, 32768), ("C2 b=4", 32, 32768)]
variants = [("default", {}), ("ctas148", {"FB_REFRESH_CTAS": "148"}),
            ("span4", {"FB_K1_MAXSPAN": "4"}), ("ctas148+span4", {"FB_REFRESH_CTAS": "148", "FB_K1_MAXSPAN": "4"}),
            ("ctas148+span5", {"FB_REFRESH_CTAS": "148", "FB_K1_MAXSPAN": "5"})]
if os.environ.get("AB_SMALL"):  # latency-bound shapes: CTA count only
    cases = [("C3 b=1 P=8", 8, 16384), ("C3 b=1 P=4", 8, 32768), ("C3 b=1 P=2", 8, 65536),
             ("C2 b=1", 8, 32768), ("C2 b=2", 16, 32768), ("C2 b=4", 32, 32768)]
    variants = [("default", {}), ("ctas148", {"FB_REFRESH_CTAS": "148"}), ("ctas144", {"FB_REFRESH_CTAS": "144"})]
res = {}
for name, groups, n in cases:
    q = r(groups, 128, 128)
    ks = [r(groups, n, 128) for _ in range(L)]
    vs = [r(groups, n, 128) for _ in range(L)]
    o, l = K.attention_partial(q, ks[0], vs[0])
    for rnd in range(2):
        for vn, env in variants:
            for k_ in ("FB_REFRESH_CTAS", "FB_K1_MAXSPAN"):
                os.environ.pop(k_, None)
            os.environ.update(env)
            t = gms(lambda: [K.attention_partial(q, ks[i], vs[i], 0, None, None, o, l) for i in range(L)])
            res.setdefault((name, vn), []).append(t)
    del ks, vs
    torch.cuda.empty_cache()
    by = 2 * groups * n * 128 * 2
    for vn, _ in variants:
        t = min(res[(name, vn)])
        print(json.dumps({"case": name, "variant": vn, "ms": t, "frac_hbm": by / (t * 1e-3) / 1e9 / HBM}), flush=True)
