"""Paged vs contiguous K1 at C2 (b=16: 128 slabs x 32,768 keys, page_rows 256,
pages scattered in a shuffled pool): CUDA-graph timing, 4 layers of distinct
KV, interleaved rounds.  One JSON line."""
import json, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K
g = torch.Generator(device="cuda").manual_seed(5)
groups, N, d, P, L = 128, 32768, 128, 256, 4
r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
q = r(groups, 128, d)
lens = torch.full((groups,), N, dtype=torch.int32, device="cuda")
mp = N // P
kc = [r(groups, N, d) for _ in range(L)]
vc = [r(groups, N, d) for _ in range(L)]
perm = torch.randperm(groups * mp, generator=torch.Generator().manual_seed(2)).cuda()
table = perm.view(groups, mp).to(torch.int32).contiguous()
kp, vp = [], []
for i in range(L):
    a = torch.empty((groups * mp, P, d), device="cuda", dtype=torch.bfloat16)
    b = torch.empty_like(a)
    a[perm] = kc[i].view(groups * mp, P, d)
    b[perm] = vc[i].view(groups * mp, P, d)
    kp.append(a); vp.append(b)
del kc[1:], vc[1:]
torch.cuda.empty_cache()
o, l = K.attention_partial_paged(q, kp[0], vp[0], table, lens)
o2, l2 = K.attention_partial_ragged(q, kc[0], vc[0], lens)
assert torch.equal(o, o2) and torch.equal(l, l2)
kc2 = [kc[0]] + [r(groups, N, d) for _ in range(L - 1)]
vc2 = [vc[0]] + [r(groups, N, d) for _ in range(L - 1)]


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


res = {"paged": [], "contiguous_ragged": []}
for _ in range(3):
    res["paged"].append(gms(lambda: [K.attention_partial_paged(q, kp[i], vp[i], table, lens, None, o, l) for i in range(L)]))
    res["contiguous_ragged"].append(gms(lambda: [K.attention_partial_ragged(q, kc2[i], vc2[i], lens, 0, None, o2, l2) for i in range(L)]))
by = 2 * groups * N * d * 2
print(json.dumps({"config": "C2 b=16 paged K1", "page_rows": P,
                  **{k + "_ms": min(v) for k, v in res.items()},
                  **{k + "_frac_hbm": by / (min(v) * 1e-3) / 1e9 / 6544.0 for k, v in res.items()},
                  "bitwise_equal": True}))
