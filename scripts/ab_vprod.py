"""Timing probe for the K1 producer split (FB_K1_VPROD, read once per
process): C2 b=16 refresh, C3 b=8 P=8 shard, C5 refresh, C4 K8 at 10/50 %
density.  Run once per setting; scripts/gpu_vprod.sh interleaves processes."""
import json, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K
g = torch.Generator(device="cuda").manual_seed(3)
r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)


def gms(fn, reps=3, per=1):
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


out = {"vprod": os.environ.get("FB_K1_VPROD", "1")}
L = 4
q = r(128, 128, 128); ks = [r(128, 32768, 128) for _ in range(L)]; vs = [r(128, 32768, 128) for _ in range(L)]
o, l = K.attention_partial(q, ks[0], vs[0])
out["c2_b16_k1_ms"] = gms(lambda: [K.attention_partial(q, ks[i], vs[i], 0, None, None, o, l) for i in range(L)], per=L)
del ks, vs
q = r(64, 128, 128); ks = [r(64, 16384, 128) for _ in range(L)]; vs = [r(64, 16384, 128) for _ in range(L)]
o, l = K.attention_partial(q, ks[0], vs[0])
out["c3_p8_k1_ms"] = gms(lambda: [K.attention_partial(q, ks[i], vs[i], 0, None, None, o, l) for i in range(L)], per=L)
del ks, vs
qv, kv, vv = r(12, 4680, 128), r(12, 56160, 128), r(12, 56160, 128)
o, l = K.attention_partial(qv, kv, vv)
out["c5_k1_ms"] = gms(lambda: K.attention_partial(qv, kv, vv, 0, None, None, o, l))
del qv, kv, vv
N = 65536
q, k, v, ki, vi = r(32, 128, 128), r(32, N, 128), r(32, N, 128), r(32, 32, 128), r(32, 32, 128)
for dens in (0.1, 0.5):
    sel = K.topk_blocks(K.block_mass(q, k, ki, N, 16), K.mask_budget(N, dens, 16))
    res = K.sparse_partitioned(q, k, v, ki, vi, N, sel)[2]
    out[f"c4_k8_{dens}_ms"] = gms(lambda: [K.sparse_attend_merge(q, k, v, ki, vi, N, sel, res) for _ in range(4)], per=4)
print(json.dumps(out), flush=True)
