"""A/B: CTA-pair K1 (cta_group::2) vs the single-CTA K1 on the tensor-bound
shapes -- C5 video refresh (12 heads x 4680 rows, 18,720 / 56,160 keys), the
C5 cached step with its 4680-key block, and block-causal prefill at the C2
attention shapes (8 kv groups x 4 heads, 8K / 32K prompt).  Interleaved
rounds, CUDA-graph timing.  Prints one JSON line per (case, variant)."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import _lib, kernels as K  # noqa: E402

lib = _lib.load()
lib.fb_debug_set_pair.argtypes = [ctypes.c_int]
dev = torch.device("cuda")
PEAK = 1601.1
try:
    PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["bf16_tflops"]
except Exception:
    pass


def gms(fn, reps=3):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        fn()
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


g = torch.Generator(device=dev).manual_seed(1)
r = lambda *s: torch.randn(s, device=dev, generator=g).to(torch.bfloat16)
cases = []
H, B = 12, 4680
qv = r(H, B, 128)
for n_ext in (18720, 56160):
    kv, vv = r(H, n_ext, 128), r(H, n_ext, 128)
    o, l = K.attention_partial(qv, kv, vv)
    cases.append((f"C5 refresh n_ext={n_ext}", 4.0 * H * B * n_ext * 128,
                  (lambda kv=kv, vv=vv, o=o, l=l: K.attention_partial(qv, kv, vv, 0, None, None, o, l))))
ki, vi = r(H, B, 128), r(H, B, 128)
oe, le = K.attention_partial(qv, kv, vv)
outb = torch.empty((H, B, 128), dtype=torch.bfloat16, device=dev)
cases.append(("C5 cached step (4680-key block)", 4.0 * H * B * B * 128,
              lambda: K.internal_merge(qv, ki, vi, oe, le, out_dtype=torch.bfloat16, out=outb)))
for n_q in (8192, 32768):
    qp, kp, vp = r(8, 4 * n_q, 128), r(8, n_q, 128), r(8, n_q, 128)
    op, lp = K.block_causal_attention(qp, kp, vp, n_q, 0, 32)
    lim = sum(min(n_q, (p // 32 + 1) * 32) for p in range(0, n_q, 32)) * 32
    cases.append((f"F4 prefill n_q={n_q}", 4.0 * 8 * 4 * lim * 128,
                  (lambda qp=qp, kp=kp, vp=vp, op=op, lp=lp, n_q=n_q:
                   K.block_causal_attention(qp, kp, vp, n_q, 0, 32, None, op, lp))))

res = {}
for rnd in range(3):
    for name, flops, fn in cases:
        for var, flag in (("pair", 1), ("single", 0)):
            lib.fb_debug_set_pair(flag)
            t = gms(fn)
            res.setdefault((name, var), []).append(t)
lib.fb_debug_set_pair(-1)
for (name, var), ts in res.items():
    flops = [c[1] for c in cases if c[0] == name][0]
    t = min(ts)
    print(json.dumps({"case": name, "variant": var, "ms": t, "ms_all": ts,
                      "tflops": flops / (t * 1e-3) / 1e12,
                      "frac_tensor": flops / (t * 1e-3) / 1e12 / PEAK}), flush=True)
