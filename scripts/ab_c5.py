"""Interleaved A/B at the C5 shapes: K1 on the single-CTA kernel (quad mode 2,
the default: two-query-tile kernel for block-causal only) vs the two-query-tile
kernel with key-tile rotation for every shape (quad mode 1).  Refresh over
n_ext keys and the large-block cached step (K1 over the 4680-key block with
the merge against the cached partial fused)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_05305_b200 import kernels as K, _lib
lib = _lib.load()
PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["bf16_tflops"]
H, D, B = 12, 128, 4680
g = torch.Generator(device="cuda").manual_seed(5)
r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
for n_ext in (56160, 18720, 0):
    q = r(H, B, D)
    if n_ext:
        k, v = r(H, n_ext, D), r(H, n_ext, D)
        o, l = K.attention_partial(q, k, v, 0, n_ext)
        fn = lambda: K.attention_partial(q, k, v, 0, n_ext, None, o, l)
        fl = 4.0 * H * B * n_ext * D
        name = f"refresh n_ext={n_ext}"
    else:
        ki, vi = r(H, B, D), r(H, B, D)
        oe = torch.randn((H, B, D), device="cuda", generator=g).to(torch.bfloat16)
        le = torch.randn((H, B), device="cuda", generator=g)
        out = torch.empty((H, B, D), device="cuda", dtype=torch.bfloat16)
        fn = lambda: K.internal_merge(q, ki, vi, oe, le, out_dtype=torch.bfloat16, out=out, ext_stable=True)
        fl = 4.0 * H * B * B * D
        name = "cached step (4680-key block)"
    graphs = {}
    for mode in (2, 1, 3):  # 3: CTA pairs (quad off, pair forced)
        lib.fb_debug_set_quad(0 if mode == 3 else mode)
        lib.fb_debug_set_pair(1 if mode == 3 else -1)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            fn(); torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                for _ in range(3):
                    fn()
        graphs[mode] = gr
    lib.fb_debug_set_quad(-1)
    lib.fb_debug_set_pair(-1)
    res = {2: [], 1: [], 3: []}
    for rnd in range(8):
        for mode in ((2, 1, 3) if rnd % 2 == 0 else (3, 1, 2)):
            graphs[mode].replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); graphs[mode].replay(); e1.record(); torch.cuda.synchronize()
            res[mode].append(e0.elapsed_time(e1) / 3)
    rec = {"shape": name}
    for mode, nm in ((2, "single"), (1, "quad_rot"), (3, "pair_rot")):
        ms = sorted(res[mode])[len(res[mode]) // 2]
        rec[nm + "_ms"] = round(ms, 4)
        rec[nm + "_frac"] = round(fl / (ms * 1e-3) / 1e12 / PEAK, 3)
    print(json.dumps(rec), flush=True)
