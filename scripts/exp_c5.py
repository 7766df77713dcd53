"""C5 refresh (video block diffusion, 12 heads x 128, block 4680) timing in one
process: run under FB_K1_QUAD / FB_QUAD_ROT to compare K1 variants."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_05305_b200 import kernels as K
PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["bf16_tflops"]
H, D, B = 12, 128, 4680
res = {}
for n_ext in (56160, 18720):
    g = torch.Generator(device="cuda").manual_seed(5)
    r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
    q, k, v = r(H, B, D), r(H, n_ext, D), r(H, n_ext, D)
    o, l = K.attention_partial(q, k, v, 0, n_ext)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        K.attention_partial(q, k, v, 0, n_ext, None, o, l); torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            for _ in range(3):
                K.attention_partial(q, k, v, 0, n_ext, None, o, l)
    ts = []
    for _ in range(5):
        gr.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); gr.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 3)
    ms = sorted(ts)[2]
    fl = 4.0 * H * B * n_ext * D
    res[n_ext] = {"ms": round(ms, 4), "tflops": round(fl / (ms * 1e-3) / 1e12, 1), "frac": round(fl / (ms * 1e-3) / 1e12 / PEAK, 3)}
    del q, k, v
print(json.dumps({"quad": os.environ.get("FB_K1_QUAD", "default"), "rot": os.environ.get("FB_QUAD_ROT", "1"), "res": res}))
