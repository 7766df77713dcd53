"""Per-CTA start / end (globaltimer) distribution of one K1 launch (C2 shapes)."""
import os, sys, ctypes, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K, _lib
lib = _lib.load(); lib.fb_debug_set_trace.argtypes = [ctypes.c_void_p]
HKV, D = 8, 128
CTX = int(os.environ.get("CTX", "32768"))
for b in [int(x) for x in sys.argv[1:]] or [16]:
    g = torch.Generator(device="cuda").manual_seed(1)
    q = torch.randn((b * HKV, 128, D), device="cuda", generator=g).to(torch.bfloat16)
    ks = [torch.randn((b * HKV, CTX, D), device="cuda", generator=g).to(torch.bfloat16) for _ in range(3)]
    vs = [torch.randn((b * HKV, CTX, D), device="cuda", generator=g).to(torch.bfloat16) for _ in range(3)]
    tr = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
    for it in range(3):
        lib.fb_debug_set_trace(tr.data_ptr() if it == 2 else None)
        K.attention_partial(q, ks[it], vs[it])
        torch.cuda.synchronize()
    lib.fb_debug_set_trace(None)
    t = tr.view(148, 8).cpu().numpy().astype(np.int64)
    t0 = t[:, 0].min()
    st = (t[:, 0] - t0) / 1e3
    end = (np.max(t[:, 1:5], axis=1) - t0) / 1e3
    q = lambda x: np.percentile(x, [0, 10, 50, 90, 100])
    print(f"b={b} start us pct0/10/50/90/100 {np.round(q(st),1)}")
    print(f"b={b} end   us pct0/10/50/90/100 {np.round(q(end),1)}  -> mean end {end.mean():.1f}, max {end.max():.1f}")
    byts = 2 * b * HKV * CTX * D * 2
    print(f"b={b} rate at median end {byts/np.median(end)/1e3:.0f} GB/s, at max end {byts/end.max()/1e3:.0f} GB/s")
    # correlation of end time with CTA index (SM placement / segment layout)
    smid_order = np.argsort(end)
    print("earliest CTAs", smid_order[:12].tolist(), "latest CTAs", smid_order[-12:].tolist())
    print("end by CTA-index decile (us):", [round(float(np.mean(end[i * 15:(i + 1) * 15])), 1) for i in range(10)])
