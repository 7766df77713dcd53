import sys, os, ctypes, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K, _lib
lib = _lib.load(); lib.fb_debug_set_trace.argtypes = [ctypes.c_void_p]
HKV, D, CTX = 8, 128, int(os.environ.get("CTX", 32768))
for b in [int(x) for x in sys.argv[1:]] or [1, 8]:
    g = torch.Generator(device="cuda").manual_seed(1)
    q = torch.randn((b * HKV, 128, D), device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn((b * HKV, CTX, D), device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn((b * HKV, CTX, D), device="cuda", generator=g).to(torch.bfloat16)
    tr = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
    for it in range(3):
        lib.fb_debug_set_trace(tr.data_ptr() if it == 2 else None)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); K.attention_partial(q, k, v); e1.record(); torch.cuda.synchronize()
    lib.fb_debug_set_trace(None)
    t = tr.view(148, 8).cpu().numpy().astype(np.int64)
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    rel = lambda x: (x - t0) / 1000.0
    st = t[:, 0]; s1 = np.where(t[:, 1] > 0, t[:, 1], 0); m1 = np.where(t[:, 2] > 0, t[:, 2], 0)
    s2 = np.where(t[:, 3] > 0, t[:, 3], 0); m2 = np.where(t[:, 4] > 0, t[:, 4], 0)
    end = np.maximum.reduce([s1, m1, s2, m2])
    print(f"b={b} event_ms={e0.elapsed_time(e1):.3f} start spread {rel(st.max()):.1f}us; "
          f"stream-end(seg0) min/med/max {rel(s1[s1>0].min()):.1f}/{rel(np.median(s1[s1>0])):.1f}/{rel(s1.max()):.1f}us; "
          f"merge-end(seg0) max {rel(m1.max()) if m1.max() else 0:.1f}; seg1 stream-end max {rel(s2.max()) if s2.max() else 0:.1f} "
          f"merge-end max {rel(m2.max()) if m2.max() else 0:.1f}; cta end max {rel(end.max()):.1f}us")
    # epilogue detail (segment 0): 5 = O accumulators final, 6 = rows stored, 7 = CTA done
    if t.shape[0] and (t[:, 5] > 0).any():
        for k, nm in ((1, "softmax done"), (5, "o_full"), (6, "stored"), (7, "cta done")):
            x = t[:, k][t[:, k] > 0]
            print(f"  {nm:13s} min/med/max {rel(x.min()):.1f}/{rel(np.median(x)):.1f}/{rel(x.max()):.1f} us")
