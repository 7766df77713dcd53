"""Per-CTA globaltimer timeline of the C4 K8 gather kernel (64K, b=4) at a density."""
import os, sys, ctypes, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K, _lib
lib = _lib.load(); lib.fb_debug_set_trace.argtypes = [ctypes.c_void_p]
HQ, HKV, D, B, N = 32, 8, 128, 32, 65536
b = 4
groups, rows = b * HKV, 4 * B
g = torch.Generator(device="cuda").manual_seed(4)
r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
q, k, v, ki, vi = r(groups, rows, D), r(groups, N, D), r(groups, N, D), r(groups, B, D), r(groups, B, D)
for dens in [float(x) for x in sys.argv[1:]] or [0.1]:
    budget = K.mask_budget(N, dens, 16)
    sel = K.topk_blocks(K.block_mass(q, k, ki, N, 16), budget)
    res = K.sparse_partitioned(q, k, v, ki, vi, N, sel)[2]
    tr = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
    for it in range(4):
        lib.fb_debug_set_trace(tr.data_ptr() if it == 3 else None)
        K.sparse_attend_merge(q, k, v, ki, vi, N, sel, res, out_dtype=torch.bfloat16)
        torch.cuda.synchronize()
    lib.fb_debug_set_trace(None)
    t = tr.view(148, 8).cpu().numpy().astype(np.int64)
    t = t[t[:, 0] > 0]  # CTAs of this launch (cluster plans use fewer than 148)
    print(f"  CTAs traced: {t.shape[0]}")
    t0 = t[:, 0].min()
    rel = lambda x: (x - t0) / 1e3
    pc = lambda x: np.round(np.percentile(x, [0, 10, 50, 90, 100]), 1)
    print(f"density {dens}: tiles/CTA ~{(groups * ((budget + 7) // 8 + 1)) / 148:.1f}")
    print("  start            ", pc(rel(t[:, 0])))
    print("  seg0 stream end  ", pc(rel(t[:, 1])))
    print("  seg0 O ready     ", pc(rel(t[:, 5])))
    print("  seg0 stored      ", pc(rel(t[:, 6])))
    last = np.max(np.where(t[:, 1:5] > 0, t[:, 1:5], 0), axis=1)
    print("  last epi end     ", pc(rel(last)))
    if os.environ.get("CLUSTER_STAMPS"):  # cluster plan: 3 = published, 4 = past the barrier, 1 = reduced
        print("  cl: published    ", pc(rel(t[:, 3])))
        print("  cl: barrier      ", pc(rel(t[:, 4])))
        print("  cl: reduced      ", pc(rel(t[:, 1])))
    print("  CTA done         ", pc(rel(t[:, 7])))
