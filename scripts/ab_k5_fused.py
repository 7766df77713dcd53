"""K5 at C4 (64K ctx, b=4: 32 groups x 128 rows): fused single-pass scoring vs
the LSE + MASS two-pass kernels (FB_K5_TWO_PASS=1, read once per process).
Times block_mass alone and block_mass + top-k at 10 % in a CUDA graph (3
layers of distinct K); the two-pass run compares its masses / selections with
the fused run's saved ones."""
import json, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K
two = os.environ.get("FB_K5_TWO_PASS", "0") == "1"
g = torch.Generator(device="cuda").manual_seed(4)
r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
N, L = 65536, 3
qs = [r(32, 128, 128) for _ in range(L)]
ks = [r(32, N, 128) for _ in range(L)]
kis = [r(32, 32, 128) for _ in range(L)]
budget = K.mask_budget(N, 0.1, 16)
s = torch.cuda.Stream()
out = {}
for name, fn in [("mass", lambda: [K.block_mass(qs[i], ks[i], kis[i], N, 16) for i in range(L)]),
                 ("mass_topk", lambda: [K.topk_blocks(K.block_mass(qs[i], ks[i], kis[i], N, 16), budget)
                                        for i in range(L)])]:
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        fn()
    gr.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record()
        gr.replay()
        e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / L)
    out[name + "_ms"] = best
out["k_bytes"] = 32 * N * 128 * 2
out["k_gbs_once"] = out["k_bytes"] / (out["mass_ms"] * 1e-3) / 1e9
masses = [K.block_mass(qs[i], ks[i], kis[i], N, 16) for i in range(L)]
sels = [K.topk_blocks(m, budget) for m in masses]
path = "gpurun_out/k5_fused_masses.pt"
if not two:
    torch.save({"m": [m.cpu() for m in masses], "s": [x.cpu() for x in sels]}, path)
elif os.path.exists(path):
    ref = torch.load(path)
    rel = max(((m.cpu() - a).abs() / a.abs().clamp_min(1e-300)).max().item() for m, a in zip(masses, ref["m"]))
    diff = sum(int((torch.sort(x.cpu(), dim=1)[0] != torch.sort(y, dim=1)[0]).any(dim=1).sum())
               for x, y in zip(sels, ref["s"]))
    out["fused_vs_two_pass_mass_rel"] = rel
    out["groups_with_different_selection"] = diff
print(json.dumps({"two_pass": two, **out}), flush=True)
