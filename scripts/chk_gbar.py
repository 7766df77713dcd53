"""Grid-barrier split-K vs the owner path on the C2-shape split test: errors of
each partial against the F32 SIMT kernel (independent implementation)."""
import os, sys, json, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_2602_05305_b200 import kernels as K
g = torch.Generator(device="cuda").manual_seed(1234)
groups, rows, d, n = 8, 128, 128, 32768
q = torch.randn((groups, rows, d), device="cuda", generator=g).to(torch.bfloat16)
k = torch.randn((groups, n, d), device="cuda", generator=g).to(torch.bfloat16)
v = torch.randn((groups, n, d), device="cuda", generator=g).to(torch.bfloat16)
a = 12345
def rel(x, y): return ((x - y).abs().max() / y.abs().max()).item()
for rng in [(0, n), (0, a), (a, n)]:
    o, l = K.attention_partial(q, k, v, *rng)
    o32, l32 = K.attention_partial(q.float(), k.float(), v.float(), *rng)
    reps = [K.attention_partial(q, k, v, *rng)[0] for _ in range(5)]
    print(json.dumps({"gbar": os.environ.get("FB_K1_GBAR", "1"), "range": rng, "rel_vs_f32": rel(o, o32),
                      "lse_vs_f32": (l.double() - l32).abs().max().item(),
                      "repeat_maxdiff": max((r - o).abs().max().item() for r in reps)}))
pa = K.attention_partial(q, k, v, 0, a); pb = K.attention_partial(q, k, v, a, n)
o, l = K.attention_partial(q, k, v)
oc, lc = K.combine([pa, pb])
print(json.dumps({"gbar": os.environ.get("FB_K1_GBAR", "1"), "combine_rel": rel(oc, o)}))
