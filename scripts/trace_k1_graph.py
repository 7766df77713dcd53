"""Per-launch kernel start/end (globaltimer) of 36 back-to-back K1 launches in a CUDA graph."""
import os, sys, ctypes, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K, _lib
lib = _lib.load(); lib.fb_debug_set_trace.argtypes = [ctypes.c_void_p]
HKV, D, CTX, L = 8, 128, 32768, 36
b = int(sys.argv[1]) if len(sys.argv) > 1 else 8
nd = int(sys.argv[2]) if len(sys.argv) > 2 else 36
groups = b * HKV
g = torch.Generator(device="cuda").manual_seed(1)
q = torch.randn((groups, 128, D), device="cuda", generator=g).to(torch.bfloat16)
ks = [torch.randn((groups, CTX, D), device="cuda", generator=g).to(torch.bfloat16) for _ in range(nd)]
vs = [torch.randn((groups, CTX, D), device="cuda", generator=g).to(torch.bfloat16) for _ in range(nd)]
o = torch.empty((groups, 128, D), device="cuda", dtype=torch.float32)
l = torch.empty((groups, 128), device="cuda", dtype=torch.float32)
tr = torch.zeros(L * 148 * 8, dtype=torch.int64, device="cuda")
fn = lambda: [K.attention_partial(q, ks[i % nd], vs[i % nd], 0, CTX, None, o, l) for i in range(L)]
fn(); torch.cuda.synchronize()
lib.fb_debug_set_trace(tr.data_ptr())
s = torch.cuda.Stream(); gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr, stream=s): fn()
lib.fb_debug_set_trace(None)
for it in range(3):
    gr.replay()
torch.cuda.synchronize()
t = tr.view(L, 148, 8).cpu().numpy().astype(np.int64)
starts = t[:, :, 0].min(axis=1); ends = np.max(t[:, :, 1:5], axis=(1, 2))
first_start = t[:, :, 0].min(); 
dur = (ends - starts) / 1e3; per = np.diff(starts) / 1e3
print(f"b={b} distinct={nd}: kernel start->last CTA end (us): median {np.median(dur):.1f} min {dur.min():.1f} max {dur.max():.1f}; launch period median {np.median(per):.1f}")
print("first 6 durations", np.round(dur[:6], 1), "periods", np.round(per[:6], 1))
