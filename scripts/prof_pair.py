"""One C5 refresh launch (12 heads x 4680 rows x 56,160 keys) with the pair
kernel (argv[1] == 'pair') or the single-CTA kernel, for ncu captures."""
import ctypes, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import _lib, kernels as K
lib = _lib.load(); lib.fb_debug_set_pair.argtypes = [ctypes.c_int]
lib.fb_debug_set_pair(1 if sys.argv[1] == "pair" else 0)
g = torch.Generator(device="cuda").manual_seed(1)
r = lambda *s: torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)
mode = sys.argv[2] if len(sys.argv) > 2 else "c5"
if mode == "c5":
    q, k, v = r(12, 4680, 128), r(12, 56160, 128), r(12, 56160, 128)
    o, l = K.attention_partial(q, k, v)
    torch.cuda.synchronize()
    o, l = K.attention_partial(q, k, v, 0, None, None, o, l)
else:
    n_q = 32768
    q, k, v = r(8, 4 * n_q, 128), r(8, n_q, 128), r(8, n_q, 128)
    o, l = K.block_causal_attention(q, k, v, n_q, 0, 32)
    torch.cuda.synchronize()
    o, l = K.block_causal_attention(q, k, v, n_q, 0, 32, None, o, l)
torch.cuda.synchronize()
print("done")
