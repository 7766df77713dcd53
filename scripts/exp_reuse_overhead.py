"""Per-call host overhead of the numpy cached step (attention_with_reuse ->
_reuse_host -> fb_internal_merge_host) at C1 shapes, split by stage."""
import os, sys, time, ctypes, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2602_05305_b200.attention as A
from paper_2602_05305_b200 import kernels as K
rng = np.random.default_rng(0)
q = rng.standard_normal((32, 64)).astype(np.float32)
k = rng.standard_normal((4128, 64)).astype(np.float32); v = rng.standard_normal((4128, 64)).astype(np.float32)
e, i = A.attention_streamed(q, k, v, 4096, 0.125); ent = A.CacheEntry(e, 0)
ki, vi = k[4096:], v[4096:]
def t(fn, n=2000):
    fn(); t0 = time.perf_counter()
    for _ in range(n): fn()
    return (time.perf_counter() - t0) / n * 1e6
print("full attention_with_reuse us", round(t(lambda: A.attention_with_reuse(q, ent, ki, vi, 0.125)), 1))
print("_reuse_host us", round(t(lambda: A._reuse_host(q, e, ki, vi, 0.125)), 1))
print("mirror check us", round(t(lambda: e._device_mirror()), 1))
print("_device us", round(t(lambda: A._device()), 1))
print("current_stream us", round(t(lambda: torch.cuda.current_stream(A._device()).cuda_stream), 1))
o_ext, l_ext = e._device_mirror()
out = np.empty(q.shape, np.float32); oi = np.empty(q.shape, np.float32); li = np.empty(32)
cnt = ctypes.c_int64(0)
lib = K._lib.load(); st = torch.cuda.current_stream().cuda_stream
args = (1, q.ctypes.data, ki.ctypes.data, vi.ctypes.data, 1, 32, 64, 32, 0.125, o_ext.data_ptr(), l_ext.data_ptr(),
        out.ctypes.data, oi.ctypes.data, li.ctypes.data, ctypes.addressof(cnt), st)
print("raw C call us", round(t(lambda: lib.fb_internal_merge_host(*args)), 1))
import flashblock.attention as R  # noqa
