import sys, os, time, numpy as np, importlib.util, torch
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "baseline", "_ref"))
import paper_2602_05305_b200.attention as new
spec = importlib.util.spec_from_file_location("paper_2602_05305_b200.attention_old", os.environ.get("OLD_ATTENTION", "scripts/_attention_old.py"))
old = importlib.util.module_from_spec(spec); sys.modules[spec.name] = old; spec.loader.exec_module(old)
import flashblock.attention as R
rng = np.random.default_rng(0)
q = rng.standard_normal((32, 64)).astype(np.float32); k = rng.standard_normal((4128, 64)).astype(np.float32); v = rng.standard_normal((4128, 64)).astype(np.float32)
def t(fn, n=200):
    fn(); t0 = time.perf_counter()
    for _ in range(n): fn()
    return (time.perf_counter() - t0) / n * 1e6
for name, M in (("new", new), ("old", old), ("cpu", R)):
    e, i = M.attention_streamed(q, k, v, 4096, 0.125)
    ent = M.CacheEntry(e, 0)
    print(name, "reuse_us", round(t(lambda: M.attention_with_reuse(q, ent, k[4096:], v[4096:], 0.125)), 1),
          "streamed_us", round(t(lambda: M.attention_streamed(q, k, v, 4096, 0.125), 50), 1),
          "merge_us", round(t(lambda: M.merge_partials(e, i)), 1))
e, i = new.attention_streamed(q, k, v, 4096, 0.125); ent = new.CacheEntry(e, 0)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(20): new.attention_with_reuse(q, ent, k[4096:], v[4096:], 0.125)
print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=25))
