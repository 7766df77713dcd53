import sys, os, numpy as np, importlib.util, torch
sys.path.insert(0, os.getcwd())
import paper_2602_05305_b200.attention as new
spec = importlib.util.spec_from_file_location("paper_2602_05305_b200.attention_old", os.environ.get("OLD_ATTENTION", "scripts/_attention_old.py"))
old = importlib.util.module_from_spec(spec); sys.modules[spec.name] = old; spec.loader.exec_module(old)
rng = np.random.default_rng(0)
for dt in (np.float32, np.float64):
    q = rng.standard_normal((8, 16)).astype(dt); k = rng.standard_normal((170, 16)).astype(dt); v = rng.standard_normal((170, 16)).astype(dt)
    for name in ("attention_dense",):
        a = getattr(new, name)(q, k, v); b = getattr(old, name)(q, k, v); print(name, dt.__name__, np.abs(a - b).max())
    a = new.attention_partial(q, k, v); b = old.attention_partial(q, k, v); print("partial", np.abs(a.out - b.out).max(), np.abs(a.lognorm - b.lognorm).max())
    sel = rng.permutation(170)[:100]
    a = new.attention_partial(q, k[sel], v[sel]); b = old.attention_partial(q, k[sel], v[sel]); print("partial sel", np.abs(a.out - b.out).max())
    e1, i1 = new.attention_streamed(q, k, v, 160); e2, i2 = old.attention_streamed(q, k, v, 160)
    print("streamed", np.abs(e1.out - e2.out).max(), np.abs(i1.out - i2.out).max(), np.abs(e1.lognorm - e2.lognorm).max())
    m1 = new.merge_partials(e1, i1); m2 = old.merge_partials(e2, i2); print("merge", np.abs(m1 - m2).max())
    ent = new.CacheEntry(e1, 0); ent2 = old.CacheEntry(e2, 0)
    o1, p1 = new.attention_with_reuse(q, ent, k[160:], v[160:]); o2, p2 = old.attention_with_reuse(q, ent2, k[160:], v[160:])
    print("reuse", np.abs(o1 - o2).max(), np.abs(p1.out - p2.out).max(), o1.dtype, o2.dtype)
