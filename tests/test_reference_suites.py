"""The reference's own invariant suite and acceptance criteria, run through the
device path.

``replay.patch_reference`` swaps the attention names that the reference's
step driver (simulator.py:28-34), sparse module (sparse.py:19-25) and
invariant suite (verification.py:14) import, so every attention evaluation
below runs in libfb200.so while the reference's own model, policy, KV cache,
counters and checks stay untouched.  Needs the unmodified reference installed
at baseline/_ref (it travels to the GPU box with the repo).

* ``verification.run_all`` (verification.py:222-247): decomposition
  exactness, merge associativity, +80 shift stability, no-KV-touch and
  baseline equivalence, each at the reference's own tolerances.
* The acceptance criteria of tests/test_acceptance.py (there) 1-8, restated
  with the same inputs, seeds and thresholds (criterion 9 is the CLI's
  byte-identical re-runs, out of scope: SURVEY §2).
"""

import os
import re
import sys
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
SEED = 20260824  # tests/test_acceptance.py:40 there


@pytest.fixture(scope="module")
def fb():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if not os.path.isdir(os.path.join(REF, "flashblock")):
        pytest.skip("reference not installed at baseline/_ref")
    sys.path.insert(0, REF)
    import flashblock
    import flashblock.analysis
    import flashblock.bench
    import flashblock.verification

    return flashblock


@pytest.fixture
def on_gpu(fb):
    from paper_2602_05305_b200 import _lib
    from paper_2602_05305_b200.replay import patch_reference

    before = _lib.load().fb_launch_count()
    with patch_reference(fb):
        yield
    # the device path really ran
    assert _lib.load().fb_launch_count() > before


def test_verification_run_all_on_device(fb, on_gpu):
    """verification.run_all (verification.py:222-247) with its default sizes."""
    results = fb.verification.run_all(seed=0)
    lines = [r.line() for r in results]
    assert [r.name for r in results] == ["decomposition-exactness", "merge-associativity",
                                         "shift-stability", "no-kv-touch", "baseline-equivalence"]
    assert all(r.passed for r in results), "\n".join(lines)


@pytest.mark.parametrize("seed", [1, 7])
def test_verification_checks_other_seeds(fb, on_gpu, seed):
    v = fb.verification
    for r in (v.check_decomposition(16, seed, max_n=512), v.check_merge_associativity(100, seed),
              v.check_shift_stability(40, seed)):
        assert r.passed, r.line()


def test_acceptance_1_split_plus_merge_matches_dense(fb, on_gpu):
    """test_acceptance.py:52-86 there: >= 1000 instances, float64 < 1e-10,
    float32 < 1e-3, under 60 s."""
    from paper_2602_05305_b200.attention import attention_dense, attention_streamed, merge_partials

    t0 = time.perf_counter()
    res = fb.verification.check_decomposition(200, seed=SEED)
    m = re.search(r"float32_err=([0-9.e+-]+) \((\d+) problems", res.detail)
    worst64, worst32, problems = res.max_err, float(m.group(1)), int(m.group(2))
    rng = np.random.Generator(np.random.Philox(SEED))
    for n in (8, 12, 16):
        for d in (8, 16, 32):
            q = rng.standard_normal((5, d))
            k = rng.standard_normal((n, d))
            v = rng.standard_normal((n, d))
            ref = attention_dense(q, k, v)
            q32, k32, v32 = (a.astype(np.float32) for a in (q, k, v))
            for boundary in range(n + 1):
                ext, inn = attention_streamed(q, k, v, boundary)
                worst64 = max(worst64, float(np.max(np.abs(merge_partials(ext, inn) - ref))))
                e32, i32 = attention_streamed(q32, k32, v32, boundary)
                worst32 = max(worst32, float(np.max(np.abs(merge_partials(e32, i32) - ref))))
                problems += 1
    elapsed = time.perf_counter() - t0
    assert problems >= 1000
    assert worst64 < 1e-10 and worst32 < 1e-3, (worst64, worst32)
    assert elapsed < 60.0 and res.passed


def test_acceptance_2_merge_order_invariant_and_shift_immune(fb, on_gpu):
    """test_acceptance.py:89-98 there."""
    assoc = fb.verification.check_merge_associativity(300, seed=SEED)
    shift = fb.verification.check_shift_stability(100, seed=SEED)
    assert assoc.passed and assoc.max_err < 1e-10, assoc.line()
    assert shift.passed and shift.max_err < 1e-6, shift.line()


def test_acceptance_3_reuse_steps_never_touch_committed_rows(fb, on_gpu):
    """test_acceptance.py:101-133 there: zero committed-row delta on reuse
    steps and the cache counters reconcile exactly."""
    model = fb.SyntheticModel(fb.ModelConfig(seed=0))
    run = fb.run_sequence(model, 64, 2, 8, 8, fb.ReuseConfig(tau=2), seed=0, unmask_per_step=1)
    reuse = [t for t in run.traces if t.decision == "Reuse"]
    assert reuse and max(t.external_rows_read for t in reuse) == 0
    assert max(abs(t.keys_attended - 8.0) for t in reuse) == 0.0
    per_pair = model.config.num_layers * model.config.num_heads
    expected = (sum(j * 8 for j in range(8)) + 64 + 72) * per_pair
    for i, t in enumerate(run.traces):
        if t.decision != "Reuse":
            expected += (64 + (i // 8) * 8) * per_pair
    c = run.kv.snapshot_counters()
    assert expected == c.key_rows_read == c.value_rows_read
    assert fb.verification.check_no_kv_touch(seed=0).passed


def test_acceptance_4_reuse_work_flat_dense_linear(fb, on_gpu):
    """test_acceptance.py:136-176 there."""
    model = fb.SyntheticModel(fb.ModelConfig(seed=0))
    contexts = (128, 512, 2048, 8192)
    dense_mean, dense_total, reuse_total, reuse_rows, reuse_counts = [], [], [], set(), []
    for context in contexts:
        dense = fb.run_sequence(model, context, 1, 8, 32, fb.ReuseConfig(tau=2, mode="always-recompute"),
                                seed=0, unmask_per_step=1)
        reuse = fb.run_sequence(model, context, 1, 8, 32, fb.ReuseConfig(tau=2), seed=0, unmask_per_step=1)
        rows_d = [t.kv_rows_read for t in dense.traces]
        dense_mean.append(float(np.mean(rows_d)))
        dense_total.append(float(np.sum(rows_d)))
        reuse_total.append(float(np.sum([t.kv_rows_read for t in reuse.traces])))
        steps = [t for t in reuse.traces if t.decision == "Reuse"]
        reuse_counts.append(len(steps))
        reuse_rows.update(t.kv_rows_read for t in steps)
    slope, intercept = np.polyfit(contexts, dense_mean, 1)
    pred = slope * np.asarray(contexts) + intercept
    r2 = 1.0 - float(np.sum((np.asarray(dense_mean) - pred) ** 2)) / \
        float(np.sum((np.asarray(dense_mean) - np.mean(dense_mean)) ** 2))
    rel = (reuse_total[-1] / reuse_total[0]) / (dense_total[-1] / dense_total[0])
    assert 0.9 <= slope <= 1.1 and r2 > 0.99
    assert reuse_rows == {8.0} and min(reuse_counts) > 0 and rel <= 0.55


def test_acceptance_5_cached_partial_size_independent_of_context(fb, on_gpu):
    """test_acceptance.py:179-193 there (the cache holds the device path's
    partials, returned in the reference's dtypes)."""
    from flashblock.simulator import denoise_step, new_block_state, prefill, prompt_ids

    sizes = {}
    for context in (128, 1024, 8192):
        model = fb.SyntheticModel(fb.ModelConfig(seed=0))
        kv = prefill(model, prompt_ids(model, context, 0), 8)
        ext = fb.ExternalAttnCache()
        state = new_block_state(0, context, 8)
        denoise_step(model, state, kv, ext, fb.ReuseConfig(tau=2), unmask_count=1)
        sizes[context] = ext.resident_bytes()
    assert len(set(sizes.values())) == 1 and sizes[128] == 4 * 4 * (8 * 16 + 8) * 8


def test_acceptance_6_cached_residual_tightens_the_sparse_gap(fb, on_gpu):
    """test_acceptance.py:196-220 there: K5/K6 select, K7/K8 attend."""
    densities = [0.1, 0.2, 0.3, 0.4, 0.5, 1.0]
    rows = fb.bench.sweep_density(densities, 100, layer=0)
    partial = [r for r in rows if r.density < 1.0]
    dominance = float(np.mean([r.l1_with_residual <= r.l1_sparse_only for r in partial]))
    full_worst = max(max(r.l1_sparse_only, r.l1_with_residual) for r in rows if r.density == 1.0)
    ms = [float(np.mean([r.l1_sparse_only for r in rows if r.density == d])) for d in densities[:5]]
    mr = [float(np.mean([r.l1_with_residual for r in rows if r.density == d])) for d in densities[:5]]
    mono = all(ms[i + 1] <= ms[i] for i in range(4)) and all(mr[i + 1] <= mr[i] for i in range(4))
    assert dominance >= 0.99 and full_worst < 1e-9 and mono, (dominance, full_worst, ms, mr)


def test_acceptance_7_match_rate_never_improves_with_larger_threshold(fb, on_gpu):
    """test_acceptance.py:223-236 there."""
    from flashblock.simulator import quality_probe

    model = fb.SyntheticModel(fb.ModelConfig(seed=0))
    dense = fb.ReuseConfig(mode="always-recompute")
    rates = [quality_probe(model, dense, fb.ReuseConfig(tau=tau), 50).match_fraction for tau in (1, 2, 4, 9)]
    assert rates[0] == 1.0 and all(rates[i + 1] <= rates[i] for i in range(3)), rates


def test_acceptance_8_external_partials_stable_under_internal_noise(fb, on_gpu):
    """test_acceptance.py:239-256 there."""
    worst_out, worst_in = 1.0, -1.0
    for model_seed, study_seed in ((3, 11), (11, 111), (42, 142)):
        model = fb.SyntheticModel(fb.ModelConfig(num_layers=1, seed=model_seed, step_scale=0.0,
                                                 internal_kv_noise=2.0))
        result = fb.analysis.stability_study(model, steps=6, seed=study_seed, unmask_per_step=0)
        assert not result.empty()
        worst_out = min(worst_out, min(r.mean_diag_out for r in result.records))
        worst_in = max(worst_in, max(r.mean_diag_in for r in result.records))
    assert worst_out >= 0.999 and worst_in < 0.9, (worst_out, worst_in)


def test_value_width_differs_from_key_width(fb, on_gpu):
    """d_v != d (the shift check's [n, 17] keys with [n, 16] values) in both
    directions, against the reference functions themselves."""
    from paper_2602_05305_b200 import attention as A

    ref = sys.modules["flashblock.attention"]
    rng = np.random.Generator(np.random.Philox(3))
    for d, dv in ((17, 16), (8, 24)):
        q = rng.standard_normal((5, d))
        k = rng.standard_normal((40, d))
        v = rng.standard_normal((40, dv))
        np.testing.assert_allclose(A.attention_dense(q, k, v), ref.attention_dense(q, k, v), atol=1e-12)
        e, i = A.attention_streamed(q, k, v, 25)
        re, ri = ref.attention_streamed(q, k, v, 25)
        assert e.out.shape == (5, dv)
        np.testing.assert_allclose(A.merge_partials(e, i), ref.merge_partials(re, ri), atol=1e-12)
        out, _ = A.attention_with_reuse(q, A.CacheEntry(e, 0, 0), k[25:], v[25:])
        rout, _ = ref.attention_with_reuse(q, ref.CacheEntry(re, 0, 0), k[25:], v[25:])
        np.testing.assert_allclose(out, rout, atol=1e-12)
