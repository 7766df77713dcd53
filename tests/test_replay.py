"""f1: the reference's own step driver (run_sequence) replayed with its
attention routed through libfb200.so.  Needs the unmodified reference
installed at baseline/_ref (it travels to the GPU box with the repo)."""

import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def ref():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if not os.path.isdir(os.path.join(REF, "flashblock")):
        pytest.skip("reference not installed at baseline/_ref")
    sys.path.insert(0, REF)
    import flashblock

    return flashblock


@pytest.mark.parametrize("dtype,tau,per_step", [(np.float64, 2, 1), (np.float64, 2, 2),
                                                (np.float32, 2, 1), (np.float64, 1, 1)])
def test_run_sequence_replay_matches_reference(ref, dtype, tau, per_step):
    from paper_2602_05305_b200.replay import patch_reference_simulator

    cfg = ref.ModelConfig(num_layers=2, num_heads=4, head_dim=64, seed=3, dtype=dtype)
    model = ref.SyntheticModel(cfg)
    args = dict(prompt_len=256, num_blocks=2, block_size=32, steps_per_block=16,
                policy=ref.ReuseConfig(tau=tau), verify=True, seed=5, unmask_per_step=per_step)
    base = ref.run_sequence(model, **args)
    with patch_reference_simulator(ref.simulator):
        gpu = ref.run_sequence(model, **args)
    assert [t.decision for t in gpu.traces] == [t.decision for t in base.traces]
    assert [t.updated_tokens for t in gpu.traces] == [t.updated_tokens for t in base.traces]
    assert [t.kv_rows_read for t in gpu.traces] == [t.kv_rows_read for t in base.traces]
    assert [t.keys_attended for t in gpu.traces] == [t.keys_attended for t in base.traces]
    np.testing.assert_array_equal(gpu.final_ids, base.final_ids)
    tol = 1e-9 if dtype == np.float64 else 1e-4
    for a, b in zip(gpu.traces, base.traces):
        assert abs(a.checksum - b.checksum) <= tol * max(1.0, abs(b.checksum))
        assert abs(a.linf_gap - b.linf_gap) <= tol * 10 + 1e-12
    # the reuse steps never touched the committed cache (tests/test_simulator.py:109-125 there)
    assert all(t.external_rows_read == 0 for t in gpu.traces if t.decision == "Reuse")


def test_sparse_gap_replay(ref):
    from paper_2602_05305_b200.replay import patch_reference_simulator

    model = ref.SyntheticModel(ref.ModelConfig(num_layers=2, num_heads=2, head_dim=8, seed=0))
    base = ref.measure_sparse_gap(model, [0.25, 0.5, 1.0], layer=0, seed=7, prompt_len=64,
                                  block_size=8)
    with patch_reference_simulator(ref.simulator, ref.sparse):
        gpu = ref.measure_sparse_gap(model, [0.25, 0.5, 1.0], layer=0, seed=7, prompt_len=64,
                                     block_size=8)
    for a, b in zip(gpu, base):
        assert a.density == b.density
        assert abs(a.l1_sparse_only - b.l1_sparse_only) <= 1e-12
        assert abs(a.l1_with_residual - b.l1_with_residual) <= 1e-12
