"""K6 stable top-k (fb_topk_blocks) against the reference rule
(sparse.py:127-128: a stable argsort of -mass truncated to the budget,
returned ascending) on adversarial mass sets: exact ties at the cut,
all-equal masses, ties spread over several radix bins, tiny / huge
exponents, zeros, and sizes around the radix early exit (<= 32 candidates
left in the k-th key's bin) and the smem / bitonic / rank fallbacks."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _ref(mass: np.ndarray, budget: int) -> np.ndarray:
    order = np.argsort(-mass, kind="stable")
    return np.sort(order[:budget])


def _cases(rng):
    nb = 4096
    yield "random", rng.random(nb) * 1e-3, 410
    m = rng.random(nb)
    m[rng.choice(nb, 300, replace=False)] = m.max() * 0.5  # a big tie block straddling the cut
    yield "tie_at_cut", m, int((m > m.max() * 0.5).sum()) + 100
    yield "all_equal", np.full(nb, 0.25), 1000
    m = np.repeat(rng.random(64), nb // 64)  # 64 distinct values, 64 copies each
    yield "repeated", rng.permutation(m), 777
    m = np.exp(rng.normal(0, 30, nb))  # exponents over many binades
    yield "wide_exponents", m, 2048
    m = rng.random(nb)
    m[: nb // 2] = 0.0
    yield "half_zero", m, 3000  # budget reaches into the zeros
    m = np.full(nb, 1.0)
    m[:40] = 2.0  # the k-th key's bin holds <= 32 keys right after the first pass
    yield "few_candidates", m, 20
    yield "budget_all", rng.random(nb), nb
    yield "budget_one", rng.random(nb), 1
    yield "tiny", rng.random(7), 3
    yield "large_nb", rng.random(30000), 3000  # beyond the smem radix path


@pytest.mark.parametrize("groups", [1, 3])
def test_topk_equals_stable_argsort(groups):
    from paper_2602_05305_b200 import kernels as K

    rng = np.random.default_rng(17)
    for name, mass, budget in _cases(rng):
        masses = np.stack([mass if g == 0 else rng.permutation(mass) for g in range(groups)])
        got = K.topk_blocks(torch.from_numpy(masses).cuda(), budget).cpu().numpy()
        for g in range(groups):
            np.testing.assert_array_equal(got[g], _ref(masses[g], budget), err_msg=name)
