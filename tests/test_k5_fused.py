"""Fused single-pass K5 (score_fused_kernel + score_mass_kernel) against the
LSE + MASS two-pass kernels and the float64 oracle (sparse.py:117-128).

The fused pass reads K once: per (row, 16-key block) exp-sums relative to the
row's quarter-tile max, weighted by exp2(max - lse2_row) once the row LSE is
final.  Same mathematics as the two passes, different fp32 rounding order, so
masses agree to ~1e-6 relative and the selections agree exactly unless two
blocks sit within that error of the cut.  Shapes cover ragged external /
current-block tails (partial quarter tiles, fully masked quarters), q_rows <
128, head_dim 64, an item split over several CTAs (stream-K LSE partials
merged in the reduce kernel), and the paged cache.
"""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import flashblock_oracle as orc  # noqa: E402


@pytest.fixture(scope="module")
def lib():
    from paper_2602_05305_b200 import _lib

    L = _lib.load()
    L.fb_debug_set_k5_mode.argtypes = [ctypes.c_int]
    L.fb_debug_k5_fused_launches.restype = ctypes.c_int64
    yield L
    L.fb_debug_set_k5_mode(-1)


def _mass(lib, mode, q, k, kin, n_ext, page_table=None):
    from paper_2602_05305_b200 import kernels as K

    lib.fb_debug_set_k5_mode(mode)
    try:
        before = lib.fb_debug_k5_fused_launches()
        m = K.block_mass(q, k, kin, n_ext, 16, page_table=page_table)
        torch.cuda.synchronize()
        fused_ran = lib.fb_debug_k5_fused_launches() > before
    finally:
        lib.fb_debug_set_k5_mode(-1)
    return m, fused_ran


@pytest.mark.parametrize("groups,q_rows,d,n_ext,n_in", [
    (4, 128, 128, 4096, 32),      # whole tiles
    (3, 128, 128, 1000, 32),      # ragged external tail (partial + fully masked quarters)
    (2, 96, 128, 2050, 0),        # q_rows < 128, no current block
    (5, 128, 128, 300, 200),      # current block spanning two tiles
    (2, 128, 64, 3000, 32),       # head_dim 64
    (40, 128, 128, 16384, 32),    # items split over several CTAs (stream-K LSE partials)
    (3, 1, 128, 17, 1),           # one query row, a 1-key tail block, a 1-key current block
    (2, 33, 64, 16, 5),           # a single external block, odd row count
])
def test_fused_mass_equals_two_pass_and_oracle(lib, groups, q_rows, d, n_ext, n_in):
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(groups * 7919 + n_ext)
    q = torch.randn((groups, q_rows, d), device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn((groups, n_ext + n_in, d), device="cuda", generator=g).to(torch.bfloat16)
    kin = k[:, n_ext:].contiguous()
    mf, fused_ran = _mass(lib, 0, q, k, kin, n_ext)
    mt, _ = _mass(lib, 1, q, k, kin, n_ext)
    assert fused_ran, "fused K5 did not run"
    assert torch.isfinite(mf).all()
    rel = ((mf - mt).abs() / mt.abs().clamp_min(1e-300)).max().item()
    assert rel <= 2e-6, rel
    # float64 oracle on two groups (bf16-exact inputs, fp32 scores on the device)
    for gi in (0, groups - 1):
        ref = orc.block_mass(q[gi].double().cpu().numpy(), k[gi].double().cpu().numpy(), n_ext, 16)
        assert np.max(np.abs(mf[gi].cpu().numpy() - ref)) <= 1e-5 * np.max(ref) + 1e-9
    # selections: equal, or differing only where two-pass masses tie within the error
    budget = K.mask_budget(n_ext, 0.1, 16)
    sf = K.topk_blocks(mf, budget).cpu().numpy()
    st = K.topk_blocks(mt, budget).cpu().numpy()
    mtn = mt.cpu().numpy()
    for gi in range(groups):
        diff = set(sf[gi].tolist()) ^ set(st[gi].tolist())
        kth = np.sort(mtn[gi])[::-1][budget - 1]
        for b in diff:
            assert abs(mtn[gi, b] - kth) <= 4 * rel * kth + 1e-300


def test_fused_mass_paged_equals_contiguous(lib):
    """Paged K pool read through a shuffled page table: bitwise equal masses."""
    groups, q_rows, d, n_ext, n_in, page = 3, 128, 128, 2000, 32, 256
    g = torch.Generator(device="cuda").manual_seed(11)
    q = torch.randn((groups, q_rows, d), device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn((groups, n_ext + n_in, d), device="cuda", generator=g).to(torch.bfloat16)
    kin = k[:, n_ext:].contiguous()
    pages_per = -(-n_ext // page)
    pool = torch.zeros((groups * pages_per + 3, page, d), device="cuda", dtype=torch.bfloat16)
    perm = torch.randperm(pool.shape[0] - 3, generator=torch.Generator().manual_seed(3)).cuda() + 3
    table = perm.view(groups, pages_per).to(torch.int32)
    for gi in range(groups):
        for p in range(pages_per):
            rows = k[gi, p * page:min((p + 1) * page, n_ext)]
            pool[table[gi, p], :rows.shape[0]] = rows
    mc, ran_c = _mass(lib, 0, q, k, kin, n_ext)
    mp, ran_p = _mass(lib, 0, q, pool, kin, n_ext, page_table=table)
    assert ran_c and ran_p
    assert torch.equal(mc, mp)


def test_fused_mass_is_deterministic(lib):
    g = torch.Generator(device="cuda").manual_seed(5)
    q = torch.randn((16, 128, 128), device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn((16, 8192 + 32, 128), device="cuda", generator=g).to(torch.bfloat16)
    kin = k[:, 8192:].contiguous()
    a, _ = _mass(lib, 0, q, k, kin, 8192)
    b, _ = _mass(lib, 0, q, k, kin, 8192)
    assert torch.equal(a, b)
