"""Cluster split-K K1 (few items: C3 b=1 shards, C2 b <= 4, C4 K8): every
item runs on one thread-block cluster whose CTAs merge their partials
through distributed shared memory (no split workspace, no merge kernel).
The merge is the reference's log-space combine (attention.py:207-233) over a
different key split than the stream-K plan's; P is rounded to bf16 against
each split's own running max, so the two paths agree to bf16 rounding of P
(not bitwise), and both match the float64 oracle within the bf16 bound."""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.fixture
def lib():
    from paper_2602_05305_b200 import _lib

    lb = _lib.load()
    yield lb
    lb.fb_debug_set_k1_cluster(-1)


def _r(g, *s):
    return torch.randn(s, device="cuda", generator=g).to(torch.bfloat16)


def _run(lib, mode, fn):
    lib.fb_debug_set_k1_cluster(mode)
    before = lib.fb_debug_k1_cluster_launches()
    res = fn()
    torch.cuda.synchronize()
    return res, lib.fb_debug_k1_cluster_launches() - before


@pytest.mark.parametrize("groups,q_rows,n", [(8, 128, 16384), (16, 128, 32768), (32, 128, 4096),
                                             (3, 256, 5000), (5, 96, 3001), (2, 128, 700)])
def test_cluster_k1_matches_stream_k_and_oracle(lib, groups, q_rows, n):
    from oracle import flashblock_oracle as orc
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(groups * 1000 + n)
    q, k, v = _r(g, groups, q_rows, 128), _r(g, groups, n, 128), _r(g, groups, n, 128)
    (o_c, l_c), nc = _run(lib, 1, lambda: K.attention_partial(q, k, v, 0, n))
    (o_s, l_s), ns = _run(lib, 0, lambda: K.attention_partial(q, k, v, 0, n))
    assert nc == 1 and ns == 0, "the forced modes did not take the intended paths"
    assert float((o_c - o_s).abs().max()) <= 5e-3 * float(o_s.abs().max())
    assert float((l_c - l_s).abs().max()) <= 1e-4
    for gi in (0, groups - 1):
        ref = orc.partial(q[gi].double().cpu().numpy(), k[gi].double().cpu().numpy(),
                          v[gi].double().cpu().numpy())
        got = o_c[gi].double().cpu().numpy()
        assert np.max(np.abs(got - ref.out)) <= 1e-2 * np.max(np.abs(ref.out))
        assert np.max(np.abs(l_c[gi].double().cpu().numpy() - ref.lognorm)) <= 1e-2


def test_cluster_k1_bf16_partial_is_fp32_rounded(lib):
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(3)
    q, k, v = _r(g, 8, 128, 128), _r(g, 8, 8192, 128), _r(g, 8, 8192, 128)
    lib.fb_debug_set_k1_cluster(1)
    o32, l32 = K.attention_partial(q, k, v)
    ob = torch.empty(o32.shape, device="cuda", dtype=torch.bfloat16)
    lb = torch.empty_like(l32)
    K.attention_partial(q, k, v, out=ob, lse=lb)
    torch.cuda.synchronize()
    assert torch.equal(ob, o32.to(torch.bfloat16)) and torch.equal(lb, l32)


def test_cluster_k1_head_gated_group_subset(lib):
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(4)
    q, k, v = _r(g, 8, 128, 128), _r(g, 8, 6000, 128), _r(g, 8, 6000, 128)
    gl = torch.tensor([6, 1, 3], device="cuda", dtype=torch.int32)
    outs = []
    for mode in (1, 0):
        o = torch.zeros((8, 128, 128), device="cuda")
        l = torch.zeros((8, 128), device="cuda")
        _, n = _run(lib, mode, lambda: K.attention_partial_groups(q, k, v, gl, 0, 6000, out=o, lse=l))
        assert n == (1 if mode == 1 else 0)
        outs.append((o, l))
    (oc, lc), (os_, ls) = outs
    assert float((oc - os_).abs().max()) <= 5e-3 * float(os_.abs().max())
    assert float((lc - ls).abs().max()) <= 1e-4
    assert torch.count_nonzero(oc[[0, 2, 4, 5, 7]]) == 0


@pytest.mark.parametrize("density", [0.1, 0.5])
@pytest.mark.parametrize("with_residual", [True, False])
def test_cluster_sparse_cached_step(lib, density, with_residual):
    """K8 (sparse.py:177-183): gathered selected blocks + current block, the
    cached residual merged in the cluster reduction itself."""
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(int(density * 100) + with_residual)
    groups, rows, n, blk = 8, 128, 16384, 32
    q, k, v = _r(g, groups, rows, 128), _r(g, groups, n, 128), _r(g, groups, n, 128)
    ki, vi = _r(g, groups, blk, 128), _r(g, groups, blk, 128)
    budget = K.mask_budget(n, density, 16)
    sel = K.topk_blocks(K.block_mass(q, k, ki, n, 16), budget)
    res = K.sparse_partitioned(q, k, v, ki, vi, n, sel)[2] if with_residual else None
    q2 = _r(g, groups, rows, 128)
    outs = []
    for mode in (1, 0):
        o, nl = _run(lib, mode, lambda: K.sparse_attend_merge(q2, k, v, ki, vi, n, sel, res, out_dtype=torch.float32))
        assert nl == (1 if mode == 1 else 0)
        outs.append(o)
    assert float((outs[0] - outs[1]).abs().max()) <= 5e-3 * float(outs[1].abs().max())


def test_cluster_large_block_cached_step_with_bf16_ext(lib):
    """Large current block (> 128 keys) over few groups: the K2 path runs K1
    over the block's keys with the merge against the bf16 cached partial
    applied in the cluster reduction."""
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(5)
    groups, q_rows, n_in = 2, 128, 4680
    q, ki, vi = _r(g, groups, q_rows, 128), _r(g, groups, n_in, 128), _r(g, groups, n_in, 128)
    ob = torch.randn((groups, q_rows, 128), device="cuda", generator=g).to(torch.bfloat16)
    le = torch.randn((groups, q_rows), device="cuda", generator=g)
    a, na = _run(lib, 1, lambda: K.internal_merge(q, ki, vi, ob, le, out_dtype=torch.float32))
    b, nb = _run(lib, 0, lambda: K.internal_merge(q, ki, vi, ob, le, out_dtype=torch.float32))
    assert na == 1 and nb == 0
    assert float((a - b).abs().max()) <= 5e-3 * float(b.abs().max())


@pytest.mark.parametrize("n_ext,n_in", [(16384, 32), (4104, 32), (4096, 24)])
def test_gather_atom_layout_is_bitwise_equal(lib, n_ext, n_in):
    """K7 / K8 with the atom smem layout (one 4 KB TMA box per 16-key block)
    compute exactly what the two-box layout does: same tiles, same MMAs."""
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(n_ext + n_in)
    groups, rows = 8, 4 * n_in
    q, k, v = _r(g, groups, rows, 128), _r(g, groups, n_ext, 128), _r(g, groups, n_ext, 128)
    ki, vi = _r(g, groups, n_in, 128), _r(g, groups, n_in, 128)
    budget = K.mask_budget(n_ext, 0.2, 16)
    sel = K.topk_blocks(K.block_mass(q, k, ki, n_ext, 16), budget)
    outs = []
    try:
        for atoms in (1, 0):
            lib.fb_debug_set_gather_atoms(atoms)
            o7, _, res = K.sparse_partitioned(q, k, v, ki, vi, n_ext, sel)
            o8 = K.sparse_attend_merge(_r(torch.Generator(device="cuda").manual_seed(1), groups, rows, 128),
                                       k, v, ki, vi, n_ext, sel, res, out_dtype=torch.float32)
            torch.cuda.synchronize()
            outs.append((o7, res[0], res[1], o8))
    finally:
        lib.fb_debug_set_gather_atoms(-1)
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a, b)


@pytest.mark.parametrize("groups,q_rows,n", [(4, 128, 4096), (3, 64, 2500)])
def test_cluster_k1_head_dim_64(lib, groups, q_rows, n):
    from oracle import flashblock_oracle as orc
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(64 + n)
    q, k, v = _r(g, groups, q_rows, 64), _r(g, groups, n, 64), _r(g, groups, n, 64)
    (o_c, l_c), nc = _run(lib, 1, lambda: K.attention_partial(q, k, v, 0, n))
    (o_s, l_s), _ = _run(lib, 0, lambda: K.attention_partial(q, k, v, 0, n))
    assert nc == 1
    assert float((o_c - o_s).abs().max()) <= 5e-3 * float(o_s.abs().max())
    for gi in range(groups):
        ref = orc.partial(q[gi].double().cpu().numpy(), k[gi].double().cpu().numpy(), v[gi].double().cpu().numpy())
        assert np.max(np.abs(o_c[gi].double().cpu().numpy() - ref.out)) <= 1e-2 * np.max(np.abs(ref.out))


@pytest.mark.parametrize("groups,n", [(8, 16384), (16, 8192), (8, 32768), (3, 6000)])
def test_grid_barrier_split_k(lib, groups, n):
    """Auto mode on few items with 8-16 CTAs each (C3 b=1 shards, C2 b=1/2):
    the item's CTAs meet at a counter in the sync-flag buffer instead of a
    cluster barrier; the counters are left zero for the next launch."""
    from oracle import flashblock_oracle as orc
    from paper_2602_05305_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(groups * 31 + n)
    q, k, v = _r(g, groups, 128, 128), _r(g, groups, n, 128), _r(g, groups, n, 128)
    outs = []
    for rep in range(2):  # twice: the counters must come back zero
        (o_a, l_a), na = _run(lib, -1, lambda: K.attention_partial(q, k, v, 0, n))
        assert na == 1, "the grid-barrier plan was not taken"
        outs.append((o_a, l_a))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    (o_s, l_s), ns = _run(lib, 0, lambda: K.attention_partial(q, k, v, 0, n))
    assert ns == 0
    o_a, l_a = outs[0]
    assert float((o_a - o_s).abs().max()) <= 5e-3 * float(o_s.abs().max())
    assert float((l_a - l_s).abs().max()) <= 1e-4
    for gi in (0, groups - 1):
        ref = orc.partial(q[gi].double().cpu().numpy(), k[gi].double().cpu().numpy(), v[gi].double().cpu().numpy())
        assert np.max(np.abs(o_a[gi].double().cpu().numpy() - ref.out)) <= 1e-2 * np.max(np.abs(ref.out))


@pytest.mark.parametrize("groups,n,expect_split_k", [
    (8, 16384, True),     # C3 b=1 P=8 shard: 8 items x 128 tiles -> 16-CTA groups (grid barrier)
    (32, 131072, False),  # C3 b=4 P=1: 32 items x 1024 tiles; a 4-CTA group would hold 256 tiles
                          # vs 222 on 148-CTA stream-K
])
def test_split_k_plan_keeps_stream_k_for_large_items(lib, groups, n, expect_split_k):
    """The per-item split-K plans (clusters / grid barrier) only for items
    whose power-of-two CTA group stays near the stream-K share of tiles; large
    items stay on 148-CTA stream-K + the split-merge kernel (the 128-CTA plan
    had cost C3 b=8 P=1 12 %).  Both plans agree with the whole-range oracle."""
    from paper_2602_05305_b200 import kernels as K
    from oracle import flashblock_oracle as orc

    g = torch.Generator(device="cuda").manual_seed(groups + n)
    q, k, v = _r(g, groups, 128, 128), _r(g, groups, n, 128), _r(g, groups, n, 128)
    (o, l), launches = _run(lib, -1, lambda: K.attention_partial(q, k, v))
    assert (launches > 0) == expect_split_k
    ref = orc.partial(q[0].double().cpu().numpy(), k[0].double().cpu().numpy(), v[0].double().cpu().numpy())
    assert np.max(np.abs(o[0].cpu().numpy() - ref.out)) <= 1e-2 * np.max(np.abs(ref.out))
    assert np.max(np.abs(l[0].cpu().numpy() - ref.lognorm)) <= 1e-3
