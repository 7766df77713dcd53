"""Split-KV exchange choreography on CPU: world_size 2 with the gloo backend.

The device kernels are replaced by oracle-backed callables (the CPU cannot
run sm_100a code); what is under test is the sharding arithmetic, the
collective layout (all_gather / all_to_all) and the merge order, against the
oracle's single-process partial over the whole key set.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import flashblock_oracle as orc
from paper_2602_05305_b200.splitkv import (SplitKVRefresh, group_chunks, least_filled,
                                           shard_bounds)


def test_shard_bounds_cover_exactly():
    for n in (0, 1, 7, 100, 131072, 131073):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def test_least_filled_and_group_chunks():
    assert least_filled([5, 3, 3, 9]) == 1
    assert group_chunks(8, 2) == [(0, 4), (4, 8)]


def _oracle_partial(q, k, v, n_local, scale, out, lse):
    if out is None:
        out = torch.empty(q.shape, dtype=torch.float64)
        lse = torch.empty(q.shape[:2], dtype=torch.float64)
    for g in range(q.shape[0]):
        p = orc.partial(q[g].numpy(), k[g, :n_local].numpy(), v[g, :n_local].numpy(), scale)
        out[g] = torch.from_numpy(p.out)
        lse[g] = torch.from_numpy(p.lognorm)
    return out, lse


def _oracle_combine(parts, out=None, lse=None):
    o, l = parts[0]
    acc = orc.Partial(o.numpy(), l.numpy())
    for o2, l2 in parts[1:]:
        acc = orc.combine(acc, orc.Partial(o2.numpy(), l2.numpy()))
    if out is not None:
        out.copy_(torch.from_numpy(acc.out))
        lse.copy_(torch.from_numpy(acc.lognorm))
        return out, lse
    return torch.from_numpy(acc.out), torch.from_numpy(acc.lognorm)


def _worker(rank, world, port, layout, n, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.Generator(np.random.Philox(77))
        groups, rows, d = 4, 6, 8
        q = torch.from_numpy(rng.standard_normal((groups, rows, d)))
        k = torch.from_numpy(rng.standard_normal((groups, n, d)))
        v = torch.from_numpy(rng.standard_normal((groups, n, d)))
        lo, hi = shard_bounds(n, world, rank)
        cap = hi - lo + 3  # slack rows past the committed length must be ignored
        ks = torch.zeros((groups, cap, d), dtype=torch.float64)
        vs = torch.full((groups, cap, d), float("nan"), dtype=torch.float64)
        ks[:, :hi - lo] = k[:, lo:hi]
        vs[:, :hi - lo] = v[:, lo:hi]
        ref = SplitKVRefresh(layout=layout, local_partial=_oracle_partial, combine=_oracle_combine)
        o, l = ref(q, ks, vs, hi - lo, None)
        chunk = group_chunks(groups, world)[rank] if layout == "all_to_all" else (0, groups)
        err = 0.0
        for gi, g in enumerate(range(*chunk)):
            full = orc.partial(q[g].numpy(), k[g].numpy(), v[g].numpy())
            err = max(err, float(np.max(np.abs(o[gi].numpy() - full.out))),
                      float(np.max(np.abs(l[gi].numpy() - full.lognorm))))
        result_q.put((rank, err))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("layout", ["all_gather", "all_to_all"])
@pytest.mark.parametrize("n,world", [(50, 2), (1, 2), (37, 4)])
def test_split_kv_gloo_matches_single_process(layout, n, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, layout, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    errs = dict(q.get(timeout=10) for _ in range(world))
    assert max(errs.values()) < 1e-12, errs


def test_split_kv_single_process_without_group():
    # no process group: the refresh is the local partial (world size 1)
    rng = np.random.Generator(np.random.Philox(5))
    q = torch.from_numpy(rng.standard_normal((2, 3, 8)))
    k = torch.from_numpy(rng.standard_normal((2, 10, 8)))
    v = torch.from_numpy(rng.standard_normal((2, 10, 8)))
    o, l = SplitKVRefresh(local_partial=_oracle_partial, combine=_oracle_combine)(q, k, v, 10)
    full = orc.partial(q[1].numpy(), k[1].numpy(), v[1].numpy())
    np.testing.assert_allclose(o[1].numpy(), full.out, atol=1e-13)
