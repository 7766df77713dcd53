"""Split-KV refresh through the real kernels in two processes sharing one GPU
(SURVEY §8e): each rank runs K1 (tcgen05) on its half of a 128K context,
the packed (O, LSE) partials go through ONE gloo exchange staged in host
memory (NCCL cannot put two ranks on one device), and K3 merges them.  The
merged partial must equal K1 over the whole key range (exact by
associativity, verification.py:99-117; here within bf16-P rounding), for
both exchange layouts.  The NCCL path runs the same code with device
buffers (bench.py --gpus N).

The ``p2p`` layout needs no collective on the data path: the two processes
map each other's partial buffers through CUDA IPC (same device here, NVLink
peers on a node), signal / wait on device flags, and K3 reads the peer's
partial in place; three refreshes with different queries exercise the
double-buffered slots and the monotone flags."""

import os
import socket

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, layout, result_q):
    import torch.distributed as dist

    from paper_2602_05305_b200 import kernels as K
    from paper_2602_05305_b200.splitkv import SplitKVRefresh, group_chunks, shard_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N, groups, rows, d = 131072, 8, 128, 128
        g = torch.Generator(device="cuda").manual_seed(2024)  # same tensors on every rank
        q = torch.randn((groups, rows, d), device="cuda", generator=g).to(torch.bfloat16)
        k = torch.randn((groups, N, d), device="cuda", generator=g).to(torch.bfloat16)
        v = torch.randn((groups, N, d), device="cuda", generator=g).to(torch.bfloat16)
        lo, hi = shard_bounds(N, world, rank)
        ks, vs = k[:, lo:hi].contiguous(), v[:, lo:hi].contiguous()
        ref = SplitKVRefresh(layout=layout)
        c0, c1 = group_chunks(groups, world)[rank] if layout in ("all_to_all", "p2p") else (0, groups)
        err_o = err_l = 0.0
        for it in range(3 if layout == "p2p" else 1):
            qi = (q.float() * (1.0 + 0.5 * it)).to(torch.bfloat16)
            o, l = ref(qi, ks, vs, hi - lo)
            assert ref.host_staged == (layout != "p2p")
            o_full, l_full = K.attention_partial(qi, k, v)
            err_o = max(err_o, ((o.float() - o_full[c0:c1]).abs().amax() / o_full[c0:c1].abs().amax()).item())
            err_l = max(err_l, (l - l_full[c0:c1]).abs().max().item())
        result_q.put((rank, err_o, err_l, tuple(o.shape)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("layout", ["all_gather", "all_to_all", "p2p"])
def test_split_kv_two_ranks_one_gpu_equals_whole_range(layout):
    import torch.multiprocessing as mp

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, layout, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    res = [q.get(timeout=10) for _ in range(2)]
    for rank, err_o, err_l, shape in res:
        assert err_o <= 5e-3 and err_l <= 1e-3, (rank, err_o, err_l)
        assert shape[0] == (8 if layout == "all_gather" else 4)
