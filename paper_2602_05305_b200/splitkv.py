"""Split-KV context parallelism for the refresh pass.

The committed context of one sequence is split along N across the P ranks
of one node.  Each rank runs K1 over its shard, giving a partial
(O_p, LSE_p) over disjoint key groups; ONE exchange moves the partials and K3
merges them -- exact by the associativity of the log-space merge
(attention.py:207-233; reference check verification.py:99-117).  Cached steps
read no KV and exchange nothing.

K1 writes O and LSE into one packed byte buffer ``[O (groups, rows, d) |
LSE (groups, rows)]`` so the exchange is a single operation:

  * ``all_gather``  -- one ``all_gather_into_tensor`` of the packed buffer;
    every rank receives all P partials and merges all groups (replicated
    O_ext; the next cached step can run on any rank).
  * ``all_to_all``  -- group-sharded: rank r receives the P partials of its
    group chunk only (groups split into P contiguous chunks) and merges those
    (each rank then owns O_ext for its kv-head shard -- the TP layout).  The
    O and LSE slices for every peer go out as one grouped point-to-point
    exchange (``batch_isend_irecv``: with NCCL one ncclGroupStart/End, one
    kernel launch); the local chunk never leaves the device.

  * ``p2p``         -- the same group-chunk result with no collective on the
    data path: every rank's packed partial lives in device memory the other
    ranks have mapped through CUDA IPC (``P2PExchange``); after K1 a rank
    signals a flag in every peer's flag array, waits until all P flags of
    this refresh are set (device-side, system-scope acquire), and K3 merges
    its group chunk reading the P partials in place over NVLink.  Partial
    buffers are double-buffered by refresh parity, so a rank's next K1 never
    overwrites a partial a peer is still merging.

The local partial and the merge default to the CUDA kernels (K1, K3); the
hooks exist so the collective choreography can be tested with world-size-2
``gloo`` process groups on CPU, where tests pass oracle-backed callables.
With a gloo group and CUDA tensors the packed buffer is staged through host
memory (``host_staged``), which lets several processes share one GPU in
tests; NCCL groups exchange device memory directly.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable

import torch
import torch.distributed as dist

from .errors import ShapeError


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous row range [lo, hi) of rank `rank` (first n % world ranks get +1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def least_filled(lengths: list[int]) -> int:
    """Rank that receives the next committed block (ties -> lowest rank)."""
    return min(range(len(lengths)), key=lambda r: (lengths[r], r))


def group_chunks(groups: int, world: int) -> list[tuple[int, int]]:
    return [shard_bounds(groups, world, r) for r in range(world)]


PartialFn = Callable[..., tuple[torch.Tensor, torch.Tensor]]
CombineFn = Callable[..., tuple[torch.Tensor, torch.Tensor]]

# (O dtype, LSE dtype) of a partial for each input dtype (kernels.PARTIAL_TYPES)
_PARTIAL_DTYPES = {torch.bfloat16: (torch.float32, torch.float32),
                   torch.float32: (torch.float32, torch.float64),
                   torch.float64: (torch.float64, torch.float64)}


def _default_partial(q, k, v, n_local, scale, out, lse):
    from . import kernels as K

    return K.attention_partial(q, k, v, 0, n_local, scale, out=out, lse=lse)


def _default_combine(parts, out=None, lse=None):
    from . import kernels as K

    return K.combine(parts, out=out, lse=lse)


class PackedPartial:
    """One byte buffer holding a partial's O [groups, rows, d] then its LSE
    [groups, rows] (LSE offset rounded up to 16 bytes, the whole record to 256
    so stacked records keep the kernels' vector alignment)."""

    def __init__(self, groups: int, rows: int, d: int, in_dtype: torch.dtype, device, lead: int = 0):
        self.ot, self.lt = _PARTIAL_DTYPES[in_dtype]
        self.shape = (groups, rows, d)
        self.o_bytes = groups * rows * d * torch.empty((), dtype=self.ot).element_size()
        self.l_off = -(-self.o_bytes // 16) * 16
        self.l_end = self.l_off + groups * rows * torch.empty((), dtype=self.lt).element_size()
        self.nbytes = -(-self.l_end // 256) * 256
        lead_shape = (lead,) if lead else ()
        self.buf = torch.empty(lead_shape + (self.nbytes,), dtype=torch.uint8, device=device)

    def views(self, buf: torch.Tensor):
        g, r, d = self.shape
        o = buf[..., :self.o_bytes].view(self.ot).view(buf.shape[:-1] + (g, r, d))
        l = buf[..., self.l_off:self.l_end].view(self.lt).view(buf.shape[:-1] + (g, r))
        return o, l


@dataclass
class SplitKVRefresh:
    """Refresh over a KV cache sharded along the sequence across a process group."""

    group: dist.ProcessGroup | None = None
    layout: str = "all_gather"
    local_partial: PartialFn = _default_partial
    combine: CombineFn = _default_combine
    # filled per call: whether the last exchange went through host memory
    host_staged: bool = field(default=False, init=False)

    def __post_init__(self):
        if self.layout not in ("all_gather", "all_to_all", "p2p"):
            raise ValueError(f"unknown layout {self.layout!r}")
        self._p2p: dict = {}

    def close(self) -> None:
        """Release the peer-memory exchanges (layout "p2p"): collective, call on
        every rank once no refresh is in flight."""
        for ex in self._p2p.values():
            ex.close()
        self._p2p.clear()

    def _stage(self, t: torch.Tensor) -> bool:
        return t.is_cuda and dist.get_backend(self.group) == "gloo"

    def __call__(self, q, k_shard, v_shard, n_local: int, scale: float | None = None, out=None, lse=None):
        """q [groups, rows, d]; k/v_shard [groups, cap_local, d] with this rank's
        n_local committed rows.  Returns (o, lse): all groups for all_gather,
        this rank's group chunk for all_to_all (written into out / lse when
        given)."""
        on = dist.is_available() and dist.is_initialized()
        world = dist.get_world_size(self.group) if on else 1
        rank = dist.get_rank(self.group) if on else 0
        groups, rows, d = q.shape
        if world == 1:  # nothing to exchange: K1 straight into the destination
            return self.local_partial(q, k_shard, v_shard, n_local, scale, out, lse)
        if self.layout == "p2p":
            key = (groups, rows, d, q.dtype, q.device)
            ex = self._p2p.get(key)
            if ex is None:
                ex = self._p2p[key] = P2PExchange(groups, rows, d, q.dtype, q.device, self.group)
            self.host_staged = False
            return ex.refresh(lambda o, l: self.local_partial(q, k_shard, v_shard, n_local, scale, o, l),
                              out, lse)
        pk = PackedPartial(groups, rows, d, q.dtype, q.device)
        o, l = pk.views(pk.buf)
        self.local_partial(q, k_shard, v_shard, n_local, scale, o, l)
        if self.layout == "all_gather":
            return self._merge(self._all_gather(pk, world), out, lse)
        chunks = group_chunks(groups, world)
        if any(hi - lo != chunks[0][1] - chunks[0][0] for lo, hi in chunks):
            raise ShapeError(f"all_to_all needs groups ({groups}) divisible by world ({world})")
        lo, hi = chunks[rank]
        parts = self._all_to_all(o, l, chunks, rank, world)
        parts[rank] = (o[lo:hi], l[lo:hi])
        return self._merge(parts, out, lse)

    def _all_gather(self, pk: PackedPartial, world: int):
        stage = self._stage(pk.buf)
        self.host_staged = stage
        src = pk.buf.cpu() if stage else pk.buf
        dst = torch.empty((world, pk.nbytes), dtype=torch.uint8, device=src.device)
        dist.all_gather_into_tensor(dst.view(-1), src, group=self.group)
        if stage:
            dst = dst.to(pk.buf.device)
        o_all, l_all = pk.views(dst)
        return [(o_all[p], l_all[p]) for p in range(world)]

    def _all_to_all(self, o, l, chunks, rank: int, world: int):
        stage = self._stage(o)
        self.host_staged = stage
        per = chunks[0][1] - chunks[0][0]
        dev = torch.device("cpu") if stage else o.device
        src_o = o.cpu() if stage else o
        src_l = l.cpu() if stage else l
        recv_o = torch.empty((world, per) + tuple(o.shape[1:]), dtype=o.dtype, device=dev)
        recv_l = torch.empty((world, per) + tuple(l.shape[1:]), dtype=l.dtype, device=dev)
        ops = []
        for p in range(world):
            if p == rank:
                continue
            plo, phi = chunks[p]
            peer = p if self.group is None else dist.get_global_rank(self.group, p)
            ops.append(dist.P2POp(dist.isend, src_o[plo:phi], peer, self.group, tag=0))
            ops.append(dist.P2POp(dist.isend, src_l[plo:phi], peer, self.group, tag=1))
            ops.append(dist.P2POp(dist.irecv, recv_o[p], peer, self.group, tag=0))
            ops.append(dist.P2POp(dist.irecv, recv_l[p], peer, self.group, tag=1))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        if stage:
            recv_o, recv_l = recv_o.to(o.device), recv_l.to(l.device)
        return [(recv_o[p], recv_l[p]) for p in range(world)]

    def _merge(self, parts, out=None, lse=None):
        # K3 takes up to 16 partials per launch; fold larger worlds in chunks
        res = None
        while True:
            chunk, parts = parts[:16], parts[16:]
            last = not parts
            res = self.combine(chunk, out=out if last else None, lse=lse if last else None)
            if last:
                return res
            parts = [res] + parts


class _CudaMem:
    """__cuda_array_interface__ of raw device bytes (a P2P allocation), so
    torch can wrap it without a copy."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


class P2PExchange:
    """Peer-memory split-KV exchange of one partial shape.

    Collective at construction (every rank of ``group``): each rank allocates
    a double-buffered packed-partial region and a flag array [world] of
    uint64 (``fb_p2p_alloc``), the 64-byte IPC handles are all-gathered, and
    every peer's region / flags are mapped (``fb_p2p_open``).  ``refresh``
    then runs with no collective:

      1. K1 writes this rank's partial into its region's slot (epoch % 2);
      2. ``fb_p2p_signal`` stores epoch + 1 into slot `rank` of every rank's
         flag array (system-scope fence + release store);
      3. ``fb_p2p_wait`` blocks the stream until all `world` flags of this
         rank reach epoch + 1 (every peer's K1 of this refresh is done);
      4. K3 (``fb_combine``) merges this rank's group chunk straight out of
         the `world` mapped partials.

    A rank's K1 of refresh e + 2 is stream-ordered after its wait of refresh
    e + 1, which saw every peer's signal e + 1, itself ordered after that
    peer's merge of refresh e -- so slot e % 2 is free again (no second
    handshake).  Requires groups divisible by the world size and <= 32 ranks.
    """

    def __init__(self, groups: int, rows: int, d: int, in_dtype: torch.dtype, device, group=None):
        from . import _lib

        self.lib = _lib.load()
        self._lib = _lib
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world > 32:
            raise ValueError("p2p exchange: at most 32 ranks")
        chunks = group_chunks(groups, self.world)
        if any(hi - lo != chunks[0][1] - chunks[0][0] for lo, hi in chunks):
            raise ShapeError(f"p2p exchange needs groups ({groups}) divisible by world ({self.world})")
        self.chunks = chunks
        self.device = torch.device(device)
        self.pk = PackedPartial(groups, rows, d, in_dtype, "meta")
        self.rows, self.d = rows, d
        self.nbytes = self.pk.nbytes
        self._opened: list[int] = []
        self._owned: list[int] = []
        region, h_region = self._alloc(2 * self.nbytes)
        flags, h_flags = self._alloc(8 * self.world)
        handles = [None] * self.world
        dist.all_gather_object(handles, (h_region, h_flags), group=group)
        self.regions, flag_ptrs = [], []
        for p, (hr, hf) in enumerate(handles):
            if p == self.rank:
                self.regions.append(region)
                flag_ptrs.append(flags)
            else:
                self.regions.append(self._open(hr))
                flag_ptrs.append(self._open(hf))
        self.my_flags = flags
        self.flag_ptrs = torch.tensor(flag_ptrs, dtype=torch.int64, device=self.device)
        local = torch.as_tensor(_CudaMem(region, 2 * self.nbytes), device=self.device)
        self.local = [local[i * self.nbytes:(i + 1) * self.nbytes] for i in range(2)]
        self.epoch = 0

    def _alloc(self, nbytes: int):
        import ctypes

        ptr = ctypes.c_void_p()
        h = (ctypes.c_ubyte * 64)()
        with torch.cuda.device(self.device):
            self._lib.call("fb_p2p_alloc", nbytes, ctypes.addressof(ptr), ctypes.addressof(h))
        self._owned.append(ptr.value)
        return ptr.value, bytes(h)

    def _open(self, handle: bytes) -> int:
        import ctypes

        ptr = ctypes.c_void_p()
        h = (ctypes.c_ubyte * 64).from_buffer_copy(handle)
        with torch.cuda.device(self.device):
            self._lib.call("fb_p2p_open", ctypes.addressof(h), ctypes.addressof(ptr))
        self._opened.append(ptr.value)
        return ptr.value

    def close(self) -> None:
        """Unmap the peers and free this rank's buffers (call on every rank
        once no refresh is in flight)."""
        torch.cuda.synchronize(self.device)
        for p in self._opened:
            self.lib.fb_p2p_close(p)
        for p in self._owned:
            self.lib.fb_p2p_free(p)
        self._opened, self._owned = [], []

    def refresh(self, local_partial, out=None, lse=None):
        from . import kernels as K

        slot = self.epoch % 2
        o, l = self.pk.views(self.local[slot])
        local_partial(o, l)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        value = self.epoch + 1
        self._lib.call("fb_p2p_signal", self.flag_ptrs.data_ptr(), self.world, self.rank, value, stream)
        self._lib.call("fb_p2p_wait", self.my_flags, self.world, value, stream)
        lo, hi = self.chunks[self.rank]
        osz, lsz = o.element_size(), l.element_size()
        o_parts = [r + slot * self.nbytes + lo * self.rows * self.d * osz for r in self.regions]
        l_parts = [r + slot * self.nbytes + self.pk.l_off + lo * self.rows * lsz for r in self.regions]
        code = K.mode_of_partial(o, l)
        shape = (hi - lo, self.rows, self.d)
        if out is None:
            out = torch.empty(shape, dtype=o.dtype, device=self.device)
        if lse is None:
            lse = torch.empty(shape[:2], dtype=l.dtype, device=self.device)
        if tuple(out.shape) != shape or tuple(lse.shape) != shape[:2] or not (out.is_contiguous()
                                                                           and lse.is_contiguous()):
            raise ShapeError(f"p2p exchange: out / lse must be contiguous {shape} / {shape[:2]}")
        K._check_partial_out(code, out, lse)
        self._lib.call("fb_combine", code, self.world, self._lib.ptr_array(o_parts), self._lib.ptr_array(l_parts),
                       (hi - lo) * self.rows, self.d, out.data_ptr(), K._OUT_CODE[out.dtype], lse.data_ptr(),
                       None, stream)
        self.epoch += 1
        return out, lse
