"""Split-KV context parallelism for the refresh pass.

The committed context of one sequence is split along N across the P ranks
of one node.  Each rank runs K1 over its shard, giving an fp32 partial
(O_p, LSE_p) over disjoint key groups; ONE collective exchanges the
partials and K3 merges them -- exact by the associativity of the log-space
merge (attention.py:207-233; reference check verification.py:99-117).
Cached steps read no KV and exchange nothing.

Two exchange layouts:
  * ``all_gather``  -- every rank receives all P partials and merges all
    groups (replicated O_ext; the next cached step can run on any rank).
  * ``all_to_all``  -- group-sharded: rank r receives the P partials of its
    groups only (groups split into P contiguous chunks) and merges those
    (each rank then owns O_ext for its kv-head shard -- the TP layout).

The local partial and the merge default to the CUDA kernels (K1, K3); the
hooks exist so the collective choreography can be tested with world-size-2
``gloo`` process groups on CPU, where tests pass oracle-backed callables.
"""

from __future__ import annotations

from dataclasses import dataclass
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
CombineFn = Callable[[list], tuple[torch.Tensor, torch.Tensor]]


def _default_partial(q, k, v, n_local, scale):
    from . import kernels as K

    return K.attention_partial(q, k, v, 0, n_local, scale)


def _default_combine(parts):
    from . import kernels as K

    return K.combine(parts)


@dataclass
class SplitKVRefresh:
    """Refresh over a KV cache sharded along the sequence across a process group."""

    group: dist.ProcessGroup | None = None
    layout: str = "all_gather"
    local_partial: PartialFn = _default_partial
    combine: CombineFn = _default_combine

    def __post_init__(self):
        if self.layout not in ("all_gather", "all_to_all"):
            raise ValueError(f"unknown layout {self.layout!r}")

    def __call__(self, q, k_shard, v_shard, n_local: int, scale: float | None = None):
        """q [groups, rows, d]; k/v_shard [groups, cap_local, d] with this rank's
        n_local committed rows.  Returns (o, lse): all groups for all_gather,
        this rank's group chunk for all_to_all."""
        on = dist.is_available() and dist.is_initialized()
        world = dist.get_world_size(self.group) if on else 1
        o, l = self.local_partial(q, k_shard, v_shard, n_local, scale)
        groups = o.shape[0]
        if world == 1:
            return o, l
        if self.layout == "all_gather":
            # concatenated along dim 0 (the form every backend accepts), viewed as [P, ...]
            o_all = torch.empty((world * o.shape[0],) + tuple(o.shape[1:]), dtype=o.dtype,
                                device=o.device)
            l_all = torch.empty((world * l.shape[0],) + tuple(l.shape[1:]), dtype=l.dtype,
                                device=l.device)
            dist.all_gather_into_tensor(o_all, o.contiguous(), group=self.group)
            dist.all_gather_into_tensor(l_all, l.contiguous(), group=self.group)
            return self._merge(o_all.view(world, *o.shape), l_all.view(world, *l.shape))
        # all_to_all: rank r gets every rank's partial for its group chunk
        chunks = group_chunks(groups, world)
        if any(hi - lo != chunks[0][1] - chunks[0][0] for lo, hi in chunks):
            raise ShapeError(f"all_to_all needs groups ({groups}) divisible by world ({world})")
        per = chunks[0][1] - chunks[0][0]
        o_in = o.contiguous().view(world, per, *o.shape[1:])
        l_in = l.contiguous().view(world, per, *l.shape[1:])
        o_out = torch.empty_like(o_in)
        l_out = torch.empty_like(l_in)
        dist.all_to_all_single(o_out, o_in, group=self.group)
        dist.all_to_all_single(l_out, l_in, group=self.group)
        return self._merge(o_out, l_out)

    def _merge(self, o_all, l_all):
        parts = [(o_all[p], l_all[p]) for p in range(o_all.shape[0])]
        out = None
        # K3 takes up to 16 partials per launch; fold larger worlds in chunks
        while len(parts) > 1 or out is None:
            chunk, parts = parts[:16], parts[16:]
            out = self.combine(chunk)
            if not parts:
                break
            parts = [out] + parts
        return out
