"""Reference-named attention API on the B200 kernels (drop-in for
flashblock/attention.py).

Same names, argument order, defaults, return types and exceptions as the
reference module (attention.py:35-321).  Inputs may be numpy arrays (results
come back as numpy, with the reference's dtypes: ``out`` in the tensor dtype,
``lognorm`` float64) or CUDA torch tensors (results stay on the device;
bfloat16 inputs give float32 partials).  Every computation runs in
libfb200.so; there is no CPU path.

``tile_size`` is validated exactly like the reference but does not change the
GPU tiling: the reference's results are tile-size independent up to float
rounding (tests/test_attention.py:128-134 there).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import kernels as K
from .errors import (BoundsError, DegenerateInputError, ReusePreconditionError,  # noqa: F401
                     ShapeError)

__all__ = [
    "DegenerateInputError",
    "ReusePreconditionError",
    "AttnPartial",
    "CacheEntry",
    "ExternalAttnCache",
    "attention_dense",
    "attention_partial",
    "attention_streamed",
    "combine_partials",
    "merge_partials",
    "attention_with_reuse",
]

DEFAULT_TILE = 64  # attention.py:49


def _is_np(x) -> bool:
    return isinstance(x, np.ndarray)


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2602_05305_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev(x, dtype=None) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x if x.is_cuda else x.to(_device())
        return t if dtype is None else t.to(dtype)
    a = np.ascontiguousarray(x)
    if a.dtype not in (np.float64, np.float32):
        a = a.astype(np.float64)
    t = torch.from_numpy(a).to(_device(), non_blocking=False)
    return t if dtype is None else t.to(dtype)


def _common_dtype(*arrs) -> torch.dtype:
    """Promotion the reference gets from numpy: float64 wins over float32."""
    kinds = set()
    for a in arrs:
        if isinstance(a, torch.Tensor):
            kinds.add(a.dtype)
        else:
            kinds.add({np.dtype(np.float32): torch.float32}.get(np.asarray(a).dtype, torch.float64))
    if torch.float64 in kinds:
        return torch.float64
    if torch.float32 in kinds:
        return torch.float32
    return torch.bfloat16


def _check_qkv(q, keys, values) -> None:
    # attention.py:104-110
    if q.ndim != 2 or keys.ndim != 2 or values.ndim != 2:
        raise ShapeError("q, keys and values must be 2-D")
    if keys.shape[1] != q.shape[1]:
        raise ShapeError(f"key dim {keys.shape[1]} != query dim {q.shape[1]}")
    if values.shape[0] != keys.shape[0]:
        raise ShapeError(f"{values.shape[0]} value rows for {keys.shape[0]} keys")


def _widen(qt, kt, vt):
    """The kernels take one head_dim for q, k and v; the reference allows a
    value width d_v != d (its shift-stability check attends [n, 17] keys with
    [n, 16] values, verification.py:137-147).  Zero columns are exact padding:
    appended to q and k they add 0 * 0 to every score, appended to v they give
    zero output columns that are sliced off.  Returns (q, k, v, d_v)."""
    d, dv = qt.shape[-1], vt.shape[-1]
    if dv == d:
        return qt, kt, vt, dv
    if dv < d:
        vt = torch.cat([vt, vt.new_zeros(vt.shape[:-1] + (d - dv,))], dim=-1)
    else:
        qt = torch.cat([qt, qt.new_zeros(qt.shape[:-1] + (dv - d,))], dim=-1)
        kt = torch.cat([kt, kt.new_zeros(kt.shape[:-1] + (dv - d,))], dim=-1)
    return qt, kt, vt, dv


@dataclass
class AttnPartial:
    """Normalised partial output plus per-row log-normaliser (attention.py:60-101).

    ``out`` [nq, d] in the tensor dtype (float32 for bf16 device inputs);
    ``lognorm`` [nq] float64 (float32 in the bf16 device mode).  Empty rows
    carry lognorm = -inf and a zero output row.
    """

    out: np.ndarray | torch.Tensor
    lognorm: np.ndarray | torch.Tensor

    @classmethod
    def empty(cls, num_queries: int, head_dim: int, dtype=np.float64) -> "AttnPartial":
        return cls(out=np.zeros((num_queries, head_dim), dtype=dtype),
                   lognorm=np.full(num_queries, -np.inf, dtype=np.float64))

    @property
    def num_queries(self) -> int:
        return self.out.shape[0]

    @property
    def head_dim(self) -> int:
        return self.out.shape[1]

    @property
    def nbytes(self) -> int:
        if isinstance(self.out, torch.Tensor):
            return self.out.numel() * self.out.element_size() + \
                self.lognorm.numel() * self.lognorm.element_size()
        return self.out.nbytes + self.lognorm.nbytes

    def empty_rows(self):
        if isinstance(self.lognorm, torch.Tensor):
            return torch.isneginf(self.lognorm)
        return np.isneginf(self.lognorm)

    def copy(self) -> "AttnPartial":
        return AttnPartial(self.out.copy() if _is_np(self.out) else self.out.clone(),
                           self.lognorm.copy() if _is_np(self.lognorm) else self.lognorm.clone())


def _partial_dev(q, keys, values, scale, begin=0, end=None):
    """Device partial of keys[begin:end] for the 2-D reference signature."""
    dt = _common_dtype(q, keys, values)
    qt, kt, vt, dv = _widen(_to_dev(q, dt), _to_dev(keys, dt), _to_dev(values, dt))
    o, l = K.attention_partial(qt, kt, vt, begin, end, scale)
    return o[..., :dv], l


def _wrap(o3, l3, as_numpy: bool, out_np_dtype=None) -> AttnPartial:
    o, l = o3[0], l3[0]
    if as_numpy:
        o_np = o.cpu().numpy()
        if out_np_dtype is not None:
            o_np = o_np.astype(out_np_dtype, copy=False)
        return AttnPartial(o_np, l.cpu().numpy().astype(np.float64, copy=False))
    return AttnPartial(o, l)


def attention_dense(q, keys, values, scale: float | None = None):
    """Full softmax attention over all keys (attention.py:113-133).

    Output is float64 for numpy inputs, as the reference; on the device the
    whole computation runs in float64 for float64/float32 inputs (the
    reference widens to float64 first) and in the bf16 tensor-core mode for
    bfloat16 tensors (float32 output).
    """
    _check_qkv(q, keys, values)
    if keys.shape[0] == 0:
        raise DegenerateInputError("dense attention needs at least one key")
    if scale is None:
        scale = 1.0 / math.sqrt(q.shape[1])
    dt = _common_dtype(q, keys, values)
    if dt != torch.bfloat16:
        dt = torch.float64
    qt, kt, vt, dv = _widen(_to_dev(q, dt), _to_dev(keys, dt), _to_dev(values, dt))
    o, _ = K.attention_partial(qt, kt, vt, 0, None, scale)
    o = o[..., :dv]
    if _is_np(q):
        return o[0].cpu().numpy().astype(np.float64, copy=False)
    return o[0]


def attention_partial(q, keys, values, scale: float | None = None,
                      tile_size: int = DEFAULT_TILE) -> AttnPartial:
    """Streamed partial over one key group (attention.py:136-182); zero keys
    give the empty sentinel."""
    _check_qkv(q, keys, values)
    if tile_size < 1:
        raise ValueError("tile_size must be >= 1")
    if scale is None:
        scale = 1.0 / math.sqrt(q.shape[1])
    o, l = _partial_dev(q, keys, values, scale)
    return _wrap(o, l, _is_np(q), q.dtype if _is_np(q) else None)


def attention_streamed(q, keys, values, boundary: int, scale: float | None = None,
                       tile_size: int = DEFAULT_TILE) -> tuple[AttnPartial, AttnPartial]:
    """(external [0, boundary), internal [boundary, end)) partials of one key
    stream (attention.py:185-204).  One device upload, two kernel ranges."""
    _check_qkv(q, keys, values)
    if not 0 <= boundary <= keys.shape[0]:
        raise BoundsError(f"boundary {boundary} outside [0, {keys.shape[0]}]")
    if tile_size < 1:
        raise ValueError("tile_size must be >= 1")
    if scale is None:
        scale = 1.0 / math.sqrt(q.shape[1])
    dt = _common_dtype(q, keys, values)
    qt, kt, vt, dv = _widen(_to_dev(q, dt), _to_dev(keys, dt), _to_dev(values, dt))
    n = kt.shape[0]
    eo, el = K.attention_partial(qt, kt, vt, 0, boundary, scale)
    io, il = K.attention_partial(qt, kt, vt, boundary, n, scale)
    eo, io = eo[..., :dv], io[..., :dv]
    np_out = q.dtype if _is_np(q) else None
    return _wrap(eo, el, _is_np(q), np_out), _wrap(io, il, _is_np(q), np_out)


def _partial_to_dev(p: AttnPartial):
    if isinstance(p.out, torch.Tensor):
        return p.out, p.lognorm
    out = np.ascontiguousarray(p.out)
    if out.dtype not in (np.float32, np.float64):
        out = out.astype(np.float64)
    return (torch.from_numpy(out).to(_device()),
            torch.from_numpy(np.ascontiguousarray(p.lognorm, dtype=np.float64)).to(_device()))


def combine_partials(a: AttnPartial, b: AttnPartial) -> AttnPartial:
    """Log-space merge of two partials over disjoint key groups
    (attention.py:207-233); one-side-empty rows pass through bitwise."""
    if tuple(a.out.shape) != tuple(b.out.shape):
        raise ShapeError(f"partial shapes differ: {tuple(a.out.shape)} vs {tuple(b.out.shape)}")
    ao, al = _partial_to_dev(a)
    bo, bl = _partial_to_dev(b)
    if ao.dtype != bo.dtype:  # numpy promotion in the reference's weighted sum
        wide = torch.float64 if torch.float64 in (ao.dtype, bo.dtype) else ao.dtype
        ao, bo = ao.to(wide), bo.to(wide)
    if al.dtype != bl.dtype:
        al, bl = al.to(torch.float64), bl.to(torch.float64)
    if ao.shape[0] == 0:
        out = (ao.clone(), al.clone())
    else:
        out = K.combine([(ao, al), (bo, bl)], out_dtype=ao.dtype)
    if _is_np(a.out):
        return AttnPartial(out[0].cpu().numpy().astype(a.out.dtype, copy=False),
                           out[1].cpu().numpy().astype(np.float64, copy=False))
    return AttnPartial(out[0], out[1])


def merge_partials(external: AttnPartial, internal: AttnPartial):
    """combine_partials(...).out, raising DegenerateInputError when a row has
    no keys on either side (attention.py:236-245)."""
    merged = combine_partials(external, internal)
    empty = merged.empty_rows()
    if bool(empty.any()):
        raise DegenerateInputError("some query rows have no keys on either side")
    return merged.out


@dataclass
class CacheEntry:
    """One cached external partial for a (layer, head) pair (attention.py:248-255)."""

    partial: AttnPartial
    step_created: int
    block_id: int = -1
    valid: bool = True


class ExternalAttnCache:
    """Per-(layer, head) store of the current block's external partials
    (attention.py:258-292).  Entries hold device or host partials by
    reference; size is nq*(d+1) scalars per entry regardless of context."""

    def __init__(self) -> None:
        self._entries: dict[tuple[int, int], CacheEntry] = {}

    def put(self, layer: int, head: int, partial: AttnPartial, step: int,
            block_id: int = -1) -> None:
        self._entries[(layer, head)] = CacheEntry(partial, step, block_id)

    def get(self, layer: int, head: int) -> CacheEntry | None:
        return self._entries.get((layer, head))

    def is_valid(self, layer: int, head: int) -> bool:
        entry = self._entries.get((layer, head))
        return entry is not None and entry.valid

    def invalidate_all(self) -> None:
        self._entries.clear()

    def resident_bytes(self) -> int:
        return sum(e.partial.nbytes for e in self._entries.values() if e.valid)


def attention_with_reuse(q, entry: CacheEntry | None, internal_keys, internal_values,
                         scale: float | None = None, tile_size: int = DEFAULT_TILE):
    """Cached step (attention.py:295-321): fresh internal partial fused with the
    merge against the cached external partial, in one kernel that never sees
    the KV cache.  Returns (merged output, internal partial)."""
    if entry is None or not entry.valid:
        raise ReusePreconditionError("no valid cached external partial")
    if entry.partial.num_queries != q.shape[0]:
        raise ReusePreconditionError(
            f"cached partial has {entry.partial.num_queries} query rows, got {q.shape[0]}")
    _check_qkv(q, internal_keys, internal_values)
    if tile_size < 1:
        raise ValueError("tile_size must be >= 1")
    if scale is None:
        scale = 1.0 / math.sqrt(q.shape[1])
    dt = _common_dtype(q, internal_keys, internal_values)
    qt, kt, vt, dv = _widen(_to_dev(q, dt), _to_dev(internal_keys, dt), _to_dev(internal_values, dt))
    eo, el = _partial_to_dev(entry.partial)
    if eo.shape[-1] != dv:
        raise ShapeError(f"cached partial has {eo.shape[-1]} value columns, internal values {dv}")
    ot, lt = K.PARTIAL_TYPES[K.dtype_code(qt)]
    eo, el = eo.to(ot), el.to(lt)
    if eo.shape[-1] < qt.shape[-1]:
        eo = torch.cat([eo, eo.new_zeros(eo.shape[:-1] + (qt.shape[-1] - dv,))], dim=-1)
    out, lse_m, (io, il) = K.internal_merge(qt, kt, vt, eo, el, scale, want_lse=True,
                                            want_internal=True)
    out, io = out[..., :dv], io[..., :dv]
    if bool(torch.isneginf(lse_m).any()):
        raise DegenerateInputError("some query rows have no keys on either side")
    if _is_np(q):
        return (out[0].cpu().numpy().astype(q.dtype, copy=False),
                AttnPartial(io[0].cpu().numpy().astype(q.dtype, copy=False),
                            il[0].cpu().numpy().astype(np.float64, copy=False)))
    return out[0], AttnPartial(io[0], il[0])
