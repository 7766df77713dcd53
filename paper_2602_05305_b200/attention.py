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

import ctypes
import math
import threading
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


_CUDA_OK = None
_DEVICES: dict[int, torch.device] = {}


def _device():
    global _CUDA_OK
    if _CUDA_OK is None:
        _CUDA_OK = torch.cuda.is_available()
    if not _CUDA_OK:
        raise RuntimeError("paper_2602_05305_b200 needs a CUDA device (no CPU fallback)")
    idx = torch.cuda.current_device()
    dev = _DEVICES.get(idx)
    if dev is None:
        dev = _DEVICES[idx] = torch.device("cuda", idx)
    return dev


def _raw_stream(dev: torch.device) -> int:
    """cudaStream_t of the current torch stream on `dev` (the cheap internal
    query when this torch build has it)."""
    get = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if get is not None:
        return get(dev.index)
    return torch.cuda.current_stream(dev).cuda_stream


def _to_dev(x, dtype=None) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x if x.is_cuda else x.to(_device())
        return t if dtype is None else t.to(dtype)
    a = np.ascontiguousarray(x)
    if a.dtype not in (np.float64, np.float32):
        a = a.astype(np.float64)
    t = torch.from_numpy(a).to(_device(), non_blocking=False)
    return t if dtype is None else t.to(dtype)


class _Staging:
    """Pinned host staging for the numpy drop-in path: a call's numpy inputs
    are packed into one pinned buffer and uploaded with ONE host->device copy;
    its results come back by async device->host copies into pinned memory and
    ONE stream synchronisation (the reference API is synchronous numpy, so a
    call must return host arrays).  Buffers are reused across calls: every
    call ends with that synchronisation, so no copy is in flight when the next
    call overwrites them.  Not shared between threads (see _ThreadStaging)."""

    def __init__(self):
        self._up: torch.Tensor | None = None
        self._down: torch.Tensor | None = None
        self._up_done: torch.cuda.Event | None = None  # the last upload's copy

    @staticmethod
    def _grow(buf, nbytes):
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes, 1 << 16) * 2, dtype=torch.uint8, pin_memory=True)
        return buf

    def upload(self, dt: torch.dtype, arrays) -> list[torch.Tensor]:
        np_dt = np.float64 if dt == torch.float64 else np.float32
        item = np.dtype(np_dt).itemsize
        sizes = [int(np.prod(a.shape)) for a in arrays]
        total = sum(sizes)
        if self._up_done is not None:  # a call that raised before its download never synchronised
            self._up_done.synchronize()
        self._up = self._grow(self._up, total * item)
        host = self._up[:total * item].numpy().view(np_dt)
        off = 0
        for a, n in zip(arrays, sizes):
            host[off:off + n] = np.asarray(a).reshape(-1)
            off += n
        dev = torch.empty(total, dtype=dt, device=_device())
        dev.copy_(self._up[:total * item].view(dt), non_blocking=True)
        if self._up_done is None:
            self._up_done = torch.cuda.Event()
        self._up_done.record()
        out, off = [], 0
        for a, n in zip(arrays, sizes):
            out.append(dev[off:off + n].view(a.shape))
            off += n
        return out

    def download(self, tensors) -> list[np.ndarray]:
        """Host copies (own memory) of device tensors, one synchronisation."""
        offs, total = [], 0
        for t in tensors:
            total = (total + 7) // 8 * 8
            offs.append(total)
            total += t.numel() * t.element_size()
        self._down = self._grow(self._down, total)
        views = []
        for t, o in zip(tensors, offs):
            nb = t.numel() * t.element_size()
            hv = self._down[o:o + nb].view(t.dtype)
            hv.copy_(t.reshape(-1), non_blocking=True)
            views.append(hv)
        torch.cuda.current_stream(_device()).synchronize()
        return [v.numpy().reshape(tuple(t.shape)).copy() for v, t in zip(views, tensors)]


class _ThreadStaging(threading.local):
    """One staging area per host thread: the reference calls its attention
    functions from worker threads (bench.sweep_density's thread_map)."""

    def __init__(self):
        self.stage = _Staging()

    def upload(self, dt, arrays):
        return self.stage.upload(dt, arrays)

    def download(self, tensors):
        return self.stage.download(tensors)


_STAGE = _ThreadStaging()


def _np_mode_dtype(*arrs) -> torch.dtype:
    """Device dtype for numpy inputs: float64 if any input is float64 (numpy
    promotion in the reference), float32 if all are float32, else float64."""
    if all(isinstance(a, np.ndarray) and a.dtype == np.float32 for a in arrs):
        return torch.float32
    return torch.float64


def _all_np(*arrs) -> bool:
    return all(isinstance(a, np.ndarray) for a in arrs)


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

    # numpy partials made by this module keep the device tensors they were
    # read back from (and host snapshots to detect in-place edits), so a later
    # cached step / merge does not upload them again
    def _set_mirror(self, o_dev: torch.Tensor, l_dev: torch.Tensor) -> "AttnPartial":
        self.__dict__["_mirror"] = (o_dev, l_dev, self.out, self.lognorm, self.out.tobytes(),
                                    self.lognorm.tobytes())
        return self

    def _device_mirror(self):
        m = self.__dict__.get("_mirror")
        if m is None:
            return None
        o_dev, l_dev, out_obj, ln_obj, out_snap, ln_snap = m
        # byte snapshots: an in-place edit (even one that keeps NaN != NaN) drops the mirror
        if self.out is not out_obj or self.lognorm is not ln_obj \
                or self.out.tobytes() != out_snap or self.lognorm.tobytes() != ln_snap:
            self.__dict__.pop("_mirror", None)
            return None
        return o_dev, l_dev

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


def _upload_qkv(q, keys, values):
    """(q, keys, values) on the device in the call's precision mode; numpy
    inputs go up in one pinned host->device copy."""
    dt = _common_dtype(q, keys, values)
    if _all_np(q, keys, values):
        return _STAGE.upload(dt, [q, keys, values])
    return [_to_dev(q, dt), _to_dev(keys, dt), _to_dev(values, dt)]


def _partial_dev(q, keys, values, scale, begin=0, end=None):
    """Device partial of keys[begin:end] for the 2-D reference signature."""
    qt, kt, vt, dv = _widen(*_upload_qkv(q, keys, values))
    o, l = K.attention_partial(qt, kt, vt, begin, end, scale)
    return o[..., :dv], l


def _wrap_many(parts, as_numpy: bool, out_np_dtype=None) -> list[AttnPartial]:
    """AttnPartials from device (o3, l3) pairs; numpy results come back with
    one synchronisation and keep their device tensors as a mirror when no
    dtype cast was applied (the mirror then equals an upload of the arrays)."""
    devs = [(o3[0], l3[0]) for o3, l3 in parts]
    if not as_numpy:
        return [AttnPartial(o, l) for o, l in devs]
    hosts = _STAGE.download([t for pair in devs for t in pair])
    res = []
    for i, (o, l) in enumerate(devs):
        o_np, l_np = hosts[2 * i], hosts[2 * i + 1]
        exact = out_np_dtype is None or np.dtype(out_np_dtype) == o_np.dtype
        if out_np_dtype is not None:
            o_np = o_np.astype(out_np_dtype, copy=False)
        exact = exact and l_np.dtype == np.float64
        p = AttnPartial(o_np, l_np.astype(np.float64, copy=False))
        if exact and o.is_contiguous() and l.is_contiguous():
            p._set_mirror(o, l)
        res.append(p)
    return res


def _wrap(o3, l3, as_numpy: bool, out_np_dtype=None) -> AttnPartial:
    return _wrap_many([(o3, l3)], as_numpy, out_np_dtype)[0]


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
    if _all_np(q, keys, values):
        qt, kt, vt, dv = _widen(*_STAGE.upload(dt, [q, keys, values]))
    else:
        qt, kt, vt, dv = _widen(_to_dev(q, dt), _to_dev(keys, dt), _to_dev(values, dt))
    o, _ = K.attention_partial(qt, kt, vt, 0, None, scale)
    o = o[..., :dv]
    if _is_np(q):
        return _STAGE.download([o[0].contiguous()])[0].astype(np.float64, copy=False)
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
    return _wrap(o.contiguous(), l, _is_np(q), q.dtype if _is_np(q) else None)


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
    qt, kt, vt, dv = _widen(*_upload_qkv(q, keys, values))
    n = kt.shape[0]
    eo, el = K.attention_partial(qt, kt, vt, 0, boundary, scale)
    io, il = K.attention_partial(qt, kt, vt, boundary, n, scale)
    if dv != eo.shape[-1]:
        eo, io = eo[..., :dv].contiguous(), io[..., :dv].contiguous()
    np_out = q.dtype if _is_np(q) else None
    ext, inn = _wrap_many([(eo, el), (io, il)], _is_np(q), np_out)
    return ext, inn


def _partial_to_dev(p: AttnPartial):
    if isinstance(p.out, torch.Tensor):
        return p.out, p.lognorm
    m = p._device_mirror()
    if m is not None:
        return m
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
        return _wrap(out[0][None], out[1][None], True, a.out.dtype)
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


def _reuse_host(q, partial: AttnPartial, k_in, v_in, scale: float):
    """The numpy cached step in ONE C-ABI call (fb_internal_merge_host: pinned
    staging, one upload, the cached step, one read-back) when the cached
    external partial is already on the device in the call's precision mode
    (a partial this module returned).  None: take the general path."""
    if not (_all_np(q, k_in, v_in) and q.shape[1] == k_in.shape[1] == v_in.shape[1]):
        return None
    m = partial._device_mirror() if isinstance(partial.out, np.ndarray) else None
    if m is None:
        return None
    dt = _np_mode_dtype(q, k_in, v_in)
    o_ext, l_ext = m
    if o_ext.dtype != dt or l_ext.dtype != torch.float64 or o_ext.shape != tuple(q.shape) \
            or o_ext.device != _device():
        return None
    np_dt = np.float64 if dt == torch.float64 else np.float32
    qa = np.ascontiguousarray(q, dtype=np_dt)
    ka = np.ascontiguousarray(k_in, dtype=np_dt)
    va = np.ascontiguousarray(v_in, dtype=np_dt)
    out = np.empty(q.shape, dtype=np_dt)
    o_int = np.empty(q.shape, dtype=np_dt)
    l_int = np.empty(q.shape[0], dtype=np.float64)
    empty = ctypes.c_int64(0)
    K._lib.call("fb_internal_merge_host", K._lib.FB_F64 if dt == torch.float64 else K._lib.FB_F32,
                qa.ctypes.data, ka.ctypes.data, va.ctypes.data, 1, q.shape[0], q.shape[1], k_in.shape[0],
                float(scale), o_ext.data_ptr(), l_ext.data_ptr(), out.ctypes.data, o_int.ctypes.data,
                l_int.ctypes.data, ctypes.addressof(empty), _raw_stream(o_ext.device))
    if empty.value > 0:
        raise DegenerateInputError("some query rows have no keys on either side")
    return out.astype(q.dtype, copy=False), AttnPartial(o_int.astype(q.dtype, copy=False), l_int)


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
    fast = _reuse_host(q, entry.partial, internal_keys, internal_values, scale)
    if fast is not None:
        return fast
    qt, kt, vt, dv = _widen(*_upload_qkv(q, internal_keys, internal_values))
    eo, el = _partial_to_dev(entry.partial)
    if eo.shape[-1] != dv:
        raise ShapeError(f"cached partial has {eo.shape[-1]} value columns, internal values {dv}")
    ot, lt = K.PARTIAL_TYPES[K.dtype_code(qt)]
    eo, el = eo.to(ot), el.to(lt)
    if eo.shape[-1] < qt.shape[-1]:
        eo = torch.cat([eo, eo.new_zeros(eo.shape[:-1] + (qt.shape[-1] - dv,))], dim=-1)
    out, lse_m, (io, il) = K.internal_merge(qt, kt, vt, eo, el, scale, want_lse=True,
                                            want_internal=True)
    if dv != out.shape[-1]:
        out, io = out[..., :dv].contiguous(), io[..., :dv].contiguous()
    if _is_np(q):
        # one synchronisation for the merged output, its lognorm (the empty
        # row check) and the internal partial
        o_np, lse_np, io_np, il_np = _STAGE.download([out[0], lse_m[0], io[0], il[0]])
        if np.isneginf(lse_np).any():
            raise DegenerateInputError("some query rows have no keys on either side")
        internal = AttnPartial(io_np.astype(q.dtype, copy=False), il_np.astype(np.float64, copy=False))
        if io_np.dtype == q.dtype and il_np.dtype == np.float64:
            internal._set_mirror(io[0], il[0])
        return o_np.astype(q.dtype, copy=False), internal
    if bool(torch.isneginf(lse_m).any()):
        raise DegenerateInputError("some query rows have no keys on either side")
    return out[0], AttnPartial(io[0], il[0])
