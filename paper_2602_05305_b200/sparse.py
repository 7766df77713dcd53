"""Reference-named sparse API on the B200 kernels (drop-in for
flashblock/sparse.py:30-212).

``build_sparse_mask`` runs K5 (float64 block mass over the full softmax) and
K6 (stable top-k) on the device; ``sparse_attention_with_residual`` runs K7
on the first step of a block and K8 (gathered selected blocks + cached
residual merge) afterwards.  Numpy inputs give numpy outputs with the
reference's dtypes; CUDA tensors stay on the device.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import kernels as K
from .attention import (AttnPartial, CacheEntry, _common_dtype, _is_np, _partial_to_dev,
                        _to_dev)
from .errors import ShapeError, StalenessError

__all__ = [
    "StalenessError",
    "SparseMask",
    "build_sparse_mask",
    "sparse_attention_with_residual",
]

DEFAULT_KEY_BLOCK = 16  # sparse.py:40


@dataclass(frozen=True)
class SparseMask:
    """Selected external key blocks for one (layer, head) and one block
    (sparse.py:47-80).  ``selected`` holds ascending block indices."""

    block_id: int
    key_block_size: int
    density: float
    selected: np.ndarray
    num_external_keys: int

    @property
    def realized_density(self) -> float:
        if self.num_external_keys == 0:
            return 0.0
        return self.selected_key_indices().size / self.num_external_keys

    def selected_key_indices(self) -> np.ndarray:
        sel = np.asarray(self.selected.cpu() if isinstance(self.selected, torch.Tensor)
                         else self.selected, dtype=np.int64)
        if sel.size == 0:
            return np.empty(0, dtype=np.int64)
        kbs, n = self.key_block_size, self.num_external_keys
        return np.concatenate([np.arange(b * kbs, min((b + 1) * kbs, n)) for b in sel])


def build_sparse_mask(q, keys, boundary: int, density: float,
                      key_block_size: int = DEFAULT_KEY_BLOCK, *, scale: float | None = None,
                      block_id: int = 0) -> SparseMask:
    """Highest-mass external key blocks from one dense evaluation
    (sparse.py:83-136): K5 block mass + K6 stable top-k on the device."""
    if not 0.0 < density <= 1.0:
        raise ValueError(f"density must be in (0, 1], got {density}")
    if key_block_size < 1:
        raise ValueError("key_block_size must be >= 1")
    if q.ndim != 2 or keys.ndim != 2 or keys.shape[1] != q.shape[1]:
        raise ShapeError("q and keys must be 2-D with matching feature dim")
    if not 0 <= boundary <= keys.shape[0]:
        raise ValueError(f"boundary {boundary} outside [0, {keys.shape[0]}]")
    if scale is None:
        scale = 1.0 / math.sqrt(q.shape[1])
    if boundary == 0:
        selected = np.empty(0, dtype=np.int64)
    else:
        dt = _common_dtype(q, keys)
        qt, kt = _to_dev(q, dt), _to_dev(keys, dt)
        k_in = kt[boundary:].contiguous()
        mass = K.block_mass(qt, kt, k_in, boundary, key_block_size, scale)
        budget = K.mask_budget(boundary, density, key_block_size)
        sel = K.topk_blocks(mass, budget)[0]
        selected = sel.cpu().numpy().astype(np.int64) if _is_np(q) else sel.to(torch.int64)
    return SparseMask(block_id=block_id, key_block_size=key_block_size, density=density,
                      selected=selected, num_external_keys=boundary)


def _sel_dev(mask: SparseMask) -> torch.Tensor:
    sel = mask.selected
    if isinstance(sel, torch.Tensor):
        return sel.to(torch.int32).reshape(1, -1)
    return torch.from_numpy(np.ascontiguousarray(sel, dtype=np.int32)).reshape(1, -1).to(
        torch.device("cuda", torch.cuda.current_device()))


def sparse_attention_with_residual(q, mask: SparseMask, keys, values,
                                   residual: CacheEntry | None = None, *,
                                   scale: float | None = None, tile_size: int = 64):
    """Sparse attention merging back the unselected keys' partial
    (sparse.py:139-183).  First step (residual None): K7 exact partition;
    later steps: K8 over the selected blocks + current block, fused with the
    cached residual.  Returns (output, residual partial in effect)."""
    n_ext = mask.num_external_keys
    if keys.shape[0] < n_ext:
        raise ShapeError(
            f"key set has {keys.shape[0]} rows but mask covers {n_ext} external keys")
    if residual is not None and (not residual.valid or residual.block_id != mask.block_id):
        raise StalenessError(
            f"residual cached for block {residual.block_id} does not match "
            f"mask block {mask.block_id}")
    if scale is None:
        scale = 1.0 / math.sqrt(q.shape[1])
    dt = _common_dtype(q, keys, values)
    qt, kt, vt = _to_dev(q, dt), _to_dev(keys, dt), _to_dev(values, dt)
    k_in, v_in = kt[n_ext:].contiguous(), vt[n_ext:].contiguous()
    sel = _sel_dev(mask)
    if residual is None:
        out, _, (o_res, l_res) = K.sparse_partitioned(qt, kt, vt, k_in, v_in, n_ext, sel,
                                                      mask.key_block_size, scale, check=True)
        if _is_np(q):
            return (out[0].cpu().numpy().astype(q.dtype, copy=False),
                    AttnPartial(o_res[0].cpu().numpy().astype(q.dtype, copy=False),
                                l_res[0].cpu().numpy().astype(np.float64, copy=False)))
        return out[0], AttnPartial(o_res[0], l_res[0])
    ro, rl = _partial_to_dev(residual.partial)
    ot, lt = K.PARTIAL_TYPES[K.dtype_code(qt)]
    out = K.sparse_attend_merge(qt, kt, vt, k_in, v_in, n_ext, sel,
                                (ro.to(ot).unsqueeze(0), rl.to(lt).unsqueeze(0)),
                                mask.key_block_size, scale, check=True)
    if _is_np(q):
        return out[0].cpu().numpy().astype(q.dtype, copy=False), residual.partial
    return out[0], residual.partial
