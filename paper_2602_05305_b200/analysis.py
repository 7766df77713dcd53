"""Cross-step similarity of attention partials on the GPU.

Mirrors the reference's analysis / calibration surface
(flashblock/analysis.py:28-148, flashblock/policy.py:184-246): the same
``pairwise_step_similarity`` and ``cosine_similarity`` semantics (zero-norm
rule of linalg.py:68-80, float64 statistics), computed by
``fb_pairwise_cosine`` / ``fb_row_cosine`` in libfb200.so, and a batched
device-side head-gate calibrator for the serving engine.
"""

from __future__ import annotations

import numpy as np
import torch

from . import kernels as K
from .errors import ShapeError
from .policy import CalibrationError, HeadGateTable

__all__ = ["pairwise_step_similarity", "row_cosine_mean", "HeadGateCalibrator"]


def _dev(x):
    if isinstance(x, torch.Tensor):
        return x
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def pairwise_step_similarity(out_s, out_s1):
    """All-pairs cosine between token outputs of adjacent steps (analysis.py:28-51):
    entry (i, j) is the similarity of token i at the later step (out_s1) with
    token j at the earlier step (out_s).  numpy in -> numpy out; 2-D or batched
    [heads, rows, d] tensors -> float64 tensor."""
    if out_s.ndim != out_s1.ndim or tuple(out_s.shape) != tuple(out_s1.shape) or out_s.ndim not in (2, 3):
        raise ShapeError(f"step outputs must share a (block, head_dim) shape: "
                         f"{tuple(out_s.shape)} vs {tuple(out_s1.shape)}")
    as_np = not isinstance(out_s, torch.Tensor)
    later, earlier = _dev(out_s1), _dev(out_s)
    if later.dtype != earlier.dtype:
        earlier = earlier.to(later.dtype)
    sim = K.pairwise_cosine(later, earlier)
    if out_s.ndim == 2:
        sim = sim[0]
    return sim.cpu().numpy() if as_np else sim


def row_cosine_mean(a, b):
    """Per-head mean over rows of cos(a[h, r], b[h, r]) (policy.py:232-240), float64."""
    return K.row_cosine(_dev(a), _dev(b))


class HeadGateCalibrator:
    """Head-gate calibration on the device (policy.py:184-246).

    The reference records every (layer, head)'s external partial at every
    step of always-recompute rollouts and, per adjacent step pair, takes the
    row-mean cosine as one sample; gates are ``mean > gamma`` over all
    samples (min kept as the conservative statistic).  Here the rollouts are
    the sequences of the engine's batch: feed ``observe(layer, o_ext)`` with
    the external partial after every refresh (``FlashBlockAttention`` does it
    when constructed with ``recorder=``); ``begin_rollout()`` separates blocks.
    Sums and minima stay on the device; only ``table()`` syncs.
    """

    def __init__(self, num_layers: int, num_q_heads: int, device=None):
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.L, self.hq = num_layers, num_q_heads
        self.sum = torch.zeros((num_layers, num_q_heads), dtype=torch.float64, device=dev)
        self.min = torch.full((num_layers, num_q_heads), float("inf"), dtype=torch.float64, device=dev)
        self.count = [0] * num_layers
        self.signal = torch.zeros((), dtype=torch.bool, device=dev)
        self.nonzero = torch.zeros((), dtype=torch.int32, device=dev)  # set by row_cosine_update
        self.prev: list = [None] * num_layers

    def begin_rollout(self) -> None:
        self.prev = [None] * self.L

    def observe(self, layer: int, o_ext: torch.Tensor, rows_per_head: int) -> None:
        """o_ext: external partial rows of one layer, [b*Hq*rows_per_head, d]
        in any view (the engine's [b*Hkv, G*B, d] is [b, Hq, B, d])."""
        x = o_ext.reshape(-1, rows_per_head, o_ext.shape[-1])
        if x.shape[0] % self.hq:
            raise ShapeError(f"{x.shape[0]} heads of rows is not a multiple of {self.hq} query heads")
        if self.prev[layer] is not None:
            # one pass: row cosines against the previous step, prev <- x, nonzero flag
            m = K.row_cosine_update(x, self.prev[layer], self.nonzero).view(-1, self.hq)  # [b, Hq]
            self.sum[layer] += m.sum(dim=0)
            self.min[layer] = torch.minimum(self.min[layer], m.min(dim=0).values)
            self.count[layer] += m.shape[0]
        else:
            self.signal |= (x != 0).any()
            self.prev[layer] = x.clone()

    def stats(self) -> dict:
        s, mn = self.sum.cpu().numpy(), self.min.cpu().numpy()
        return {(l, h): (float(s[l, h] / self.count[l]), float(mn[l, h]))
                for l in range(self.L) if self.count[l] for h in range(self.hq)}

    def table(self, gamma: float) -> HeadGateTable:
        if not (bool(self.signal) or bool(self.nonzero)):
            raise CalibrationError("all recorded external partials are zero")
        return HeadGateTable.from_similarities(gamma, self.stats())
