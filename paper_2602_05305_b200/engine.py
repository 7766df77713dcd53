"""Batched FlashBlock attention engine for one GPU (the per-step caller).

This is the device-resident counterpart of the reference step driver's
attention routing (simulator.py:400-441): per (layer) and diffusion step, a
refresh step streams the committed KV cache once (K1) and merges the
current block (K2), storing the external partial; a cached step runs only
K2 against the stored partial and never touches the KV cache.  All heads
of a layer share one decision in token-threshold mode, so a layer is one
batched launch pair.

Layouts: Q [b, Hq, B, d], KV cache [b, Hkv, N_cap, d], current-block K/V
[b, Hkv, B, d] -- all bf16 (or f32/f64 for parity runs); the external
partial per layer is O_ext [b, Hq, B, d] fp32 + LSE_ext [b, Hq, B] fp32
(the reference's cache entry, attention.py:248-292, batched).
"""

from __future__ import annotations

import math

import torch

from . import kernels as K
from .errors import ReusePreconditionError, ShapeError
from .policy import Decision, ReuseConfig, decide


class FlashBlockAttention:
    def __init__(self, num_layers: int, batch: int, num_q_heads: int, num_kv_heads: int,
                 block_len: int, head_dim: int, device=None, dtype=torch.bfloat16,
                 out_dtype: torch.dtype | None = None, scale: float | None = None,
                 config: ReuseConfig | None = None):
        if num_q_heads % num_kv_heads:
            raise ShapeError("num_q_heads must be a multiple of num_kv_heads")
        self.L, self.b, self.hq, self.hkv = num_layers, batch, num_q_heads, num_kv_heads
        self.B, self.d = block_len, head_dim
        self.G = num_q_heads // num_kv_heads
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self.dtype = dtype
        code = K._CODE[dtype]
        self.ot, self.lt = K.PARTIAL_TYPES[code]
        self.out_dtype = out_dtype or (torch.bfloat16 if dtype == torch.bfloat16 else self.ot)
        self.scale = 1.0 / math.sqrt(head_dim) if scale is None else float(scale)
        self.config = config or ReuseConfig()
        groups, rows = batch * num_kv_heads, self.G * block_len
        self.o_ext = torch.zeros((num_layers, groups, rows, head_dim), dtype=self.ot, device=self.device)
        self.lse_ext = torch.full((num_layers, groups, rows), -math.inf, dtype=self.lt, device=self.device)
        self.valid = [False] * num_layers
        self.block_id = 0

    # -- cache lifecycle (ExternalAttnCache.invalidate_all, simulator.py:562-563)
    def begin_block(self, block_id: int) -> None:
        self.block_id = block_id
        self.valid = [False] * self.L

    def is_valid(self, layer: int) -> bool:
        return self.valid[layer]

    def resident_bytes(self) -> int:
        per = self.o_ext[0].numel() * self.o_ext.element_size() + \
            self.lse_ext[0].numel() * self.lse_ext.element_size()
        return per * sum(self.valid)

    def _groups(self, q, k_in, v_in):
        if q.shape != (self.b, self.hq, self.B, self.d):
            raise ShapeError(f"q {tuple(q.shape)} != {(self.b, self.hq, self.B, self.d)}")
        if k_in.shape != (self.b, self.hkv, self.B, self.d) or v_in.shape != k_in.shape:
            raise ShapeError("current-block K/V must be [b, Hkv, B, d]")
        return K.gqa_view(q, self.hkv), k_in.reshape(self.b * self.hkv, self.B, self.d), \
            v_in.reshape(self.b * self.hkv, self.B, self.d)

    def refresh(self, layer: int, q, k_cache, v_cache, n_ext: int, k_in, v_in, out=None):
        """Refresh step: K1 over cache rows [0, n_ext) + K2; stores the
        external partial for `layer`.  Returns out [b, Hq, B, d]."""
        qg, kg, vg = self._groups(q, k_in, v_in)
        kc = k_cache.reshape(self.b * self.hkv, k_cache.shape[-2], self.d)
        vc = v_cache.reshape(self.b * self.hkv, v_cache.shape[-2], self.d)
        o = out.view(qg.shape) if out is not None else None
        res, _, _ = K.full_attention(qg, kc, vc, n_ext, kg, vg, self.scale, self.out_dtype,
                                     o_ext=self.o_ext[layer], lse_ext=self.lse_ext[layer], out=o)
        self.valid[layer] = True
        return res.view(self.b, self.hq, self.B, self.d)

    def cached(self, layer: int, q, k_in, v_in, out=None):
        """Cached step: K2 only -- internal partial merged with the stored
        external partial; the KV cache is not an argument."""
        if not self.valid[layer]:
            raise ReusePreconditionError(f"no valid cached external partial for layer {layer}")
        qg, kg, vg = self._groups(q, k_in, v_in)
        o = out.view(qg.shape) if out is not None else None
        res = K.internal_merge(qg, kg, vg, self.o_ext[layer], self.lse_ext[layer], self.scale,
                               self.out_dtype, out=o)
        return res.view(self.b, self.hq, self.B, self.d)

    def step(self, layer: int, q, k_cache, v_cache, n_ext: int, k_in, v_in, *,
             first_visit: bool, updated_tokens: int, out=None):
        """Route one layer through the reuse policy (simulator.py:412-434)."""
        choice = decide(self.config, self.valid[layer], first_visit, updated_tokens)
        if choice is Decision.REUSE:
            return self.cached(layer, q, k_in, v_in, out), choice
        return self.refresh(layer, q, k_cache, v_cache, n_ext, k_in, v_in, out), choice

    def full_recompute(self, q, k_cache, v_cache, n_ext: int, k_in, v_in, out=None,
                       o_scratch=None, lse_scratch=None):
        """Baseline: full attention every step (same K1+K2 launch pair as a
        refresh, partial kept in scratch instead of the cache)."""
        qg, kg, vg = self._groups(q, k_in, v_in)
        kc = k_cache.reshape(self.b * self.hkv, k_cache.shape[-2], self.d)
        vc = v_cache.reshape(self.b * self.hkv, v_cache.shape[-2], self.d)
        o = out.view(qg.shape) if out is not None else None
        res, _, _ = K.full_attention(qg, kc, vc, n_ext, kg, vg, self.scale, self.out_dtype,
                                     o_ext=o_scratch, lse_ext=lse_scratch, out=o)
        return res.view(self.b, self.hq, self.B, self.d)
