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
partial per layer is O_ext [b, Hq, B, d] + LSE_ext [b, Hq, B] fp32 (the
reference's cache entry, attention.py:248-292, batched).  In bf16 mode O_ext
is stored in bf16 by default (ext_dtype): the reference keeps a partial's out
in the tensor dtype (attention.py:70-71), and every cached step re-reads it.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import kernels as K
from .errors import BoundsError, ReusePreconditionError, ShapeError, StalenessError
from .policy import Decision, ReuseConfig, decide


@dataclass
class AccessCounters:
    """Counted cache traffic, the reference's AccessCounters (kv_cache.py:28-52):
    key / value rows read from the committed cache (per kv slab, as the
    reference counts per (layer, head) read_range), rows appended, and bytes
    resident.  Cached steps read no cache rows (tests/test_acceptance.py:132-176
    there); the kernels of a cached step never receive the cache pointer."""

    key_rows_read: int = 0
    value_rows_read: int = 0
    rows_appended: int = 0
    cache_bytes_resident: int = 0

    def copy(self) -> "AccessCounters":
        return AccessCounters(self.key_rows_read, self.value_rows_read, self.rows_appended,
                              self.cache_bytes_resident)


class FlashBlockAttention:
    def __init__(self, num_layers: int, batch: int, num_q_heads: int, num_kv_heads: int,
                 block_len: int, head_dim: int, device=None, dtype=torch.bfloat16,
                 out_dtype: torch.dtype | None = None, scale: float | None = None,
                 config: ReuseConfig | None = None, recorder=None,
                 ext_dtype: torch.dtype | None = None):
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
        # cached external partial's O: bf16 in bf16 mode where the tcgen05
        # kernels run (head_dim 64 / 128), else the mode's partial type
        if ext_dtype is None:
            ext_dtype = torch.bfloat16 if (dtype == torch.bfloat16 and head_dim in (64, 128)) else self.ot
        if ext_dtype not in (self.ot, torch.bfloat16) or (ext_dtype == torch.bfloat16 and dtype != torch.bfloat16):
            raise ShapeError(f"ext_dtype {ext_dtype} is not a partial type of {dtype} mode")
        self.ext_dtype = ext_dtype
        self.o_ext = torch.zeros((num_layers, groups, rows, head_dim), dtype=ext_dtype, device=self.device)
        self.lse_ext = torch.full((num_layers, groups, rows), -math.inf, dtype=self.lt, device=self.device)
        self.valid = [False] * num_layers
        self.block_id = 0
        # optional HeadGateCalibrator: sees every refreshed external partial
        self.recorder = recorder
        self._glists: dict = {}
        # cache rows read (host count for uniform lengths, device count for ragged)
        self._rows_read = 0
        self._rows_read_dev = None

    def _count_rows(self, rows) -> None:
        if isinstance(rows, torch.Tensor):
            if self._rows_read_dev is None:
                self._rows_read_dev = torch.zeros((), dtype=torch.int64, device=self.device)
            self._rows_read_dev += rows.to(torch.int64).sum()
        else:
            self._rows_read += int(rows)

    def snapshot_counters(self) -> AccessCounters:
        """Rows read so far (syncs once if ragged refreshes were counted on the device)."""
        n = self._rows_read + (int(self._rows_read_dev) if self._rows_read_dev is not None else 0)
        return AccessCounters(key_rows_read=n, value_rows_read=n)

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

    def _group_lengths(self, n_ext):
        """int -> None (uniform); tensor [b] (per sequence) or [b*Hkv] -> int32 [b*Hkv]."""
        if isinstance(n_ext, int):
            return None
        t = n_ext.to(torch.int32).reshape(-1)
        if t.numel() == self.b:
            t = t.repeat_interleave(self.hkv)
        if t.numel() != self.b * self.hkv:
            raise ShapeError(f"lengths must have {self.b} or {self.b * self.hkv} entries")
        return t.contiguous()

    def refresh(self, layer: int, q, k_cache, v_cache, n_ext, k_in, v_in, out=None):
        """Refresh step: K1 over the committed cache rows + K2; stores the
        external partial for `layer`.  n_ext is one context length for the
        batch (int) or per-sequence lengths (CUDA int32 tensor [b] or
        [b*Hkv], ragged -- SURVEY 8f row f2).  k_cache may instead be a
        PagedKVCache (v_cache and n_ext are then ignored: the cache's page
        tables and lengths are used).  Returns out [b, Hq, B, d]."""
        qg, kg, vg = self._groups(q, k_in, v_in)
        if isinstance(k_cache, PagedKVCache):  # paged serving cache: v_cache / n_ext unused
            o = out.view(qg.shape) if out is not None else None
            self._count_rows(k_cache.lengths[layer])
            K.attention_partial_paged(qg, k_cache.k[layer], k_cache.v[layer], k_cache.table[layer],
                                      k_cache.lengths[layer], self.scale, out=self.o_ext[layer],
                                      lse=self.lse_ext[layer])
            res = K.internal_merge(qg, kg, vg, self.o_ext[layer], self.lse_ext[layer], self.scale,
                                   self.out_dtype, out=o)
            self.valid[layer] = True
            if self.recorder is not None:
                self.recorder.observe(layer, self.o_ext[layer], self.B)
            return res.view(self.b, self.hq, self.B, self.d)
        kc = k_cache.reshape(self.b * self.hkv, k_cache.shape[-2], self.d)
        vc = v_cache.reshape(self.b * self.hkv, v_cache.shape[-2], self.d)
        o = out.view(qg.shape) if out is not None else None
        lens = self._group_lengths(n_ext)
        if lens is None:
            self._count_rows(self.b * self.hkv * int(n_ext))
            # K1 (in-kernel split merge through the device's sync flags) then K2
            K.attention_partial(qg, kc, vc, 0, int(n_ext), self.scale, out=self.o_ext[layer],
                                lse=self.lse_ext[layer])
            res = K.internal_merge(qg, kg, vg, self.o_ext[layer], self.lse_ext[layer], self.scale,
                                   self.out_dtype, out=o)
        else:
            self._count_rows(lens.clamp(max=kc.shape[1]))
            K.attention_partial_ragged(qg, kc, vc, lens, 0, self.scale, out=self.o_ext[layer],
                                       lse=self.lse_ext[layer])
            res = K.internal_merge(qg, kg, vg, self.o_ext[layer], self.lse_ext[layer], self.scale,
                                   self.out_dtype, out=o)
        self.valid[layer] = True
        if self.recorder is not None:
            self.recorder.observe(layer, self.o_ext[layer], self.B)
        return res.view(self.b, self.hq, self.B, self.d)

    def cached(self, layer: int, q, k_in, v_in, out=None):
        """Cached step: K2 only -- internal partial merged with the stored
        external partial; the KV cache is not an argument."""
        if not self.valid[layer]:
            raise ReusePreconditionError(f"no valid cached external partial for layer {layer}")
        qg, kg, vg = self._groups(q, k_in, v_in)
        o = out.view(qg.shape) if out is not None else None
        # the external partial was written at the last refresh, never by the
        # kernel right before this one (refresh ends with K2), so K2 may
        # prefetch it before its PDL wait
        res = K.internal_merge(qg, kg, vg, self.o_ext[layer], self.lse_ext[layer], self.scale,
                               self.out_dtype, out=o, ext_stable=True)
        return res.view(self.b, self.hq, self.B, self.d)

    # -- token-major variants: q / k_in / v_in as [b, B, H, d] views of a fused
    # QKV projection output and the output token-major for the O projection,
    # so the attention layer needs no head-major copies on cached steps
    def cached_tokmajor(self, layer: int, q_tok, k_tok, v_tok, out_tok):
        """cached() on token-major tensors (fb_internal_merge_tok)."""
        if not self.valid[layer]:
            raise ReusePreconditionError(f"no valid cached external partial for layer {layer}")
        K.internal_merge_tok(q_tok, k_tok, v_tok, self.o_ext[layer], self.lse_ext[layer], out_tok, self.scale,
                             ext_stable=True)
        return out_tok

    def refresh_tokmajor(self, layer: int, q_tok, k_cache, v_cache, n_ext: int, k_tok, v_tok, out_tok):
        """refresh() on token-major tensors: K1 on a head-major copy of the
        queries (one copy per refresh step), K2 token-major."""
        q = q_tok.permute(0, 2, 1, 3).contiguous()
        qg = K.gqa_view(q, self.hkv)
        kc = k_cache.reshape(self.b * self.hkv, k_cache.shape[-2], self.d)
        vc = v_cache.reshape(self.b * self.hkv, v_cache.shape[-2], self.d)
        self._count_rows(self.b * self.hkv * int(n_ext))
        K.attention_partial(qg, kc, vc, 0, int(n_ext), self.scale, out=self.o_ext[layer], lse=self.lse_ext[layer])
        K.internal_merge_tok(q_tok, k_tok, v_tok, self.o_ext[layer], self.lse_ext[layer], out_tok, self.scale)
        self.valid[layer] = True
        return out_tok

    def step(self, layer: int, q, k_cache, v_cache, n_ext, k_in, v_in, *,
             first_visit: bool, updated_tokens: int, out=None):
        """Route one layer through the reuse policy (simulator.py:412-434)."""
        choice = decide(self.config, self.valid[layer], first_visit, updated_tokens)
        if choice is Decision.REUSE:
            return self.cached(layer, q, k_in, v_in, out), choice
        return self.refresh(layer, q, k_cache, v_cache, n_ext, k_in, v_in, out), choice

    def prefill(self, q, k_cache, v_cache, n_prefix: int = 0, out=None, lse=None):
        """Prefill / commit attention over a prompt: the
        reference's per-block commit passes (simulator.py:297-354) in one
        block-causal launch.  q [b, Hq, n_q, d]; the caches already hold the
        prompt's K/V at rows [n_prefix, n_prefix + n_q).  Block size = the
        engine's block.  Returns the attention output [b, Hq, n_q, d] in the
        partial dtype (fp32 for bf16 inputs)."""
        b, hq, n_q, d = q.shape
        if (b, hq, d) != (self.b, self.hq, self.d):
            raise ShapeError(f"queries {tuple(q.shape)} do not match the engine")
        qg = q.reshape(self.b * self.hkv, (self.hq // self.hkv) * n_q, self.d)
        kc = k_cache.reshape(self.b * self.hkv, k_cache.shape[-2], self.d)
        vc = v_cache.reshape(self.b * self.hkv, v_cache.shape[-2], self.d)
        o = out.view(qg.shape) if out is not None else None
        # the reference's commit passes read the committed prefix of every block
        # (simulator.py:316-317): sum over blocks j of n_prefix + j * B rows
        nblk = -(-n_q // self.B)
        self._count_rows(self.b * self.hkv * (nblk * n_prefix + self.B * nblk * (nblk - 1) // 2))
        res, _ = K.block_causal_attention(qg, kc, vc, n_q, n_prefix, self.B, self.scale, out=o, lse=lse)
        return res.view(b, hq, n_q, d)

    def prefill_paged(self, q, cache: "PagedKVCache", layer: int, n_prefix: int = 0, out=None, lse=None):
        """prefill() with the prompt's K/V read through a PagedKVCache's page
        tables for `layer` (commit the prompt into the cache first; every slab
        must hold n_prefix + n_q rows)."""
        b, hq, n_q, d = q.shape
        if (b, hq, d) != (self.b, self.hq, self.d):
            raise ShapeError(f"queries {tuple(q.shape)} do not match the engine")
        qg = q.reshape(self.b * self.hkv, (self.hq // self.hkv) * n_q, self.d)
        o = out.view(qg.shape) if out is not None else None
        nblk = -(-n_q // self.B)
        self._count_rows(self.b * self.hkv * (nblk * n_prefix + self.B * nblk * (nblk - 1) // 2))
        res, _ = K.block_causal_attention_paged(qg, cache.k[layer], cache.v[layer], cache.table[layer], n_q,
                                                n_prefix, self.B, self.scale, out=o, lse=lse)
        return res.view(b, hq, n_q, d)

    # -- sparse + residual reuse (sparse.py:83-183), batched over the engine's groups
    def sparse_first_step(self, layer: int, q, k_cache, v_cache, n_ext: int, k_in, v_in,
                          density: float, key_block_size: int = 16, out=None):
        """First step of a block with the sparse variant: K5 + K6 select the
        top-k external key blocks per kv group (pooled over the group's rows,
        build_sparse_mask, sparse.py:83-136), K7 computes the exact partition
        (selected + current block, and the residual over the unselected
        blocks, sparse.py:166-175) and the output; the selection and the
        residual partial are kept for `layer`'s later steps.  k_cache may be a
        PagedKVCache (v_cache ignored; uniform n_ext).  Returns out
        [b, Hq, B, d]."""
        qg, kg, vg = self._groups(q, k_in, v_in)
        kc, vc, pt = self._sparse_kv(layer, k_cache, v_cache)
        budget = K.mask_budget(int(n_ext), density, key_block_size)
        mass = K.block_mass(qg, kc, kg, int(n_ext), key_block_size, self.scale, page_table=pt)
        sel = K.topk_blocks(mass, budget)
        res, _, resid = K.sparse_partitioned(qg, kc, vc, kg, vg, int(n_ext), sel, key_block_size,
                                             self.scale, self.out_dtype, page_table=pt)
        if not hasattr(self, "_sparse"):
            self._sparse = {}
        self._sparse[layer] = (sel, resid, int(n_ext), key_block_size, self.block_id)
        self._count_rows(self.b * self.hkv * int(n_ext))
        if out is not None:
            out.view(res.shape).copy_(res)
            return out
        return res.view(self.b, self.hq, self.B, self.d)

    def sparse_cached_step(self, layer: int, q, k_cache, v_cache, k_in, v_in, out=None):
        """Later steps: K8 attends the stored selected blocks + the current
        block with the current queries and merges the cached residual
        (sparse.py:177-183).  StalenessError when `layer` has no residual for
        this block (sparse.py:177-181)."""
        st = getattr(self, "_sparse", {}).get(layer)
        if st is None or st[4] != self.block_id:
            raise StalenessError(f"no residual for layer {layer} in block {self.block_id}")
        sel, resid, n_ext, kbs, _ = st
        qg, kg, vg = self._groups(q, k_in, v_in)
        kc, vc, pt = self._sparse_kv(layer, k_cache, v_cache)
        res = K.sparse_attend_merge(qg, kc, vc, kg, vg, n_ext, sel, resid, kbs, self.scale,
                                    self.out_dtype, page_table=pt)
        # exactly the selected committed rows, the tail block clipped at n_ext
        # (read_selected_rows, sparse.py:186-212)
        self._count_rows((n_ext - sel.to(torch.int64) * kbs).clamp(min=0, max=kbs))
        if out is not None:
            out.view(res.shape).copy_(res)
            return out
        return res.view(self.b, self.hq, self.B, self.d)

    def _sparse_kv(self, layer: int, k_cache, v_cache):
        if isinstance(k_cache, PagedKVCache):
            return k_cache.k[layer], k_cache.v[layer], k_cache.table[layer]
        kc = k_cache.reshape(self.b * self.hkv, k_cache.shape[-2], self.d)
        vc = v_cache.reshape(self.b * self.hkv, v_cache.shape[-2], self.d)
        return kc, vc, None

    def step_gated(self, layer: int, q, k_cache, v_cache, n_ext: int, k_in, v_in, *,
                   first_visit: bool, updated_tokens: int, gates, out=None):
        """Head-gated mode: every query head decides on its
        own (decide with its gate, policy.py:71-94; simulator.py:399-405); a kv
        group is refreshed when any of its query heads recomputes, the others
        keep their cached external partial.  With 1:1 heads (G = 1) this is
        the reference's per-(layer, head) behaviour exactly.  K1 runs on the
        refreshed groups only (fb_attention_partial_groups), then K2 merges
        every group with its external partial.  Returns (out, per-head
        decisions)."""
        heads = [decide(self.config, self.valid[layer], first_visit, updated_tokens,
                        gates.is_enabled(layer, h)) for h in range(self.hq)]
        kv_refresh = [any(heads[kv * self.G + j] is Decision.RECOMPUTE for j in range(self.G))
                      for kv in range(self.hkv)]
        if all(kv_refresh):
            return self.refresh(layer, q, k_cache, v_cache, n_ext, k_in, v_in, out), heads
        if not any(kv_refresh):
            return self.cached(layer, q, k_in, v_in, out), heads
        key = tuple(kv_refresh)
        gl = self._glists.get(key)
        if gl is None:
            ids = [bi * self.hkv + kv for bi in range(self.b) for kv in range(self.hkv) if kv_refresh[kv]]
            gl = torch.tensor(ids, dtype=torch.int32, device=self.device)
            self._glists[key] = gl
        qg, kg, vg = self._groups(q, k_in, v_in)
        if isinstance(k_cache, PagedKVCache):  # paged serving cache: v_cache / n_ext unused
            # K1 over the refreshed groups only: their queries, page-table rows and
            # lengths gathered into a sub-batch, the partials scattered back into
            # the layer's external partial (other groups keep their cached rows)
            gl64 = gl.to(torch.int64)
            lens = k_cache.lengths[layer].index_select(0, gl64)
            self._count_rows(lens)
            o_sub = torch.empty((gl64.numel(),) + tuple(self.o_ext.shape[2:]), dtype=self.o_ext.dtype,
                                device=self.device)
            o_sub, l_sub = K.attention_partial_paged(qg.index_select(0, gl64), k_cache.k[layer],
                                                     k_cache.v[layer],
                                                     k_cache.table[layer].index_select(0, gl64), lens,
                                                     self.scale, out=o_sub)
            self.o_ext[layer].index_copy_(0, gl64, o_sub)
            self.lse_ext[layer].index_copy_(0, gl64, l_sub)
        else:
            kc = k_cache.reshape(self.b * self.hkv, k_cache.shape[-2], self.d)
            vc = v_cache.reshape(self.b * self.hkv, v_cache.shape[-2], self.d)
            self._count_rows(gl.numel() * int(n_ext))
            K.attention_partial_groups(qg, kc, vc, gl, 0, int(n_ext), self.scale,
                                       out=self.o_ext[layer], lse=self.lse_ext[layer])
        o = out.view(qg.shape) if out is not None else None
        res = K.internal_merge(qg, kg, vg, self.o_ext[layer], self.lse_ext[layer], self.scale,
                               self.out_dtype, out=o)
        return res.view(self.b, self.hq, self.B, self.d), heads

    def full_recompute(self, q, k_cache, v_cache, n_ext: int, k_in, v_in, out=None,
                       o_scratch=None, lse_scratch=None, layer: int | None = None):
        """Baseline: full attention every step (same K1+K2 launch pair as a
        refresh, partial kept in scratch instead of the cache -- the layer's
        cached external partial and its valid flag are left alone).  k_cache
        may be a PagedKVCache; then `layer` selects its page tables (v_cache
        and n_ext are unused)."""
        qg, kg, vg = self._groups(q, k_in, v_in)
        o = out.view(qg.shape) if out is not None else None
        if isinstance(k_cache, PagedKVCache):  # paged serving cache: v_cache / n_ext unused
            if layer is None:
                raise ValueError("full_recompute on a PagedKVCache needs layer=")
            self._count_rows(k_cache.lengths[layer])
            o_ext, l_ext = K.attention_partial_paged(qg, k_cache.k[layer], k_cache.v[layer],
                                                     k_cache.table[layer], k_cache.lengths[layer],
                                                     self.scale, out=o_scratch, lse=lse_scratch)
        else:
            kc = k_cache.reshape(self.b * self.hkv, k_cache.shape[-2], self.d)
            vc = v_cache.reshape(self.b * self.hkv, v_cache.shape[-2], self.d)
            self._count_rows(self.b * self.hkv * int(n_ext))
            o_ext, l_ext = K.attention_partial(qg, kc, vc, 0, int(n_ext), self.scale, out=o_scratch,
                                               lse=lse_scratch)
        res = K.internal_merge(qg, kg, vg, o_ext, l_ext, self.scale, self.out_dtype, out=o)
        return res.view(self.b, self.hq, self.B, self.d)


class KVCache:
    """Device KV cache with per-sequence committed lengths (the step after the
    path; reference KvCache, kv_cache.py:80-217).

    Per layer: K, V [b, Hkv, capacity, d] and int32 lengths [b*Hkv] (one per
    kv slab, like the reference's per-(layer, head) row counts).  Blocks are
    appended on the device (fb_commit_block); committed rows are immutable.
    Allocated with zeros, though the kernels never read past a slab's length.
    """

    def __init__(self, num_layers: int, batch: int, num_kv_heads: int, capacity: int,
                 head_dim: int, device=None, dtype=torch.bfloat16):
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.L, self.b, self.hkv, self.cap, self.d = num_layers, batch, num_kv_heads, capacity, head_dim
        self.k = [torch.zeros((batch, num_kv_heads, capacity, head_dim), dtype=dtype, device=dev)
                  for _ in range(num_layers)]
        self.v = [torch.zeros_like(t) for t in self.k]
        self.lengths = [torch.zeros(batch * num_kv_heads, dtype=torch.int32, device=dev)
                        for _ in range(num_layers)]
        # host mirror of the (uniform) committed length per layer: every commit
        # advances every slab by the block's rows, so overflow is caught before
        # the launch without a device sync
        self._len = [0] * num_layers
        self.rows_appended = 0

    def commit_block(self, layer: int, k_block, v_block, check: bool = False) -> None:
        """Append one finished block's rows [b, Hkv, B, d] for `layer`.  Raises
        BoundsError (before launching) when the block would run past the
        capacity -- committed rows are never dropped (kv_cache.py:121-144).
        check=True additionally reads the device overflow counter back."""
        if k_block.shape[:2] != (self.b, self.hkv) or k_block.shape[-1] != self.d:
            raise ShapeError(f"block {tuple(k_block.shape)} does not match the cache")
        rows = k_block.shape[-2]
        if self._len[layer] + rows > self.cap:
            raise BoundsError(f"commit of {rows} rows at length {self._len[layer]} exceeds capacity {self.cap}")
        K.commit_block(self.k[layer].view(self.b * self.hkv, self.cap, self.d),
                       self.v[layer].view(self.b * self.hkv, self.cap, self.d),
                       k_block.reshape(self.b * self.hkv, -1, self.d),
                       v_block.reshape(self.b * self.hkv, -1, self.d), self.lengths[layer], check)
        self._len[layer] += rows
        self.rows_appended += self.b * self.hkv * rows

    def snapshot_counters(self) -> AccessCounters:
        """Rows appended and bytes resident (committed rows of every slab; syncs)."""
        rows = sum(int(t.clamp(max=self.cap).to(torch.int64).sum()) for t in self.lengths)
        return AccessCounters(rows_appended=self.rows_appended,
                              cache_bytes_resident=rows * 2 * self.d * self.k[0].element_size())

    def sequence_lengths(self, layer: int = 0) -> torch.Tensor:
        return self.lengths[layer].view(self.b, self.hkv)[:, 0]


class PagedKVCache:
    """Paged device KV cache (the serving layout): per layer
    one page pool K, V [num_pages, page_rows, d] shared by every (sequence,
    kv-head) slab, an int32 page table [b*Hkv, max_pages] and int32 committed
    lengths [b*Hkv] on the device.  Pages are handed out from a host free list
    when a block is committed and returned when a sequence is released, so
    sequences of very different lengths share one pool.  Attention reads the
    pages through the table inside K1 (fb_attention_partial_paged); the results
    equal the contiguous-slab ragged path on the same rows."""

    def __init__(self, num_layers: int, batch: int, num_kv_heads: int, num_pages: int,
                 page_rows: int, head_dim: int, max_pages_per_slab: int, device=None,
                 dtype=torch.bfloat16):
        if page_rows % 128:
            raise ShapeError("page_rows must be a multiple of 128")
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.L, self.b, self.hkv, self.P, self.d = num_layers, batch, num_kv_heads, page_rows, head_dim
        self.groups = batch * num_kv_heads
        self.max_pages = max_pages_per_slab
        self.k = [torch.zeros((num_pages, page_rows, head_dim), dtype=dtype, device=dev)
                  for _ in range(num_layers)]
        self.v = [torch.zeros_like(t) for t in self.k]
        self.table = [torch.full((self.groups, max_pages_per_slab), -1, dtype=torch.int32, device=dev)
                      for _ in range(num_layers)]
        self.lengths = [torch.zeros(self.groups, dtype=torch.int32, device=dev) for _ in range(num_layers)]
        self._len = [[0] * self.groups for _ in range(num_layers)]
        self._pages = [[[] for _ in range(self.groups)] for _ in range(num_layers)]
        self._free = [list(range(num_pages - 1, -1, -1)) for _ in range(num_layers)]

    def _reserve(self, layer: int, rows: int) -> None:
        changed = False
        for g in range(self.groups):
            need = -(-(self._len[layer][g] + rows) // self.P)
            while len(self._pages[layer][g]) < need:
                if len(self._pages[layer][g]) >= self.max_pages:
                    raise BoundsError("slab would exceed max_pages_per_slab")
                if not self._free[layer]:
                    raise BoundsError("page pool exhausted")
                self._pages[layer][g].append(self._free[layer].pop())
                changed = True
        if changed:
            host = torch.full((self.groups, self.max_pages), -1, dtype=torch.int32)
            for g, pages in enumerate(self._pages[layer]):
                host[g, :len(pages)] = torch.tensor(pages, dtype=torch.int32)
            self.table[layer].copy_(host, non_blocking=False)

    def commit_block(self, layer: int, k_block, v_block) -> None:
        """Append one finished block's rows [b, Hkv, B, d] for `layer`."""
        if k_block.shape[:2] != (self.b, self.hkv) or k_block.shape[-1] != self.d:
            raise ShapeError(f"block {tuple(k_block.shape)} does not match the cache")
        rows = k_block.shape[-2]
        self._reserve(layer, rows)
        K.commit_block_paged(self.k[layer], self.v[layer], self.table[layer],
                             k_block.reshape(self.groups, rows, self.d),
                             v_block.reshape(self.groups, rows, self.d), self.lengths[layer])
        for g in range(self.groups):
            self._len[layer][g] += rows

    def release(self, seq: int) -> None:
        """Return sequence `seq`'s pages (all layers) to the pools; its slabs restart empty."""
        for layer in range(self.L):
            for g in range(seq * self.hkv, (seq + 1) * self.hkv):
                self._free[layer].extend(reversed(self._pages[layer][g]))
                self._pages[layer][g] = []
                self._len[layer][g] = 0
            self.table[layer][seq * self.hkv:(seq + 1) * self.hkv] = -1
            self.lengths[layer][seq * self.hkv:(seq + 1) * self.hkv] = 0

    def attention_partial(self, layer: int, q):
        """K1 (refresh) for `layer`: q [b, Hq, B, d] -> (O_ext, LSE_ext) over
        every slab's committed rows, read through the page table."""
        q3 = K.gqa_view(q, self.hkv)
        return K.attention_partial_paged(q3, self.k[layer], self.v[layer], self.table[layer],
                                         self.lengths[layer])

    def free_pages(self, layer: int = 0) -> int:
        return len(self._free[layer])
