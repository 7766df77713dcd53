"""Batched device API over the C ABI: torch tensors in, torch tensors out.

Layouts (see include/flashblock_b200.h): a call processes ``groups`` pairs of
(query block [q_rows, d], key/value slab [kv_rows_cap, d]).  For a GQA layer
with Q [b, Hq, B, d] and a KV cache [b, Hkv, N_cap, d], use
``gqa_view`` -- groups = b*Hkv, q_rows = (Hq/Hkv)*B.

Every function here launches on the current torch CUDA stream and never
synchronises the host unless ``check=True`` (which reads the degenerate-row
counter back to raise ``DegenerateInputError`` like the reference).
"""

from __future__ import annotations

import math

import torch

from . import _lib
from .errors import DegenerateInputError, ShapeError

_CODE = {torch.float64: _lib.FB_F64, torch.float32: _lib.FB_F32, torch.bfloat16: _lib.FB_BF16}
# (partial out dtype, lognorm dtype) per mode
PARTIAL_TYPES = {
    _lib.FB_F64: (torch.float64, torch.float64),
    _lib.FB_F32: (torch.float32, torch.float64),
    _lib.FB_BF16: (torch.float32, torch.float32),
}
_OUT_CODE = {torch.float64: _lib.FB_F64, torch.float32: _lib.FB_F32, torch.bfloat16: _lib.FB_BF16}


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _CODE[t.dtype]
    except KeyError:
        raise ShapeError(f"unsupported dtype {t.dtype}; expected float64, float32 or bfloat16")


def mode_of_partial(out: torch.Tensor, lse: torch.Tensor) -> int:
    key = (out.dtype, lse.dtype)
    for code, types in PARTIAL_TYPES.items():
        if types == key:
            return code
    raise ShapeError(f"partial dtypes {key} match no precision mode")


def _partial_code(code: int, o: torch.Tensor) -> int:
    """The mode code, with FB_PARTIAL_BF16 when a BF16-mode partial's O is bf16
    (the reference keeps a partial's out in the tensor dtype, attention.py:70-71)."""
    if code == _lib.FB_BF16 and o.dtype == torch.bfloat16:
        return code | _lib.FB_PARTIAL_BF16
    return code


def _check_partial_out(code: int, out: torch.Tensor, lse: torch.Tensor) -> None:
    ot, lt = PARTIAL_TYPES[code]
    ok_o = out.dtype == ot or (code == _lib.FB_BF16 and out.dtype == torch.bfloat16)
    if not ok_o or lse.dtype != lt:
        raise ShapeError(f"partial out {out.dtype} / lognorm {lse.dtype} do not match the mode")
    if not (out.is_contiguous() and lse.is_contiguous()):
        raise ShapeError("partial out / lognorm must be contiguous")


def require_cuda(*ts: torch.Tensor) -> None:
    for t in ts:
        if t is not None and not t.is_cuda:
            raise RuntimeError("paper_2602_05305_b200 runs on CUDA tensors only (no CPU fallback)")


def _p(t):
    return None if t is None else t.data_ptr()


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


class _Workspace:
    """Scratch buffer for split-KV partials per (device, stream), grown on demand.

    Keyed by the launching stream, so kernels on different streams never share
    scratch.  A buffer that was outgrown is kept alive (not freed): a CUDA graph
    captured earlier may still hold its pointer and replay into it.  Graphs that
    are replayed concurrently must therefore be captured on distinct streams."""

    def __init__(self):
        self._bufs: dict[tuple[int, int], torch.Tensor] = {}
        self._retired: list[torch.Tensor] = []

    def get(self, device: torch.device, nbytes: int) -> torch.Tensor:
        idx = device.index if device.index is not None else torch.cuda.current_device()
        key = (idx, torch.cuda.current_stream(idx).cuda_stream)
        buf = self._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            if buf is not None:
                self._retired.append(buf)
            buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
            self._bufs[key] = buf
        return buf


WORKSPACE = _Workspace()


class _SyncFlags:
    """Ready-flag buffer for K1's in-kernel split merge per (device, stream):
    zeroed once, left zeroed by every launch, never shared with other scratch
    or with launches on another stream (the flag protocol assumes one K1 in
    flight per buffer; launches on one stream are ordered)."""

    def __init__(self):
        self._bufs: dict[tuple[int, int], torch.Tensor] = {}

    def get(self, device: torch.device) -> torch.Tensor:
        idx = device.index if device.index is not None else torch.cuda.current_device()
        key = (idx, torch.cuda.current_stream(idx).cuda_stream)
        buf = self._bufs.get(key)
        if buf is None:
            n = int(_lib.load().fb_sync_flags_count())
            buf = torch.zeros(n, dtype=torch.int64, device=device)
            self._bufs[key] = buf
        return buf


SYNC_FLAGS = _SyncFlags()


def gqa_view(q: torch.Tensor, num_kv_heads: int) -> torch.Tensor:
    """[b, Hq, B, d] -> [b*Hkv, (Hq/Hkv)*B, d] (no copy)."""
    b, hq, blk, d = q.shape
    if hq % num_kv_heads:
        raise ShapeError(f"{hq} query heads not divisible by {num_kv_heads} kv heads")
    return q.contiguous().view(b * num_kv_heads, (hq // num_kv_heads) * blk, d)


def _as3(x: torch.Tensor, name: str) -> torch.Tensor:
    if x.dim() == 2:
        return x.unsqueeze(0)
    if x.dim() == 3:
        return x
    if x.dim() == 4:
        return x.reshape(x.shape[0] * x.shape[1], x.shape[2], x.shape[3])
    raise ShapeError(f"{name} must be 2-, 3- or 4-D, got {x.dim()}-D")


def _check_kv(q3, k3, v3):
    if k3.shape != v3.shape:
        raise ShapeError(f"keys {tuple(k3.shape)} and values {tuple(v3.shape)} differ")
    if k3.shape[0] != q3.shape[0] or k3.shape[2] != q3.shape[2]:
        raise ShapeError(f"queries {tuple(q3.shape)} do not match keys {tuple(k3.shape)}")
    if not (q3.dtype == k3.dtype == v3.dtype):
        raise ShapeError("q, k, v must share one dtype")


def attention_partial(q, k, v, key_begin: int = 0, key_end: int | None = None,
                      scale: float | None = None, out=None, lse=None):
    """K1: normalised partial over slab rows [key_begin, key_end) for every group.

    q [groups, q_rows, d] (or [q_rows, d]); k, v [groups, cap, d].
    Returns (o, lse) in the mode's partial types.
    """
    q3, k3, v3 = _as3(q, "q"), _as3(k, "k"), _as3(v, "v")
    require_cuda(q3, k3, v3)
    _check_kv(q3, k3, v3)
    q3, k3, v3 = q3.contiguous(), k3.contiguous(), v3.contiguous()
    groups, q_rows, d = q3.shape
    cap = k3.shape[1]
    key_end = cap if key_end is None else int(key_end)
    code = dtype_code(q3)
    ot, lt = PARTIAL_TYPES[code]
    if out is None:
        out = torch.empty((groups, q_rows, d), dtype=ot, device=q3.device)
    if lse is None:
        lse = torch.empty((groups, q_rows), dtype=lt, device=q3.device)
    _check_partial_out(code, out, lse)
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    wsb = _lib.load().fb_partial_workspace_bytes(code, groups, q_rows, d, max(0, key_end - key_begin))
    ws = WORKSPACE.get(q3.device, wsb) if wsb else None
    flags = SYNC_FLAGS.get(q3.device)
    _lib.call("fb_attention_partial_sync", _partial_code(code, out), _p(q3), _p(k3), _p(v3), groups, q_rows, d, cap,
              int(key_begin), key_end, scale, _p(out), _p(lse), _p(ws),
              0 if ws is None else ws.numel(), _p(flags), flags.numel(), _stream(q3))
    return out, lse


def attention_partial_ragged(q, k, v, key_end: torch.Tensor, key_begin: int = 0,
                             scale: float | None = None, out=None, lse=None):
    """K1 over per-group (ragged) committed lengths: group g attends slab rows
    [key_begin, key_end[g]).  key_end: int32 CUDA tensor [groups]."""
    q3, k3, v3 = _as3(q, "q"), _as3(k, "k"), _as3(v, "v")
    require_cuda(q3, k3, v3, key_end)
    _check_kv(q3, k3, v3)
    q3, k3, v3 = q3.contiguous(), k3.contiguous(), v3.contiguous()
    groups, q_rows, d = q3.shape
    ends = key_end.reshape(-1).to(torch.int32).contiguous()
    if ends.numel() != groups:
        raise ShapeError(f"key_end has {ends.numel()} entries for {groups} groups")
    code = dtype_code(q3)
    ot, lt = PARTIAL_TYPES[code]
    if out is None:
        out = torch.empty((groups, q_rows, d), dtype=ot, device=q3.device)
    if lse is None:
        lse = torch.empty((groups, q_rows), dtype=lt, device=q3.device)
    _check_partial_out(code, out, lse)
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    wsb = _lib.load().fb_ragged_workspace_bytes(code, groups, q_rows, d, k3.shape[1])
    ws = WORKSPACE.get(q3.device, wsb) if wsb else None
    _lib.call("fb_attention_partial_ragged", _partial_code(code, out), _p(q3), _p(k3), _p(v3), groups, q_rows, d,
              k3.shape[1], int(key_begin), _p(ends), scale, _p(out), _p(lse), _p(ws),
              0 if ws is None else ws.numel(), _stream(q3))
    return out, lse


def attention_partial_paged(q, k_pages, v_pages, page_table: torch.Tensor, key_len: torch.Tensor,
                            scale: float | None = None, out=None, lse=None):
    """K1 over a paged KV cache: group g attends its logical
    rows [0, key_len[g]), row r stored at row r % P of page page_table[g, r // P]
    of the pools k_pages / v_pages [num_pages, P, d] (P a multiple of 128).
    bf16 only; same outputs as attention_partial_ragged on contiguous slabs."""
    q3 = _as3(q, "q").contiguous()
    require_cuda(q3, k_pages, v_pages, page_table, key_len)
    if k_pages.dim() != 3 or k_pages.shape != v_pages.shape or k_pages.shape[2] != q3.shape[2]:
        raise ShapeError("page pools must be [num_pages, page_rows, head_dim] and match q")
    if q3.dtype != torch.bfloat16 or k_pages.dtype != torch.bfloat16 or v_pages.dtype != torch.bfloat16:
        raise ShapeError("the paged path is bf16")
    kp, vp = k_pages.contiguous(), v_pages.contiguous()
    groups, q_rows, d = q3.shape
    table = page_table.reshape(groups, -1).to(torch.int32).contiguous()
    lens = key_len.reshape(-1).to(torch.int32).contiguous()
    if lens.numel() != groups:
        raise ShapeError(f"key_len has {lens.numel()} entries for {groups} groups")
    if out is None:
        out = torch.empty((groups, q_rows, d), dtype=torch.float32, device=q3.device)
    if lse is None:
        lse = torch.empty((groups, q_rows), dtype=torch.float32, device=q3.device)
    _check_partial_out(_lib.FB_BF16, out, lse)
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    wsb = _lib.load().fb_paged_workspace_bytes(_CODE[torch.bfloat16], groups, q_rows, d)
    ws = WORKSPACE.get(q3.device, wsb) if wsb else None
    _lib.call("fb_attention_partial_paged", _partial_code(_lib.FB_BF16, out), _p(q3), _p(kp), _p(vp), kp.shape[0],
              kp.shape[1], _p(table), table.shape[1], groups, q_rows, d, _p(lens), scale, _p(out),
              _p(lse), _p(ws), 0 if ws is None else ws.numel(), _stream(q3))
    return out, lse


def block_causal_attention_paged(q, k_pages, v_pages, page_table: torch.Tensor, n_q: int,
                                 n_prefix: int = 0, block_size: int = 32, scale: float | None = None,
                                 out=None, lse=None):
    """Prefill / commit attention (block_causal_attention) with the keys read
    through a paged cache's page tables (the prompt committed into the pages
    first).  bf16; q [groups, heads_per_group * n_q, d]."""
    q3 = _as3(q, "q").contiguous()
    require_cuda(q3, k_pages, v_pages, page_table)
    if k_pages.dim() != 3 or k_pages.shape != v_pages.shape or k_pages.shape[2] != q3.shape[2]:
        raise ShapeError("page pools must be [num_pages, page_rows, head_dim] and match q")
    if q3.dtype != torch.bfloat16 or k_pages.dtype != torch.bfloat16:
        raise ShapeError("the paged path is bf16")
    kp, vp = k_pages.contiguous(), v_pages.contiguous()
    groups, q_rows, d = q3.shape
    table = page_table.reshape(groups, -1).to(torch.int32).contiguous()
    if out is None:
        out = torch.empty((groups, q_rows, d), dtype=torch.float32, device=q3.device)
    if lse is None:
        lse = torch.empty((groups, q_rows), dtype=torch.float32, device=q3.device)
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    wsb = _lib.load().fb_paged_workspace_bytes(_CODE[torch.bfloat16], groups, q_rows, d)
    ws = WORKSPACE.get(q3.device, wsb) if wsb else None
    _lib.call("fb_block_causal_attention_paged", _CODE[torch.bfloat16], _p(q3), _p(kp), _p(vp),
              kp.shape[0], kp.shape[1], _p(table), table.shape[1], groups, q_rows, int(n_q), d,
              int(n_prefix), int(block_size), scale, _p(out), _p(lse), _p(ws),
              0 if ws is None else ws.numel(), _stream(q3))
    return out, lse


def commit_block_paged(k_pages, v_pages, page_table: torch.Tensor, k_block, v_block,
                       lengths: torch.Tensor, check: bool = False) -> None:
    """Append a finished block's K/V ([groups, B, d]) to each group's pages at
    logical row lengths[g]; lengths advance by B (kv_cache.py:121-144)."""
    kb, vb = _as3(k_block, "k_block").contiguous(), _as3(v_block, "v_block").contiguous()
    require_cuda(k_pages, v_pages, page_table, kb, vb, lengths)
    if not (k_pages.is_contiguous() and v_pages.is_contiguous()) or k_pages.shape != v_pages.shape:
        raise ShapeError("page pools must be contiguous and alike")
    groups = kb.shape[0]
    table = page_table.reshape(groups, -1)
    if table.dtype != torch.int32 or not table.is_contiguous():
        raise ShapeError("page_table must be a contiguous int32 tensor [groups, max_pages]")
    if lengths.dtype != torch.int32 or lengths.numel() != groups:
        raise ShapeError("lengths must be an int32 tensor [groups]")
    cnt = _empty_counter(kb.device) if check else None
    _lib.call("fb_commit_block_paged", dtype_code(kb), _p(k_pages), _p(v_pages), k_pages.shape[1],
              _p(table), table.shape[1], groups, kb.shape[2], _p(kb), _p(vb), kb.shape[1],
              _p(lengths), _p(cnt), _stream(kb))
    if cnt is not None and int(cnt.item()) > 0:
        from .errors import BoundsError
        raise BoundsError("block commit runs past the allocated pages")


def attention_partial_groups(q, k, v, group_list: torch.Tensor, key_begin: int = 0,
                             key_end: int | None = None, scale: float | None = None, out=None,
                             lse=None):
    """K1 over the groups in group_list only (head-gated refresh, SURVEY 8f
    row f3): rows of the other groups in out / lse are left untouched.
    group_list: CUDA int32 tensor of distinct group indices.  F64 / BF16."""
    q3, k3, v3 = _as3(q, "q"), _as3(k, "k"), _as3(v, "v")
    require_cuda(q3, k3, v3)
    _check_kv(q3, k3, v3)
    q3, k3, v3 = q3.contiguous(), k3.contiguous(), v3.contiguous()
    groups, q_rows, d = q3.shape
    cap = k3.shape[1]
    key_end = cap if key_end is None else int(key_end)
    code = dtype_code(q3)
    ot, lt = PARTIAL_TYPES[code]
    if out is None:
        out = torch.empty((groups, q_rows, d), dtype=ot, device=q3.device)
    if lse is None:
        lse = torch.empty((groups, q_rows), dtype=lt, device=q3.device)
    gl = group_list.to(device=q3.device, dtype=torch.int32).contiguous()
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    _check_partial_out(code, out, lse)
    wsb = _lib.load().fb_partial_workspace_bytes(code, gl.numel(), q_rows, d,
                                                 max(0, key_end - key_begin))
    ws = WORKSPACE.get(q3.device, wsb) if wsb else None
    _lib.call("fb_attention_partial_groups", _partial_code(code, out), _p(q3), _p(k3), _p(v3), groups, q_rows, d, cap,
              int(key_begin), key_end, _p(gl), gl.numel(), scale, _p(out), _p(lse), _p(ws),
              0 if ws is None else ws.numel(), _stream(q3))
    return out, lse


def _sim_code(t: torch.Tensor) -> int:
    return {torch.float64: _lib.FB_F64, torch.float32: _lib.FB_F32,
            torch.bfloat16: _lib.FB_BF16}[t.dtype]


def row_cosine(a, b, want_rows: bool = False):
    """Per-row cosine of a, b [heads, rows, d] (zero-norm rule of linalg.py:68-80)
    and its per-head mean, float64.  Returns head_mean [heads] (and row_cos)."""
    a3, b3 = _as3(a, "a").contiguous(), _as3(b, "b").contiguous()
    require_cuda(a3, b3)
    if a3.shape != b3.shape or a3.dtype != b3.dtype:
        raise ShapeError(f"step outputs differ: {tuple(a3.shape)} vs {tuple(b3.shape)}")
    heads, rows, d = a3.shape
    mean = torch.empty(heads, dtype=torch.float64, device=a3.device)
    rc = torch.empty((heads, rows), dtype=torch.float64, device=a3.device)
    _lib.call("fb_row_cosine", _sim_code(a3), _p(a3), _p(b3), heads, rows, d, _p(rc), _p(mean),
              _stream(a3))
    return (mean, rc) if want_rows else mean


def row_cosine_update(a, prev, nonzero=None):
    """row_cosine(a, prev)'s per-head mean [heads] (float64), then prev <- a in
    the same pass (fb_row_cosine_update); nonzero (int32 scalar tensor, optional)
    is set to 1 if a has a nonzero row.  prev must be contiguous, a's shape."""
    a3 = _as3(a, "a").contiguous()
    require_cuda(a3, prev)
    if not prev.is_contiguous() or prev.shape != a3.shape or prev.dtype != a3.dtype:
        raise ShapeError(f"previous step copy must be a contiguous {tuple(a3.shape)} {a3.dtype} tensor")
    heads, rows, d = a3.shape
    mean = torch.empty(heads, dtype=torch.float64, device=a3.device)
    rc = torch.empty((heads, rows), dtype=torch.float64, device=a3.device)
    _lib.call("fb_row_cosine_update", _sim_code(a3), _p(a3), _p(prev), heads, rows, d, _p(rc), _p(mean),
              None if nonzero is None else _p(nonzero), _stream(a3))
    return mean


def pairwise_cosine(later, earlier):
    """All-pairs cosine [heads, rows, rows] between a later and an earlier
    step's rows (analysis.py:28-51), float64."""
    a3, b3 = _as3(later, "later").contiguous(), _as3(earlier, "earlier").contiguous()
    require_cuda(a3, b3)
    if a3.shape != b3.shape or a3.dtype != b3.dtype:
        raise ShapeError(f"step outputs must share a (block, head_dim) shape: "
                         f"{tuple(a3.shape)} vs {tuple(b3.shape)}")
    heads, rows, d = a3.shape
    out = torch.empty((heads, rows, rows), dtype=torch.float64, device=a3.device)
    _lib.call("fb_pairwise_cosine", _sim_code(a3), _p(a3), _p(b3), heads, rows, d, _p(out),
              _stream(a3))
    return out


def block_causal_attention(q, k, v, n_q: int, n_prefix: int = 0, block_size: int = 32,
                           scale: float | None = None, out=None, lse=None):
    """Prefill / commit attention (simulator.py:297-354).

    q [groups, heads_per_group * n_q, d]: a kv group's query heads stacked,
    each n_q positions; k, v [groups, cap, d] hold the committed prefix in rows
    [0, n_prefix) and the new positions' keys in [n_prefix, n_prefix + n_q).
    Row at position p attends rows [0, n_prefix + min(n_q, (p // B + 1) * B)).
    Returns (out, lse) in the mode's partial types (fp32 for bf16 inputs).
    """
    q3, k3, v3 = _as3(q, "q"), _as3(k, "k"), _as3(v, "v")
    require_cuda(q3, k3, v3)
    _check_kv(q3, k3, v3)
    q3, k3, v3 = q3.contiguous(), k3.contiguous(), v3.contiguous()
    groups, q_rows, d = q3.shape
    code = dtype_code(q3)
    ot, lt = PARTIAL_TYPES[code]
    if out is None:
        out = torch.empty((groups, q_rows, d), dtype=ot, device=q3.device)
    if lse is None:
        lse = torch.empty((groups, q_rows), dtype=lt, device=q3.device)
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    wsb = _lib.load().fb_block_causal_workspace_bytes(code, groups, q_rows, d)
    ws = WORKSPACE.get(q3.device, wsb) if wsb else None
    _lib.call("fb_block_causal_attention", code, _p(q3), _p(k3), _p(v3), groups, q_rows, int(n_q),
              d, k3.shape[1], int(n_prefix), int(block_size), scale, _p(out), _p(lse), _p(ws),
              0 if ws is None else ws.numel(), _stream(q3))
    return out, lse


def commit_block(k_cache, v_cache, k_block, v_block, lengths: torch.Tensor,
                 check: bool = False) -> None:
    """Append a finished block's K/V ([groups, B, d]) to each group's slab of
    the cache ([groups, N_cap, d]) at row lengths[g]; lengths advance by B."""
    kc, vc = _as3(k_cache, "k_cache"), _as3(v_cache, "v_cache")
    kb, vb = _as3(k_block, "k_block").contiguous(), _as3(v_block, "v_block").contiguous()
    require_cuda(kc, vc, kb, vb, lengths)
    if not (kc.is_contiguous() and vc.is_contiguous()):
        raise ShapeError("the KV cache must be contiguous")
    if kc.shape != vc.shape or kb.shape != vb.shape or kb.shape[0] != kc.shape[0] \
            or kb.shape[2] != kc.shape[2] or lengths.numel() != kc.shape[0]:
        raise ShapeError("cache / block / lengths shapes do not line up")
    if lengths.dtype != torch.int32 or not lengths.is_contiguous():
        raise ShapeError("lengths must be a contiguous int32 tensor")
    cnt = _empty_counter(kc.device) if check else None
    _lib.call("fb_commit_block", dtype_code(kc), _p(kc), _p(vc), kc.shape[0], kc.shape[1],
              kc.shape[2], _p(kb), _p(vb), kb.shape[1], _p(lengths), _p(cnt), _stream(kc))
    if cnt is not None and int(cnt.item()) > 0:
        from .errors import BoundsError
        raise BoundsError("block commit overflows the KV cache capacity")


def _empty_counter(device):
    return torch.zeros(1, dtype=torch.int32, device=device)


def _raise_if_empty(counter, what):
    if counter is not None and int(counter.item()) > 0:
        raise DegenerateInputError(f"{what}: some query rows have no keys on either side")


def internal_merge(q, k_in, v_in, o_ext, lse_ext, scale: float | None = None,
                   out_dtype: torch.dtype | None = None, want_lse: bool = False,
                   want_internal: bool = False, check: bool = False, out=None,
                   ext_stable: bool = False):
    """K2: block-internal partial fused with the merge against the cached
    external partial.  Returns out, or a tuple (out, lse_merged?, (o_int, lse_int)?).

    ext_stable: o_ext/lse_ext were not written by the kernel launched
    immediately before this one on the stream (FB_EXT_STABLE; true for cached
    steps), so the kernel may load them before its PDL wait."""
    q3, k3, v3 = _as3(q, "q"), _as3(k_in, "k_in"), _as3(v_in, "v_in")
    require_cuda(q3, k3, v3, o_ext, lse_ext)
    _check_kv(q3, k3, v3)
    q3, k3, v3 = q3.contiguous(), k3.contiguous(), v3.contiguous()
    groups, q_rows, d = q3.shape
    code = dtype_code(q3)
    ot, lt = PARTIAL_TYPES[code]
    o_ext = o_ext.contiguous()
    lse_ext = lse_ext.contiguous()
    o_ok = o_ext.dtype == ot or (code == _lib.FB_BF16 and o_ext.dtype == torch.bfloat16)
    if not o_ok or lse_ext.dtype != lt or o_ext.numel() != groups * q_rows * d \
            or lse_ext.numel() != groups * q_rows:
        raise ShapeError("cached partial does not match the queries (shape or precision)")
    if want_internal and o_ext.dtype != ot:
        raise ShapeError("want_internal needs the mode's fp32 cached partial")
    if out_dtype is None:
        out_dtype = ot
    if out is None:
        out = torch.empty((groups, q_rows, d), dtype=out_dtype, device=q3.device)
    lse_m = torch.empty((groups, q_rows), dtype=lt, device=q3.device) if want_lse else None
    o_int = torch.empty((groups, q_rows, d), dtype=ot, device=q3.device) if want_internal else None
    l_int = torch.empty((groups, q_rows), dtype=lt, device=q3.device) if want_internal else None
    cnt = _empty_counter(q3.device) if check else None
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    wsb = _lib.load().fb_internal_merge_workspace_bytes(code, groups, q_rows, d, k3.shape[1])
    ws = WORKSPACE.get(q3.device, wsb) if wsb else None
    _lib.call("fb_internal_merge_ex", _partial_code(code, o_ext), _p(q3), _p(k3), _p(v3), groups, q_rows, d, k3.shape[1],
              scale, _p(o_ext), _p(lse_ext), _p(out), _OUT_CODE[out.dtype], _p(lse_m), _p(o_int),
              _p(l_int), _p(cnt), _p(ws), 0 if ws is None else ws.numel(),
              _lib.FB_EXT_STABLE if ext_stable else 0, _stream(q3))
    _raise_if_empty(cnt, "internal_merge")
    if not (want_lse or want_internal):
        return out
    res = [out]
    if want_lse:
        res.append(lse_m)
    if want_internal:
        res.append((o_int, l_int))
    return tuple(res)


def _tok_stride(t: torch.Tensor, name: str) -> int:
    """Token stride of a token-major [b, B, H, d] view (heads x d contiguous)."""
    if t.dim() != 4 or t.stride(-1) != 1 or t.stride(-2) != t.shape[-1] \
            or t.stride(0) != t.shape[1] * t.stride(1):
        raise ShapeError(f"{name} must be a token-major [b, B, H, d] view with contiguous heads x d")
    return t.stride(1)


def internal_merge_tok(q_tok, k_tok, v_tok, o_ext, lse_ext, out_tok, scale: float | None = None,
                       ext_stable: bool = False):
    """K2 on token-major tensors (fb_internal_merge_tok): q_tok [b, B, Hq, d],
    k_tok / v_tok [b, B, Hkv, d] (views into a fused QKV projection output),
    out_tok [b, B, Hq, d] (the O projection's input); o_ext / lse_ext keep the
    stacked [b*Hkv, G*B, d] layout.  Same arithmetic as internal_merge."""
    require_cuda(q_tok, k_tok, v_tok, o_ext, lse_ext, out_tok)
    b, B, hq, d = q_tok.shape
    hkv = k_tok.shape[2]
    if k_tok.shape != (b, B, hkv, d) or v_tok.shape != k_tok.shape or out_tok.shape != q_tok.shape:
        raise ShapeError("token-major q / k / v / out shapes do not line up")
    qs, ks, vs, os_ = (_tok_stride(q_tok, "q"), _tok_stride(k_tok, "k_in"), _tok_stride(v_tok, "v_in"),
                       _tok_stride(out_tok, "out"))
    if o_ext.dtype not in (torch.float32, torch.bfloat16) or o_ext.numel() != b * hq * B * d \
            or lse_ext.numel() != b * hq * B:
        raise ShapeError("cached partial does not match the queries")
    if lse_ext.dtype != torch.float32 or not (o_ext.is_contiguous() and lse_ext.is_contiguous()):
        raise ShapeError("the cached partial must be contiguous (o_ext float32 or bfloat16, lse_ext float32)")
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    _lib.call("fb_internal_merge_tok", _partial_code(_CODE[q_tok.dtype], o_ext), _p(q_tok), qs, _p(k_tok), ks, _p(v_tok), vs, b, B,
              hq, hkv, d, scale, _p(o_ext), _p(lse_ext), _p(out_tok), _OUT_CODE[out_tok.dtype], os_,
              _lib.FB_EXT_STABLE if ext_stable else 0, _stream(q_tok))
    return out_tok


def combine(parts, out_dtype: torch.dtype | None = None, want_lse: bool = True,
            check: bool = False, out=None, lse=None):
    """K3: log-space merge of partials [(o, lse), ...] over disjoint key groups.
    out / lse: optional contiguous destinations (out's dtype is the output dtype)."""
    if not 1 <= len(parts) <= 16:
        raise ValueError("combine takes 1..16 partials")
    o0, l0 = parts[0]
    require_cuda(o0, l0)
    code = mode_of_partial(o0, l0)
    os_, ls_ = [], []
    for o, l in parts:
        if o.shape != o0.shape or l.shape != l0.shape:
            raise ShapeError(f"partial shapes differ: {tuple(o0.shape)} vs {tuple(o.shape)}")
        if mode_of_partial(o, l) != code:
            raise ShapeError("partials of different precision modes")
        os_.append(o.contiguous())
        ls_.append(l.contiguous())
    d = o0.shape[-1]
    rows = l0.numel()
    ot, lt = PARTIAL_TYPES[code]
    if out is not None:
        out_dtype = out.dtype
        if out.shape != o0.shape or not out.is_contiguous():
            raise ShapeError("combine: out must be a contiguous tensor of the partials' shape")
    out_dtype = ot if out_dtype is None else out_dtype
    if out is None:
        out = torch.empty(o0.shape, dtype=out_dtype, device=o0.device)
    if lse is not None:
        if lse.shape != l0.shape or lse.dtype != lt or not lse.is_contiguous():
            raise ShapeError("combine: lse must be a contiguous tensor of the lognorms' shape and dtype")
    elif want_lse:
        lse = torch.empty(l0.shape, dtype=lt, device=o0.device)
    cnt = _empty_counter(o0.device) if check else None
    _lib.call("fb_combine", code, len(parts), _lib.ptr_array([_p(o) for o in os_]),
              _lib.ptr_array([_p(l) for l in ls_]), rows, d, _p(out), _OUT_CODE[out_dtype], _p(lse),
              _p(cnt), _stream(o0))
    _raise_if_empty(cnt, "combine")
    return out, lse


def full_attention(q, k, v, n_ext: int, k_in, v_in, scale: float | None = None,
                   out_dtype: torch.dtype | None = None, o_ext=None, lse_ext=None,
                   check: bool = False, out=None):
    """K4 / refresh step: attention over [cache rows 0..n_ext) | current block],
    normalised output; the refreshed external partial lands in (o_ext, lse_ext)."""
    q3, k3, v3 = _as3(q, "q"), _as3(k, "k"), _as3(v, "v")
    ki3, vi3 = _as3(k_in, "k_in").contiguous(), _as3(v_in, "v_in").contiguous()
    require_cuda(q3, k3, v3, ki3, vi3)
    _check_kv(q3, k3, v3)
    _check_kv(q3, ki3, vi3)
    q3, k3, v3 = q3.contiguous(), k3.contiguous(), v3.contiguous()
    groups, q_rows, d = q3.shape
    code = dtype_code(q3)
    ot, lt = PARTIAL_TYPES[code]
    if o_ext is None:
        o_ext = torch.empty((groups, q_rows, d), dtype=ot, device=q3.device)
    if lse_ext is None:
        lse_ext = torch.empty((groups, q_rows), dtype=lt, device=q3.device)
    out_dtype = ot if out_dtype is None else out_dtype
    if out is None:
        out = torch.empty((groups, q_rows, d), dtype=out_dtype, device=q3.device)
    cnt = _empty_counter(q3.device) if check else None
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    lib = _lib.load()
    wsb = max(lib.fb_partial_workspace_bytes(code, groups, q_rows, d, int(n_ext)),
              lib.fb_internal_merge_workspace_bytes(code, groups, q_rows, d, ki3.shape[1]))
    ws = WORKSPACE.get(q3.device, wsb) if wsb else None
    _lib.call("fb_full_attention", code, _p(q3), _p(k3), _p(v3), groups, q_rows, d, k3.shape[1],
              int(n_ext), _p(ki3), _p(vi3), ki3.shape[1], scale, _p(o_ext), _p(lse_ext), _p(out),
              _OUT_CODE[out.dtype], _p(cnt), _p(ws), 0 if ws is None else ws.numel(), _stream(q3))
    _raise_if_empty(cnt, "full_attention")
    return out, o_ext, lse_ext


# ------------------------------------------------------------------ sparse


def mask_budget(n_ext: int, density: float, key_block_size: int) -> int:
    """min(nb, max(1, ceil(density*n_ext/kbs))) evaluated in double (sparse.py:126)."""
    return int(_lib.load().fb_mask_budget(int(n_ext), float(density), int(key_block_size)))


def _paged_table(page_table, groups):
    t = page_table.reshape(groups, -1)
    if t.dtype != torch.int32:
        t = t.to(torch.int32)
    return t.contiguous()


def block_mass(q, k, k_in, n_ext: int, key_block_size: int = 16, scale: float | None = None, *,
               page_table=None):
    """K5: float64 softmax mass per external key block, summed over each group's rows.
    With page_table ([groups, max_pages] int32), k is a page pool
    [num_pages, page_rows, d] read through the table (paged serving cache)."""
    q3, k3, ki3 = _as3(q, "q").contiguous(), _as3(k, "k").contiguous(), _as3(k_in, "k_in").contiguous()
    require_cuda(q3, k3, ki3)
    groups, q_rows, d = q3.shape
    if (page_table is None and k3.shape[0] != groups) or k3.shape[2] != d or ki3.shape[0] != groups \
            or ki3.shape[2] != d:
        raise ShapeError("q and keys must be 2-D with matching feature dim")
    code = dtype_code(q3)
    nb = -(-int(n_ext) // int(key_block_size))
    mass = torch.empty((groups, nb), dtype=torch.float64, device=q3.device)
    wsb = _lib.load().fb_block_mass_workspace_bytes_ex(code, groups, q_rows, d, int(n_ext),
                                                       ki3.shape[1], int(key_block_size))
    ws = WORKSPACE.get(q3.device, wsb)
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    if page_table is not None:
        require_cuda(page_table)
        t = _paged_table(page_table, groups)
        _lib.call("fb_block_mass_paged", code, _p(q3), _p(k3), _p(ki3), k3.shape[0], k3.shape[1], _p(t),
                  t.shape[1], groups, q_rows, d, int(n_ext), ki3.shape[1], int(key_block_size), scale,
                  _p(mass), _p(ws), ws.numel(), _stream(q3))
        return mass
    _lib.call("fb_block_mass", code, _p(q3), _p(k3), _p(ki3), groups, q_rows, d, k3.shape[1],
              int(n_ext), ki3.shape[1], int(key_block_size), scale, _p(mass), _p(ws), ws.numel(),
              _stream(q3))
    return mass


def topk_blocks(mass: torch.Tensor, budget: int) -> torch.Tensor:
    """K6: stable top-`budget` blocks per group (mass desc, index asc), ascending int32."""
    require_cuda(mass)
    m2 = mass.reshape(-1, mass.shape[-1]).contiguous()
    sel = torch.empty((m2.shape[0], int(budget)), dtype=torch.int32, device=mass.device)
    _lib.call("fb_topk_blocks", _p(m2), m2.shape[0], m2.shape[1], int(budget), _p(sel), _stream(m2))
    return sel


def sparse_partitioned(q, k, v, k_in, v_in, n_ext: int, selected: torch.Tensor,
                       key_block_size: int = 16, scale: float | None = None,
                       out_dtype: torch.dtype | None = None, check: bool = False, *, page_table=None):
    """K7: first sparse step -- (out, selected partial, residual partial).
    With page_table, k / v are page pools read through it (see block_mass)."""
    q3, k3, v3 = _as3(q, "q").contiguous(), _as3(k, "k").contiguous(), _as3(v, "v").contiguous()
    ki3, vi3 = _as3(k_in, "k_in").contiguous(), _as3(v_in, "v_in").contiguous()
    require_cuda(q3, k3, v3, ki3, vi3, selected)
    if page_table is None:
        _check_kv(q3, k3, v3)
    _check_kv(q3, ki3, vi3)
    groups, q_rows, d = q3.shape
    if page_table is None and k3.shape[1] < n_ext:
        raise ShapeError(f"key set has {k3.shape[1]} rows but mask covers {n_ext} external keys")
    sel = selected.reshape(groups, -1).to(torch.int32).contiguous()
    code = dtype_code(q3)
    ot, lt = PARTIAL_TYPES[code]
    mk = lambda: (torch.empty((groups, q_rows, d), dtype=ot, device=q3.device),
                  torch.empty((groups, q_rows), dtype=lt, device=q3.device))
    o_sel, l_sel = mk()
    o_res, l_res = mk()
    out_dtype = ot if out_dtype is None else out_dtype
    out = torch.empty((groups, q_rows, d), dtype=out_dtype, device=q3.device)
    cnt = _empty_counter(q3.device) if check else None
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    wsb = _lib.load().fb_sparse_workspace_bytes(code, groups, q_rows, d, int(n_ext), sel.shape[1],
                                                ki3.shape[1], int(key_block_size))
    ws = WORKSPACE.get(q3.device, wsb) if wsb else None
    if page_table is not None:
        t = _paged_table(page_table, groups)
        _lib.call("fb_sparse_partitioned_paged", code, _p(q3), _p(k3), _p(v3), _p(ki3), _p(vi3),
                  k3.shape[0], k3.shape[1], _p(t), t.shape[1], groups, q_rows, d, int(n_ext),
                  ki3.shape[1], _p(sel), sel.shape[1], int(key_block_size), scale, _p(o_sel), _p(l_sel),
                  _p(o_res), _p(l_res), _p(out), _OUT_CODE[out_dtype], _p(cnt), _p(ws),
                  0 if ws is None else ws.numel(), _stream(q3))
    else:
        _lib.call("fb_sparse_partitioned", code, _p(q3), _p(k3), _p(v3), _p(ki3), _p(vi3), groups,
                  q_rows, d, k3.shape[1], int(n_ext), ki3.shape[1], _p(sel), sel.shape[1],
                  int(key_block_size), scale, _p(o_sel), _p(l_sel), _p(o_res), _p(l_res), _p(out),
                  _OUT_CODE[out_dtype], _p(cnt), _p(ws), 0 if ws is None else ws.numel(), _stream(q3))
    _raise_if_empty(cnt, "sparse_partitioned")
    return out, (o_sel, l_sel), (o_res, l_res)


def sparse_attend_merge(q, k, v, k_in, v_in, n_ext: int, selected: torch.Tensor,
                        residual=None, key_block_size: int = 16, scale: float | None = None,
                        out_dtype: torch.dtype | None = None, check: bool = False, *, page_table=None):
    """K8: later sparse steps -- selected blocks + current block, merged with
    the cached residual (or renormalised sparse-only when residual is None)."""
    q3, k3, v3 = _as3(q, "q").contiguous(), _as3(k, "k").contiguous(), _as3(v, "v").contiguous()
    ki3, vi3 = _as3(k_in, "k_in").contiguous(), _as3(v_in, "v_in").contiguous()
    require_cuda(q3, k3, v3, ki3, vi3, selected)
    if page_table is None:
        _check_kv(q3, k3, v3)
    _check_kv(q3, ki3, vi3)
    groups, q_rows, d = q3.shape
    if page_table is None and k3.shape[1] < n_ext:
        raise ShapeError(f"key set has {k3.shape[1]} rows but mask covers {n_ext} external keys")
    sel = selected.reshape(groups, -1).to(torch.int32).contiguous()
    code = dtype_code(q3)
    ot, lt = PARTIAL_TYPES[code]
    o_res = l_res = None
    if residual is not None:
        o_res, l_res = residual[0].contiguous(), residual[1].contiguous()
        if (o_res.dtype, l_res.dtype) != (ot, lt):
            raise ShapeError("residual precision does not match the queries")
    out_dtype = ot if out_dtype is None else out_dtype
    out = torch.empty((groups, q_rows, d), dtype=out_dtype, device=q3.device)
    cnt = _empty_counter(q3.device) if check else None
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    wsb = _lib.load().fb_sparse_workspace_bytes(code, groups, q_rows, d, int(n_ext), sel.shape[1],
                                                ki3.shape[1], int(key_block_size))
    ws = WORKSPACE.get(q3.device, wsb) if wsb else None
    if page_table is not None:
        t = _paged_table(page_table, groups)
        _lib.call("fb_sparse_attend_merge_paged", code, _p(q3), _p(k3), _p(v3), _p(ki3), _p(vi3),
                  k3.shape[0], k3.shape[1], _p(t), t.shape[1], groups, q_rows, d, int(n_ext),
                  ki3.shape[1], _p(sel), sel.shape[1], int(key_block_size), scale, _p(o_res), _p(l_res),
                  _p(out), _OUT_CODE[out_dtype], _p(cnt), _p(ws), 0 if ws is None else ws.numel(),
                  _stream(q3))
    else:
        _lib.call("fb_sparse_attend_merge", code, _p(q3), _p(k3), _p(v3), _p(ki3), _p(vi3), groups,
                  q_rows, d, k3.shape[1], int(n_ext), ki3.shape[1], _p(sel), sel.shape[1],
                  int(key_block_size), scale, _p(o_res), _p(l_res), _p(out), _OUT_CODE[out_dtype],
                  _p(cnt), _p(ws), 0 if ws is None else ws.numel(), _stream(q3))
    _raise_if_empty(cnt, "sparse_attend_merge")
    return out
