"""ctypes binding of libfb200.so (the C ABI in include/flashblock_b200.h).

There is no CPU fallback: if the library is missing, or no CUDA device is
present, calls raise.  The library is built in-tree by
``python -m paper_2602_05305_b200.build`` (or ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import (BoundsError, DegenerateInputError, ReusePreconditionError, ShapeError,
                     StalenessError)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libfb200.so")
# diagnostics only (A/B of two builds on one box): FB_LIB_PATH overrides the in-tree library
LIB_PATH = os.environ.get("FB_LIB_PATH", LIB_PATH)

FB_OK, FB_ERR_SHAPE, FB_ERR_BOUNDS, FB_ERR_DEGENERATE = 0, 1, 2, 3
FB_ERR_REUSE, FB_ERR_STALE, FB_ERR_CUDA, FB_ERR_VALUE, FB_ERR_UNSUPPORTED = 4, 5, 6, 7, 8
FB_F64, FB_F32, FB_BF16 = 0, 1, 2
FB_EXT_STABLE = 1  # fb_internal_merge_ex flag
FB_PARTIAL_BF16 = 0x100  # OR'ed into FB_BF16: the partial's O is stored as bf16

vp, i64, i32, dbl, sz = C.c_void_p, C.c_int64, C.c_int, C.c_double, C.c_size_t

# name -> (restype, argtypes); mirrors include/flashblock_b200.h
SIGNATURES = {
    "fb_last_error": (C.c_char_p, []),
    "fb_p2p_alloc": (i32, [sz, vp, vp]),
    "fb_p2p_free": (i32, [vp]),
    "fb_p2p_open": (i32, [vp, vp]),
    "fb_p2p_close": (i32, [vp]),
    "fb_p2p_signal": (i32, [vp, i32, i32, C.c_uint64, vp]),
    "fb_p2p_wait": (i32, [vp, i32, C.c_uint64, vp]),
    "fb_internal_merge_host": (i32, [i32, vp, vp, vp, i64, i64, i64, i64, dbl, vp, vp, vp, vp, vp,
                                     vp, vp]),
    "fb_version": (C.c_char_p, []),
    "fb_launch_count": (i64, []),
    "fb_partial_workspace_bytes": (sz, [i32, i64, i64, i64, i64]),
    "fb_attention_partial_sync": (i32, [i32, vp, vp, vp, i64, i64, i64, i64, i64, i64, dbl, vp, vp,
                                        vp, sz, vp, i64, vp]),
    "fb_sync_flags_count": (i64, []),
    "fb_attention_partial": (i32, [i32, vp, vp, vp, i64, i64, i64, i64, i64, i64, dbl, vp, vp,
                                   vp, sz, vp]),
    "fb_attention_partial_ragged": (i32, [i32, vp, vp, vp, i64, i64, i64, i64, i64, vp, dbl, vp,
                                          vp, vp, sz, vp]),
    "fb_ragged_workspace_bytes": (sz, [i32, i64, i64, i64, i64]),
    "fb_block_causal_attention": (i32, [i32, vp, vp, vp, i64, i64, i64, i64, i64, i64, i64, dbl,
                                        vp, vp, vp, sz, vp]),
    "fb_block_causal_workspace_bytes": (sz, [i32, i64, i64, i64]),
    "fb_attention_partial_groups": (i32, [i32, vp, vp, vp, i64, i64, i64, i64, i64, i64, vp, i64,
                                          dbl, vp, vp, vp, sz, vp]),
    "fb_row_cosine": (i32, [i32, vp, vp, i64, i64, i64, vp, vp, vp]),
    "fb_row_cosine_update": (i32, [i32, vp, vp, i64, i64, i64, vp, vp, vp, vp]),
    "fb_pairwise_cosine": (i32, [i32, vp, vp, i64, i64, i64, vp, vp]),
    "fb_commit_block": (i32, [i32, vp, vp, i64, i64, i64, vp, vp, i64, vp, vp, vp]),
    "fb_attention_partial_paged": (i32, [i32, vp, vp, vp, i64, i64, vp, i64, i64, i64, i64, vp, dbl,
                                         vp, vp, vp, sz, vp]),
    "fb_paged_workspace_bytes": (sz, [i32, i64, i64, i64]),
    "fb_block_causal_attention_paged": (i32, [i32, vp, vp, vp, i64, i64, vp, i64, i64, i64, i64, i64,
                                              i64, i64, dbl, vp, vp, vp, sz, vp]),
    "fb_block_mass_paged": (i32, [i32, vp, vp, vp, i64, i64, vp, i64, i64, i64, i64, i64, i64, i64,
                                  dbl, vp, vp, sz, vp]),
    "fb_sparse_partitioned_paged": (i32, [i32, vp, vp, vp, vp, vp, i64, i64, vp, i64, i64, i64, i64,
                                          i64, i64, vp, i64, i64, dbl, vp, vp, vp, vp, vp, i32, vp, vp,
                                          sz, vp]),
    "fb_sparse_attend_merge_paged": (i32, [i32, vp, vp, vp, vp, vp, i64, i64, vp, i64, i64, i64, i64,
                                           i64, i64, vp, i64, i64, dbl, vp, vp, vp, i32, vp, vp, sz,
                                           vp]),
    "fb_internal_merge_tok": (i32, [i32, vp, i64, vp, i64, vp, i64, i64, i64, i64, i64, i64, dbl, vp, vp,
                                    vp, i32, i64, i32, vp]),
    "fb_commit_block_paged": (i32, [i32, vp, vp, i64, vp, i64, i64, i64, vp, vp, i64, vp, vp, vp]),
    "fb_internal_merge": (i32, [i32, vp, vp, vp, i64, i64, i64, i64, dbl, vp, vp, vp, i32, vp,
                                vp, vp, vp, vp, sz, vp]),
    "fb_internal_merge_ex": (i32, [i32, vp, vp, vp, i64, i64, i64, i64, dbl, vp, vp, vp, i32, vp,
                                   vp, vp, vp, vp, sz, i32, vp]),
    "fb_internal_merge_workspace_bytes": (sz, [i32, i64, i64, i64, i64]),
    "fb_combine": (i32, [i32, i32, vp, vp, i64, i64, vp, i32, vp, vp, vp]),
    "fb_full_attention": (i32, [i32, vp, vp, vp, i64, i64, i64, i64, i64, vp, vp, i64, dbl, vp,
                                vp, vp, i32, vp, vp, sz, vp]),
    "fb_block_mass": (i32, [i32, vp, vp, vp, i64, i64, i64, i64, i64, i64, i64, dbl, vp, vp, sz,
                            vp]),
    "fb_block_mass_workspace_bytes": (sz, [i64, i64]),
    "fb_block_mass_workspace_bytes_ex": (sz, [i32, i64, i64, i64, i64, i64, i64]),
    "fb_topk_blocks": (i32, [vp, i64, i64, i64, vp, vp]),
    "fb_mask_budget": (i64, [i64, dbl, i64]),
    "fb_sparse_partitioned": (i32, [i32, vp, vp, vp, vp, vp, i64, i64, i64, i64, i64, i64, vp,
                                    i64, i64, dbl, vp, vp, vp, vp, vp, i32, vp, vp, sz, vp]),
    "fb_sparse_attend_merge": (i32, [i32, vp, vp, vp, vp, vp, i64, i64, i64, i64, i64, i64, vp,
                                     i64, i64, dbl, vp, vp, vp, i32, vp, vp, sz, vp]),
    "fb_sparse_workspace_bytes": (sz, [i32, i64, i64, i64, i64, i64, i64, i64]),
}

_lib = None


def load() -> C.CDLL:
    """Load libfb200.so (once) and declare every exported signature."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2602_05305_b200.build` "
                "(no CPU fallback exists)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error() -> str:
    msg = load().fb_last_error()
    return msg.decode() if msg else ""


_STATUS_EXC = {
    FB_ERR_SHAPE: ShapeError,
    FB_ERR_BOUNDS: BoundsError,
    FB_ERR_DEGENERATE: DegenerateInputError,
    FB_ERR_REUSE: ReusePreconditionError,
    FB_ERR_STALE: StalenessError,
    FB_ERR_VALUE: ValueError,
    FB_ERR_UNSUPPORTED: NotImplementedError,
}


def check(status: int, what: str) -> None:
    """Map a non-OK fb_status to the reference-named exception."""
    if status == FB_OK:
        return
    exc = _STATUS_EXC.get(status, RuntimeError)
    raise exc(f"{what}: {last_error()} (fb_status={status})")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def ptr_array(ptrs) -> C.Array:
    arr = (C.c_void_p * len(ptrs))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr
