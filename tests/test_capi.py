"""CPU-side checks of the C-ABI boundary: the library loads, exports every
symbol include/flashblock_b200.h declares, and its host-only logic (argument
validation, budget arithmetic) matches the reference.  No kernel launches."""

import ctypes
import os
import re

import pytest

from oracle import flashblock_oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "flashblock_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"FB_API\s+[\w\s\*]+?\b(fb_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2602_05305_b200 import _lib

    return _lib.load()


def test_header_declares_the_hot_path():
    syms = header_symbols()
    for name in ("fb_attention_partial", "fb_internal_merge", "fb_combine", "fb_full_attention",
                 "fb_block_mass", "fb_topk_blocks", "fb_sparse_partitioned",
                 "fb_sparse_attend_merge", "fb_last_error"):
        assert name in syms


def test_library_exports_every_declared_symbol(lib):
    from paper_2602_05305_b200 import _lib

    for name in header_symbols():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"


def test_version_string(lib):
    assert b"sm_100a" in lib.fb_version()


@pytest.mark.parametrize("n_ext,density,kbs", [(160, 0.001, 16), (160, 0.1, 16), (160, 0.2, 16),
                                               (160, 0.5, 16), (160, 1.0, 16), (20, 1.0, 16),
                                               (65536, 0.3, 16), (1000, 0.07, 16), (7, 0.5, 3)])
def test_mask_budget_matches_reference(lib, n_ext, density, kbs):
    nb = -(-n_ext // kbs)
    assert lib.fb_mask_budget(n_ext, density, kbs) == orc.mask_budget(nb, density, n_ext, kbs)


def test_validation_errors_need_no_device(lib):
    from paper_2602_05305_b200 import _lib

    # unknown dtype
    assert lib.fb_attention_partial(9, None, None, None, 1, 1, 8, 4, 0, 4, 1.0, None, None, None,
                                     0, None) == _lib.FB_ERR_VALUE
    # key range outside the slab -> BoundsError
    assert lib.fb_attention_partial(_lib.FB_F32, None, None, None, 1, 1, 8, 4, 0, 5, 1.0, None,
                                     None, None, 0, None) == _lib.FB_ERR_BOUNDS
    assert "outside" in _lib.last_error()
    # too many combine parts
    assert lib.fb_combine(_lib.FB_F32, 17, None, None, 1, 8, None, _lib.FB_F32, None, None,
                          None) == _lib.FB_ERR_VALUE
    # bad budget
    assert lib.fb_topk_blocks(None, 1, 4, 5, None, None) == _lib.FB_ERR_VALUE
    with pytest.raises(ValueError):
        _lib.check(_lib.FB_ERR_VALUE, "x")


def test_prefill_subset_and_similarity_validation_need_no_device(lib):
    from paper_2602_05305_b200 import _lib

    bc = lib.fb_block_causal_attention
    # q_rows not a multiple of n_q -> ShapeError
    assert bc(_lib.FB_BF16, None, None, None, 2, 100, 32, 128, 64, 0, 32, 1.0, None, None, None, 0,
              None) == _lib.FB_ERR_SHAPE
    # prompt does not fit the slab -> BoundsError
    assert bc(_lib.FB_BF16, None, None, None, 2, 64, 32, 128, 40, 10, 32, 1.0, None, None, None, 0,
              None) == _lib.FB_ERR_BOUNDS
    # block size < 1 -> ValueError
    assert bc(_lib.FB_BF16, None, None, None, 2, 64, 32, 128, 64, 0, 0, 1.0, None, None, None, 0,
              None) == _lib.FB_ERR_VALUE
    gp = lib.fb_attention_partial_groups
    # list longer than the batch of groups -> ShapeError; no list -> ValueError
    assert gp(_lib.FB_BF16, None, None, None, 2, 128, 128, 64, 0, 64, None, 3, 1.0, None, None,
              None, 0, None) == _lib.FB_ERR_SHAPE
    assert gp(_lib.FB_BF16, None, None, None, 2, 128, 128, 64, 0, 64, None, 1, 1.0, None, None,
              None, 0, None) == _lib.FB_ERR_VALUE
    assert gp(_lib.FB_BF16, None, None, None, 2, 128, 128, 64, 0, 65, None, 1, 1.0, None, None,
              None, 0, None) == _lib.FB_ERR_BOUNDS
    # row cosine needs its row buffer
    assert lib.fb_row_cosine(_lib.FB_F32, None, None, 2, 3, 8, None, None, None) == _lib.FB_ERR_VALUE
    assert lib.fb_row_cosine_update(_lib.FB_F32, None, None, 2, 3, 8, None, None, None, None) == _lib.FB_ERR_VALUE
    # token-major cached step: bf16 only, GQA divisibility, d 128 and G * B <= 128 (checked before any launch)
    tok = lambda dt, b, blk, hq, hkv, d, od=_lib.FB_BF16, fl=0: lib.fb_internal_merge_tok(
        dt, None, 6144, None, 6144, None, 6144, b, blk, hq, hkv, d, 1.0, None, None, None, od, 4096, fl, None)
    assert tok(_lib.FB_F32, 2, 32, 32, 8, 128) == _lib.FB_ERR_UNSUPPORTED
    assert tok(_lib.FB_BF16, 2, 32, 32, 6, 128) == _lib.FB_ERR_SHAPE
    assert tok(_lib.FB_BF16, 2, 32, 32, 8, 64) == _lib.FB_ERR_UNSUPPORTED
    # supported shape but null device pointers -> ValueError before any tensor map is built
    assert tok(_lib.FB_BF16, 2, 32, 32, 8, 128) == _lib.FB_ERR_VALUE
    assert tok(_lib.FB_BF16, 2, 64, 32, 8, 128) == _lib.FB_ERR_UNSUPPORTED  # G * B = 256 rows
    assert tok(_lib.FB_BF16, 2, 32, 32, 8, 128, fl=8) == _lib.FB_ERR_VALUE
    assert tok(_lib.FB_BF16, 0, 32, 32, 8, 128) == _lib.FB_OK  # empty batch: nothing to do
    # unknown cached-step flags
    assert lib.fb_internal_merge_ex(_lib.FB_BF16, None, None, None, 1, 1, 128, 32, 1.0, None, None,
                                    None, _lib.FB_BF16, None, None, None, None, None, 0, 8,
                                    None) == _lib.FB_ERR_VALUE


def test_status_maps_to_reference_exception_types():
    from paper_2602_05305_b200 import _lib
    from paper_2602_05305_b200.errors import (BoundsError, DegenerateInputError,
                                              ReusePreconditionError, ShapeError, StalenessError)

    for code, exc, base in [(_lib.FB_ERR_SHAPE, ShapeError, ValueError),
                            (_lib.FB_ERR_BOUNDS, BoundsError, IndexError),
                            (_lib.FB_ERR_DEGENERATE, DegenerateInputError, ValueError),
                            (_lib.FB_ERR_REUSE, ReusePreconditionError, RuntimeError),
                            (_lib.FB_ERR_STALE, StalenessError, RuntimeError)]:
        with pytest.raises(exc):
            _lib.check(code, "probe")
        assert issubclass(exc, base)
