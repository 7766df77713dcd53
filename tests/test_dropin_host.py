"""The numpy drop-in path (attention.py on host arrays): one host<->device
round trip per reference call.

* fb_internal_merge_host (C-ABI cached step on host buffers) argument checks
  run without a GPU;
* on the GPU: the host-buffer cached step equals the general device path
  bit for bit; a partial returned by this module is used from its device
  mirror, and an in-place edit of the host arrays invalidates the mirror
  (the edited values are what the next call sees, as in the reference);
  rows with no keys on either side raise DegenerateInputError.
"""

import ctypes

import numpy as np
import pytest

from paper_2602_05305_b200 import _lib


@pytest.fixture(scope="module")
def lib():
    try:
        return _lib.load()
    except OSError as e:  # pragma: no cover - the build step provides the library
        pytest.skip(f"libfb200.so not built: {e}")


def test_host_merge_rejects_bf16_and_null_pointers(lib):
    null = None
    rc = lib.fb_internal_merge_host(_lib.FB_BF16, null, null, null, 1, 4, 8, 4, 0.5, null, null, null,
                                    null, null, null, null)
    assert rc == _lib.FB_ERR_UNSUPPORTED
    rc = lib.fb_internal_merge_host(_lib.FB_F32, null, null, null, 1, 4, 8, 4, 0.5, null, null, null,
                                    null, null, null, null)
    assert rc == _lib.FB_ERR_VALUE
    rc = lib.fb_internal_merge_host(_lib.FB_F64, null, null, null, 1, 4, 0, 4, 0.5, null, null, null,
                                    null, null, null, null)
    assert rc == _lib.FB_ERR_SHAPE
    # empty query block: nothing to do, nothing touched
    cnt = ctypes.c_int64(7)
    rc = lib.fb_internal_merge_host(_lib.FB_F64, null, null, null, 1, 0, 8, 4, 0.5, null, null, null,
                                    null, null, ctypes.addressof(cnt), null)
    assert rc == _lib.FB_OK and cnt.value == 0


@pytest.mark.gpu
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_host_cached_step_equals_device_path(lib, dt):
    import torch

    from paper_2602_05305_b200 import attention as A

    rng = np.random.default_rng(3)
    q = rng.standard_normal((32, 64)).astype(dt)
    k = rng.standard_normal((1000 + 32, 64)).astype(dt)
    v = rng.standard_normal((1000 + 32, 64)).astype(dt)
    ext, _ = A.attention_streamed(q, k, v, 1000, 0.125)
    assert ext._device_mirror() is not None
    before = lib.fb_launch_count()
    out_h, int_h = A.attention_with_reuse(q, A.CacheEntry(ext, 0), k[1000:], v[1000:], 0.125)
    assert lib.fb_launch_count() > before
    # the general device path on torch tensors, same precision mode
    dev = torch.device("cuda")
    ot = torch.from_numpy(ext.out).to(dev)
    lt = torch.from_numpy(ext.lognorm).to(dev)
    out_d, int_d = A.attention_with_reuse(torch.from_numpy(q).to(dev), A.CacheEntry(A.AttnPartial(ot, lt), 0),
                                          torch.from_numpy(k[1000:]).to(dev), torch.from_numpy(v[1000:]).to(dev),
                                          0.125)
    np.testing.assert_array_equal(out_h, out_d.cpu().numpy())
    np.testing.assert_array_equal(int_h.out, int_d.out.cpu().numpy())
    np.testing.assert_array_equal(int_h.lognorm, int_d.lognorm.cpu().numpy())
    assert out_h.dtype == dt and int_h.lognorm.dtype == np.float64


@pytest.mark.gpu
def test_mirror_follows_in_place_edits(lib):
    from paper_2602_05305_b200 import attention as A

    rng = np.random.default_rng(4)
    q = rng.standard_normal((16, 32))
    k = rng.standard_normal((300, 32))
    v = rng.standard_normal((300, 32))
    ext, _ = A.attention_streamed(q, k, v, 280)
    ext.out *= 2.0  # edit the host partial in place: the mirror must not be used
    assert ext._device_mirror() is None
    out_a, _ = A.attention_with_reuse(q, A.CacheEntry(ext, 0), k[280:], v[280:])
    fresh = A.AttnPartial(ext.out.copy(), ext.lognorm.copy())  # no mirror: uploaded
    out_b, _ = A.attention_with_reuse(q, A.CacheEntry(fresh, 0), k[280:], v[280:])
    np.testing.assert_array_equal(out_a, out_b)


@pytest.mark.gpu
def test_host_cached_step_raises_on_degenerate_rows(lib):
    from paper_2602_05305_b200 import attention as A
    from paper_2602_05305_b200.errors import DegenerateInputError

    rng = np.random.default_rng(5)
    q = rng.standard_normal((8, 16))
    k = rng.standard_normal((0, 16))
    ext, _ = A.attention_streamed(q, k, k, 0)  # empty external partial (sentinel rows)
    assert ext._device_mirror() is not None
    with pytest.raises(DegenerateInputError):
        A.attention_with_reuse(q, A.CacheEntry(ext, 0), k, k)


@pytest.mark.gpu
def test_host_cached_step_mixed_dtypes_and_value_width(lib):
    """Mixed numpy dtypes promote like the reference (float64 wins); a value
    width != key width takes the general device path; both equal the oracle."""
    from oracle import flashblock_oracle as orc
    from paper_2602_05305_b200 import attention as A

    rng = np.random.default_rng(7)
    q = rng.standard_normal((12, 16)).astype(np.float32)
    k = rng.standard_normal((200, 16))           # float64
    v = rng.standard_normal((200, 16)).astype(np.float32)
    ext, _ = A.attention_streamed(q, k, v, 180)
    out, internal = A.attention_with_reuse(q, A.CacheEntry(ext, 0), k[180:], v[180:])
    ref = orc.dense(q.astype(np.float64), k, v.astype(np.float64))
    assert out.dtype == np.float32 and internal.lognorm.dtype == np.float64
    np.testing.assert_allclose(out, ref, rtol=0, atol=1e-5 * np.abs(ref).max())
    # value width 12 != key width 16
    v12 = rng.standard_normal((200, 12))
    ext12, _ = A.attention_streamed(q.astype(np.float64), k, v12, 180)
    out12, _ = A.attention_with_reuse(q.astype(np.float64), A.CacheEntry(ext12, 0), k[180:], v12[180:])
    np.testing.assert_allclose(out12, orc.dense(q.astype(np.float64), k, v12), rtol=0, atol=1e-10)
