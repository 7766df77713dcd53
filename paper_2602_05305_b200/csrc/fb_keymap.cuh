// Key-row maps: which key/value rows a partial attends, in which order.
//
// A partial is "softmax attention over a key group" (attention.py:60-101).
// The groups the hot path needs are
//   RangeMap      contiguous committed rows [begin, end)        (attention.py:202)
//   SelectedMap   mask-selected 16-row blocks of the committed rows, then
//                 every current-block row from a separate k_in/v_in slab
//                                                          (sparse.py:167,171,182)
//   ResidualMap   the committed rows NOT in the selected blocks (sparse.py:170-174)
// Each map turns a dense key ordinal t in [0, count) into a row pointer.
#pragma once

#include <stdint.h>

namespace fb {

template <typename T>
struct RangeMap {
  const T* k;          // group 0 slab base
  const T* v;
  int64_t slab_stride; // elements between groups' slabs (kv_rows_cap*d)
  int64_t begin, end;
  int64_t d;
  __device__ __forceinline__ int64_t count(int64_t) const { return end - begin; }
  __device__ __forceinline__ void row(int64_t g, int64_t t, const T*& kr, const T*& vr) const {
    const int64_t off = g * slab_stride + (begin + t) * d;
    kr = k + off;
    vr = v + off;
  }
};

// Per-sequence (ragged) committed lengths: group g attends slab rows
// [begin, min(ends[g], cap)) -- the serving layout where every sequence of the
// batch has its own context length.
template <typename T>
struct RaggedMap {
  const T* k;
  const T* v;
  const int32_t* ends;  // device [groups]
  int64_t slab_stride, begin, cap, d;
  __device__ __forceinline__ int64_t count(int64_t g) const {
    const int64_t e = min((int64_t)ends[g], cap);
    return e > begin ? e - begin : 0;
  }
  __device__ __forceinline__ void row(int64_t g, int64_t t, const T*& kr, const T*& vr) const {
    const int64_t off = g * slab_stride + (begin + t) * d;
    kr = k + off;
    vr = v + off;
  }
};

// Committed rows [0, n_ext) of the slab, then the n_in current-block rows of
// a separate [groups, n_in, d] tensor: the full key stream of a step
// (simulator.py:425-429) without materialising the concatenation.
template <typename T>
struct ConcatMap {
  const T* k;
  const T* v;
  const T* k_in;
  const T* v_in;
  int64_t slab_stride, n_ext, n_in, d;
  __device__ __forceinline__ int64_t count(int64_t) const { return n_ext + n_in; }
  __device__ __forceinline__ void row(int64_t g, int64_t t, const T*& kr, const T*& vr) const {
    if (t < n_ext) {
      const int64_t off = g * slab_stride + t * d;
      kr = k + off;
      vr = v ? v + off : nullptr;
    } else {
      const int64_t off = (g * n_in + (t - n_ext)) * d;
      kr = k_in + off;
      vr = v_in ? v_in + off : nullptr;
    }
  }
};

// Block-causal prefill / commit keys (simulator.py:297-354): slab rows
// [0, n_prefix + n_q); query row r (position p = r % n_q of its head) attends
// rows [0, n_prefix + min(n_q, (p / blk + 1) * blk)).
template <typename T>
struct CausalMap {
  const T* k;
  const T* v;
  int64_t slab_stride, d, n_q, blk, n_prefix;
  static constexpr bool kCausal = true;
  __device__ __forceinline__ int64_t count(int64_t) const { return n_prefix + n_q; }
  __device__ __forceinline__ void row(int64_t g, int64_t t, const T*& kr, const T*& vr) const {
    const int64_t off = g * slab_stride + t * d;
    kr = k + off;
    vr = v + off;
  }
  __device__ __forceinline__ int64_t row_limit(int64_t grow) const {
    const int64_t p = grow % n_q;
    const int64_t e = (p / blk + 1) * blk;
    return n_prefix + (e < n_q ? e : n_q);
  }
};

template <typename M, typename = void>
struct is_causal_map { static constexpr bool value = false; };
template <typename M>
struct is_causal_map<M, decltype((void)M::kCausal)> { static constexpr bool value = M::kCausal; };

// Number of external rows covered by `n_sel` ascending selected blocks; only the
// last selected block can be the clipped tail block (sparse.py:69-80).
__device__ __forceinline__ int64_t selected_rows(const int32_t* sel, int64_t n_sel, int64_t kbs,
                                                 int64_t n_ext) {
  if (n_sel == 0) return 0;
  const int64_t last = sel[n_sel - 1];
  const int64_t last_rows = min(kbs, n_ext - last * kbs);
  return (n_sel - 1) * kbs + last_rows;
}

template <typename T>
struct SelectedMap {
  const T* k;
  const T* v;
  const T* k_in;       // [groups, n_in, d]
  const T* v_in;
  const int32_t* sel;  // [groups, n_sel]
  int64_t n_sel, kbs, n_ext, n_in, slab_stride, d;
  __device__ __forceinline__ int64_t count(int64_t g) const {
    return selected_rows(sel + g * n_sel, n_sel, kbs, n_ext) + n_in;
  }
  __device__ __forceinline__ void row(int64_t g, int64_t t, const T*& kr, const T*& vr) const {
    const int32_t* s = sel + g * n_sel;
    const int64_t n_ext_sel = selected_rows(s, n_sel, kbs, n_ext);
    if (t < n_ext_sel) {
      const int64_t r = (int64_t)s[t / kbs] * kbs + (t % kbs);
      const int64_t off = g * slab_stride + r * d;
      kr = k + off;
      vr = v + off;
    } else {
      const int64_t off = (g * n_in + (t - n_ext_sel)) * d;
      kr = k_in + off;
      vr = v_in + off;
    }
  }
};

template <typename T>
struct ResidualMap {
  const T* k;
  const T* v;
  const int32_t* sel;
  int64_t n_sel, kbs, n_ext, slab_stride, d;
  __device__ __forceinline__ int64_t count(int64_t g) const {
    return n_ext - selected_rows(sel + g * n_sel, n_sel, kbs, n_ext);
  }
  // t-th unselected external row: unselected block u = t / kbs is the smallest
  // block b with b - |{selected < b}| == u (binary search over the ascending list).
  __device__ __forceinline__ void row(int64_t g, int64_t t, const T*& kr, const T*& vr) const {
    const int32_t* s = sel + g * n_sel;
    const int64_t u = t / kbs;
    int64_t lo = 0, hi = n_sel;  // count of selected blocks below the answer
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)s[mid] - mid <= u) lo = mid + 1; else hi = mid;
    }
    const int64_t b = u + lo;
    const int64_t r = b * kbs + (t % kbs);
    const int64_t off = g * slab_stride + r * d;
    kr = k + off;
    vr = v + off;
  }
};

}  // namespace fb
