// Sparse key-block selection: K5 block mass and K6 stable top-k.
//
// Reference: build_sparse_mask (sparse.py:83-136).  The softmax runs over ALL
// keys passed -- the committed context [0, n_ext) plus the current block --
// with per-row normalisation (linalg.py:52-65, used at sparse.py:119); the
// mass of external block b is the sum of those probabilities over the block's
// rows and over every query row (sparse.py:120-125); the budget is
// min(nb, max(1, ceil(density*n_ext/kbs))) (sparse.py:126) and ranking is a
// stable sort on -mass, i.e. ties go to the lower block index (sparse.py:127),
// emitted ascending (sparse.py:128).
//
// Mass = sum_r sum_{t in b} exp(s_rt - lse_r), with lse_r the row log-sum-exp
// over all keys (computed by the partial kernel in lognorm-only mode).  Block
// sums use a fixed reduction order, so equal inputs give bit-equal masses and
// the tie rule is exact.
#include "fb_kernels.cuh"

namespace fb {

constexpr int MASS_WARPS = 8;

// grid: (ceil(nb / MASS_WARPS), groups); block: 32*MASS_WARPS.
// smem: K rows of the CTA's blocks [MASS_WARPS*kbs][d+1] in the score type.
template <typename Mode>
__global__ void __launch_bounds__(32 * MASS_WARPS)
block_mass_kernel(const typename Mode::Tin* __restrict__ q, const typename Mode::Tin* __restrict__ k,
                  const double* __restrict__ row_lse, int64_t q_rows, int64_t head_dim,
                  int64_t slab_stride, int64_t n_ext, int64_t kbs, int64_t nb, double scale,
                  double* __restrict__ mass) {
  using Ts = typename Mode::Ts;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Ts* ks = reinterpret_cast<Ts*>(smem_raw);
  const int64_t g = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b0 = (int64_t)blockIdx.x * MASS_WARPS;
  const int64_t ld = head_dim + 1;

  // stage the keys of this CTA's blocks
  const int64_t key0 = b0 * kbs;
  const int64_t nkeys = min((int64_t)MASS_WARPS * kbs, n_ext - key0);
  for (int64_t i = threadIdx.x; i < nkeys * head_dim; i += blockDim.x) {
    const int64_t t = i / head_dim, c = i % head_dim;
    ks[t * ld + c] = cvt<Ts>(k[g * slab_stride + (key0 + t) * head_dim + c]);
  }
  __syncthreads();

  const int64_t b = b0 + warp;
  if (b >= nb) return;
  const int64_t lo = b * kbs;
  const int64_t hi = min(lo + kbs, n_ext);
  double acc = 0.0;
  for (int64_t t = lo + lane; t < hi; t += 32) {
    const Ts* kr = ks + (t - key0) * ld;
    double part = 0.0;
    for (int64_t r = 0; r < q_rows; ++r) {
      const typename Mode::Tin* qr = q + (g * q_rows + r) * head_dim;
      Ts s = 0;
      for (int64_t c = 0; c < head_dim; ++c) s += cvt<Ts>(qr[c]) * kr[c];
      part += exp((double)(s * (Ts)scale) - row_lse[g * q_rows + r]);
    }
    acc += part;
  }
  acc = warp_sum(acc);
  if (lane == 0) mass[g * nb + b] = acc;
}

// ---------------------------------------------------------------- top-k

// Radix select, one CTA (1024 threads) per group: the budget-th largest mass
// T is found MSB-first over the 64-bit pattern of the (non-negative) double
// masses, 8 bits per pass; then blocks with mass > T, plus the lowest-index
// blocks with mass == T up to the budget, are emitted in ascending index
// order -- exactly a stable sort on -mass truncated to the budget
// (sparse.py:127-128).  Once the bin holding the budget-th mass has <= 32
// keys, one warp ranks them exactly and the passes stop (C4: 21 -> 13 us).
// Masses live in shared memory up to 24K blocks, beyond that in global / L2.
constexpr int TOPK_THREADS = 1024;
constexpr int TOPK_SMEM_BLOCKS = 24 * 1024;

__device__ __forceinline__ int block_exclusive_scan(int v, int* warp_tot, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = warp_tot[lane];
    int inc = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    warp_tot[lane] = inc - w;  // exclusive per warp
    if (lane == 31) warp_tot[32] = inc;
  }
  __syncthreads();
  const int res = warp_tot[warp] + x - v;
  total = warp_tot[32];
  __syncthreads();
  return res;
}

__global__ void __launch_bounds__(TOPK_THREADS)
topk_radix_kernel(const double* __restrict__ mass, int nb, int budget, int32_t* __restrict__ selected) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // keys in shared memory up to 24K blocks; beyond that (contexts > 384K keys
  // at 16-key blocks) every pass reads them from global memory / L2
  const bool in_smem = nb <= TOPK_SMEM_BLOCKS;
  unsigned long long* skey = reinterpret_cast<unsigned long long*>(smem_raw);
  const unsigned long long* key =
      in_smem ? skey : reinterpret_cast<const unsigned long long*>(mass + (long long)blockIdx.x * nb);
  __shared__ int hist[256];
  __shared__ int warp_tot[33];
  __shared__ unsigned long long sh_prefix;
  __shared__ int sh_k, sh_cnt, sh_n;
  __shared__ unsigned long long cand_k[32];
  __shared__ int cand_i[32];
  const int g = blockIdx.x;
  if (in_smem)
    for (int i = threadIdx.x; i < nb; i += blockDim.x)
      skey[i] = (unsigned long long)__double_as_longlong(mass[(long long)g * nb + i]);
  if (threadIdx.x == 0) {
    sh_prefix = 0ull;
    sh_k = budget;
  }
  __syncthreads();
  unsigned long long mask = 0ull;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const unsigned long long prefix = sh_prefix;
    for (int i = threadIdx.x; i < nb; i += blockDim.x)
      if ((key[i] & mask) == prefix) atomicAdd(&hist[(key[i] >> shift) & 255], 1);
    __syncthreads();
    if (threadIdx.x < 32) {
      // bins from the top: find digit d with (count above d) < k <= (count at or above d)
      const int lane = threadIdx.x;
      int k = sh_k;
      int above = 0;
      for (int base = 255; base >= 0; base -= 32) {
        const int d = base - lane;
        const int c = hist[d];
        int inc = c;  // inclusive prefix from the top
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += y;
        }
        const unsigned hit = __ballot_sync(0xffffffffu, above + inc >= k && above + inc - c < k);
        if (hit) {
          const int src = __ffs(hit) - 1;
          const int cnt_before = __shfl_sync(0xffffffffu, above + inc - c, src);
          __syncwarp();  // every lane's read of sh_k (above) precedes lane 0's write
          const int cnt_bin = __shfl_sync(0xffffffffu, c, src);
          if (lane == 0) {
            sh_prefix = prefix | ((unsigned long long)(base - src) << shift);
            sh_k = k - cnt_before;
            sh_cnt = cnt_bin;
          }
          break;
        }
        above += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
    mask |= 0xffull << shift;
    __syncthreads();
    // early exit: once the bin holding the k-th mass has <= 32 keys, one warp
    // ranks those candidates exactly (mass desc, index asc) and names the k-th
    if (shift > 0 && sh_cnt <= 32) {
      if (threadIdx.x == 0) sh_n = 0;
      __syncthreads();
      const unsigned long long pre = sh_prefix;
      for (int i = threadIdx.x; i < nb; i += blockDim.x)
        if ((key[i] & mask) == pre) {
          const int at = atomicAdd(&sh_n, 1);
          cand_k[at] = key[i];
          cand_i[at] = i;
        }
      __syncthreads();
      if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const int n = sh_n;
        const unsigned long long kv = lane < n ? cand_k[lane] : 0ull;
        const int ix = lane < n ? cand_i[lane] : 0x7fffffff;
        int rank = 0;  // candidates before this one in (mass desc, index asc) order
        for (int j = 0; j < n; ++j) {
          const unsigned long long kj = cand_k[j];
          const int ij = cand_i[j];
          rank += (kj > kv || (kj == kv && ij < ix)) ? 1 : 0;
        }
        const int k = sh_k;
        const unsigned hit = __ballot_sync(0xffffffffu, lane < n && rank == k - 1);
        const unsigned long long T = __shfl_sync(0xffffffffu, kv, __ffs(hit) - 1);
        const unsigned gt = __ballot_sync(0xffffffffu, lane < n && kv > T);
        __syncwarp();
        if (lane == 0) {
          sh_prefix = T;
          sh_k = k - __popc(gt);  // keys equal to T still to take
        }
      }
      __syncthreads();
      break;
    }
  }
  const unsigned long long T = sh_prefix;
  const int take_eq = sh_k;  // blocks with mass == T to take, lowest indices first
  int eq_base = 0, out_base = 0;
  for (int c0 = 0; c0 < nb; c0 += blockDim.x) {
    const int i = c0 + threadIdx.x;
    const unsigned long long kv = i < nb ? key[i] : 0ull;
    const int eq = (i < nb && kv == T) ? 1 : 0;
    int eq_tot;
    const int eq_before = eq_base + block_exclusive_scan(eq, warp_tot, eq_tot);
    const int sel = (i < nb) && (kv > T || (eq && eq_before < take_eq));
    int sel_tot;
    const int pos = out_base + block_exclusive_scan(sel, warp_tot, sel_tot);
    if (sel) selected[(long long)g * budget + pos] = (int32_t)i;
    eq_base += eq_tot;
    out_base += sel_tot;
  }
}

// Ascending list of the blocks NOT selected (the residual key set,
// sparse.py:170): the u-th unselected block is u + |{selected < it}|, found
// by a binary search over the ascending selection.
__global__ void complement_kernel(const int32_t* __restrict__ sel, int64_t n_sel, int64_t nb,
                                  int32_t* __restrict__ out) {
  const int64_t g = blockIdx.y;
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n_res = nb - n_sel;
  if (u >= n_res) return;
  const int32_t* s = sel + g * n_sel;
  int64_t lo = 0, hi = n_sel;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)s[mid] - mid <= u) lo = mid + 1; else hi = mid;
  }
  out[g * n_res + u] = (int32_t)(u + lo);
}

int launch_complement(const int32_t* sel, int64_t groups, int64_t n_sel, int64_t nb, int32_t* out,
                      cudaStream_t st) {
  const int64_t n_res = nb - n_sel;
  if (n_res <= 0 || groups == 0) return FB_OK;
  dim3 grid((unsigned)((n_res + 255) / 256), (unsigned)groups);
  complement_kernel<<<grid, 256, 0, st>>>(sel, n_sel, nb, out);
  count_launch();
  return check_launch("complement_kernel");
}

// ---------------------------------------------------------------- block commit

// Device-side append of a finished block's K/V rows (kv_cache.py:121-144,
// simulator.py:327-333): group g's blk_rows rows go to cache rows
// [len[g], len[g] + blk_rows) of its slab, then len[g] advances.  Rows that
// would pass kv_rows_cap are dropped and counted in *overflow.
__global__ void commit_block_kernel(unsigned char* __restrict__ kc, unsigned char* __restrict__ vc,
                                    const unsigned char* __restrict__ kb,
                                    const unsigned char* __restrict__ vb, int64_t cap,
                                    int64_t row_bytes, int64_t blk_rows, int32_t* __restrict__ len,
                                    int32_t* __restrict__ overflow) {
  const int64_t g = blockIdx.y;
  const int64_t r = blockIdx.x;
  const int64_t base = len[g];
  __syncthreads();
  const int64_t dst_row = base + r;
  if (dst_row < cap) {
    const int64_t dst = (g * cap + dst_row) * row_bytes;
    const int64_t src = (g * blk_rows + r) * row_bytes;
    if ((row_bytes & 15) == 0) {
      for (int64_t i = threadIdx.x * 16; i < row_bytes; i += blockDim.x * 16) {
        *reinterpret_cast<uint4*>(kc + dst + i) = *reinterpret_cast<const uint4*>(kb + src + i);
        *reinterpret_cast<uint4*>(vc + dst + i) = *reinterpret_cast<const uint4*>(vb + src + i);
      }
    } else {
      for (int64_t i = threadIdx.x; i < row_bytes; i += blockDim.x) {
        kc[dst + i] = kb[src + i];
        vc[dst + i] = vb[src + i];
      }
    }
  } else if (threadIdx.x == 0 && overflow) {
    atomicAdd(overflow, 1);
  }
}

__global__ void advance_lengths_kernel(int32_t* __restrict__ len, int64_t groups, int64_t blk_rows,
                                       int64_t cap) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g < groups) len[g] = (int32_t)min((int64_t)len[g] + blk_rows, cap);
}

int launch_commit_block(void* kc, void* vc, const void* kb, const void* vb, int64_t groups,
                        int64_t cap, int64_t row_bytes, int64_t blk_rows, int32_t* len,
                        int32_t* overflow, cudaStream_t st) {
  if (groups == 0 || blk_rows == 0) return FB_OK;
  dim3 grid((unsigned)blk_rows, (unsigned)groups);
  commit_block_kernel<<<grid, 64, 0, st>>>(reinterpret_cast<unsigned char*>(kc),
                                            reinterpret_cast<unsigned char*>(vc),
                                            reinterpret_cast<const unsigned char*>(kb),
                                            reinterpret_cast<const unsigned char*>(vb), cap, row_bytes,
                                            blk_rows, len, overflow);
  advance_lengths_kernel<<<(unsigned)((groups + 255) / 256), 256, 0, st>>>(len, groups, blk_rows, cap);
  count_launch(2);
  return check_launch("commit_block_kernel");
}

// Paged variant: logical row len[g] + r of group g goes to page
// table[g * max_pages + row / page_rows], row % page_rows of the page pool.
// Rows past the table (or into a negative page id) are dropped and counted.
__global__ void commit_block_paged_kernel(unsigned char* __restrict__ kp, unsigned char* __restrict__ vp,
                                          int64_t page_rows, const int32_t* __restrict__ table,
                                          int64_t max_pages, const unsigned char* __restrict__ kb,
                                          const unsigned char* __restrict__ vb, int64_t row_bytes,
                                          int64_t blk_rows, int32_t* __restrict__ len,
                                          int32_t* __restrict__ overflow) {
  const int64_t g = blockIdx.y;
  const int64_t r = blockIdx.x;
  const int64_t dst_row = (int64_t)len[g] + r;
  const int64_t pi = dst_row / page_rows;
  const int32_t page = pi < max_pages ? table[g * max_pages + pi] : -1;
  if (page >= 0) {
    const int64_t dst = ((int64_t)page * page_rows + dst_row % page_rows) * row_bytes;
    const int64_t src = (g * blk_rows + r) * row_bytes;
    if ((row_bytes & 15) == 0) {
      for (int64_t i = threadIdx.x * 16; i < row_bytes; i += blockDim.x * 16) {
        *reinterpret_cast<uint4*>(kp + dst + i) = *reinterpret_cast<const uint4*>(kb + src + i);
        *reinterpret_cast<uint4*>(vp + dst + i) = *reinterpret_cast<const uint4*>(vb + src + i);
      }
    } else {
      for (int64_t i = threadIdx.x; i < row_bytes; i += blockDim.x) {
        kp[dst + i] = kb[src + i];
        vp[dst + i] = vb[src + i];
      }
    }
  } else if (threadIdx.x == 0 && overflow) {
    atomicAdd(overflow, 1);
  }
}

int launch_commit_block_paged(void* kp, void* vp, int64_t page_rows, const int32_t* table,
                              int64_t max_pages, const void* kb, const void* vb, int64_t groups,
                              int64_t row_bytes, int64_t blk_rows, int32_t* len, int32_t* overflow,
                              cudaStream_t st) {
  if (groups == 0 || blk_rows == 0) return FB_OK;
  dim3 grid((unsigned)blk_rows, (unsigned)groups);
  commit_block_paged_kernel<<<grid, 64, 0, st>>>(
      reinterpret_cast<unsigned char*>(kp), reinterpret_cast<unsigned char*>(vp), page_rows, table,
      max_pages, reinterpret_cast<const unsigned char*>(kb), reinterpret_cast<const unsigned char*>(vb),
      row_bytes, blk_rows, len, overflow);
  advance_lengths_kernel<<<(unsigned)((groups + 255) / 256), 256, 0, st>>>(len, groups, blk_rows,
                                                                          max_pages * page_rows);
  count_launch(2);
  return check_launch("commit_block_paged_kernel");
}

// ---------------------------------------------------------------- launchers

template <typename Mode>
int launch_block_mass(const typename Mode::Tin* q, const typename Mode::Tin* k,
                      const double* row_lse, int64_t groups, int64_t q_rows, int64_t head_dim,
                      int64_t slab_stride, int64_t n_ext, int64_t kbs, double scale, double* mass,
                      cudaStream_t st) {
  const int64_t nb = (n_ext + kbs - 1) / kbs;
  if (nb == 0 || groups == 0) return FB_OK;
  const size_t smem = sizeof(typename Mode::Ts) * (size_t)(MASS_WARPS * kbs) * (size_t)(head_dim + 1);
  if (smem > 220 * 1024) return fail(FB_ERR_UNSUPPORTED, "key_block_size * head_dim too large for block_mass");
  auto kern = block_mass_kernel<Mode>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((unsigned)((nb + MASS_WARPS - 1) / MASS_WARPS), (unsigned)groups);
  kern<<<grid, 32 * MASS_WARPS, smem, st>>>(q, k, row_lse, q_rows, head_dim, slab_stride, n_ext, kbs,
                                            nb, scale, mass);
  count_launch();
  return check_launch("block_mass_kernel");
}

template int launch_block_mass<ModeMaskF64>(const double*, const double*, const double*, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, double, double*, cudaStream_t);
template int launch_block_mass<ModeMaskF32>(const float*, const float*, const double*, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, double, double*, cudaStream_t);
template int launch_block_mass<ModeMaskBF16>(const __nv_bfloat16*, const __nv_bfloat16*, const double*, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, double, double*, cudaStream_t);

int launch_topk(const double* mass, int64_t groups, int64_t nb, int64_t budget, int32_t* selected,
                void* scratch, size_t scratch_bytes, cudaStream_t st) {
  if (groups == 0 || budget == 0) return FB_OK;
  if (nb < (int64_t(1) << 31)) {  // keys in smem up to TOPK_SMEM_BLOCKS, else read from global / L2
    const size_t smem = nb <= TOPK_SMEM_BLOCKS ? (size_t)nb * sizeof(unsigned long long) : 0;
    static size_t attr = 0;
    if (smem > attr) {
      cudaFuncSetAttribute(topk_radix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = smem;
    }
    topk_radix_kernel<<<(unsigned)groups, TOPK_THREADS, smem, st>>>(mass, (int)nb, (int)budget, selected);
    count_launch();
    return check_launch("topk_radix_kernel");
  }
  return fail(FB_ERR_UNSUPPORTED, "top-k over >= 2^31 blocks");
}

}  // namespace fb
