// Cross-step similarity of attention partials: the
// statistics behind head-gate calibration and the stability study.
//
//  * row_cosine_kernel      per-row cosine between two partial outputs of the
//                           same rows (consecutive denoising steps), with the
//                           reference's zero-norm rule (linalg.py:68-80), and
//                           its per-head mean over rows (policy.py:232-240).
//  * pairwise_cosine_kernel all-pairs cosine matrix between the rows of a
//                           later and an earlier step (analysis.py:28-51).
// Everything accumulates in float64 (the reference's statistics are float64
// means of cosines); reductions run in a fixed order, so results are
// bitwise reproducible.
#include "fb_kernels.cuh"

namespace fb {

constexpr double ZERO_NORM_EPS = 1e-12;  // linalg.py:25

template <typename T>
__device__ __forceinline__ double ld64(const T* p) { return cvt<double>(*p); }
template <>
__device__ __forceinline__ double ld64<double>(const double* p) { return *p; }

// grid: ceil(heads*rows / 8); block 256: one warp per row (all rows of all
// heads in parallel) -> row_cos[h*rows + r]
template <typename T>
__global__ void __launch_bounds__(256)
row_cosine_kernel(const T* __restrict__ a, T* b, int64_t n_rows, int64_t d,
                  double* __restrict__ row_cos, int update, int* __restrict__ nonzero) {
  const int lane = threadIdx.x & 31;
  bool any = false;
  // grid-stride over rows (the grid is capped at 8 blocks per SM, so the
  // nonzero flag is written at most once per block, not once per row: one
  // address written by every warp serialises in its L2 slice)
  for (int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); r < n_rows; r += (int64_t)gridDim.x * 8) {
    const T* u = a + r * d;
    T* v = b + r * d;
    double uu = 0.0, vv = 0.0, uv = 0.0;
    // 128 columns per pass with all 8 loads of a lane issued before the math
    // (same per-lane order c = lane, lane + 32, ... as a plain loop)
    for (int64_t c0 = 0; c0 < d; c0 += 128) {
      T xr[4], yr[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t c = c0 + lane + 32 * i;
        if (c < d) {
          xr[i] = u[c];
          yr[i] = v[c];
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (c0 + lane + 32 * i < d) {
          const double x = ld64(&xr[i]), y = ld64(&yr[i]);
          uu += x * x;
          vv += y * y;
          uv += x * y;
        }
      }
      // calibrator step (update): b becomes a for the next step's comparison,
      // read above before written by the same thread
      if (update) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (c0 + lane + 32 * i < d) v[c0 + lane + 32 * i] = xr[i];
      }
    }
    uu = warp_sum(uu);
    vv = warp_sum(vv);
    uv = warp_sum(uv);
    any |= uu != 0.0;
    const double nu = sqrt(uu), nv = sqrt(vv);
    if (lane == 0) row_cos[r] = (nu < ZERO_NORM_EPS || nv < ZERO_NORM_EPS) ? 0.0 : uv / (nu * nv);
  }
  if (nonzero != nullptr && __syncthreads_or(any) && threadIdx.x == 0) *nonzero = 1;
}

// grid: heads; block 256: head_mean[h] = mean of row_cos[h, :], summed in a
// fixed order (per-thread strided sums, then a fixed tree)
__global__ void __launch_bounds__(256)
head_mean_kernel(const double* __restrict__ row_cos, int64_t rows, double* __restrict__ head_mean) {
  __shared__ double part[256];
  const int64_t h = blockIdx.x;
  double s = 0.0;
#pragma unroll 8
  for (int64_t r = threadIdx.x; r < rows; r += 256) s += row_cos[h * rows + r];  // loads batched, adds in order
  part[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) head_mean[h] = rows > 0 ? part[0] / (double)rows : 0.0;
}

// grid: (ceil(n/16), ceil(n/16), heads); block 16x16; out[h, i, j] =
// cos(later_i, earlier_j); rows with norm < eps give 0 (analysis.py:41-50)
template <typename T>
__global__ void __launch_bounds__(256)
pairwise_cosine_kernel(const T* __restrict__ later, const T* __restrict__ earlier, int64_t n,
                       int64_t d, double* __restrict__ out) {
  constexpr int TL = 16, DC = 32;  // rows per tile, columns per chunk
  __shared__ double sa[TL][DC + 1], sb[TL][DC + 1];
  __shared__ double na[TL], nb[TL];
  const int64_t h = blockIdx.z;
  const int64_t i0 = (int64_t)blockIdx.y * TL, j0 = (int64_t)blockIdx.x * TL;
  const int ty = threadIdx.x / TL, tx = threadIdx.x % TL;
  double dot = 0.0, nsa = 0.0, nsb = 0.0;
  for (int64_t c0 = 0; c0 < d; c0 += DC) {
    __syncthreads();
    for (int e = threadIdx.x; e < TL * DC; e += 256) {
      const int rr = e / DC, cc = e % DC;
      const int64_t col = c0 + cc;
      const int64_t ia = i0 + rr, jb = j0 + rr;
      sa[rr][cc] = (ia < n && col < d) ? ld64(later + (h * n + ia) * d + col) : 0.0;
      sb[rr][cc] = (jb < n && col < d) ? ld64(earlier + (h * n + jb) * d + col) : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int cc = 0; cc < DC; ++cc) dot += sa[ty][cc] * sb[tx][cc];
    if (tx == 0) {
      for (int cc = 0; cc < DC; ++cc) nsa += sa[ty][cc] * sa[ty][cc];
    }
    if (ty == 0) {
      for (int cc = 0; cc < DC; ++cc) nsb += sb[tx][cc] * sb[tx][cc];
    }
  }
  if (tx == 0) na[ty] = sqrt(nsa);
  if (ty == 0) nb[tx] = sqrt(nsb);
  __syncthreads();
  const int64_t i = i0 + ty, j = j0 + tx;
  if (i < n && j < n) {
    const double den = na[ty] * nb[tx];
    double s = 0.0;
    if (na[ty] >= ZERO_NORM_EPS && nb[tx] >= ZERO_NORM_EPS && den >= ZERO_NORM_EPS * ZERO_NORM_EPS)
      s = dot / den;
    out[(h * n + i) * n + j] = s;
  }
}

template <typename T>
int launch_row_cosine(const void* a, const void* b, int64_t heads, int64_t rows, int64_t d,
                      double* row_cos, double* head_mean, cudaStream_t st, bool update, int* nonzero) {
  const int64_t n = heads * rows;
  if (n > 0) {
    row_cosine_kernel<T><<<(unsigned)std::min<int64_t>((n + 7) / 8, (int64_t)num_sms() * 8), 256, 0, st>>>(
        reinterpret_cast<const T*>(a), const_cast<T*>(reinterpret_cast<const T*>(b)), n, d, row_cos,
        update ? 1 : 0, nonzero);
    count_launch();
    if (int rc = check_launch("row_cosine_kernel")) return rc;
  }
  if (head_mean == nullptr) return FB_OK;
  head_mean_kernel<<<(unsigned)heads, 256, 0, st>>>(row_cos, rows, head_mean);
  count_launch();
  return check_launch("head_mean_kernel");
}

template <typename T>
int launch_pairwise_cosine(const void* later, const void* earlier, int64_t heads, int64_t n,
                           int64_t d, double* out, cudaStream_t st) {
  const unsigned t = (unsigned)((n + 15) / 16);
  pairwise_cosine_kernel<T><<<dim3(t, t, (unsigned)heads), 256, 0, st>>>(
      reinterpret_cast<const T*>(later), reinterpret_cast<const T*>(earlier), n, d, out);
  count_launch();
  return check_launch("pairwise_cosine_kernel");
}

template int launch_row_cosine<double>(const void*, const void*, int64_t, int64_t, int64_t, double*, double*, cudaStream_t,
                                       bool, int*);
template int launch_row_cosine<float>(const void*, const void*, int64_t, int64_t, int64_t, double*, double*, cudaStream_t,
                                       bool, int*);
template int launch_row_cosine<__nv_bfloat16>(const void*, const void*, int64_t, int64_t, int64_t, double*, double*, cudaStream_t,
                                       bool, int*);
template int launch_pairwise_cosine<double>(const void*, const void*, int64_t, int64_t, int64_t, double*, cudaStream_t);
template int launch_pairwise_cosine<float>(const void*, const void*, int64_t, int64_t, int64_t, double*, cudaStream_t);
template int launch_pairwise_cosine<__nv_bfloat16>(const void*, const void*, int64_t, int64_t, int64_t, double*, cudaStream_t);

}  // namespace fb
