// K2 -- cached step on sm_100a: block-internal attention fused with the
// log-space merge against the cached external partial.
//
// Reference: attention_with_reuse (attention.py:295-321) = attention_partial
// over the current block's keys (:320) + merge_partials with the cached
// external partial (:321, :207-245).  The KV cache is not an argument.
//
// One CTA per (group, 128-row query tile, output-column slice), 160 threads:
//   warps 0..3  softmax + merge epilogue, thread = query row = TMEM lane;
//               each thread loads its row of the cached O_ext slice and its
//               LSE_ext straight into registers at kernel start;
//   warp 4      TMA (Q, K_in, V_in, 128B swizzled) and the tcgen05.mma issue.
// S = Q K_in^T (N = NT <= 128 keys) lands in TMEM; P (bf16) overwrites S;
// O = P V_in (TS MMA) lands in TMEM; the epilogue normalises O, merges it
// with O_ext / LSE_ext in fp32 and writes bf16 (or fp32) output.  ~45 KB of
// shared memory, so the next launch's CTAs fit beside this one's (PDL).
// ext_early: the caller guarantees the external partial was not written by
// the kernel immediately preceding this launch in the stream (true for every
// cached step), so its loads are issued before griddepcontrol.wait and
// overlap the predecessor's tail.
#include "fb_kernels.cuh"
#include "fb_sm100_ptx.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

namespace fb {
namespace sm100k2 {

constexpr int BM = 128;
constexpr int THREADS = 160;  // warps 0-3 softmax/epilogue, warp 4 TMA + MMA
constexpr int BOX = 64;  // bf16 columns per 128-byte swizzle span

// The output columns of a query tile are split over SPLIT CTAs (each
// recomputes the cheap S = Q K^T and softmax, then does P V, the merge and
// the stores for its D/SPLIT columns): twice the CTAs, a third fewer bytes each.
template <int D, int NT, int SPLIT_ = 1>
struct Cfg {
  static constexpr int SPLIT = SPLIT_;
  static constexpr int DC = D / SPLIT;                  // output columns per CTA
  // O_ext columns prefetched into registers (fewer beside a 128-key score row)
#ifndef FB_K2_PRE_MAX
#define FB_K2_PRE_MAX 64  // diagnostics build knob (O_ext columns prefetched into registers)
#endif
  static constexpr int PRE = NT >= 128 ? 32 : (DC > FB_K2_PRE_MAX ? FB_K2_PRE_MAX : DC);
  static constexpr int NB = D / BOX;                    // 64-col boxes per bf16 row
  static constexpr int NBV = DC / BOX;                  // V boxes per CTA
  static constexpr uint32_t QBOX = BM * 128;            // 16 KB
  static constexpr uint32_t KBOX = NT * 128;            // NT rows x 128 B
  static constexpr uint32_t OFF_Q = 0;
  static constexpr uint32_t OFF_K = OFF_Q + NB * QBOX;
  static constexpr uint32_t OFF_V = OFF_K + NB * KBOX;
  static constexpr uint32_t OFF_BAR = OFF_V + NBV * KBOX;
  static constexpr uint32_t SMEM = OFF_BAR + 128 + 1024;
  static constexpr uint32_t COL_S = 0, COL_O = NT < 32 ? 32 : NT;  // P stores span >= 32 cols
  static constexpr uint32_t TMEM_COLS = (COL_O + DC) <= 128 ? 128 : (COL_O + DC) <= 256 ? 256 : 512;
  static constexpr uint32_t TX_QKV = NB * (QBOX + KBOX) + NBV * KBOX;
  static constexpr uint32_t TX_V = NBV * KBOX;
};

struct Bars {
  uint64_t load_qkv, s_full, p_ready, o_full, load_v;
  uint32_t tmem_base;
};

// Token-major layout (TOK): Q / K_in / V_in are strided views of a QKV
// projection output [b * B, ...] and the output is written token-major
// ([b * B, out_ts], head h of kv group kvh at columns (kvh * G + h) * D), so
// the attention layer needs no head-major copies around its GEMMs.
struct TokLayout {
  int B, G, Hkv;
  long long out_ts;  // output token stride (elements)
};

#ifndef FB_K2_MIN_BLOCKS
#define FB_K2_MIN_BLOCKS 2  // diagnostics build knob
#endif
// EXTB: the cached external partial's O is bf16 (fp32 LSE), half the bytes of
// the fp32 layout; the merge arithmetic stays fp32.
template <int D, int NT, int SPLIT, bool TRACE = false, bool TOK = false, bool EXTB = false>
__global__ void __launch_bounds__(THREADS, FB_K2_MIN_BLOCKS)  // (3 CTAs/SM at 136 regs: 8 % slower, C2 b=16)
internal_merge_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v, const void* __restrict__ o_ext_,
                      const float* __restrict__ lse_ext, int q_rows, int m_tiles, int n_in,
                      float scale_log2, void* __restrict__ out, int out_bf16,
                      float* __restrict__ lse_merged, float* __restrict__ o_int,
                      float* __restrict__ lse_int, int* __restrict__ empty_rows, int ext_early,
                      unsigned long long* __restrict__ trace, TokLayout tl) {
  using C = Cfg<D, NT, SPLIT>;
  // diagnostics (TRACE): per-CTA globaltimer stamps, 8 per CTA
  auto stamp = [&](int i) {
    if constexpr (TRACE) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      trace[blockIdx.x * 8 + i] = t;
    }
  };
  if (threadIdx.x == 128) stamp(0);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Bars* bar = reinterpret_cast<Bars*>(smem + C::OFF_BAR);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.x % C::SPLIT;  // output-column slice
  const int g = (blockIdx.x / C::SPLIT) / m_tiles;
  const int mt = (blockIdx.x / C::SPLIT) % m_tiles;
  const int col0 = h * C::DC;
  const int row = (warp & 3) * 32 + lane;
  const int grow = mt * BM + row;
  const bool live_row = warp < 4 && grow < q_rows;
  const long long rr = (long long)g * q_rows + grow;
  // output row offset (elements): stacked [groups, q_rows, D] or token-major
  long long orr = rr * D;
  if constexpr (TOK) {
    const int bi = g / tl.Hkv, kvh = g % tl.Hkv, hh = grow / tl.B, tt = grow % tl.B;
    orr = (long long)(bi * tl.B + tt) * tl.out_ts + (long long)(kvh * tl.G + hh) * D;
  }

  // this thread's row of the cached external partial (its column slice)
  float le = -INFINITY;
  const float* o_ext = reinterpret_cast<const float*>(o_ext_);
  const __nv_bfloat16* o_extb = reinterpret_cast<const __nv_bfloat16*>(o_ext_);
  float oe[EXTB ? 1 : C::PRE];
  uint32_t ob[EXTB ? C::PRE / 2 : 1];  // bf16x2 words
  auto load_ext = [&]() {
    if constexpr (EXTB) {
      if (live_row) {
        le = __ldg(lse_ext + rr);
        const __nv_bfloat16* srow = o_extb + rr * D + col0;
        if ((reinterpret_cast<uintptr_t>(srow) & 31) == 0 && C::PRE % 16 == 0) {  // 256-bit loads
#pragma unroll
          for (int j = 0; j < C::PRE / 16; ++j) ptx::ld_v8_nc_b32(srow + 16 * j, ob + 8 * j);
        } else {
          const uint4* src = reinterpret_cast<const uint4*>(srow);
#pragma unroll
          for (int j = 0; j < C::PRE / 8; ++j) {
            const uint4 v4 = __ldg(src + j);
            ob[4 * j] = v4.x; ob[4 * j + 1] = v4.y; ob[4 * j + 2] = v4.z; ob[4 * j + 3] = v4.w;
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < C::PRE / 2; ++i) ob[i] = 0u;
      }
      return;
    }
    if (live_row) {
      le = __ldg(lse_ext + rr);
      const float* srow = o_ext + rr * D + col0;
      if ((reinterpret_cast<uintptr_t>(srow) & 31) == 0 && C::PRE % 8 == 0) {  // 256-bit loads
#pragma unroll
        for (int j = 0; j < C::PRE / 8; ++j) ptx::ld_v8_nc(srow + 8 * j, oe + 8 * j);
      } else {
        const float4* src = reinterpret_cast<const float4*>(srow);
#pragma unroll
        for (int j = 0; j < C::PRE / 4; ++j) {
          const float4 v4 = __ldg(src + j);
          oe[4 * j] = v4.x; oe[4 * j + 1] = v4.y; oe[4 * j + 2] = v4.z; oe[4 * j + 3] = v4.w;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < C::PRE; ++i) oe[i] = 0.f;
    }
  };
  const bool pdl_late = (ext_early & 2) != 0;  // see internal_merge_v2_kernel
  const bool vsplit = (ext_early & 4) != 0;    // V_in on its own barrier (as v2)
  ext_early &= 1;
  if (ext_early) load_ext();

  if (threadIdx.x == 128) {
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
    ptx::mbar_init(&bar->load_qkv, 1);
    ptx::mbar_init(&bar->s_full, 1);
    ptx::mbar_init(&bar->p_ready, 128);
    ptx::mbar_init(&bar->o_full, 1);
    ptx::mbar_init(&bar->load_v, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 4) ptx::tmem_alloc(&bar->tmem_base, C::TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = bar->tmem_base;
  if (threadIdx.x == 128) stamp(1);
  ptx::pdl_wait();               // inputs of this launch are final from here on
  if (!pdl_late) ptx::pdl_launch_dependents();
  if (threadIdx.x == 128) stamp(2);

  if (warp == 4) {
    if (lane == 0) {
      const uint64_t pol = ptx::policy_evict_first();
      // (TOK: the Q box holds G * B rows, not BM, so fewer bytes land)
      uint64_t* bar_v = vsplit ? &bar->load_v : &bar->load_qkv;
      ptx::mbar_expect_tx(&bar->load_qkv, (TOK ? C::TX_QKV - C::NB * (uint32_t)(BM - tl.B * tl.G) * 128u
                                               : C::TX_QKV) - (vsplit ? C::TX_V : 0u));
      if (vsplit) ptx::mbar_expect_tx(bar_v, C::TX_V);
      if constexpr (TOK) {  // 5-D Q {d, B, G, Hkv, b}, 4-D K / V {d, B, Hkv, b}
        const int bi = g / tl.Hkv, kvh = g % tl.Hkv;
        for (int b = 0; b < C::NB; ++b) {
          ptx::tma_load_5d(smem + C::OFF_Q + b * C::QBOX, &tm_q, &bar->load_qkv, b * BOX, 0, 0, kvh, bi, pol);
          ptx::tma_load_4d(smem + C::OFF_K + b * C::KBOX, &tm_k, &bar->load_qkv, b * BOX, 0, kvh, bi, pol);
        }
        for (int b = 0; b < C::NBV; ++b)
          ptx::tma_load_4d(smem + C::OFF_V + b * C::KBOX, &tm_v, bar_v, col0 + b * BOX, 0, kvh, bi, pol);
      } else {
        for (int b = 0; b < C::NB; ++b) {
          ptx::tma_load_3d(smem + C::OFF_Q + b * C::QBOX, &tm_q, &bar->load_qkv, b * BOX, mt * BM, g, pol);
          ptx::tma_load_3d(smem + C::OFF_K + b * C::KBOX, &tm_k, &bar->load_qkv, b * BOX, 0, g, pol);
        }
        for (int b = 0; b < C::NBV; ++b)
          ptx::tma_load_3d(smem + C::OFF_V + b * C::KBOX, &tm_v, bar_v, col0 + b * BOX, 0, g, pol);
      }

      constexpr uint32_t IDESC_S = ptx::idesc_bf16_f32(BM, NT, false);
      constexpr uint32_t IDESC_O = ptx::idesc_bf16_f32(BM, C::DC, true);
      ptx::mbar_wait(&bar->load_qkv, 0);
      if (pdl_late) ptx::pdl_launch_dependents();
      stamp(3);
      ptx::tc_fence_after();
      const uint32_t q_base = ptx::smem_u32(smem + C::OFF_Q);
      const uint32_t k_base = ptx::smem_u32(smem + C::OFF_K);
      const uint32_t v_base = ptx::smem_u32(smem + C::OFF_V);
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        ptx::mma_ss(tmem + C::COL_S,
                    ptx::sdesc_sw128(q_base + (kk / 4) * C::QBOX + (kk % 4) * 32, 16, 1024),
                    ptx::sdesc_sw128(k_base + (kk / 4) * C::KBOX + (kk % 4) * 32, 16, 1024),
                    IDESC_S, kk > 0);
      }
      ptx::tc_commit(&bar->s_full);
      if (vsplit) ptx::mbar_wait(&bar->load_v, 0);
      ptx::mbar_wait(&bar->p_ready, 0);
      ptx::tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < NT / 16; ++kk) {
        ptx::mma_ts(tmem + C::COL_O, tmem + C::COL_S + kk * 8,
                    ptx::sdesc_sw128(v_base + kk * 2048, C::KBOX, 1024), IDESC_O, kk > 0);
      }
      ptx::tc_commit(&bar->o_full);
    }
  } else if (warp < 4) {
    // ------------------------------------------------ softmax + merge epilogue
    if (!ext_early) load_ext();
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    uint32_t r[32];
    float s[NT];
    ptx::mbar_wait(&bar->s_full, 0);
    if (threadIdx.x == 0) stamp(4);
    ptx::tc_fence_after();
#pragma unroll
    for (int c = 0; c < NT / 32 + (NT % 32 ? 1 : 0); ++c) {
      if constexpr (NT >= 32) {
        ptx::tmem_ld32(tmem + lane_off + C::COL_S + c * 32, r);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(r[i]);
      } else {
        ptx::tmem_ld32(tmem + lane_off + C::COL_S, r);  // 16 valid columns, rest unused TMEM
        ptx::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < NT; ++i) s[i] = __uint_as_float(r[i]);
      }
    }
    float mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < NT; ++i) {
      if (i >= n_in) s[i] = -INFINITY;
      mx = fmaxf(mx, s[i]);
    }
    const float m2 = mx * scale_log2;  // -inf when n_in == 0
    const float neg = (n_in > 0) ? -m2 : 0.f;
    float l = 0.f;
#pragma unroll
    for (int c = 0; c < (NT + 63) / 64; ++c) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int j = c * 64 + 2 * i;
        float p0 = 0.f, p1 = 0.f;
        if (j < NT) {
          p0 = ptx::ex2(fmaf(s[j], scale_log2, neg));
          p1 = ptx::ex2(fmaf(s[j + 1], scale_log2, neg));
        }
        l += p0 + p1;
        r[i] = ptx::pack_bf16(p0, p1);
      }
      ptx::tmem_st32(tmem + lane_off + C::COL_S + c * 32, r);
    }
    ptx::tmem_wait_st();
    ptx::tc_fence_before();
    ptx::mbar_arrive(&bar->p_ready);
    if (threadIdx.x == 0) stamp(5);

    // internal partial statistics (natural log), rounded as stored (fp32)
    const bool has_int = n_in > 0;
    const float li = has_int ? (m2 + log2f(l)) * 0.69314718055994530942f : -INFINITY;
    const float inv = has_int ? 1.f / l : 0.f;
    const float mm = fmaxf(le, li);
    const bool live = mm != -INFINITY;
    const float we = live ? __expf(le - mm) : 0.f;
    const float wi = live ? __expf(li - mm) : 0.f;
    const float z = we + wi;
    const float iz = live ? 1.f / z : 0.f;

    ptx::mbar_wait(&bar->o_full, 0);
    if (threadIdx.x == 0) stamp(6);
    ptx::tc_fence_after();
#pragma unroll
    for (int c = 0; c < C::DC / 32; ++c) {
      ptx::tmem_ld32(tmem + lane_off + C::COL_O + c * 32, r);
      float oc[32];
      if constexpr (EXTB) {
        if (c * 32 < C::PRE) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const uint32_t u = ob[((c * 32) % C::PRE) / 2 + i];
            oc[2 * i] = ptx::bf16_lo(u);
            oc[2 * i + 1] = ptx::bf16_hi(u);
          }
        } else if (live_row) {  // columns past the prefetched ones
          const uint4* src = reinterpret_cast<const uint4*>(o_extb + rr * D + col0 + c * 32);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint4 v4 = __ldg(src + j);
            const uint32_t w[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              oc[8 * j + 2 * k] = ptx::bf16_lo(w[k]);
              oc[8 * j + 2 * k + 1] = ptx::bf16_hi(w[k]);
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) oc[i] = 0.f;
        }
      } else if (c * 32 < C::PRE) {
#pragma unroll
        for (int i = 0; i < 32; ++i) oc[i] = oe[(c * 32 + i) % C::PRE];
      } else if (live_row) {  // columns past the prefetched ones (unsplit D = 128)
        const float4* src = reinterpret_cast<const float4*>(o_ext + rr * D + col0 + c * 32);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 v4 = __ldg(src + j);
          oc[4 * j] = v4.x; oc[4 * j + 1] = v4.y; oc[4 * j + 2] = v4.z; oc[4 * j + 3] = v4.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) oc[i] = 0.f;
      }
      ptx::tmem_wait_ld();
      float val[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float oi = __uint_as_float(r[i]) * inv;
        val[i] = live ? (__fmul_rn(we, oc[i]) + __fmul_rn(wi, oi)) * iz : 0.f;
        r[i] = __float_as_uint(oi);
      }
      if (live_row) {
        if (out_bf16) {
          __nv_bfloat16* drow = reinterpret_cast<__nv_bfloat16*>(out) + orr + col0 + c * 32;
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) pk[j] = ptx::pack_bf16(val[2 * j], val[2 * j + 1]);
          if ((reinterpret_cast<uintptr_t>(drow) & 31) == 0) {  // 256-bit stores
            ptx::st_v8_b32(drow, pk[0], pk[1], pk[2], pk[3], pk[4], pk[5], pk[6], pk[7]);
            ptx::st_v8_b32(drow + 16, pk[8], pk[9], pk[10], pk[11], pk[12], pk[13], pk[14], pk[15]);
          } else {
            uint4* dst = reinterpret_cast<uint4*>(drow);
#pragma unroll
            for (int j = 0; j < 4; ++j) dst[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
          }
        } else {
          ptx::st_row32(reinterpret_cast<float*>(out) + orr + col0 + c * 32, val);
        }
        if (o_int) {
          float4* di = reinterpret_cast<float4*>(o_int + rr * D + col0 + c * 32);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            di[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
        }
      }
    }
    if (threadIdx.x == 0) stamp(7);
    if (live_row && h == 0) {
      if (lse_int) lse_int[rr] = li;
      if (lse_merged) lse_merged[rr] = live ? mm + logf(z) : -INFINITY;
      if (!live && empty_rows) atomicAdd(empty_rows, 1);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, C::TMEM_COLS);
  }
}


// ---------------------------------------------------------------- K2 v2
// d = 128: one CTA per (group, 128-row query tile) with the cached external
// partial prefetched into shared memory by TMA (fp32, 128B-swizzled boxes of
// 32 columns: the epilogue's row-per-thread reads are bank-conflict free)
// instead of registers.  On cached steps (ext_early) that 64 KB load is issued
// before griddepcontrol.wait, and at ~115 KB of shared memory two CTAs fit per
// SM, so at C2 (128 CTAs) the next layer's whole grid is resident and
// prefetching while this one computes.  288 threads: warps 0-3 and 4-7 run the
// merge epilogue on output columns 0-63 / 64-127 of the same rows (TMEM lane
// quarter = warp % 4); warps 0-3 also run the softmax; warp 8 allocates TMEM,
// issues the TMA loads and the two MMAs.  Loads land on up to three
// barriers (Q / K columns 0-63, columns 64-127, V_in), so S = Q K^T starts on
// the first half while the rest is in flight; when the grid exceeds the SMs
// the bf16 output goes out as one bulk tensor store per (CTA, column half)
// from the Q tile, which is dead once o_full has fired.
constexpr int V2_THREADS = 288;

template <int NT, bool EXTB = false>
struct CfgV2 {
  static constexpr int D = 128;
  static constexpr uint32_t QBOX = BM * 128;   // 16 KB (128 rows x 64 bf16)
  static constexpr uint32_t KBOX = NT * 128;   // NT rows x 64 bf16
  static constexpr uint32_t EBOX = BM * 128;   // 16 KB (128 rows x 32 fp32, or x 64 bf16)
  static constexpr int NE = EXTB ? 2 : 4;      // O_ext boxes per 128-column row
  static constexpr int ECOLS = EXTB ? 64 : 32; // O_ext columns per box
  // barriers sit below the 1024-aligned tile area (dynamic shared memory
  // starts 1024-aligned after the 1 KB system reservation, so the tiles begin
  // at base + 1024); two CTAs per SM need SMEM <= 115,712 B
  static constexpr uint32_t OFF_Q = 0;  // offsets from the aligned tile base
  static constexpr uint32_t OFF_K = OFF_Q + 2 * QBOX;
  static constexpr uint32_t OFF_V = OFF_K + 2 * KBOX;
  static constexpr uint32_t OFF_E = (OFF_V + 2 * KBOX + 1023) / 1024 * 1024;
  static constexpr uint32_t OFF_X = OFF_K;  // [2][128] floats of WG0, over K (dead after S = Q K^T)
  static constexpr uint32_t TILES = OFF_E + NE * EBOX;
  static constexpr uint32_t SMEM = 1024 + TILES;
  static constexpr uint32_t COL_S = 0, COL_O = NT < 32 ? 32 : NT;
  static constexpr uint32_t TMEM_COLS = (COL_O + D) <= 256 ? 256 : 512;
  static constexpr uint32_t TX_QKV = 2 * (QBOX + 2 * KBOX);
  static constexpr uint32_t TX_QK = 2 * (QBOX + KBOX), TX_V = 2 * KBOX, TX_H = QBOX + KBOX;
  static constexpr uint32_t TX_E = NE * EBOX;
};

struct BarsV2 {
  uint64_t load_qkv, load_e, s_full, p_ready, o_full, load_v, load_h1;
  uint32_t tmem_base;
};

template <int NT, bool EXTB = false>
__global__ void __launch_bounds__(V2_THREADS, 2)
internal_merge_v2_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_e,
                         const __grid_constant__ CUtensorMap tm_o,
                         const float* __restrict__ lse_ext, int q_rows, int m_tiles, int n_in,
                         float scale_log2, void* __restrict__ out, int out_bf16,
                         float* __restrict__ lse_merged, float* __restrict__ o_int,
                         float* __restrict__ lse_int, int* __restrict__ empty_rows, int ext_early,
                         int tma_out) {
  using C = CfgV2<NT, EXTB>;
  constexpr int D = C::D;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  BarsV2* bar = reinterpret_cast<BarsV2*>(smem_raw);
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + sizeof(BarsV2) + 1023) & ~uintptr_t(1023));
  if (smem + C::TILES > smem_raw + C::SMEM) __trap();  // base not 1024-aligned: layout bug
  float* xch = reinterpret_cast<float*>(smem + C::OFF_X);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x / m_tiles;
  const int mt = blockIdx.x % m_tiles;
  const int wq = warp & 3, wg = warp >> 2;  // epilogue: lane quarter, column half
  const int row = wq * 32 + lane;
  const int grow = mt * BM + row;
  const bool live_row = warp < 8 && grow < q_rows;
  const long long rr = (long long)g * q_rows + grow;

  // ext_early bit 1 (pdl_late): signal the dependent launch only once this
  // CTA's Q / K / V have landed, so the next launch's O_ext prefetch does not
  // compete with this launch's post-wait loads
  const bool pdl_late = (ext_early & 2) != 0;
  // bit 2: V_in on its own barrier, so S = Q K^T starts once Q and K landed;
  // bit 3 as well: the two 64-column halves of Q and K on their own barriers,
  // so the first half of S = Q K^T starts once Q / K columns 0-63 landed
  const bool vsplit = (ext_early & 4) != 0;
  const bool hsplit = vsplit && (ext_early & 8) != 0;
  ext_early &= 1;
  float le = -INFINITY;
  if (ext_early && live_row) le = __ldg(lse_ext + rr);
  if (threadIdx.x == 256) {
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
    ptx::tma_prefetch_desc(&tm_e);
    ptx::mbar_init(&bar->load_qkv, 1);
    ptx::mbar_init(&bar->load_e, 1);
    ptx::mbar_init(&bar->s_full, 1);
    ptx::mbar_init(&bar->p_ready, 128);
    ptx::mbar_init(&bar->o_full, 1);
    ptx::mbar_init(&bar->load_v, 1);
    ptx::mbar_init(&bar->load_h1, 1);
    ptx::fence_barrier_init();
    if (ext_early) {  // the cached partial is final before this launch: fetch it now
      const uint64_t pol = ptx::policy_evict_first();
      ptx::mbar_expect_tx(&bar->load_e, C::TX_E);
      for (int b = 0; b < C::NE; ++b)
        ptx::tma_load_3d(smem + C::OFF_E + b * C::EBOX, &tm_e, &bar->load_e, b * C::ECOLS, mt * BM, g, pol);
    }
  }
  if (warp == 8) ptx::tmem_alloc(&bar->tmem_base, C::TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = bar->tmem_base;
  ptx::pdl_wait();
  if (!pdl_late) ptx::pdl_launch_dependents();

  if (warp == 8) {
    if (lane == 0) {
      const uint64_t pol = ptx::policy_evict_first();
      if (!ext_early) {
        ptx::mbar_expect_tx(&bar->load_e, C::TX_E);
        for (int b = 0; b < C::NE; ++b)
          ptx::tma_load_3d(smem + C::OFF_E + b * C::EBOX, &tm_e, &bar->load_e, b * C::ECOLS, mt * BM, g, pol);
      }
      uint64_t* bar_v = vsplit ? &bar->load_v : &bar->load_qkv;
      uint64_t* bar_h1 = hsplit ? &bar->load_h1 : &bar->load_qkv;
      ptx::mbar_expect_tx(&bar->load_qkv, hsplit ? C::TX_H : vsplit ? C::TX_QK : C::TX_QKV);
      if (hsplit) ptx::mbar_expect_tx(bar_h1, C::TX_H);
      if (vsplit) ptx::mbar_expect_tx(bar_v, C::TX_V);
      for (int b = 0; b < 2; ++b) {
        uint64_t* bh = b == 0 ? &bar->load_qkv : bar_h1;
        ptx::tma_load_3d(smem + C::OFF_Q + b * C::QBOX, &tm_q, bh, b * BOX, mt * BM, g, pol);
        ptx::tma_load_3d(smem + C::OFF_K + b * C::KBOX, &tm_k, bh, b * BOX, 0, g, pol);
      }
      for (int b = 0; b < 2; ++b)
        ptx::tma_load_3d(smem + C::OFF_V + b * C::KBOX, &tm_v, bar_v, b * BOX, 0, g, pol);
      constexpr uint32_t IDESC_S = ptx::idesc_bf16_f32(BM, NT, false);
      constexpr uint32_t IDESC_O = ptx::idesc_bf16_f32(BM, D, true);
      ptx::mbar_wait(&bar->load_qkv, 0);
      if (pdl_late) ptx::pdl_launch_dependents();
      ptx::tc_fence_after();
      const uint32_t q_base = ptx::smem_u32(smem + C::OFF_Q);
      const uint32_t k_base = ptx::smem_u32(smem + C::OFF_K);
      const uint32_t v_base = ptx::smem_u32(smem + C::OFF_V);
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        if (kk == 4 && hsplit) {
          ptx::mbar_wait(&bar->load_h1, 0);
          ptx::tc_fence_after();
        }
        ptx::mma_ss(tmem + C::COL_S,
                    ptx::sdesc_sw128(q_base + (kk / 4) * C::QBOX + (kk % 4) * 32, 16, 1024),
                    ptx::sdesc_sw128(k_base + (kk / 4) * C::KBOX + (kk % 4) * 32, 16, 1024),
                    IDESC_S, kk > 0);
      }
      ptx::tc_commit(&bar->s_full);
      if (vsplit) ptx::mbar_wait(&bar->load_v, 0);
      ptx::mbar_wait(&bar->p_ready, 0);
      ptx::tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < NT / 16; ++kk)
        ptx::mma_ts(tmem + C::COL_O, tmem + C::COL_S + kk * 8,
                    ptx::sdesc_sw128(v_base + kk * 2048, C::KBOX, 1024), IDESC_O, kk > 0);
      ptx::tc_commit(&bar->o_full);
    }
  } else {
    if (!ext_early && live_row) le = __ldg(lse_ext + rr);
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    uint32_t r[32];
    if (wg == 0) {
      // ------------------------------------------------ softmax (WG0)
      float s[NT];
      ptx::mbar_wait(&bar->s_full, 0);
      ptx::tc_fence_after();
#pragma unroll
      for (int c = 0; c < NT / 32 + (NT % 32 ? 1 : 0); ++c) {
        ptx::tmem_ld32(tmem + lane_off + C::COL_S + c * 32, r);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (c * 32 + i < NT) s[c * 32 + i] = __uint_as_float(r[i]);
      }
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < NT; ++i) {
        if (i >= n_in) s[i] = -INFINITY;
        mx = fmaxf(mx, s[i]);
      }
      const float m2 = mx * scale_log2;
      const float neg = (n_in > 0) ? -m2 : 0.f;
      float l = 0.f;
#pragma unroll
      for (int c = 0; c < (NT + 63) / 64; ++c) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int j = c * 64 + 2 * i;
          float p0 = 0.f, p1 = 0.f;
          if (j < NT) {
            p0 = ptx::ex2(fmaf(s[j], scale_log2, neg));
            p1 = ptx::ex2(fmaf(s[j + 1], scale_log2, neg));
          }
          l += p0 + p1;
          r[i] = ptx::pack_bf16(p0, p1);
        }
        ptx::tmem_st32(tmem + lane_off + C::COL_S + c * 32, r);
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&bar->p_ready);
      xch[row] = m2;
      xch[BM + row] = l;
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    const float m2 = xch[row], l = xch[BM + row];
    const bool has_int = n_in > 0;
    const float li = has_int ? (m2 + log2f(l)) * 0.69314718055994530942f : -INFINITY;
    const float inv = has_int ? 1.f / l : 0.f;
    const float mm = fmaxf(le, li);
    const bool live = mm != -INFINITY;
    const float we = live ? __expf(le - mm) : 0.f;
    const float wi = live ? __expf(li - mm) : 0.f;
    const float z = we + wi;
    const float iz = live ? 1.f / z : 0.f;
    ptx::mbar_wait(&bar->load_e, 0);
    ptx::mbar_wait(&bar->o_full, 0);
    ptx::tc_fence_after();
    const unsigned char* erow = smem + C::OFF_E + row * 128;
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      const int c = wg * 2 + cc;  // 32-column chunk = fp32 box c
      ptx::tmem_ld32(tmem + lane_off + C::COL_O + c * 32, r);
      float oc[32];
      if constexpr (EXTB) {  // box c / 2, 16-byte chunks (c % 2) * 4 + j (8 bf16 each)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint4 v4 = *reinterpret_cast<const uint4*>(erow + (c >> 1) * C::EBOX +
                                                           ((((c & 1) * 4 + j) ^ (row & 7)) << 4));
          const uint32_t w[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            oc[8 * j + 2 * k] = ptx::bf16_lo(w[k]);
            oc[8 * j + 2 * k + 1] = ptx::bf16_hi(w[k]);
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 v4 = *reinterpret_cast<const float4*>(erow + c * C::EBOX + ((j ^ (row & 7)) << 4));
          oc[4 * j] = v4.x; oc[4 * j + 1] = v4.y; oc[4 * j + 2] = v4.z; oc[4 * j + 3] = v4.w;
        }
      }
      ptx::tmem_wait_ld();
      float val[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float oi = __uint_as_float(r[i]) * inv;
        val[i] = live ? (__fmul_rn(we, oc[i]) + __fmul_rn(wi, oi)) * iz : 0.f;
        r[i] = __float_as_uint(oi);
      }
      if (tma_out) {
        // bf16 row -> the dead Q tile (box wg, 128B-swizzled like the TMA
        // load that filled it; MMA 1 finished reading it before o_full), one
        // bulk tensor store per warpgroup below; rows past q_rows are clipped
        unsigned char* orow = smem + C::OFF_Q + wg * C::QBOX + row * 128;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          *reinterpret_cast<uint4*>(orow + (((cc * 4 + j) ^ (row & 7)) << 4)) =
              make_uint4(ptx::pack_bf16(val[8 * j], val[8 * j + 1]), ptx::pack_bf16(val[8 * j + 2], val[8 * j + 3]),
                         ptx::pack_bf16(val[8 * j + 4], val[8 * j + 5]), ptx::pack_bf16(val[8 * j + 6], val[8 * j + 7]));
      } else if (live_row) {
        if (out_bf16) {
          __nv_bfloat16* drow = reinterpret_cast<__nv_bfloat16*>(out) + rr * D + c * 32;
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) pk[j] = ptx::pack_bf16(val[2 * j], val[2 * j + 1]);
          if ((reinterpret_cast<uintptr_t>(drow) & 31) == 0) {  // 256-bit stores
            ptx::st_v8_b32(drow, pk[0], pk[1], pk[2], pk[3], pk[4], pk[5], pk[6], pk[7]);
            ptx::st_v8_b32(drow + 16, pk[8], pk[9], pk[10], pk[11], pk[12], pk[13], pk[14], pk[15]);
          } else {
            uint4* dst = reinterpret_cast<uint4*>(drow);
#pragma unroll
            for (int j = 0; j < 4; ++j) dst[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
          }
        } else {
          ptx::st_row32(reinterpret_cast<float*>(out) + rr * D + c * 32, val);
        }
      }
      if (live_row && o_int) {
        float4* di = reinterpret_cast<float4*>(o_int + rr * D + c * 32);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          di[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                              __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
      }
    }
    if (tma_out) {
      ptx::fence_proxy_async_smem();
      asm volatile("bar.sync %0, 128;" ::"r"(3 + wg) : "memory");
      if (row == 0) {
        ptx::tma_store_3d(&tm_o, smem + C::OFF_Q + wg * C::QBOX, wg * 64, mt * BM, g);
        ptx::bulk_commit();
        ptx::bulk_wait_read();  // the tile must outlive the CTA's shared memory
      }
    }
    if (live_row && wg == 0) {
      if (lse_int) lse_int[rr] = li;
      if (lse_merged) lse_merged[rr] = live ? mm + logf(z) : -INFINITY;
      if (!live && empty_rows) atomicAdd(empty_rows, 1);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, C::TMEM_COLS);
  }
}
}  // namespace sm100k2

// host: tensor maps shared with the refresh kernel's encoder
int make_tmap_3d(CUtensorMap* map, const void* base, int dtype_bytes, int64_t inner, int64_t dim1,
                 int64_t dim1_stride_elems, int64_t dim2, int box_inner, int box_rows);

static int g_k2_v2_override = -1;
void set_k2_v2(int v) { g_k2_v2_override = v; }
// v2 output stores: -1 (default) / 1 one bulk tensor store per (CTA, column
// half) from shared memory, 0 row-per-thread 256-bit global stores.  C2 b=32
// cached step 8.62 -> 8.42 us, b=64 16.36 -> 16.21 (scripts/ab_k2_store.py)
static int g_k2_store = -1;
void set_k2_store(int v) { g_k2_store = v; }
// v2 V_in on its own load barrier (S = Q K^T issued once Q and K landed):
// -1 (default) / 1 on, 2 also the Q / K column halves, 0 one barrier for Q, K and V
static int g_k2_vsplit = -1;
void set_k2_vsplit(int v) { g_k2_vsplit = v; }
// the defaults above can be overridden from the environment (A/B inside whole
// programs such as bench.py): FB_K2_STORE=0/1, FB_K2_VSPLIT=0/1
static int k2_env(const char* name, int v) {
  if (v != -1) return v;
  const char* e = getenv(name);
  return (e != nullptr && e[0] >= '0' && e[0] <= '2') ? e[0] - '0' : -1;
}
// vsplit level 2 (FB_K2_VSPLIT=2): also the Q / K column halves on their own
// barriers.  Default (-1): level 2 when the grid exceeds the SMs (two CTAs per
// SM: b=32 8.24 -> 8.08 us), else level 1 (b=4 3.73 -> 3.68 us)
static int k2_vsplit_bits(int64_t ctas = 0) {
  int v = k2_env("FB_K2_VSPLIT", g_k2_vsplit);
  if (v == -1) v = ctas > num_sms() ? 2 : 1;
  return v == 0 ? 0 : v == 2 ? 4 | 8 : 4;
}
// diagnostics: FB_K2_PDL_LATE=1 signals the dependent launch after the Q/K/V loads landed
static int k2_pdl_late() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FB_K2_PDL_LATE");
    v = (e != nullptr && e[0] == '1') ? 1 : 0;
  }
  return v;
}

bool sm100_k2_supported(int64_t head_dim, int64_t n_in) {
  // n_in == 0 (no current-block keys) takes the SIMT path: there is nothing to load
  return (head_dim == 128 || head_dim == 64) && n_in >= 1 && n_in <= 128;
}

static unsigned long long* g_k2_trace = nullptr;  // diagnostics: fb_debug_set_k2_trace
static int g_k2_trace_n = 0, g_k2_trace_i = 0;
void set_k2_trace(void* p, int launches) {
  g_k2_trace = reinterpret_cast<unsigned long long*>(p);
  g_k2_trace_n = launches;
  g_k2_trace_i = 0;
}

template <int D, int NT, int SPLIT>
static int launch_k2(const __nv_bfloat16* q, const __nv_bfloat16* k_in, const __nv_bfloat16* v_in,
                     int64_t groups, int64_t q_rows, int64_t n_in, double scale, const void* o_ext,
                     const float* lse_ext, void* out, bool out_bf16, float* lse_merged, float* o_int,
                     float* lse_int, int32_t* empty, bool ext_early, bool extb, cudaStream_t st) {
  using C = sm100k2::Cfg<D, NT, SPLIT>;
  CUtensorMap mq, mk, mv;
  int rc;
  if ((rc = make_tmap_3d(&mq, q, 2, D, q_rows, q_rows, groups, sm100k2::BOX, sm100k2::BM))) return rc;
  const int64_t nin_eff = n_in > 0 ? n_in : 1;  // zero-row maps are invalid; rows are masked
  if ((rc = make_tmap_3d(&mk, k_in, 2, D, nin_eff, nin_eff, groups, sm100k2::BOX, NT))) return rc;
  if ((rc = make_tmap_3d(&mv, v_in, 2, D, nin_eff, nin_eff, groups, sm100k2::BOX, NT))) return rc;
  unsigned long long* trace = nullptr;
  if (g_k2_trace != nullptr && g_k2_trace_i < g_k2_trace_n)
    trace = g_k2_trace + (size_t)(g_k2_trace_i++) * 1024 * 8;  // slab per traced launch
  auto kern = trace ? (extb ? sm100k2::internal_merge_kernel<D, NT, SPLIT, true, false, true>
                            : sm100k2::internal_merge_kernel<D, NT, SPLIT, true>)
                    : (extb ? sm100k2::internal_merge_kernel<D, NT, SPLIT, false, false, true>
                            : sm100k2::internal_merge_kernel<D, NT, SPLIT, false>);
  static bool attr[4] = {false, false, false, false};
  const int ai = (trace ? 1 : 0) + (extb ? 2 : 0);
  if (!attr[ai]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    attr[ai] = true;
  }
  const int m_tiles = (int)((q_rows + sm100k2::BM - 1) / sm100k2::BM);
  const float scale_log2 = (float)(scale * 1.4426950408889634);
  launch_pdl(kern, dim3((unsigned)(groups * m_tiles * C::SPLIT)), dim3(sm100k2::THREADS), C::SMEM, st,
             mq, mk, mv, o_ext, lse_ext, (int)q_rows, m_tiles, (int)n_in, scale_log2, out,
             out_bf16 ? 1 : 0, lse_merged, o_int, lse_int, reinterpret_cast<int*>(empty),
             (ext_early ? 1 : 0) | (k2_pdl_late() ? 2 : 0) | (k2_vsplit_bits() & 4), trace,
             sm100k2::TokLayout{1, 1, 1, 0});
  count_launch();
  return check_launch("internal_merge_kernel(sm100)");
}

template <int NT, bool EXTB>
static int launch_k2_v2(const __nv_bfloat16* q, const __nv_bfloat16* k_in, const __nv_bfloat16* v_in,
                        int64_t groups, int64_t q_rows, int64_t n_in, double scale, const void* o_ext,
                        const float* lse_ext, void* out, bool out_bf16, float* lse_merged, float* o_int,
                        float* lse_int, int32_t* empty, bool ext_early, cudaStream_t st) {
  using C = sm100k2::CfgV2<NT, EXTB>;
  constexpr int D = 128;
  CUtensorMap mq, mk, mv, me;
  int rc;
  if ((rc = make_tmap_3d(&mq, q, 2, D, q_rows, q_rows, groups, sm100k2::BOX, sm100k2::BM))) return rc;
  const int64_t nin_eff = n_in > 0 ? n_in : 1;
  if ((rc = make_tmap_3d(&mk, k_in, 2, D, nin_eff, nin_eff, groups, sm100k2::BOX, NT))) return rc;
  if ((rc = make_tmap_3d(&mv, v_in, 2, D, nin_eff, nin_eff, groups, sm100k2::BOX, NT))) return rc;
  if ((rc = make_tmap_3d(&me, o_ext, EXTB ? 2 : 4, D, q_rows, q_rows, groups, C::ECOLS, sm100k2::BM))) return rc;
  // bf16 output through one bulk tensor store per (CTA, column half)
  // default (-1): TMA store only when the grid exceeds the SMs (b=16, one CTA
  // per SM: 5.78 -> 6.08 us with it; b=32 8.56 -> 8.38)
  const int store = k2_env("FB_K2_STORE", g_k2_store);
  const int64_t ctas = groups * ((q_rows + sm100k2::BM - 1) / sm100k2::BM);
  const bool tma_out = out_bf16 && (store == 1 || (store == -1 && ctas > num_sms())) &&
                       (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  CUtensorMap mo = me;  // unused unless tma_out
  if (tma_out && (rc = make_tmap_3d(&mo, out, 2, D, q_rows, q_rows, groups, sm100k2::BOX, sm100k2::BM))) return rc;
  auto kern = sm100k2::internal_merge_v2_kernel<NT, EXTB>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    attr = true;
  }
  const int m_tiles = (int)((q_rows + sm100k2::BM - 1) / sm100k2::BM);
  const float scale_log2 = (float)(scale * 1.4426950408889634);
  launch_pdl(kern, dim3((unsigned)(groups * m_tiles)), dim3(sm100k2::V2_THREADS), C::SMEM, st, mq, mk,
             mv, me, mo, lse_ext, (int)q_rows, m_tiles, (int)n_in, scale_log2, out, out_bf16 ? 1 : 0,
             lse_merged, o_int, lse_int, reinterpret_cast<int*>(empty),
             (ext_early ? 1 : 0) | (k2_pdl_late() ? 2 : 0) | k2_vsplit_bits(ctas), tma_out ? 1 : 0);
  count_launch();
  return check_launch("internal_merge_v2_kernel(sm100)");
}

int make_tmap_nd(CUtensorMap* map, const void* base, int rank, const int64_t* dims,
                 const int64_t* stride_bytes, const int* box);

// Token-major cached step (TokLayout): q / k_in / v_in are [batch, B, H, d]
// views with token strides q_ts / k_ts / v_ts (elements; e.g. the row pitch of
// a fused QKV projection output) and the output is [batch, B, Hq, d] with
// token stride out_ts.  d = 128, G * B <= 128, B <= 64.
template <int NT>
static int launch_k2_tok(const __nv_bfloat16* q, int64_t q_ts, const __nv_bfloat16* k, int64_t k_ts,
                         const __nv_bfloat16* v, int64_t v_ts, int64_t batch, int64_t B, int64_t Hq,
                         int64_t Hkv, double scale, const void* o_ext, const float* lse_ext, void* out,
                         int64_t out_ts, bool out_bf16, bool ext_early, bool extb, cudaStream_t st) {
  constexpr int D = 128, SPLIT = 2;
  using C = sm100k2::Cfg<D, NT, SPLIT>;
  const int64_t G = Hq / Hkv;
  CUtensorMap mq, mk, mv;
  int rc;
  {
    const int64_t dims[5] = {D, B, G, Hkv, batch};
    const int64_t str[5] = {2, q_ts * 2, D * 2, G * D * 2, B * q_ts * 2};
    const int box[5] = {sm100k2::BOX, (int)B, (int)G, 1, 1};
    if ((rc = make_tmap_nd(&mq, q, 5, dims, str, box))) return rc;
  }
  {
    const int64_t dims[4] = {D, B, Hkv, batch};
    const int64_t sk[4] = {2, k_ts * 2, D * 2, B * k_ts * 2};
    const int64_t sv[4] = {2, v_ts * 2, D * 2, B * v_ts * 2};
    const int box[4] = {sm100k2::BOX, NT, 1, 1};
    if ((rc = make_tmap_nd(&mk, k, 4, dims, sk, box))) return rc;
    if ((rc = make_tmap_nd(&mv, v, 4, dims, sv, box))) return rc;
  }
  auto kern = extb ? sm100k2::internal_merge_kernel<D, NT, SPLIT, false, true, true>
                   : sm100k2::internal_merge_kernel<D, NT, SPLIT, false, true>;
  static bool attr[2] = {false, false};
  if (!attr[extb ? 1 : 0]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    attr[extb ? 1 : 0] = true;
  }
  const int64_t groups = batch * Hkv, q_rows = G * B;
  const float scale_log2 = (float)(scale * 1.4426950408889634);
  launch_pdl(kern, dim3((unsigned)(groups * SPLIT)), dim3(sm100k2::THREADS), C::SMEM, st, mq, mk, mv, o_ext,
             lse_ext, (int)q_rows, 1, (int)B, scale_log2, out, out_bf16 ? 1 : 0, (float*)nullptr,
             (float*)nullptr, (float*)nullptr, (int*)nullptr,
             (ext_early ? 1 : 0) | (k2_pdl_late() ? 2 : 0) | (k2_vsplit_bits() & 4),
             (unsigned long long*)nullptr, sm100k2::TokLayout{(int)B, (int)G, (int)Hkv, (long long)out_ts});
  count_launch();
  return check_launch("internal_merge_kernel(sm100, token-major)");
}

int launch_internal_merge_tok_sm100(const __nv_bfloat16* q, int64_t q_ts, const __nv_bfloat16* k,
                                    int64_t k_ts, const __nv_bfloat16* v, int64_t v_ts, int64_t batch,
                                    int64_t B, int64_t Hq, int64_t Hkv, int64_t d, double scale,
                                    const void* o_ext, const float* lse_ext, void* out, int64_t out_ts,
                                    bool out_bf16, bool ext_early, bool extb, cudaStream_t st) {
  if (d != 128 || Hkv <= 0 || Hq % Hkv != 0 || (Hq / Hkv) * B > 128 || B < 1 || B > 64)
    return fail(FB_ERR_UNSUPPORTED, "token-major cached step: d 128, (Hq/Hkv)*B <= 128, 1 <= B <= 64");
  if (B <= 16)
    return launch_k2_tok<16>(q, q_ts, k, k_ts, v, v_ts, batch, B, Hq, Hkv, scale, o_ext, lse_ext, out, out_ts,
                             out_bf16, ext_early, extb, st);
  if (B <= 32)
    return launch_k2_tok<32>(q, q_ts, k, k_ts, v, v_ts, batch, B, Hq, Hkv, scale, o_ext, lse_ext, out, out_ts,
                             out_bf16, ext_early, extb, st);
  return launch_k2_tok<64>(q, q_ts, k, k_ts, v, v_ts, batch, B, Hq, Hkv, scale, o_ext, lse_ext, out, out_ts,
                           out_bf16, ext_early, extb, st);
}

int launch_internal_merge_sm100(const __nv_bfloat16* q, const __nv_bfloat16* k_in,
                                const __nv_bfloat16* v_in, int64_t groups, int64_t q_rows,
                                int64_t head_dim, int64_t n_in, double scale, const void* o_ext,
                                const float* lse_ext, void* out, bool out_bf16, float* lse_merged,
                                float* o_int, float* lse_int, int32_t* empty, bool ext_early,
                                bool extb, cudaStream_t st) {
#define FB_K2(DD, NN)                                                                           \
  return split ? launch_k2<DD, NN, (DD == 128 ? 2 : 1)>(q, k_in, v_in, groups, q_rows, n_in, scale, \
                                                        o_ext, lse_ext, out, out_bf16, lse_merged,  \
                                                        o_int, lse_int, empty, ext_early, extb, st) \
               : launch_k2<DD, NN, 1>(q, k_in, v_in, groups, q_rows, n_in, scale, o_ext, lse_ext,   \
                                      out, out_bf16, lse_merged, o_int, lse_int, empty, ext_early,  \
                                      extb, st)
  // split the output columns over 2 CTAs: measured faster at every batch
  // (C2 b=16: 5.7 vs 8.2 us; b=24: 9.9 vs 10.8; b=32: 11.3 vs 14.5, 1.7 waves)
  bool split = true;
  if (const char* e = getenv("FB_K2_SPLIT")) split = e[0] == '1';  // diagnostics
  // v2 (O_ext prefetched into smem by TMA, whole rows per CTA, two CTAs per
  // SM) once the query tiles outnumber the SMs: measured at C2 (36 layers x 31
  // cached steps in one graph) b=32 9.2 vs 11.3 us per launch, while at b=16 /
  // b=4 (128 / 32 tiles) v1's column split over 2 CTAs stays faster (5.7 vs
  // 6.0 us, 4.2 vs 5.1 us).  FB_K2_V2=0 / 1 forces v1 / v2 (diagnostics).
  static int v2_env = -2;
  if (v2_env == -2) {
    const char* e = getenv("FB_K2_V2");
    v2_env = e == nullptr ? -1 : (e[0] == '0' ? 0 : 1);
  }
  const int v2 = g_k2_v2_override >= 0 ? g_k2_v2_override : v2_env;
  const int64_t k2_tiles = groups * ((q_rows + sm100k2::BM - 1) / sm100k2::BM);
  // with a bf16 cached partial (FB_PARTIAL_BF16) v2's O_ext tile is 32 KB and
  // it wins as soon as v1's column-split grid (2 CTAs per tile) exceeds the
  // SMs: C2 b=16 5.42 vs 6.12 us (v1), b=32 8.09 vs 10.57; b=4 v1 3.70 vs 4.66
  const bool use_v2 = v2 == 1 || (v2 == -1 && (extb ? 2 * k2_tiles > num_sms() : k2_tiles > num_sms()));
  if (head_dim == 128 && use_v2 && n_in <= 64 && (reinterpret_cast<uintptr_t>(o_ext) & 15) == 0) {
#define FB_K2V2(NN)                                                                                     \
  return extb ? launch_k2_v2<NN, true>(q, k_in, v_in, groups, q_rows, n_in, scale, o_ext, lse_ext, out,  \
                                       out_bf16, lse_merged, o_int, lse_int, empty, ext_early, st)       \
              : launch_k2_v2<NN, false>(q, k_in, v_in, groups, q_rows, n_in, scale, o_ext, lse_ext, out, \
                                        out_bf16, lse_merged, o_int, lse_int, empty, ext_early, st)
    if (n_in <= 16) FB_K2V2(16);
    if (n_in <= 32) FB_K2V2(32);
    if (n_in <= 64) FB_K2V2(64);
#undef FB_K2V2
    // (n_in > 64: the 128-key score row does not fit beside 96 registers; v1)
  }
  if (head_dim == 128) {
    if (n_in <= 16) FB_K2(128, 16);
    if (n_in <= 32) FB_K2(128, 32);
    if (n_in <= 64) FB_K2(128, 64);
    FB_K2(128, 128);
  }
  if (n_in <= 16) FB_K2(64, 16);
  if (n_in <= 32) FB_K2(64, 32);
  if (n_in <= 64) FB_K2(64, 64);
  FB_K2(64, 128);
#undef FB_K2
}

}  // namespace fb
