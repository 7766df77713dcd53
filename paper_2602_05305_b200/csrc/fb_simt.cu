// SIMT kernels of the FlashBlock hot path: any head_dim, F64 / F32 / BF16.
//
//  * partial_simt     -- online-softmax partial over a key map, optionally
//                        split along the keys (split-KV within the GPU) and
//                        optionally fused with the log-space merge against a
//                        cached partial (the K2 "internal + merge" epilogue).
//  * combine_parts    -- P-way log-space merge (K3), sentinel aware.
//  * fill_sentinel    -- the empty partial (out 0, lognorm -inf).
//
// Algorithm restated from the reference: tile-streamed softmax with running
// max / normaliser / accumulator and exp(m_old - m_new) rescaling
// (attention.py:156-182); merge weights exp(L - max L) (attention.py:207-233).
// The score product runs in the mode's score type (the tensor dtype, as
// attention.py:166); statistics and accumulation in the accumulate type.
#include "fb_kernels.cuh"

namespace fb {

constexpr int SIMT_WARPS = 4;
constexpr int SIMT_ROWS_PER_WARP = 4;
constexpr int SIMT_ROWS = SIMT_WARPS * SIMT_ROWS_PER_WARP;  // query rows per CTA
constexpr int SIMT_KT = 32;                                  // keys per tile (one per lane)

template <int D, typename Ts, typename Ta>
constexpr size_t simt_smem_bytes() {
  return sizeof(Ts) * (SIMT_ROWS * D + SIMT_KT * (D + 1)) + sizeof(Ta) * SIMT_KT * D;
}

// Products that must round before they are summed (no FMA contraction), so a
// two-way merge is bitwise symmetric like the reference's wa*A + wb*B.
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

// Element type -> 16-byte chunk unpacking into the score / accumulate types.
template <typename Tin>
struct Chunk {
  static constexpr int E = 16 / sizeof(Tin);
  template <typename To>
  static __device__ __forceinline__ void unpack(const uint4& u, To* dst) {
    const Tin* e = reinterpret_cast<const Tin*>(&u);
#pragma unroll
    for (int i = 0; i < E; ++i) dst[i] = cvt<To>(e[i]);
  }
};

// grid: (ceil(q_rows/SIMT_ROWS), splits, groups); block: 32*SIMT_WARPS.
// Split s of group g covers key ordinals [s*per_split, min((s+1)*per_split, count)).
// Without MERGE the normalised partial goes to (po, pl) at slot
// [s][g*q_rows + row]; with MERGE (splits == 1) it is merged with the cache.
// `vec`: every row pointer is 16-byte aligned and head_dim*sizeof(Tin) % 16 == 0,
// so tiles move as 16-byte chunks with all loads of a batch issued up front.
template <typename Mode, int D, bool MERGE, bool NO_V, typename Map>
__global__ void __launch_bounds__(32 * SIMT_WARPS)
partial_simt(const typename Mode::Tin* __restrict__ q, Map map, int64_t q_rows, int64_t head_dim,
             int64_t per_split, typename Mode::Ta scale, typename Mode::Ta* po,
             typename Mode::Tl* pl, int64_t rows_total, MergeOut<Mode> mo, bool vec,
             const int32_t* __restrict__ glist) {
  using Tin = typename Mode::Tin;
  using Ts = typename Mode::Ts;
  using Ta = typename Mode::Ta;
  using To = typename Mode::To;
  using Tl = typename Mode::Tl;
  constexpr int C = D / 32;  // output columns per lane
  constexpr int E = Chunk<Tin>::E;
  constexpr int NT = 32 * SIMT_WARPS;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  Ts* qs = reinterpret_cast<Ts*>(smem_raw);                // [SIMT_ROWS][D]
  Ts* ks = qs + SIMT_ROWS * D;                              // [KT][D+1]
  Ta* vs = reinterpret_cast<Ta*>(ks + SIMT_KT * (D + 1));   // [KT][D]
  __shared__ const Tin* kptr[SIMT_KT];
  __shared__ const Tin* vptr[SIMT_KT];

  const int64_t g = glist != nullptr ? (int64_t)glist[blockIdx.z] : (int64_t)blockIdx.z;  // group subset
  const int split = blockIdx.y;
  const int64_t row0 = (int64_t)blockIdx.x * SIMT_ROWS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int64_t n_keys = map.count(g);
  const int64_t kb = min((int64_t)split * per_split, n_keys);
  int64_t ke = min(kb + per_split, n_keys);
  constexpr bool CAUSAL = is_causal_map<Map>::value;
  // block-causal rows: this warp's rows end at their own limits (the CTA stops
  // at the largest one); launched unsplit, so every row has key 0
  int64_t row_end[SIMT_ROWS_PER_WARP];
#pragma unroll
  for (int i = 0; i < SIMT_ROWS_PER_WARP; ++i) row_end[i] = ke;
  if constexpr (CAUSAL) {
    int64_t cta_end = 0;
    for (int r = 0; r < SIMT_ROWS; ++r) {
      const int64_t gr = min(row0 + r, q_rows - 1);
      cta_end = max(cta_end, map.row_limit(gr));
    }
    ke = min(ke, cta_end);
#pragma unroll
    for (int i = 0; i < SIMT_ROWS_PER_WARP; ++i)
      row_end[i] = min(ke, map.row_limit(min(row0 + warp * SIMT_ROWS_PER_WARP + i, q_rows - 1)));
  }

  // merge operands first: their latency overlaps the tile loads
  Ta oe[SIMT_ROWS_PER_WARP][C];
  Ta le[SIMT_ROWS_PER_WARP];
  if constexpr (MERGE) {
#pragma unroll
    for (int i = 0; i < SIMT_ROWS_PER_WARP; ++i) {
      const int64_t gr = row0 + warp * SIMT_ROWS_PER_WARP + i;
      const int64_t rr = g * q_rows + gr;
      const bool ok = gr < q_rows && mo.lse_ext != nullptr;
      le[i] = ok ? (Ta)mo.lse_ext[rr] : Num<Ta>::ninf();
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const int col = lane + 32 * c;
        oe[i][c] = (ok && col < head_dim) ? (Ta)mo.o_ext[rr * head_dim + col] : (Ta)0;
      }
    }
  }

  // stage the CTA's query rows (zero-padded to D)
  const int cpr = (int)(head_dim / E);  // 16-byte chunks per row (vec path)
  if (vec) {
    for (int ci = threadIdx.x; ci < SIMT_ROWS * cpr; ci += NT) {
      const int r = ci / cpr, cc = ci % cpr;
      const int64_t gr = row0 + r;
      uint4 u = make_uint4(0, 0, 0, 0);
      if (gr < q_rows) u = *reinterpret_cast<const uint4*>(q + (g * q_rows + gr) * head_dim + cc * E);
      Chunk<Tin>::unpack(u, qs + r * D + cc * E);
    }
    for (int i = threadIdx.x; i < SIMT_ROWS * (D - (int)head_dim); i += NT) {
      const int r = i / (D - (int)head_dim), c = (int)head_dim + i % (D - (int)head_dim);
      qs[r * D + c] = 0;
    }
  } else {
    for (int i = threadIdx.x; i < SIMT_ROWS * D; i += NT) {
      const int r = i / D, c = i % D;
      const int64_t gr = row0 + r;
      Ts val = 0;
      if (gr < q_rows && c < head_dim) val = cvt<Ts>(q[(g * q_rows + gr) * head_dim + c]);
      qs[i] = val;
    }
  }

  Ta m[SIMT_ROWS_PER_WARP], l[SIMT_ROWS_PER_WARP], acc[SIMT_ROWS_PER_WARP][C];
#pragma unroll
  for (int i = 0; i < SIMT_ROWS_PER_WARP; ++i) {
    m[i] = Num<Ta>::ninf();
    l[i] = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) acc[i][c] = 0;
  }

  for (int64_t t0 = kb; t0 < ke; t0 += SIMT_KT) {
    __syncthreads();  // previous tile fully consumed
    if (threadIdx.x < SIMT_KT) {
      const int64_t t = t0 + threadIdx.x;
      const Tin* kr = nullptr;
      const Tin* vr = nullptr;
      if (t < ke) map.row(g, t, kr, vr);
      kptr[threadIdx.x] = kr;
      vptr[threadIdx.x] = vr;
    }
    __syncthreads();
    if (vec) {
      constexpr int NB = 4;  // chunks per thread per batch (per K and V)
      for (int base = 0; base < SIMT_KT * cpr; base += NB * NT) {
        uint4 ku[NB], vu[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          const int ci = base + b * NT + threadIdx.x;
          ku[b] = vu[b] = make_uint4(0, 0, 0, 0);
          if (ci < SIMT_KT * cpr) {
            const int j = ci / cpr, cc = ci % cpr;
            if (kptr[j] != nullptr) {
              ku[b] = *reinterpret_cast<const uint4*>(kptr[j] + cc * E);
              if constexpr (!NO_V) vu[b] = *reinterpret_cast<const uint4*>(vptr[j] + cc * E);
            }
          }
        }
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          const int ci = base + b * NT + threadIdx.x;
          if (ci < SIMT_KT * cpr) {
            const int j = ci / cpr, cc = ci % cpr;
            Chunk<Tin>::unpack(ku[b], ks + j * (D + 1) + cc * E);
            if constexpr (!NO_V) Chunk<Tin>::unpack(vu[b], vs + j * D + cc * E);
          }
        }
      }
      for (int i = threadIdx.x; i < SIMT_KT * (D - (int)head_dim); i += NT) {
        const int j = i / (D - (int)head_dim), c = (int)head_dim + i % (D - (int)head_dim);
        ks[j * (D + 1) + c] = 0;
        if constexpr (!NO_V) vs[j * D + c] = 0;
      }
    } else {
      for (int j = warp; j < SIMT_KT; j += SIMT_WARPS) {
        const Tin* kr = kptr[j];
        const Tin* vr = vptr[j];
        for (int c = lane; c < D; c += 32) {
          Ts kv = 0;
          Ta vv = 0;
          if (kr != nullptr && c < head_dim) {
            kv = cvt<Ts>(kr[c]);
            if constexpr (!NO_V) vv = cvt<Ta>(vr[c]);
          }
          ks[j * (D + 1) + c] = kv;
          if constexpr (!NO_V) vs[j * D + c] = vv;
        }
      }
    }
    __syncthreads();
    const bool key_ok = (t0 + lane) < ke;

    Ts s[SIMT_ROWS_PER_WARP];
#pragma unroll
    for (int i = 0; i < SIMT_ROWS_PER_WARP; ++i) s[i] = 0;
    const Ts* krow = ks + lane * (D + 1);
#pragma unroll 8
    for (int c = 0; c < D; ++c) {
      const Ts kc = krow[c];
#pragma unroll
      for (int i = 0; i < SIMT_ROWS_PER_WARP; ++i)
        s[i] += qs[(warp * SIMT_ROWS_PER_WARP + i) * D + c] * kc;
    }
#pragma unroll
    for (int i = 0; i < SIMT_ROWS_PER_WARP; ++i) {
      // scores in the tensor dtype, then widened (attention.py:166)
      const bool ok = CAUSAL ? (t0 + lane) < row_end[i] : key_ok;
      const Ta si = ok ? (Ta)(s[i] * (Ts)scale) : Num<Ta>::ninf();
      const Ta m_new = fmax(m[i], warp_max(si));
      const Ta alpha = Num<Ta>::exp_(m[i] - m_new);  // exp(-inf) = 0 for the first tile
      const Ta p = ok ? Num<Ta>::exp_(si - m_new) : (Ta)0;
      l[i] = l[i] * alpha + warp_sum(p);
      if constexpr (!NO_V) {
#pragma unroll
        for (int c = 0; c < C; ++c) acc[i][c] *= alpha;
#pragma unroll 8
        for (int j = 0; j < SIMT_KT; ++j) {
          const Ta pj = __shfl_sync(0xffffffffu, p, j);
          const Ta* vrow = vs + j * D + lane;
#pragma unroll
          for (int c = 0; c < C; ++c) acc[i][c] += pj * vrow[c * 32];
        }
      }
      m[i] = m_new;
    }
  }

  // epilogue
#pragma unroll
  for (int i = 0; i < SIMT_ROWS_PER_WARP; ++i) {
    const int64_t gr = row0 + warp * SIMT_ROWS_PER_WARP + i;
    if (gr >= q_rows) continue;
    const int64_t rr = g * q_rows + gr;  // global row
    const bool empty = (ke <= kb);
    const Ta inv = empty ? (Ta)0 : (Ta)1 / l[i];
    const Ta lse = empty ? Num<Ta>::ninf() : m[i] + Num<Ta>::log_(l[i]);
    if constexpr (!MERGE) {
      if constexpr (!NO_V) {
        Ta* dst = po + ((int64_t)split * rows_total + rr) * head_dim;
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const int col = lane + 32 * c;
          if (col < head_dim) dst[col] = acc[i][c] * inv;
        }
      }
      if (lane == 0) pl[(int64_t)split * rows_total + rr] = (Tl)lse;
    } else {
      // internal partial rounded to its stored type first, as the reference
      // merges the partial it returns (attention.py:180, :320-321)
      const Ta li = (Ta)(Tl)lse;
      const Ta mx = fmax(le[i], li);
      const bool live = mx != Num<Ta>::ninf();
      const Ta we = live ? Num<Ta>::exp_(le[i] - mx) : (Ta)0;
      const Ta wi = live ? Num<Ta>::exp_(li - mx) : (Ta)0;
      const Ta z = we + wi;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const int col = lane + 32 * c;
        if (col >= head_dim) continue;
        const To oi = (To)(acc[i][c] * inv);
        if (mo.o_int) mo.o_int[rr * head_dim + col] = oi;
        Ta val = 0;
        if (live) val = (mul_rn(we, oe[i][c]) + mul_rn(wi, (Ta)oi)) / z;
        if (mo.out_bf16)
          reinterpret_cast<__nv_bfloat16*>(mo.out)[rr * head_dim + col] = cvt<__nv_bfloat16>(val);
        else
          reinterpret_cast<To*>(mo.out)[rr * head_dim + col] = (To)val;
      }
      if (lane == 0) {
        if (mo.lse_int) mo.lse_int[rr] = (Tl)lse;
        if (mo.lse_merged) mo.lse_merged[rr] = live ? (Tl)(mx + Num<Ta>::log_(z)) : (Tl)Num<Ta>::ninf();
        if (!live && mo.empty_rows) atomicAdd(mo.empty_rows, 1);
      }
    }
  }
}

// ------------------------------------------------------------------ combine

// One warp per row.  Parts come either from a pointer list (API combine) or
// from a strided workspace (split-KV partials).
template <typename Tp, typename Tlp, typename Ta, typename To, typename Tlo>
__global__ void combine_parts(CombineList list, int64_t rows, int64_t head_dim, To* o_out,
                              Tlo* l_out, int32_t* empty_rows, bool vec) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  auto optr = [&](int p) -> const Tp* {
    return list.strided ? reinterpret_cast<const Tp*>(list.o[0]) + (int64_t)p * list.o_stride
                        : reinterpret_cast<const Tp*>(list.o[p]);
  };
  auto lptr = [&](int p) -> const Tlp* {
    return list.strided ? reinterpret_cast<const Tlp*>(list.l[0]) + (int64_t)p * list.l_stride
                        : reinterpret_cast<const Tlp*>(list.l[p]);
  };
  if (list.n <= FB_MAX_PARTS) {
    // lane p holds part p's lognorm and merge weight, computed once per row and
    // broadcast by shuffle; all parts' loads in flight before the sum; products
    // rounded before summing, so a two-way merge stays bitwise symmetric like
    // the reference's wa*A + wb*B
    const Ta lp = lane < list.n ? (Ta)lptr(lane)[row] : Num<Ta>::ninf();
    const Ta mx = warp_max(lp);
    const bool live = mx != Num<Ta>::ninf();
    const Ta w = (live && lane < list.n) ? Num<Ta>::exp_(lp - mx) : (Ta)0;
    const Ta z = warp_sum(w);
    Ta wv[FB_MAX_PARTS];
#pragma unroll
    for (int p = 0; p < FB_MAX_PARTS; ++p) wv[p] = __shfl_sync(0xffffffffu, w, p);
    if (vec) {
      // 16-byte loads: a lane owns VW consecutive columns, all parts in flight
      constexpr int VW = 16 / sizeof(Tp);
      for (int64_t c = (int64_t)lane * VW; c < head_dim; c += 32 * VW) {
        Tp vals[FB_MAX_PARTS][VW];
#pragma unroll
        for (int p = 0; p < FB_MAX_PARTS; ++p) {
          if (live && p < list.n) {
            const uint4 u = *reinterpret_cast<const uint4*>(optr(p) + row * head_dim + c);
            const Tp* e = reinterpret_cast<const Tp*>(&u);
#pragma unroll
            for (int i = 0; i < VW; ++i) vals[p][i] = e[i];
          } else {
#pragma unroll
            for (int i = 0; i < VW; ++i) vals[p][i] = (Tp)0;
          }
        }
#pragma unroll
        for (int i = 0; i < VW; ++i) {
          Ta num = 0;
          if (live) {
#pragma unroll
            for (int p = 0; p < FB_MAX_PARTS; ++p)
              if (p < list.n) num += mul_rn(wv[p], (Ta)vals[p][i]);
            num = num / z;
          }
          o_out[row * head_dim + c + i] = cvt<To>(num);
        }
      }
    } else
    for (int64_t c = lane; c < head_dim; c += 32) {
      Ta vals[FB_MAX_PARTS];
#pragma unroll
      for (int p = 0; p < FB_MAX_PARTS; ++p)
        vals[p] = (live && p < list.n) ? (Ta)optr(p)[row * head_dim + c] : (Ta)0;
      Ta num = 0;
      if (live) {
#pragma unroll
        for (int p = 0; p < FB_MAX_PARTS; ++p)
          if (p < list.n) num += mul_rn(wv[p], vals[p]);
        num = num / z;
      }
      o_out[row * head_dim + c] = cvt<To>(num);
    }
    if (lane == 0) {
      if (l_out) l_out[row] = live ? (Tlo)(mx + Num<Ta>::log_(z)) : (Tlo)Num<Ta>::ninf();
      if (!live && empty_rows) atomicAdd(empty_rows, 1);
    }
    return;
  }
  // many parts (in-GPU SIMT split-KV partials): sequential over parts
  Ta mx = Num<Ta>::ninf();
  for (int p = 0; p < list.n; ++p) mx = fmax(mx, (Ta)lptr(p)[row]);
  const bool live = mx != Num<Ta>::ninf();
  Ta z = 0;
  for (int p = 0; p < list.n; ++p) z += live ? Num<Ta>::exp_((Ta)lptr(p)[row] - mx) : (Ta)0;
  for (int64_t c = lane; c < head_dim; c += 32) {
    Ta num = 0;
    if (live) {
      for (int p = 0; p < list.n; ++p) {
        const Ta w = Num<Ta>::exp_((Ta)lptr(p)[row] - mx);
        num += mul_rn(w, (Ta)optr(p)[row * head_dim + c]);
      }
      num = num / z;
    }
    o_out[row * head_dim + c] = cvt<To>(num);
  }
  if (lane == 0) {
    if (l_out) l_out[row] = live ? (Tlo)(mx + Num<Ta>::log_(z)) : (Tlo)Num<Ta>::ninf();
    if (!live && empty_rows) atomicAdd(empty_rows, 1);
  }
}

template <typename To, typename Tl>
__global__ void fill_sentinel(To* o, Tl* l, int64_t rows, int64_t head_dim) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < rows * head_dim) o[i] = cvt<To>(0.0f);
  if (l && i < rows) l[i] = (Tl)(-INFINITY);
}

// ------------------------------------------------------------------ launchers

static inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
template <typename T>
static bool rows_ok(const T* q, int64_t d) {
  return al16(q) && (d * (int64_t)sizeof(T)) % 16 == 0;
}
template <typename T>
static bool map_vec_ok(const RangeMap<T>& m, const T* q, int64_t d) {
  return rows_ok(q, d) && al16(m.k) && al16(m.v);
}
template <typename T>
static bool map_vec_ok(const RaggedMap<T>& m, const T* q, int64_t d) {
  return rows_ok(q, d) && al16(m.k) && al16(m.v);
}
template <typename T>
static bool map_vec_ok(const ConcatMap<T>& m, const T* q, int64_t d) {
  return rows_ok(q, d) && al16(m.k) && al16(m.k_in) && (m.v == nullptr || al16(m.v)) &&
         (m.v_in == nullptr || al16(m.v_in));
}
template <typename T>
static bool map_vec_ok(const SelectedMap<T>& m, const T* q, int64_t d) {
  return rows_ok(q, d) && al16(m.k) && al16(m.v) && al16(m.k_in) && al16(m.v_in);
}
template <typename T>
static bool map_vec_ok(const CausalMap<T>& m, const T* q, int64_t d) {
  return rows_ok(q, d) && al16(m.k) && al16(m.v);
}
template <typename T>
static bool map_vec_ok(const ResidualMap<T>& m, const T* q, int64_t d) {
  return rows_ok(q, d) && al16(m.k) && al16(m.v);
}

template <typename Mode, int D, bool MERGE, bool NO_V, typename Map>
static int launch_partial_d(const typename Mode::Tin* q, const Map& map, int64_t groups,
                            int64_t q_rows, int64_t head_dim, int64_t per_split, int splits,
                            double scale, typename Mode::Ta* po, typename Mode::Tl* pl,
                            const MergeOut<Mode>& mo, cudaStream_t st, const int32_t* glist) {
  constexpr size_t smem = simt_smem_bytes<D, typename Mode::Ts, typename Mode::Ta>();
  auto kern = partial_simt<Mode, D, MERGE, NO_V, Map>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  dim3 grid((unsigned)((q_rows + SIMT_ROWS - 1) / SIMT_ROWS), (unsigned)splits, (unsigned)groups);
  const bool vec = map_vec_ok(map, q, head_dim);
  kern<<<grid, 32 * SIMT_WARPS, smem, st>>>(q, map, q_rows, head_dim, per_split,
                                            (typename Mode::Ta)scale, po, pl, groups * q_rows, mo,
                                            vec, glist);
  count_launch();
  return check_launch("partial_simt");
}

template <typename Mode, bool MERGE, bool NO_V, typename Map>
int launch_partial_simt(const typename Mode::Tin* q, const Map& map, int64_t groups,
                        int64_t q_rows, int64_t head_dim, int64_t per_split, int splits,
                        double scale, typename Mode::Ta* po, typename Mode::Tl* pl,
                        const MergeOut<Mode>& mo, cudaStream_t st, const int32_t* glist) {
  if (head_dim <= 32)
    return launch_partial_d<Mode, 32, MERGE, NO_V>(q, map, groups, q_rows, head_dim, per_split, splits, scale, po, pl, mo, st, glist);
  if (head_dim <= 64)
    return launch_partial_d<Mode, 64, MERGE, NO_V>(q, map, groups, q_rows, head_dim, per_split, splits, scale, po, pl, mo, st, glist);
  if (head_dim <= 128)
    return launch_partial_d<Mode, 128, MERGE, NO_V>(q, map, groups, q_rows, head_dim, per_split, splits, scale, po, pl, mo, st, glist);
  if (head_dim <= 256)
    return launch_partial_d<Mode, 256, MERGE, NO_V>(q, map, groups, q_rows, head_dim, per_split, splits, scale, po, pl, mo, st, glist);
  return fail(FB_ERR_UNSUPPORTED, "head_dim > 256 is not supported");
}

template <typename Tp, typename Tlp, typename Ta, typename To, typename Tlo>
int launch_combine(const CombineList& list, int64_t rows, int64_t head_dim, To* o_out, Tlo* l_out,
                   int32_t* empty_rows, cudaStream_t st) {
  if (rows == 0) return FB_OK;
  const int warps = 8;
  const unsigned blocks = (unsigned)((rows + warps - 1) / warps);
  // 16-byte vector loads when every part's rows are 16-byte aligned
  bool vec = (head_dim * (int64_t)sizeof(Tp)) % 16 == 0 && list.n <= FB_MAX_PARTS;
  for (int p = 0; p < list.n && vec; ++p) {
    const void* base = list.strided ? (const void*)(reinterpret_cast<const Tp*>(list.o[0]) + (int64_t)p * list.o_stride)
                                    : list.o[p];
    vec = (reinterpret_cast<uintptr_t>(base) & 15u) == 0;
  }
  combine_parts<Tp, Tlp, Ta, To, Tlo><<<blocks, 32 * warps, 0, st>>>(list, rows, head_dim, o_out,
                                                                      l_out, empty_rows, vec);
  count_launch();
  return check_launch("combine_parts");
}

template <typename To, typename Tl>
int launch_fill_sentinel(To* o, Tl* l, int64_t rows, int64_t head_dim, cudaStream_t st) {
  const int64_t n = rows * head_dim > rows ? rows * head_dim : rows;
  if (n == 0) return FB_OK;
  fill_sentinel<To, Tl><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(o, l, rows, head_dim);
  count_launch();
  return check_launch("fill_sentinel");
}

// ------------------------------------------------------------------ instantiations

#define FB_INST_PARTIAL(MODE, MERGE, MAP)                                                      \
  template int launch_partial_simt<MODE, MERGE, false, MAP<MODE::Tin>>(                       \
      const MODE::Tin*, const MAP<MODE::Tin>&, int64_t, int64_t, int64_t, int64_t, int, double, \
      MODE::Ta*, MODE::Tl*, const MergeOut<MODE>&, cudaStream_t, const int32_t*);

#define FB_INST_MODE(MODE)                  \
  FB_INST_PARTIAL(MODE, false, RangeMap)    \
  FB_INST_PARTIAL(MODE, false, RaggedMap)   \
  FB_INST_PARTIAL(MODE, false, CausalMap)   \
  FB_INST_PARTIAL(MODE, true, RangeMap)     \
  FB_INST_PARTIAL(MODE, false, SelectedMap) \
  FB_INST_PARTIAL(MODE, true, SelectedMap)  \
  FB_INST_PARTIAL(MODE, false, ResidualMap) \
  FB_INST_PARTIAL(MODE, true, ResidualMap)

FB_INST_MODE(ModeF64)
FB_INST_MODE(ModeF32)
FB_INST_MODE(ModeBF16)

// block-causal (prefill / commit) in F32 mode: float64 scores as attention_dense
template int launch_partial_simt<ModeMaskF32, false, false, CausalMap<float>>(const float*, const CausalMap<float>&, int64_t, int64_t, int64_t, int64_t, int, double, double*, double*, const MergeOut<ModeMaskF32>&, cudaStream_t, const int32_t*);

// lognorm-only passes for the sparse mask (scores in double for F64/F32 inputs,
// as sparse.py:117-118 widens before the product)
template int launch_partial_simt<ModeMaskF64, false, true, ConcatMap<double>>(const double*, const ConcatMap<double>&, int64_t, int64_t, int64_t, int64_t, int, double, double*, double*, const MergeOut<ModeMaskF64>&, cudaStream_t, const int32_t*);
template int launch_partial_simt<ModeMaskF32, false, true, ConcatMap<float>>(const float*, const ConcatMap<float>&, int64_t, int64_t, int64_t, int64_t, int, double, double*, double*, const MergeOut<ModeMaskF32>&, cudaStream_t, const int32_t*);
template int launch_partial_simt<ModeMaskBF16, false, true, ConcatMap<__nv_bfloat16>>(const __nv_bfloat16*, const ConcatMap<__nv_bfloat16>&, int64_t, int64_t, int64_t, int64_t, int, double, double*, double*, const MergeOut<ModeMaskBF16>&, cudaStream_t, const int32_t*);

// combine: (part out, part lse, accumulate, out, lse out)
template int launch_combine<double, double, double, double, double>(const CombineList&, int64_t, int64_t, double*, double*, int32_t*, cudaStream_t);
template int launch_combine<float, double, double, float, double>(const CombineList&, int64_t, int64_t, float*, double*, int32_t*, cudaStream_t);
template int launch_combine<float, float, float, float, float>(const CombineList&, int64_t, int64_t, float*, float*, int32_t*, cudaStream_t);
template int launch_combine<float, float, float, __nv_bfloat16, float>(const CombineList&, int64_t, int64_t, __nv_bfloat16*, float*, int32_t*, cudaStream_t);
template int launch_combine<double, double, double, float, double>(const CombineList&, int64_t, int64_t, float*, double*, int32_t*, cudaStream_t);

template int launch_fill_sentinel<double, double>(double*, double*, int64_t, int64_t, cudaStream_t);
template int launch_fill_sentinel<float, double>(float*, double*, int64_t, int64_t, cudaStream_t);
template int launch_fill_sentinel<float, float>(float*, float*, int64_t, int64_t, cudaStream_t);
template int launch_fill_sentinel<__nv_bfloat16, float>(__nv_bfloat16*, float*, int64_t, int64_t, cudaStream_t);

}  // namespace fb
