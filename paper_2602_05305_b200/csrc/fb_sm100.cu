// K1 -- block-external ("refresh") partial attention on sm_100a.
//
// Computes, per group g (a kv head of one sequence, its G query heads stacked
// into 128-row query tiles), the normalised online-softmax partial over keys
// [kb, ke) of the slab -- the reference's attention_partial over the committed
// context (attention.py:136-182, called at :202).  At C2 this is the HBM-bound
// kernel: the KV cache is streamed exactly once.
//
// Structure (persistent: one CTA per SM, stream-K over (item, key tile); 384
// threads):
//   warp 0      TMA producer: Q tile once per segment, then K/V 128-key tiles
//               into a STAGES-deep ring (128B-swizzled boxes of 64 columns);
//               on the gathered path warp 3 issues the V tiles.
//   warp 1      MMA issuer (one thread): S_j = Q K_j^T (SS, tcgen05.mma into
//               TMEM, double-buffered S), then O += P_{j-1} V_{j-1} with P
//               read straight from TMEM (TS form) -- QK^T of tile j overlaps
//               the softmax of tile j-1.
//   warp 2      TMEM allocator (512 columns: S0 | S1 | O0 | O1).
//   warps 4-11  two softmax warpgroups on alternate key tiles: thread t owns
//               query row t (TMEM lane t); reads S, keeps (max, sum) in
//               registers, writes P (bf16) back over S, rescales its O in
//               TMEM only when the running max grows by more than 2^8 (exact:
//               the same max is used for l and O); the segment epilogue merges
//               the two warpgroups' partials and writes the fp32 partial and
//               the natural-log lognorm (or a split partial for the merge).
// Key sources: contiguous slabs, ragged lengths, page tables (Paged), block-
// causal row limits (Causal) and mask-selected 16-key blocks (Gather, K7/K8).
// The CTA-pair (cta_group::2) variant lives in fb_sm100_pair.cuh.
#include "fb_kernels.cuh"
#include "fb_sm100_ptx.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

namespace fb {
namespace sm100 {

constexpr int BM = 128;       // query rows per tile (TMEM lanes)
constexpr int BN = 128;       // keys per tile
constexpr int THREADS = 384;  // 4 control warps + 2 softmax warpgroups
constexpr int BOX_COLS = 64;  // 128-byte swizzle span in bf16
constexpr uint32_t TMEM_COLS = 512;
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units: P stays <= 256

template <int D>
struct Cfg {
  static constexpr int STAGES = D == 128 ? 3 : 6;
  static constexpr int NBOX = D / BOX_COLS;
  static constexpr uint32_t BOX_BYTES = BM * BOX_COLS * 2;  // 16 KB (128 rows x 128 B)
  static constexpr uint32_t TILE_BYTES = NBOX * BOX_BYTES;  // one Q / K / V tile
  static constexpr uint32_t OFF_Q = 0;
  static constexpr uint32_t OFF_K = OFF_Q + TILE_BYTES;
  static constexpr uint32_t OFF_V = OFF_K + STAGES * TILE_BYTES;
  static constexpr uint32_t OFF_BAR = OFF_V + STAGES * TILE_BYTES;
  static constexpr uint32_t BAR_BYTES = 512;
  static constexpr uint32_t OFF_XCH = OFF_BAR + BAR_BYTES;    // [3][128] fp32 epilogue exchange
  static constexpr uint32_t SMEM = OFF_XCH + 3 * BM * 4 + 1024;  // + alignment slack
  static constexpr uint32_t COL_S0 = 0, COL_S1 = 128, COL_O0 = 256, COL_O1 = 256 + D;
  // cluster split-K: the CTA's normalised partial staged over the idle K/V ring
  // as 128B-swizzled fp32 boxes of 32 columns x 128 rows (row-per-thread
  // stores conflict free), the TMA store source
  static constexpr uint32_t OFF_STG = OFF_K;
  static constexpr uint32_t STG_BOX = BM * 128;  // 16 KB
  static_assert((D / 32) * STG_BOX <= 2 * STAGES * TILE_BYTES, "staging exceeds the ring");
};

struct Barriers {
  uint64_t q_full, q_empty;
  uint64_t k_full[6], k_empty[6], v_full[6], v_empty[6];
  uint64_t s_full[2], p_ready[2];
  uint64_t pv_done[2], o_full, o_empty;
  uint32_t tmem_base;
};

// Stream-K schedule: the flattened (item, key tile) space of T tiles is cut
// into `ctas` equal contiguous ranges, one per CTA (one CTA per SM), so every
// SM streams the same number of KV bytes whatever b*Hkv is.  A CTA's range
// covers one or more "segments" (the part of one item inside it).  Items
// have a uniform tile count (tpi) or, for ragged per-sequence context
// lengths, tile offsets `prefix[items+1]` in device memory (T = prefix[items]).
// Only a CTA's first and last segment can belong to an item that other CTAs
// share, so split partials need just two workspace slots per CTA.
struct Sched {
  long long T;             // total tiles (ragged: filled in-kernel from prefix)
  int tpi;                 // tiles per item (uniform)
  int m_tiles;             // 128-row query tiles per group
  int items;
  int ctas;
  const long long* prefix; // ragged item offsets, or nullptr
  const int* glist;        // group subset (head-gated refresh): item group -> slab, or nullptr
  int kv_keep;             // K/V tiles re-read by other query tiles of the group: keep in L2
  int rr;                  // pair kernel: round-robin whole items (block-causal), no stream-K
  int vprod;               // refresh kernel: warp 3 issues the V tiles (warp 0 Q and K)
  int o_bf16;              // final partial O rows stored as bf16 (FB_PARTIAL_BF16)
  int clus;                // cluster split-K: CTAs per item (one cluster each), 0 = stream-K
  int gbar;                // ... with the item's CTAs meeting at a counter in global memory
                           // instead of a cluster barrier (any co-resident CTAs, no GPC placement)
  int rot;                 // two-query-tile kernel: rotate each segment's key tiles (Seg::shift)
  int fin_whole;           // refresh kernel: items one CTA finishes apply the MergeFinal in its
                           // epilogue; the merge kernel then finishes split items only
  __device__ __forceinline__ void resolve() {
    if (prefix != nullptr) T = prefix[items];
  }
  __device__ __forceinline__ long long start(int c) const {
    if (clus > 0) {  // item-aligned: CTA c takes part c % clus of item c / clus
      const int it = c / clus, r = c % clus;
      return (long long)it * tpi + (long long)r * tpi / clus;
    }
    return (long long)c * T / ctas;
  }
  // largest c with start(c) <= x
  __device__ __forceinline__ int cta_of(long long x) const {
    return (int)(((x + 1) * ctas - 1) / T);
  }
  __device__ __forceinline__ long long item_begin(int i) const {
    return prefix ? prefix[i] : (long long)i * tpi;
  }
  __device__ __forceinline__ long long item_end(int i) const {
    return prefix ? prefix[i + 1] : (long long)(i + 1) * tpi;
  }
  // item holding tile t (ragged: last i with prefix[i] <= t, skipping empty items)
  __device__ __forceinline__ int item_of(long long t) const {
    if (prefix == nullptr) return (int)(t / tpi);
    int lo = 0, hi = items;  // prefix[lo] <= t < prefix[hi]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (prefix[mid] <= t) lo = mid; else hi = mid;
    }
    return lo;
  }
  // Item order is group major: item i = (group i / m_tiles, query tile
  // i % m_tiles).  (Query-tile-major order was measured: C5 refresh within
  // noise, block-causal prefill 12 % slower.)
  __device__ __forceinline__ int group_of(int i) const {
    const int gi = i / m_tiles;
    return glist != nullptr ? __ldg(glist + gi) : gi;
  }
  __device__ __forceinline__ int mtile_of(int i) const { return i % m_tiles; }
  // the item after `prev` holding tile t (segments of a CTA are consecutive
  // items: advance past empty ragged items instead of searching again)
  __device__ __forceinline__ int item_next(long long t, int prev) const {
    if (prefix == nullptr) return (int)(t / tpi);
    if (prev < 0) return item_of(t);
    int i = prev + 1;
    while (prefix[i + 1] <= t) ++i;
    return i;
  }
  // workspace slot of item i's segment inside CTA c
  __device__ __forceinline__ long long slot(int c, int i) const {
    return 2ll * c + (item_begin(i) <= start(c) ? 0 : 1);
  }
};

static_assert(sizeof(Barriers) <= 512, "barrier block overflows its smem slot");
static_assert(Cfg<128>::SMEM <= 232448, "K1 shared memory exceeds the 227 KB opt-in limit");

// In-kernel split merge (stream-K fix-up): the CTA holding an item's first
// tile finishes it last (it is that CTA's last segment), so it merges the
// other CTAs' partials of the item -- each written in that CTA's FIRST
// segment, long before -- instead of a separate merge kernel.  Ready flags
// live in a caller-owned buffer that is zero before the launch: a writer CTA
// sets its flag to 1 (release), the merging CTA waits for 1 (acquire) and
// sets it back to 0, so the buffer is zero again after every launch.  (The
// grid's %gridid is NOT a usable per-launch token: CUDA-graph replays of one
// node repeat it -- scripts/micro/gridid.cu.)
__device__ __forceinline__ void flag_signal(unsigned long long* f, unsigned long long v) {
  __threadfence();
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(f), "l"(v) : "memory");
}
__device__ __forceinline__ void flag_wait(const unsigned long long* f, unsigned long long v) {
  uint32_t polls = 0;
  while (true) {
    unsigned long long x;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(f) : "memory");
    if (x == v) break;
    if (++polls == (1u << 26)) __trap();  // a schedule bug must not hang the GPU
    __nanosleep(100);
  }
}

__device__ __forceinline__ void flag_wait_ge(const unsigned long long* f, unsigned long long v) {
  uint32_t polls = 0;
  while (true) {
    unsigned long long x;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(f) : "memory");
    if (x >= v) break;
    if (++polls == (1u << 26)) __trap();  // a schedule bug must not hang the GPU
    __nanosleep(64);
  }
}

// Gathered key source (sparse K7/K8, sparse.py:167-183): an item's first
// sel_tiles tiles are 8 mask-selected 16-key blocks each (read straight from
// the cache by block index: one 16-row TMA box per block; missing entries
// point past the slab end so TMA zero-fills them), followed by the current
// block's keys from the k_in / v_in tensors in 128-row tiles.
struct Gather {
  const int32_t* list;  // [groups, n_list] ascending block ids
  int n_list, n_ext, n_in, sel_tiles;
  // Atom layout (d = 128): a K / V tile is 16 atoms of 8 keys x [2 d-halves x
  // 128 B] (2 KB each), so a whole 16-key block -- both d-halves, two atoms --
  // is ONE 4 KB TMA box of a 5-D view {64 cols, 8 rows, 2 halves, atoms,
  // slabs} instead of two 64-column boxes (scripts/micro/tma_gather.cu: 5.07
  // vs 4.22 TB/s of pure gather streaming).  MMA descriptors: K-major K with
  // the d-half 1 KB apart and SBO 2 KB; MN-major V with LBO 1 KB, SBO 2 KB.
  int atoms;
};

// Paged KV cache (serving layout): a group's logical key row
// r lives in page table[g * max_pages + r / page_rows] at row r % page_rows of
// a shared page pool [num_pages, page_rows, d]; page_rows is a multiple of 128,
// so every 128-key tile sits inside one page (one TMA box per 64 columns).
struct Paged {
  const int32_t* table;  // [groups, max_pages] page ids, or nullptr (contiguous slabs)
  int max_pages, page_rows;
};

// DIAG (diagnostics only, fb_debug_set_k1_diag): 1 = softmax warps load S but skip
// the softmax math, 2 = they skip the TMEM load too (pure TMA + MMA pipeline).
// Block-causal rows (prefill / commit attention, simulator.py:297-354): query
// row r of a group sits at position p = r % n_q of its head and attends keys
// [0, n_prefix + min(n_q, (p / blk + 1) * blk)) -- every earlier block plus its
// own block.  blk == 0: off (every row attends the item's whole key range).
struct Causal {
  int n_q, blk, n_prefix;
  __device__ __forceinline__ int row_limit(int grow) const {
    const int p = grow % n_q;
    return n_prefix + min(n_q, (p / blk + 1) * blk);
  }
};

// POLY: every POLY-th pair of P values per thread takes 2^x on the FMA pipes
// (ptx::ex2_poly) instead of MUFU; 0 = MUFU only.
constexpr int K1_POLY = 0;  // measured: the extra FMA-pipe instructions cost more than MUFU

// Cluster split-K reduction.  The CLS CTAs of an item's cluster publish their
// staged normalised partials to global slots (coalesced 512 B rows), meet at
// the cluster barrier, and CTA `rank` merges rows [rank*128/CLS, ...) over all
// of them in rank order -- the log-space merge of combine_partials
// (attention.py:207-233) -- then applies the MergeFinal merge if any and
// writes the finished rows.  The 8 softmax warps each take 16/CLS rows, all
// at once: a row is spread over 2*CLS lanes of D/(2*CLS) columns each; every
// lane loads the row's CLS LSEs and its column slice of the CLS partials (all
// in flight), so the merge costs one L2 round trip per warp.  (DSMEM instead
// of L2 measured equal; one row per warp at a time was 2-4x slower.)
template <int CLS, int D>
__device__ __forceinline__ void cluster_reduce(int rank, const Sched& sc, int item, int w8, int lane, int q_rows,
                                               const unsigned char* stg_box, const CUtensorMap* tm_ws,
                                               float* __restrict__ ws_o,
                                               float* __restrict__ ws_l, float* __restrict__ o_out,
                                               float* __restrict__ lse_out, const MergeFinal& fin,
                                               unsigned long long* trace, unsigned long long* counters) {
  // diagnostics (trace != nullptr): globaltimer after publishing (slot 3) and after the barrier (slot 4)
  auto stamp = [&](int slot) {
    if (trace != nullptr && w8 == 0 && lane == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      trace[blockIdx.x * 8 + slot] = t;
    }
  };
  constexpr int NRW = 16 / CLS;      // rows per warp (rows_per = BM / CLS over 8 warps)
  constexpr int LPR = 32 / NRW;      // lanes per row
  constexpr int NV = (D / 4 + LPR - 1) / LPR;  // float4 chunks per lane: chunk v = columns 4 * (v * LPR + lsub)
  constexpr int ROWS_PER = BM / CLS;
  static_assert(NV >= 1 && NRW * LPR == 32 && (D / 4) % LPR == 0 || NV == 1, "cluster_reduce mapping");
  const int g = sc.group_of(item), mt = sc.mtile_of(item);
  const int rsub = lane / LPR, lsub = lane % LPR;
  const int row = rank * ROWS_PER + w8 + rsub * 8;  // this lane's row (tile-local)
  const bool ok = mt * BM + row < q_rows;
  const long long orow = (long long)g * q_rows + mt * BM + row;
  auto colv = [&](int v) { return 4 * (v * LPR + lsub); };  // coalesced: a row's lanes read adjacent 16 B
  const bool cok = colv(0) < D;  // (d = 64 on 16-CTA clusters: half the lanes idle)
  // the MergeFinal (o2, l2) rows are final before this launch: load them first
  float l2 = -INFINITY;
  float4 o2[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) o2[v] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (ok && fin.out != nullptr && fin.l2 != nullptr) {
    l2 = __ldg(fin.l2 + orow);
    if (l2 != -INFINITY && cok) {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        if (fin.o2_bf16) {
          const uint2 u = __ldg(reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(fin.o2) +
                                                               orow * D + colv(v)));
          o2[v] = make_float4(ptx::bf16_lo(u.x), ptx::bf16_hi(u.x), ptx::bf16_lo(u.y), ptx::bf16_hi(u.y));
        } else {
          o2[v] = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(fin.o2) + orow * D + colv(v)));
        }
      }
    }
  }
  // publish this CTA's partial: the staged swizzled boxes -> its global slot
  // by TMA (the LSEs went straight to the slot from the epilogue).  Measured
  // at C4 K8 10 %: 1.9 us from staged to published vs 2.2 with a coalesced
  // copy loop; reading the peers' staging through DSMEM instead took 3.4 us.
  ptx::fence_proxy_async_smem();
  asm volatile("bar.sync 5, 256;" ::: "memory");
  if (w8 == 0 && lane == 0) {
#pragma unroll
    for (int b = 0; b < D / 32; ++b)
      ptx::tma_store_3d(tm_ws, stg_box + b * (BM * 128), b * 32, 0, (int)blockIdx.x);
    ptx::bulk_commit();
    ptx::bulk_wait_all();
    ptx::fence_proxy_async_global();
  }
  stamp(3);
  if (sc.gbar) {
    // grid barrier of the item's CLS CTAs (all co-resident: one CTA per SM,
    // ctas <= SMs): arrive (release) and wait for CLS arrivals (acquire); the
    // last CTA to leave resets both counters, so every launch finds them zero
    unsigned long long* arrive = counters + 2 * item;
    if (w8 == 0 && lane == 0) {
      __threadfence();
      atomicAdd(arrive, 1ull);
      flag_wait_ge(arrive, (unsigned long long)CLS);
    }
    asm volatile("bar.sync 6, 256;" ::: "memory");
    __threadfence();
  } else {
    ptx::cluster_sync();  // release / acquire (cluster scope; invalidates L1): every CTA of the cluster published
  }
  stamp(4);
  const float* part_o = ws_o + (long long)item * CLS * BM * D;
  const float* part_l = ws_l + (long long)item * CLS * BM;
  float li[CLS];
  float4 x[CLS][NV];
#pragma unroll
  for (int i = 0; i < CLS; ++i) {
    li[i] = ok ? __ldcg(part_l + (long long)i * BM + row) : -INFINITY;
#pragma unroll
    for (int v = 0; v < NV; ++v)
      x[i][v] = (ok && cok) ? __ldcg(reinterpret_cast<const float4*>(part_o + ((long long)i * BM + row) * D + colv(v)))
                            : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (sc.gbar) {  // every read of the item's slots is issued and complete (values in registers)
    asm volatile("bar.sync 6, 256;" ::: "memory");
    if (w8 == 0 && lane == 0) {
      unsigned long long* arrive = counters + 2 * item;
      if (atomicAdd(arrive + 1, 1ull) == (unsigned long long)CLS - 1) {  // the last CTA to leave
        atomicExch(arrive, 0ull);
        atomicExch(arrive + 1, 0ull);
      }
    }
  }
  if (!ok) return;
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < CLS; ++i) mx = fmaxf(mx, li[i]);
  float w[CLS], z = 0.f;
#pragma unroll
  for (int i = 0; i < CLS; ++i) {
    w[i] = li[i] != -INFINITY ? __expf(li[i] - mx) : 0.f;
    z += w[i];
  }
  const float iz = z > 0.f ? 1.f / z : 0.f;
  float4 acc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int i = 0; i < CLS; ++i) {  // rank order
      acc[v].x += w[i] * x[i][v].x; acc[v].y += w[i] * x[i][v].y;
      acc[v].z += w[i] * x[i][v].z; acc[v].w += w[i] * x[i][v].w;
    }
    acc[v] = make_float4(acc[v].x * iz, acc[v].y * iz, acc[v].z * iz, acc[v].w * iz);
  }
  const float L = z > 0.f ? mx + logf(z) : -INFINITY;
  if (fin.out == nullptr || !fin.skip_partial) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (!cok) break;
      if (sc.o_bf16) {
        uint2 u;
        u.x = ptx::pack_bf16(acc[v].x, acc[v].y);
        u.y = ptx::pack_bf16(acc[v].z, acc[v].w);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(o_out) + orow * D + colv(v)) = u;
      } else {
        *reinterpret_cast<float4*>(o_out + orow * D + colv(v)) = acc[v];
      }
    }
    if (lsub == 0) lse_out[orow] = L;
  }
  if (fin.out != nullptr) {  // fused final merge with (o2, l2), as final_merge_row
    const float m = fmaxf(L, l2);
    const bool flive = m != -INFINITY;
    const float wp = (flive && L != -INFINITY) ? __expf(L - m) : 0.f;
    const float w2 = (flive && l2 != -INFINITY) ? __expf(l2 - m) : 0.f;
    const float fiz = flive ? 1.f / (wp + w2) : 0.f;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (!cok) break;
      const float4 f = make_float4((__fmul_rn(wp, acc[v].x) + __fmul_rn(w2, o2[v].x)) * fiz,
                                   (__fmul_rn(wp, acc[v].y) + __fmul_rn(w2, o2[v].y)) * fiz,
                                   (__fmul_rn(wp, acc[v].z) + __fmul_rn(w2, o2[v].z)) * fiz,
                                   (__fmul_rn(wp, acc[v].w) + __fmul_rn(w2, o2[v].w)) * fiz);
      if (fin.out_bf16) {
        uint2 u;
        u.x = ptx::pack_bf16(f.x, f.y);
        u.y = ptx::pack_bf16(f.z, f.w);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(fin.out) + orow * D + colv(v)) = u;
      } else {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(fin.out) + orow * D + colv(v)) = f;
      }
    }
    if (!flive && lsub == 0 && fin.empty_rows) atomicAdd(fin.empty_rows, 1);
  }
}

// CL: cluster split-K variant (Sched::clus > 0); AT: atom-layout gather
// (Gather::atoms).  Compile-time, so the common kernels stay lean: the extra
// code in one kernel cost the gathered K7 residual pass 50 % through
// instruction-cache misses (ncu: no-instruction stalls 0.43 -> 2.26 per issue).
template <int D, bool GATHER, int DIAG = 0, int POLY = K1_POLY, bool CL = false, bool AT = false>
__global__ void __launch_bounds__(THREADS, 1)
refresh_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
               const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_ki,
               const __grid_constant__ CUtensorMap tm_vi, Gather ga, Paged pg, Causal cz, Sched sc, int q_rows, int key_begin,
               int key_end, const int* __restrict__ key_len, float scale_log2, float* __restrict__ o_out,
               float* __restrict__ lse_out, float* __restrict__ ws_o,
               float* __restrict__ ws_l, unsigned long long* __restrict__ trace,
               unsigned long long* __restrict__ flags, MergeFinal fin,
               const __grid_constant__ CUtensorMap tm_ws) {
  using C = Cfg<D>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Barriers* bar = reinterpret_cast<Barriers*>(smem + C::OFF_BAR);
  float* xch = reinterpret_cast<float*>(smem + C::OFF_XCH);  // [2][128] epilogue exchange

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  sc.resolve();
  const long long t_begin = sc.start(blockIdx.x);
  const long long t_end = sc.start(blockIdx.x + 1);
  // diagnostics (FB_REFRESH_TRACE): globaltimer at start / per-segment stream end / merge end
  auto stamp = [&](int slot) {
    if (trace != nullptr) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      trace[blockIdx.x * 8 + slot] = t;
    }
  };
  if (threadIdx.x == 0) stamp(0);

  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
    ptx::mbar_init(&bar->q_full, 1);
    ptx::mbar_init(&bar->q_empty, 1);
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&bar->k_full[s], 1);
      ptx::mbar_init(&bar->k_empty[s], 1);
      ptx::mbar_init(&bar->v_full[s], 1);
      ptx::mbar_init(&bar->v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&bar->s_full[b], 1);
      ptx::mbar_init(&bar->p_ready[b], 128);
      ptx::mbar_init(&bar->pv_done[b], 1);
    }
    ptx::mbar_init(&bar->o_full, 1);
    ptx::mbar_init(&bar->o_empty, 256);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(&bar->tmem_base, TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = bar->tmem_base;
  ptx::pdl_wait();               // inputs of this launch are final from here on
  ptx::pdl_launch_dependents();  // let the next kernel's prologue start
  // registers: control warpgroup 72/thread, softmax warpgroups 216 (64,512 of 65,536; at 56 / 224
  // the gathered producer spilled and K7 streamed ~25 % slower)
  if (warp < 4) {
  ptx::setmaxnreg_dec<72>();
  if (warp == 0 || (warp == 3 && sc.vprod)) {
    // ------------------------------------------------------------ TMA producer
    // warp 0 issues Q and K; V comes from warp 3 when sc.vprod (two issuing
    // threads: a V slot wait never delays the next K tile's issue, and the
    // gathered path's 16 small boxes per K / V tile go out in parallel)
    if (lane == 0) {
      const bool do_k = warp == 0, do_v = warp == 3 || !sc.vprod;
      const uint64_t keep = ptx::policy_evict_last();
      // K/V: streamed once (evict first), except block-causal prefill where
      // every later query tile of the group re-reads them (keep in L2)
      const uint64_t stream = (cz.blk > 0 || sc.kv_keep) ? ptx::policy_evict_last() : ptx::policy_evict_first();
      int j = 0, seg = 0, item = -1;
      for (long long t = t_begin; t < t_end; ++seg) {
        item = sc.item_next(t, item);
        const long long ib = sc.item_begin(item);
        const long long seg_end = min(t_end, sc.item_end(item));
        const int g = sc.group_of(item), mt = sc.mtile_of(item);
        if (do_k) {
          if (seg > 0) ptx::mbar_wait(&bar->q_empty, (seg - 1) & 1);
          ptx::mbar_expect_tx(&bar->q_full, C::TILE_BYTES);
          for (int b = 0; b < C::NBOX; ++b)
            ptx::tma_load_3d(smem + C::OFF_Q + b * C::BOX_BYTES, &tm_q, &bar->q_full, b * BOX_COLS,
                             mt * BM, g, keep);
        }
        for (; t < seg_end; ++t, ++j) {
          const int s = j % C::STAGES;
          const uint32_t ph = (j / C::STAGES) & 1;
          const int lt = (int)(t - ib);
          if constexpr (!GATHER) {
            int row = key_begin + lt * BN;
            int slab = g;
            if (pg.table != nullptr) {  // paged: the tile's page, row inside it
              slab = __ldg(pg.table + (long long)g * pg.max_pages + row / pg.page_rows);
              row %= pg.page_rows;
            }
            if (do_k) {
              ptx::mbar_wait(&bar->k_empty[s], ph ^ 1);
              ptx::mbar_expect_tx(&bar->k_full[s], C::TILE_BYTES);
              for (int b = 0; b < C::NBOX; ++b)
                ptx::tma_load_3d(smem + C::OFF_K + s * C::TILE_BYTES + b * C::BOX_BYTES, &tm_k,
                                 &bar->k_full[s], b * BOX_COLS, row, slab, stream);
            }
            if (do_v) {
              ptx::mbar_wait(&bar->v_empty[s], ph ^ 1);
              ptx::mbar_expect_tx(&bar->v_full[s], C::TILE_BYTES);
              for (int b = 0; b < C::NBOX; ++b)
                ptx::tma_load_3d(smem + C::OFF_V + s * C::TILE_BYTES + b * C::BOX_BYTES, &tm_v,
                                 &bar->v_full[s], b * BOX_COLS, row, slab, stream);
            }
          } else if (lt < ga.sel_tiles) {
            int rows[8], slabs[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int e = lt * 8 + i;
              rows[i] = e < ga.n_list ? __ldg(ga.list + (long long)g * ga.n_list + e) * 16 : ga.n_ext;
              slabs[i] = g;
              if (pg.table != nullptr) {  // paged cache: block -> (page, row); none -> past a page
                if (e < ga.n_list) {
                  slabs[i] = __ldg(pg.table + (long long)g * pg.max_pages + rows[i] / pg.page_rows);
                  rows[i] %= pg.page_rows;
                } else {
                  slabs[i] = 0;
                  rows[i] = pg.page_rows;
                }
              }
            }
            if (do_k) {
              ptx::mbar_wait(&bar->k_empty[s], ph ^ 1);
              ptx::mbar_expect_tx(&bar->k_full[s], C::TILE_BYTES);
              if constexpr (AT) {
#pragma unroll
                for (int i = 0; i < 8; ++i)
                  ptx::tma_load_5d(smem + C::OFF_K + s * C::TILE_BYTES + i * 4096, &tm_k, &bar->k_full[s], 0, 0,
                                   0, rows[i] / 8, slabs[i], stream);
              } else {
                for (int b = 0; b < C::NBOX; ++b)
#pragma unroll
                  for (int i = 0; i < 8; ++i)
                    ptx::tma_load_3d(smem + C::OFF_K + s * C::TILE_BYTES + b * C::BOX_BYTES + i * 2048,
                                     &tm_k, &bar->k_full[s], b * BOX_COLS, rows[i], slabs[i], stream);
              }
            }
            if (do_v) {
              ptx::mbar_wait(&bar->v_empty[s], ph ^ 1);
              ptx::mbar_expect_tx(&bar->v_full[s], C::TILE_BYTES);
              if constexpr (AT) {
#pragma unroll
                for (int i = 0; i < 8; ++i)
                  ptx::tma_load_5d(smem + C::OFF_V + s * C::TILE_BYTES + i * 4096, &tm_v, &bar->v_full[s], 0, 0,
                                   0, rows[i] / 8, slabs[i], stream);
              } else {
                for (int b = 0; b < C::NBOX; ++b)
#pragma unroll
                  for (int i = 0; i < 8; ++i)
                    ptx::tma_load_3d(smem + C::OFF_V + s * C::TILE_BYTES + b * C::BOX_BYTES + i * 2048,
                                     &tm_v, &bar->v_full[s], b * BOX_COLS, rows[i], slabs[i], stream);
              }
            }
          } else {
            const int row = (lt - ga.sel_tiles) * BN;
            if (do_k) {
              ptx::mbar_wait(&bar->k_empty[s], ph ^ 1);
              ptx::mbar_expect_tx(&bar->k_full[s], C::TILE_BYTES);
              if constexpr (AT)
                ptx::tma_load_5d(smem + C::OFF_K + s * C::TILE_BYTES, &tm_ki, &bar->k_full[s], 0, 0, 0, row / 8, g,
                                 stream);
              else
                for (int b = 0; b < C::NBOX; ++b)
                  ptx::tma_load_3d(smem + C::OFF_K + s * C::TILE_BYTES + b * C::BOX_BYTES, &tm_ki,
                                   &bar->k_full[s], b * BOX_COLS, row, g, stream);
            }
            if (do_v) {
              ptx::mbar_wait(&bar->v_empty[s], ph ^ 1);
              ptx::mbar_expect_tx(&bar->v_full[s], C::TILE_BYTES);
              if constexpr (AT)
                ptx::tma_load_5d(smem + C::OFF_V + s * C::TILE_BYTES, &tm_vi, &bar->v_full[s], 0, 0, 0, row / 8, g,
                                 stream);
              else
                for (int b = 0; b < C::NBOX; ++b)
                  ptx::tma_load_3d(smem + C::OFF_V + s * C::TILE_BYTES + b * C::BOX_BYTES, &tm_vi,
                                   &bar->v_full[s], b * BOX_COLS, row, g, stream);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // Tile j goes to softmax warpgroup w = j & 1: S_j -> TMEM S[w], O[w] += P_j V_j.
    if (lane == 0) {
      constexpr uint32_t IDESC_S = ptx::idesc_bf16_f32(BM, BN, false);
      constexpr uint32_t IDESC_O = ptx::idesc_bf16_f32(BM, D, true);
      const uint32_t q_base = ptx::smem_u32(smem + C::OFF_Q);
      int jg = 0, seg = 0, item = -1;
      for (long long t0 = t_begin; t0 < t_end; ++seg) {
        item = sc.item_next(t0, item);
        const int n = (int)(min(t_end, sc.item_end(item)) - t0);
        // ragged contexts: V rows past the sequence end are zeroed in smem before
        // P V (masked P is 0, but 0 * NaN from uninitialised cache rows is not)
        const int v_valid_last = key_len ? min(key_len[sc.group_of(item)], key_end) - key_begin -
                                               (int)(t0 + n - 1 - sc.item_begin(item)) * BN
                                         : BN;
        ptx::mbar_wait(&bar->q_full, seg & 1);
        ptx::tc_fence_after();
        for (int t = 0; t <= n; ++t) {
          if (t < n) {
            const int j = jg + t;
            const int s = j % C::STAGES;
            ptx::mbar_wait(&bar->k_full[s], (j / C::STAGES) & 1);
            ptx::tc_fence_after();
            const uint32_t k_base = ptx::smem_u32(smem + C::OFF_K + s * C::TILE_BYTES);
            const uint32_t d_s = tmem + ((j & 1) ? C::COL_S1 : C::COL_S0);
            constexpr bool at = GATHER && AT;
            const uint32_t k_half = at ? 1024u : C::BOX_BYTES, k_sbo = at ? 2048u : 1024u;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              // K-major SW128: a 16-element K step is +32 B inside a 64-column box
              const uint32_t off = (kk / 4) * C::BOX_BYTES + (kk % 4) * 32;
              const uint32_t koff = (kk / 4) * k_half + (kk % 4) * 32;
              ptx::mma_ss(d_s, ptx::sdesc_sw128(q_base + off, 16, 1024),
                          ptx::sdesc_sw128(k_base + koff, 16, k_sbo), IDESC_S, kk > 0);
            }
            ptx::tc_commit(&bar->k_empty[s]);
            ptx::tc_commit(&bar->s_full[j & 1]);
            if (t == n - 1) ptx::tc_commit(&bar->q_empty);  // Q no longer read
          }
          if (t > 0) {
            const int jj = jg + t - 1;
            const int s = jj % C::STAGES;
            ptx::mbar_wait(&bar->p_ready[jj & 1], (jj >> 1) & 1);
            ptx::mbar_wait(&bar->v_full[s], (jj / C::STAGES) & 1);
            if (t == 1 && seg > 0) ptx::mbar_wait(&bar->o_empty, (seg - 1) & 1);  // O drained
            if (t == n && v_valid_last < BN) {
              unsigned char* vt = smem + C::OFF_V + s * C::TILE_BYTES;
              for (int b = 0; b < C::NBOX; ++b)
                for (int off = max(v_valid_last, 0) * 128; off < BN * 128; off += 16)
                  *reinterpret_cast<uint4*>(vt + b * C::BOX_BYTES + off) = make_uint4(0, 0, 0, 0);
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            }
            ptx::tc_fence_after();
            const uint32_t v_base = ptx::smem_u32(smem + C::OFF_V + s * C::TILE_BYTES);
            const uint32_t p_tmem = tmem + ((jj & 1) ? C::COL_S1 : C::COL_S0);
            const uint32_t o_tmem = tmem + ((jj & 1) ? C::COL_O1 : C::COL_O0);
            if constexpr (DIAG != 3) {  // DIAG 3 (diagnostics): no P V MMA, S = Q K^T only
              constexpr bool at = GATHER && AT;
#pragma unroll
              for (int kk = 0; kk < BN / 16; ++kk) {
                // MN-major SW128 V: 16 keys = 16 rows of 128 B; d halves LBO apart
                // (the first two tiles of a segment start their warpgroup's O afresh);
                // atom layout: 16 keys = two 2 KB atoms, d halves 1 KB apart
                ptx::mma_ts(o_tmem, p_tmem + kk * 8,
                            at ? ptx::sdesc_sw128(v_base + kk * 4096, 1024, 2048)
                               : ptx::sdesc_sw128(v_base + kk * 2048, C::BOX_BYTES, 1024),
                            IDESC_O, (t > 2 || kk > 0) ? 1u : 0u);
              }
            }
            ptx::tc_commit(&bar->v_empty[s]);
            ptx::tc_commit(&bar->pv_done[jj & 1]);
            if (t == n) ptx::tc_commit(&bar->o_full);
          }
        }
        jg += n;
        t0 += n;
      }
    }
  }
  if constexpr (CL) {  // the cluster reduction's barrier (softmax warps do the work)
    if (!sc.gbar) ptx::cluster_sync();
  }
  } else {
    ptx::setmaxnreg_inc<216>();
    // ------------------------------------------------------------ softmax
    // Two warpgroups take alternate key tiles, each with its own running
    // (max, sum) and O accumulator, so one's softmax overlaps the other's.
    const int wg = (warp - 4) >> 2;                // 0: warps 4-7, 1: warps 8-11
    const int wq = warp & 3;                       // TMEM lane quarter
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const int row = wq * 32 + lane;                // row inside the 128-row tile
    const uint32_t s_col = wg ? C::COL_S1 : C::COL_S0;
    const uint32_t o_col = wg ? C::COL_O1 : C::COL_O0;
    uint32_t r[32];
    float s[BN];
    int jg = 0, seg = 0, item = -1;
    for (long long t0 = t_begin; t0 < t_end; ++seg) {
      item = sc.item_next(t0, item);
      const long long ib = sc.item_begin(item);
      const int lt0 = (int)(t0 - ib);
      const int n = (int)(min(t_end, sc.item_end(item)) - t0);
      const int kb = key_begin + lt0 * BN;
      int ke = min(kb + n * BN, key_len ? min(key_len[sc.group_of(item)], key_end) : key_end);
      if (cz.blk > 0) ke = min(ke, cz.row_limit(sc.mtile_of(item) * BM + row));  // this row's end
      float m_used = -INFINITY;  // running max, log2-scaled
      float l = 0.f;
      int last_rows = 16;  // valid rows of the list's last block (gather mode)
      if constexpr (GATHER) {
        if (ga.n_list > 0) {
          const int last = __ldg(ga.list + (long long)sc.group_of(item) * ga.n_list + ga.n_list - 1);
          last_rows = min(16, ga.n_ext - last * 16);
        }
      }
      for (int t = ((jg & 1) == wg) ? 0 : 1; t < n; t += 2) {
        const int j = jg + t;
        ptx::mbar_wait(&bar->s_full[wg], (j >> 1) & 1);
        ptx::tc_fence_after();
        if constexpr (DIAG > 0) {
          if constexpr (DIAG == 1) {
#pragma unroll
            for (int c = 0; c < BN / 32; ++c)
              ptx::tmem_ld32(tmem + lane_off + s_col + c * 32, reinterpret_cast<uint32_t*>(s) + c * 32);
            ptx::tmem_wait_ld();
            if (s[0] == 12345.f) l += 1.f;  // keep the load live
          }
          m_used = 0.f;
          l += 1.f;
          ptx::tc_fence_before();
          ptx::mbar_arrive(&bar->p_ready[wg]);
          continue;
        }
#pragma unroll
        for (int c = 0; c < BN / 32; ++c)  // all four loads in flight, one wait
          ptx::tmem_ld32(tmem + lane_off + s_col + c * 32, reinterpret_cast<uint32_t*>(s) + c * 32);
        ptx::tmem_wait_ld();
        if constexpr (!GATHER) {
          const int valid = ke - (kb + t * BN);
          if (valid < BN) {
#pragma unroll
            for (int i = 0; i < BN; ++i)
              if (i >= valid) s[i] = -INFINITY;
          }
        } else {
          const int lt = lt0 + t;
          if (lt < ga.sel_tiles) {
            // 16 rows per listed block; entries past the list are empty; only the
            // last entry of the ascending list can be the slab's clipped tail block
            const int e0 = lt * 8;
            if (e0 + 8 >= ga.n_list) {  // this tile holds the list's end
              int vr[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int e = e0 + i;
                vr[i] = e < ga.n_list - 1 ? 16 : (e == ga.n_list - 1 ? last_rows : 0);
              }
#pragma unroll
              for (int i = 0; i < BN; ++i)
                if ((i & 15) >= vr[i >> 4]) s[i] = -INFINITY;
            }
          } else {
            const int valid = ga.n_in - (lt - ga.sel_tiles) * BN;
            if (valid < BN) {
#pragma unroll
              for (int i = 0; i < BN; ++i)
                if (i >= valid) s[i] = -INFINITY;
            }
          }
        }
        // P = 2^(s*scale - m) into TMEM over S (bf16 pairs); returns the row sum.
        // x = s * scale - m and the sum on packed pairs (FFMA2 / FADD2).
        auto exp_tile = [&](float neg) -> float {
          const uint64_t sc2 = ptx::f2_pack(scale_log2, scale_log2), ng2 = ptx::f2_pack(neg, neg);
          uint64_t ls4[4] = {0, 0, 0, 0};  // 4 independent pair chains (+0.0f bits)
#pragma unroll
          for (int c = 0; c < BN / 64; ++c) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const uint64_t x2 = ptx::f2_fma(ptx::f2_pack(s[c * 64 + 2 * i], s[c * 64 + 2 * i + 1]), sc2, ng2);
              float x0, x1;
              ptx::f2_unpack(x2, x0, x1);
              float p0, p1;
              if (POLY > 0 && (i % (POLY > 0 ? POLY : 1)) == (POLY > 0 ? POLY : 1) - 1) {
                ptx::ex2_poly2(x2, p0, p1);
              } else {
                p0 = ptx::ex2(x0);
                p1 = ptx::ex2(x1);
              }
              ls4[i & 3] = ptx::f2_add(ls4[i & 3], ptx::f2_pack(p0, p1));
              r[i] = ptx::pack_bf16(p0, p1);
            }
            ptx::tmem_st32(tmem + lane_off + s_col + c * 32, r);
          }
          const uint64_t a2 = ptx::f2_add(ptx::f2_add(ls4[0], ls4[1]), ptx::f2_add(ls4[2], ls4[3]));
          float a0, a1;
          ptx::f2_unpack(a2, a0, a1);
          return a0 + a1;
        };
        // Fast path: exponentiate against the running max without a max pass.
        // The max is exact in the result either way (l and O share it); it only
        // has to keep P finite.  A row whose scores rose more than 2^32 / 128
        // (log2: ~25) past it -- or inf / NaN -- shows in the tile sum, and
        // the warp redoes the tile through the max pass below.
        float lt = 0.f;
        bool full = __any_sync(0xffffffffu, m_used == -INFINITY);
        if (!full) {
          lt = exp_tile(-m_used);
          full = __any_sync(0xffffffffu, !(lt <= 4294967296.f));
        }
        if (full) {
          // row max as 8 independent chains
          float mx8[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) mx8[k] = s[k];
#pragma unroll
          for (int i = 8; i < BN; ++i) mx8[i & 7] = fmaxf(mx8[i & 7], s[i]);
          const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                 fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
          const float m_new = fmaxf(m_used, mx * scale_log2);
          const bool need = m_new > m_used + RESCALE_THRESHOLD;
          if (__any_sync(0xffffffffu, need)) {
            // a row with no key yet on both sides (m_used = m_new = -inf) keeps l = 0:
            // ex2(-inf - -inf) would be NaN
            const float alpha = m_new == -INFINITY ? 1.f : ptx::ex2(m_used - m_new);
            if (t >= 2) {
              // O[wg] holds this segment's P V so far: wait for its last PV (tile j-2)
              ptx::mbar_wait(&bar->pv_done[wg], ((j - 2) >> 1) & 1);
              ptx::tc_fence_after();
#pragma unroll 1
              for (int c = 0; c < D / 32; ++c) {
                const uint32_t a = tmem + lane_off + o_col + c * 32;
                ptx::tmem_ld32(a, r);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
                ptx::tmem_st32(a, r);
              }
              ptx::tmem_wait_st();
            }
            l *= alpha;
            m_used = m_new;
          }
          // a row with no key yet (block-causal segment past its end) keeps p = 0
          lt = exp_tile(m_used == -INFINITY ? 0.f : -m_used);
        }
        l += lt;
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&bar->p_ready[wg]);
      }
      jg += n;
      t0 += n;
      if (row == 0 && wg == 0) stamp(1 + 2 * (seg & 1));

      // ---------------------------------------------------------- segment epilogue
      // Merge the two warpgroups' partials (exact log-space merge): WG0 posts
      // (m0, l0), WG1 forms the weights and posts WG0's; each WG then writes
      // half of the output columns from both O accumulators.
      const bool whole = ib >= t_begin && sc.item_end(item) <= t_end;  // item not shared
      const int g = sc.group_of(item), mt = sc.mtile_of(item);
      const int grow = mt * BM + row;
      const bool live = grow < q_rows;
      const long long orow = (long long)g * q_rows + grow;
      float c_own, c_oth, lse = 0.f;
      if (wg == 0) {
        xch[row] = m_used;
        xch[BM + row] = l;
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (wg == 1) {
        const float m0 = xch[row], l0 = xch[BM + row];
        const float m = fmaxf(m0, m_used);
        const float a0 = l0 > 0.f ? ptx::ex2(m0 - m) : 0.f;
        const float a1 = l > 0.f ? ptx::ex2(m_used - m) : 0.f;
        const float z = a0 * l0 + a1 * l;
        const float iz = z > 0.f ? 1.f / z : 0.f;  // z == 0: no key in this segment (empty partial)
        c_own = a1 * iz;
        c_oth = a0 * iz;
        lse = z > 0.f ? (m + log2f(z)) * 0.69314718055994530942f : -INFINITY;
        xch[row] = c_oth;
        xch[BM + row] = c_own;
        xch[2 * BM + row] = lse;
      }
      asm volatile("bar.sync 2, 256;" ::: "memory");
      if (wg == 0) {
        c_own = xch[row];
        c_oth = xch[BM + row];
        lse = xch[2 * BM + row];
      }
      // coefficient of O0 and O1 (a warpgroup without tiles in this segment has
      // weight 0 and a stale accumulator, so it is selected out, not multiplied)
      float c0 = wg == 0 ? c_own : c_oth;
      float c1 = wg == 0 ? c_oth : c_own;
      // in-kernel split merge: the item's first CTA (this segment is its last)
      // merges the partials of CTAs cb+1..ce, written in their first segments
      const bool owner = !CL && flags != nullptr && !whole && ib >= t_begin;
      const int cb = blockIdx.x + 1, ce = owner ? sc.cta_of(sc.item_end(item) - 1) : 0;
      float* dst;
      float* stg = reinterpret_cast<float*>(smem + C::OFF_STG);  // cluster split-K staging
      if constexpr (CL) {
        dst = stg;  // (swizzled boxes below)
        if (wg == 1) ws_l[(long long)blockIdx.x * BM + row] = lse;  // this CTA's LSE slot (coalesced)
      } else if (whole || owner) {
        dst = live ? o_out + orow * D : nullptr;
      } else {
        const long long slot = sc.slot(blockIdx.x, item) * BM + row;
        dst = ws_o + slot * D;
        if (wg == 1) ws_l[slot] = lse;
      }
      float mmax = lse, inv_z = 1.f;
      if (owner) {
        if (wg == 0 && row == 0) {
          for (int cc = cb; cc <= ce; ++cc) {
            flag_wait(flags + cc, 1ull);
            flags[cc] = 0ull;  // consumed: zero again for the next launch
          }
        }
        asm volatile("bar.sync 3, 256;" ::: "memory");
        // merge weights over this CTA's partial and the others' (same
        // arithmetic in both warpgroups, so both get identical weights)
        for (int cc = cb; cc <= ce; ++cc)
          mmax = fmaxf(mmax, __ldcg(ws_l + sc.slot(cc, item) * BM + row));
        float z = lse == -INFINITY ? 0.f : __expf(lse - mmax);
        const float w_own = z;
        for (int cc = cb; cc <= ce; ++cc) {
          const float lk = __ldcg(ws_l + sc.slot(cc, item) * BM + row);
          z += lk == -INFINITY ? 0.f : __expf(lk - mmax);
        }
        inv_z = 1.f / z;
        c0 *= w_own * inv_z;
        c1 *= w_own * inv_z;
        lse = mmax + logf(z);
      }
      // whole item with a fused final merge (fin_whole): this row's partial
      // (v below, lse) is merged with (o2, l2) here and written as the output,
      // the same arithmetic as final_merge_row
      const bool fw = !CL && sc.fin_whole && whole && live;
      float f_wp = 0.f, f_w2 = 0.f, f_iz = 0.f;
      if (fw) {
        const float l2 = fin.l2 ? fin.l2[orow] : -INFINITY;
        const float m = fmaxf(lse, l2);
        const bool flive = m != -INFINITY;
        f_wp = (flive && lse != -INFINITY) ? __expf(lse - m) : 0.f;
        f_w2 = (flive && l2 != -INFINITY) ? __expf(l2 - m) : 0.f;
        f_iz = flive ? 1.f / (f_wp + f_w2) : 0.f;
        if (!flive && wg == 1 && fin.empty_rows) atomicAdd(fin.empty_rows, 1);
      }
      ptx::mbar_wait(&bar->o_full, seg & 1);
      ptx::tc_fence_after();
      if (row == 0 && wg == 0 && seg == 0) stamp(5);
      uint32_t r1[32];
#pragma unroll 1
      for (int c = wg * (D / 64); c < (wg + 1) * (D / 64); ++c) {
        ptx::tmem_ld32(tmem + lane_off + C::COL_O0 + c * 32, r);
        ptx::tmem_ld32(tmem + lane_off + C::COL_O1 + c * 32, r1);
        ptx::tmem_wait_ld();
        if (dst != nullptr) {
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i)
            v[i] = (c0 != 0.f ? c0 * __uint_as_float(r[i]) : 0.f) +
                   (c1 != 0.f ? c1 * __uint_as_float(r1[i]) : 0.f);
          if (owner) {
            for (int cc = cb; cc <= ce; ++cc) {
              const long long sl = sc.slot(cc, item) * BM + row;
              const float lk = __ldcg(ws_l + sl);
              const float w = lk == -INFINITY ? 0.f : __expf(lk - mmax) * inv_z;
              const float4* src = reinterpret_cast<const float4*>(ws_o + sl * D + c * 32);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const float4 x = __ldcg(src + i);
                v[4 * i] += w * x.x; v[4 * i + 1] += w * x.y; v[4 * i + 2] += w * x.z; v[4 * i + 3] += w * x.w;
              }
            }
          }
          if constexpr (CL) {  // box c, row `row`, 16-byte chunk j at (j ^ (row % 8))
            unsigned char* brow = smem + C::OFF_STG + c * C::STG_BOX + row * 128;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<float4*>(brow + ((j ^ (row & 7)) << 4)) =
                  make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          } else if (fw) {
            if (!fin.skip_partial) ptx::st_row32(dst + c * 32, v);
            float o2[32];
            if (f_w2 != 0.f) {
              if (fin.o2_bf16) {
                const uint4* src = reinterpret_cast<const uint4*>(
                    reinterpret_cast<const __nv_bfloat16*>(fin.o2) + orow * D + c * 32);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const uint4 u = __ldg(src + j);
                  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                  for (int k = 0; k < 4; ++k) {
                    o2[8 * j + 2 * k] = ptx::bf16_lo(w[k]);
                    o2[8 * j + 2 * k + 1] = ptx::bf16_hi(w[k]);
                  }
                }
              } else {
                const float4* src = reinterpret_cast<const float4*>(
                    reinterpret_cast<const float*>(fin.o2) + orow * D + c * 32);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  const float4 x = __ldg(src + j);
                  o2[4 * j] = x.x; o2[4 * j + 1] = x.y; o2[4 * j + 2] = x.z; o2[4 * j + 3] = x.w;
                }
              }
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i) o2[i] = 0.f;
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = (__fmul_rn(f_wp, v[i]) + __fmul_rn(f_w2, o2[i])) * f_iz;
            if (fin.out_bf16)
              ptx::st_row32_bf16(reinterpret_cast<__nv_bfloat16*>(fin.out) + orow * D + c * 32, v);
            else
              ptx::st_row32(reinterpret_cast<float*>(fin.out) + orow * D + c * 32, v);
          } else if (sc.o_bf16 && (whole || owner)) {  // final row into a bf16 partial
            ptx::st_row32_bf16(reinterpret_cast<__nv_bfloat16*>(o_out) + orow * D + c * 32, v);
          } else {
            ptx::st_row32(dst + c * 32, v);
          }
        }
      }
      if (row == 0 && wg == 0 && seg == 0) stamp(6);
      ptx::tc_fence_before();
      ptx::mbar_arrive(&bar->o_empty);  // MMA may overwrite O for the next segment
      if (!CL && flags != nullptr && !whole && !owner) {
        // this CTA's share of an item begun by an earlier CTA: publish it
        asm volatile("bar.sync 3, 256;" ::: "memory");
        if (wg == 0 && row == 0) flag_signal(flags + blockIdx.x, 1ull);
      }
      if (!CL && (whole || owner) && live && wg == 1 && !(fw && fin.skip_partial)) lse_out[orow] = lse;
      if (row == 0 && wg == 0) stamp(2 + 2 * (seg & 1));
    }
    if constexpr (CL) {
      // Cluster split-K reduction (see cluster_reduce); the CTA's rows are
      // staged in shared memory by the epilogue above
      const int item = blockIdx.x / sc.clus;
      const int rk = sc.gbar ? (int)(blockIdx.x % sc.clus) : (int)ptx::cluster_ctarank();
      unsigned long long* counters = flags + 512;  // grid-barrier counters (two per item)
      const unsigned char* stgb = smem + C::OFF_STG;
      switch (sc.clus) {
        case 2: cluster_reduce<2, D>(rk, sc, item, warp - 4, lane, q_rows, stgb, &tm_ws, ws_o, ws_l, o_out, lse_out, fin, trace, counters); break;
        case 4: cluster_reduce<4, D>(rk, sc, item, warp - 4, lane, q_rows, stgb, &tm_ws, ws_o, ws_l, o_out, lse_out, fin, trace, counters); break;
        case 8: cluster_reduce<8, D>(rk, sc, item, warp - 4, lane, q_rows, stgb, &tm_ws, ws_o, ws_l, o_out, lse_out, fin, trace, counters); break;
        default: cluster_reduce<16, D>(rk, sc, item, warp - 4, lane, q_rows, stgb, &tm_ws, ws_o, ws_l, o_out, lse_out, fin, trace, counters); break;
      }
      if (row == 0 && wg == 0) stamp(1);  // reduction done
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) stamp(7);
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, TMEM_COLS);
  }
}

// A row's split partials, merged in segment order: max and sum of the
// weights exp(L_k - max) and the weighted sum of the 4 columns at lane*4.
// Lane u resolves segment k0 + u's workspace row (two 64-bit divisions) once
// per 32-segment chunk and broadcasts it by shuffle; every lane then keeps 16
// segments' loads in flight.  (Resolving every segment in every lane cost
// ~100 dependent 64-bit divisions per lane: the C3 b=1 merge took 16 us.)
// Same arithmetic and order as a plain per-segment loop.
__device__ __forceinline__ long long seg_row(const Sched& sc, int item, int row, int bm, int c) {
  const long long s0 = sc.start(c), s1 = sc.start(c + 1);
  if (s1 <= s0) return -1;  // CTAs with empty ranges hold no partial
  return (2ll * c + (sc.item_begin(item) <= s0 ? 0 : 1)) * bm + row;
}

__device__ __forceinline__ float4 merge_segments(const Sched& sc, int item, int row, int bm, int D,
                                                 int c_first, int nseg, const float* __restrict__ ws_o,
                                                 const float* __restrict__ ws_l, int lane, float& mx_out,
                                                 float& z_out) {
  constexpr unsigned FULL = 0xffffffffu;
  const int c = lane * 4;
  const bool col = c < D;
  float mx = -INFINITY;
  const long long sl0 = lane < nseg ? seg_row(sc, item, row, bm, c_first + lane) : -1;
  const float lk0 = sl0 >= 0 ? ws_l[sl0] : -INFINITY;  // first chunk's LSEs, kept for the sum
  if (sl0 >= 0) mx = lk0;
  for (int k0 = 32; k0 < nseg; k0 += 32) {
    const long long sl = k0 + lane < nseg ? seg_row(sc, item, row, bm, c_first + k0 + lane) : -1;
    if (sl >= 0) mx = fmaxf(mx, ws_l[sl]);
  }
  mx = warp_max(mx);
  float z = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int k0 = 0; k0 < nseg; k0 += 32) {
    const long long sl = k0 == 0 ? sl0 : k0 + lane < nseg ? seg_row(sc, item, row, bm, c_first + k0 + lane) : -1;
    const float w = sl >= 0 ? __expf((k0 == 0 ? lk0 : ws_l[sl]) - mx) : 0.f;
    z += w;
    const int n = min(32, nseg - k0);
    for (int u0 = 0; u0 < n; u0 += 16) {  // 16 segments' loads in flight
      float wu[16];
      float4 v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const long long su = __shfl_sync(FULL, sl, (u0 + u) & 31);
        wu[u] = __shfl_sync(FULL, w, (u0 + u) & 31);
        v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (u0 + u < n && su >= 0) {
          if (col) v[u] = *reinterpret_cast<const float4*>(ws_o + su * D + c);
        } else {
          wu[u] = 0.f;
        }
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        acc.x += wu[u] * v[u].x; acc.y += wu[u] * v[u].y; acc.z += wu[u] * v[u].z; acc.w += wu[u] * v[u].w;
      }
    }
  }
  mx_out = mx;
  z_out = warp_sum(z);
  return acc;
}

// Fused final merge (MergeFinal): the row's K1 partial -- merged from the
// split workspace and stored to (o_k1, l_k1) like the plain merge, or the
// whole-item partial K1 already wrote there -- is merged with (o2, l2) and
// written as the attention output in the same pass.  Two-way log-space merge
// as K3 (attention.py:207-233), products rounded before the sum; a row empty
// on both sides gives 0 and is counted (merge_partials' DegenerateInputError).
__device__ __forceinline__ void final_merge_row(const Sched& sc, int item, int row, long long orow,
                                                int D, int bm, const float* __restrict__ ws_o,
                                                const float* __restrict__ ws_l, float* __restrict__ o_k1,
                                                float* __restrict__ l_k1, const MergeFinal& fin, int lane) {
  const long long ib = sc.item_begin(item), ie = sc.item_end(item);
  const int c_first = ib < ie ? sc.cta_of(ib) : 0;
  const int c_last = ib < ie ? sc.cta_of(ie - 1) : 0;
  const bool split = ib < ie && c_last > c_first;
  if (sc.fin_whole && ib < ie && !split) return;  // finished by its CTA's epilogue
  const int c = lane * 4;  // this lane's 4 columns (D <= 128)
  const bool col = c < D;
  float lp;
  float4 pv = make_float4(0.f, 0.f, 0.f, 0.f);
  if (ib == ie) {  // no keys: the empty partial
    lp = -INFINITY;
    if (col) *reinterpret_cast<float4*>(o_k1 + orow * D + c) = pv;
    if (lane == 0) l_k1[orow] = lp;
  } else if (!split) {
    lp = l_k1[orow];
    if (col) pv = *reinterpret_cast<const float4*>(o_k1 + orow * D + c);
  } else {
    const int nseg = c_last - c_first + 1;
    float mx, z;
    pv = merge_segments(sc, item, row, bm, D, c_first, nseg, ws_o, ws_l, lane, mx, z);
    const float iz = 1.f / z;
    if (col) {
      pv = make_float4(pv.x * iz, pv.y * iz, pv.z * iz, pv.w * iz);
      *reinterpret_cast<float4*>(o_k1 + orow * D + c) = pv;
    }
    lp = mx + logf(z);
    if (lane == 0) l_k1[orow] = lp;
  }
  const float l2 = fin.l2 ? fin.l2[orow] : -INFINITY;
  const float m = fmaxf(lp, l2);
  const bool live = m != -INFINITY;
  const float wp = (live && lp != -INFINITY) ? __expf(lp - m) : 0.f;
  const float w2 = (live && l2 != -INFINITY) ? __expf(l2 - m) : 0.f;
  const float iz = live ? 1.f / (wp + w2) : 0.f;
  if (col) {
    float4 o2 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (w2 != 0.f) {
      if (fin.o2_bf16) {
        const uint2 u = *reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(fin.o2) + orow * D + c);
        o2 = make_float4(ptx::bf16_lo(u.x), ptx::bf16_hi(u.x), ptx::bf16_lo(u.y), ptx::bf16_hi(u.y));
      } else {
        o2 = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(fin.o2) + orow * D + c);
      }
    }
    const float4 o = make_float4((__fmul_rn(wp, pv.x) + __fmul_rn(w2, o2.x)) * iz,
                                 (__fmul_rn(wp, pv.y) + __fmul_rn(w2, o2.y)) * iz,
                                 (__fmul_rn(wp, pv.z) + __fmul_rn(w2, o2.z)) * iz,
                                 (__fmul_rn(wp, pv.w) + __fmul_rn(w2, o2.w)) * iz);
    if (fin.out_bf16) {
      uint2 u;
      u.x = ptx::pack_bf16(o.x, o.y);
      u.y = ptx::pack_bf16(o.z, o.w);
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(fin.out) + orow * D + c) = u;
    } else {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(fin.out) + orow * D + c) = o;
    }
  }
  if (!live && lane == 0 && fin.empty_rows) atomicAdd(fin.empty_rows, 1);
}

// Split merge for items covered by several CTAs: one warp per query row,
// lanes over columns (coalesced 512 B per partial row); the partials are
// merged in segment order, so the result does not depend on CTA timing.
// Same log-space merge as K3 (attention.py:207-233).
__global__ void __launch_bounds__(256)
refresh_merge_kernel(Sched sc, int q_rows, int D, const float* __restrict__ ws_o,
                     const float* __restrict__ ws_l, float* __restrict__ o_out,
                     float* __restrict__ lse_out, int bm, MergeFinal fin) {
  ptx::pdl_wait();
  ptx::pdl_launch_dependents();
  sc.resolve();
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // item*bm + row
  const int lane = threadIdx.x & 31;
  const int item = (int)(gw / bm);
  const int row = (int)(gw % bm);
  if (item >= sc.items) return;
  const int g = sc.group_of(item), mt = sc.mtile_of(item);
  const int grow = mt * bm + row;
  if (grow >= q_rows) return;
  const long long orow = (long long)g * q_rows + grow;
  const long long ib = sc.item_begin(item), ie = sc.item_end(item);
  if (fin.out != nullptr) {  // fused final merge: this row's partial(s) + (o2, l2) -> out
    final_merge_row(sc, item, row, orow, D, bm, ws_o, ws_l, o_out, lse_out, fin, lane);
    return;
  }
  if (ib == ie) {  // no keys (ragged length 0): the empty partial
    if (sc.o_bf16)
      for (int c = lane; c < D; c += 32) reinterpret_cast<__nv_bfloat16*>(o_out)[orow * D + c] = __float2bfloat16(0.f);
    else
      for (int c = lane; c < D; c += 32) o_out[orow * D + c] = 0.f;
    if (lane == 0) lse_out[orow] = -INFINITY;
    return;
  }
  const int c_first = sc.cta_of(ib);
  const int c_last = sc.cta_of(ie - 1);
  if (c_first == c_last) return;  // written whole by its CTA
  const int nseg = c_last - c_first + 1;
  float mx, z;
  const float4 acc = merge_segments(sc, item, row, bm, D, c_first, nseg, ws_o, ws_l, lane, mx, z);
  const float iz = 1.f / z;
  if (lane * 4 < D) {
    if (sc.o_bf16) {
      uint2 u;
      u.x = ptx::pack_bf16(acc.x * iz, acc.y * iz);
      u.y = ptx::pack_bf16(acc.z * iz, acc.w * iz);
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(o_out) + orow * D + lane * 4) = u;
    } else {
      *reinterpret_cast<float4*>(o_out + orow * D + lane * 4) =
          make_float4(acc.x * iz, acc.y * iz, acc.z * iz, acc.w * iz);
    }
  }
  if (lane == 0) lse_out[orow] = mx + logf(z);
}

#include "fb_sm100_pair.cuh"  // K1 on CTA pairs (tensor-bound shapes)
#include "fb_sm100_quad.cuh"  // K1 with two query tiles per CTA (experimental)

// ---------------------------------------------------------------- K5 scoring
//
// Sparse block selection scores (sparse.py:117-125) on the tensor cores.
// Two-pass form (score_kernel<D, MODE>, MODE 0 / 1; kept for A/B behind
// fb_debug_set_k5_mode(1) / FB_K5_TWO_PASS=1):
//   LSE pass  : per query row, log2-domain log-sum-exp of the scaled scores over
//               ALL keys (committed [0,n_ext) + current block [0,n_in)), as
//               stream-K split partials merged by score_lse_merge_kernel;
//   MASS pass : per external 16-key block, sum over the block's keys and over
//               the tile's 128 query rows of exp2(s*c - lse2_row); rows reduce in
//               double in a fixed order (bit-equal masses for equal inputs).
// K tiles only (no V, no PV): Q + a 6-deep K ring in smem, S double-buffered
// in TMEM, the softmax warps release each S buffer after reading it.
//   FUSED pass (score_fused_kernel, the default): ONE read of K.  Four
//               score warpgroups take 32 columns (two 16-key blocks) of every
//               S tile each; a thread takes its row's quarter-tile max mt,
//               sums p = exp2(s*c - mt) per block (A; optionally part of the
//               exp2 pairs on the FMA pipes, off by default) and over the
//               quarter (the row's running
//               LSE, rescaled by two exp2 per tile), and stores A and mt for
//               the external tiles; score_mass_kernel weights A by
//               exp2(mt - lse2_row) once the row LSE is final and sums the
//               rows.  K bytes once plus 6 KB of A / mt per 32 KB K tile.
template <int D>
struct ScoreCfg {
  static constexpr int STAGES = 6;
  static constexpr int NBOX = D / BOX_COLS;
  static constexpr uint32_t BOX_BYTES = BM * BOX_COLS * 2;
  static constexpr uint32_t TILE_BYTES = NBOX * BOX_BYTES;
  static constexpr uint32_t OFF_Q = 0;
  static constexpr uint32_t OFF_K = OFF_Q + TILE_BYTES;
  static constexpr uint32_t OFF_BAR = OFF_K + STAGES * TILE_BYTES;
  static constexpr uint32_t OFF_RED = OFF_BAR + 512;  // [2][8][4] doubles + [2][128] floats
  static constexpr uint32_t SMEM = OFF_RED + 2 * 8 * 4 * 8 + 2 * 128 * 4 + 1024;
};

struct ScoreBars {
  uint64_t q_full, q_empty;
  uint64_t k_full[6], k_empty[6];
  uint64_t s_full[2], s_free[2];
  uint32_t tmem_base;
};

constexpr int SCORE_THREADS = 384;  // 4 control warps + 2 score warpgroups

template <int D, int MODE>
__global__ void __launch_bounds__(SCORE_THREADS, 1)
score_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
             const __grid_constant__ CUtensorMap tm_ki, Paged pg, Sched sc, int q_rows, int n_ext, int n_in,
             int ext_tiles, float scale_log2, const float* __restrict__ lse2_in,
             float* __restrict__ lse2_out, float* __restrict__ ws_l, double* __restrict__ mass,
             int nb) {
  using C = ScoreCfg<D>;
  constexpr bool MASS = MODE == 1;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  ScoreBars* bar = reinterpret_cast<ScoreBars*>(smem + C::OFF_BAR);
  double* red = reinterpret_cast<double*>(smem + C::OFF_RED);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long t_begin = sc.start(blockIdx.x), t_end = sc.start(blockIdx.x + 1);  // uniform items

  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::mbar_init(&bar->q_full, 1);
    ptx::mbar_init(&bar->q_empty, 1);
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&bar->k_full[s], 1);
      ptx::mbar_init(&bar->k_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&bar->s_full[b], 1);
      ptx::mbar_init(&bar->s_free[b], 256);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(&bar->tmem_base, 256);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = bar->tmem_base;
  ptx::pdl_wait();
  ptx::pdl_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t keep = ptx::policy_evict_last(), stream = ptx::policy_evict_first();
      int j = 0, seg = 0;
      for (long long t = t_begin; t < t_end; ++seg) {
        const int item = (int)(t / sc.tpi);
        const long long seg_end = min(t_end, (long long)(item + 1) * sc.tpi);
        const int g = sc.group_of(item), mt = sc.mtile_of(item);
        if (seg > 0) ptx::mbar_wait(&bar->q_empty, (seg - 1) & 1);
        ptx::mbar_expect_tx(&bar->q_full, C::TILE_BYTES);
        for (int b = 0; b < C::NBOX; ++b)
          ptx::tma_load_3d(smem + C::OFF_Q + b * C::BOX_BYTES, &tm_q, &bar->q_full, b * BOX_COLS,
                           mt * BM, g, keep);
        for (; t < seg_end; ++t, ++j) {
          const int s = j % C::STAGES;
          const int lt = (int)(t - (long long)item * sc.tpi);
          const bool ext = lt < ext_tiles;
          int row = ext ? lt * BN : (lt - ext_tiles) * BN;
          int slab = g;
          if (ext && pg.table != nullptr) {  // paged cache: the tile's page, row inside it
            slab = __ldg(pg.table + (long long)g * pg.max_pages + row / pg.page_rows);
            row %= pg.page_rows;
          }
          ptx::mbar_wait(&bar->k_empty[s], ((j / C::STAGES) & 1) ^ 1);
          ptx::mbar_expect_tx(&bar->k_full[s], C::TILE_BYTES);
          for (int b = 0; b < C::NBOX; ++b)
            ptx::tma_load_3d(smem + C::OFF_K + s * C::TILE_BYTES + b * C::BOX_BYTES,
                             ext ? &tm_k : &tm_ki, &bar->k_full[s], b * BOX_COLS, row, slab, stream);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t IDESC_S = ptx::idesc_bf16_f32(BM, BN, false);
      const uint32_t q_base = ptx::smem_u32(smem + C::OFF_Q);
      int j = 0, seg = 0;
      for (long long t0 = t_begin; t0 < t_end; ++seg) {
        const int item = (int)(t0 / sc.tpi);
        const int n = (int)(min(t_end, (long long)(item + 1) * sc.tpi) - t0);
        ptx::mbar_wait(&bar->q_full, seg & 1);
        ptx::tc_fence_after();
        for (int t = 0; t < n; ++t, ++j) {
          const int s = j % C::STAGES;
          ptx::mbar_wait(&bar->k_full[s], (j / C::STAGES) & 1);
          if (j >= 2) ptx::mbar_wait(&bar->s_free[j & 1], ((j >> 1) - 1) & 1);
          ptx::tc_fence_after();
          const uint32_t k_base = ptx::smem_u32(smem + C::OFF_K + s * C::TILE_BYTES);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk / 4) * C::BOX_BYTES + (kk % 4) * 32;
            ptx::mma_ss(tmem + (j & 1) * 128, ptx::sdesc_sw128(q_base + off, 16, 1024),
                        ptx::sdesc_sw128(k_base + off, 16, 1024), IDESC_S, kk > 0);
          }
          ptx::tc_commit(&bar->k_empty[s]);
          ptx::tc_commit(&bar->s_full[j & 1]);
          if (t == n - 1) ptx::tc_commit(&bar->q_empty);
        }
        t0 += n;
      }
    }
  } else if (warp >= 4) {
    // two score warpgroups: WG0 (warps 4-7) columns 0-63, WG1 (warps 8-11)
    // columns 64-127 of every S tile; the same 128 rows (TMEM lanes).
    constexpr int HALF = BN / 2;
    const int wq = warp & 3;
    const int wg = (warp - 4) >> 2;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const int row = wq * 32 + lane;
    float* xch = reinterpret_cast<float*>(red + 2 * 8 * 4);  // [2][128] (m, l) of WG1
    uint32_t r[32];
    float s[HALF];
    int j = 0, seg = 0;
    for (long long t0 = t_begin; t0 < t_end; ++seg) {
      const int item = (int)(t0 / sc.tpi);
      const int lt0 = (int)(t0 - (long long)item * sc.tpi);
      const int n = (int)(min(t_end, (long long)(item + 1) * sc.tpi) - t0);
      const int g = sc.group_of(item), mt = sc.mtile_of(item);
      const int grow = mt * BM + row;
      const bool live = grow < q_rows;
      const long long orow = (long long)g * q_rows + grow;
      float m = -INFINITY, l = 0.f;
      const float lse2 = MASS ? (live ? lse2_in[orow] : INFINITY) : 0.f;
      for (int t = 0; t < n; ++t, ++j) {
        const int lt = lt0 + t;
        ptx::mbar_wait(&bar->s_full[j & 1], (j >> 1) & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int c = 0; c < HALF / 32; ++c)
          ptx::tmem_ld32(tmem + lane_off + (j & 1) * 128 + wg * HALF + c * 32,
                         reinterpret_cast<uint32_t*>(s) + c * 32);
        ptx::tmem_wait_ld();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&bar->s_free[j & 1]);
        const bool ext = lt < ext_tiles;
        const int valid = (ext ? n_ext - lt * BN : n_in - (lt - ext_tiles) * BN) - wg * HALF;
        if constexpr (!MASS) {
          float mx8[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) mx8[k] = -INFINITY;
#pragma unroll
          for (int i = 0; i < HALF; ++i) {
            if (i >= valid) s[i] = -INFINITY;
            mx8[i & 7] = fmaxf(mx8[i & 7], s[i]);
          }
          const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                 fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
          const float m_new = fmaxf(m, mx * scale_log2);
          if (m_new != -INFINITY) {  // a half tile may be fully masked
            float a8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int i = 0; i < HALF; ++i) a8[i & 7] += ptx::ex2(fmaf(s[i], scale_log2, -m_new));
            const float acc = ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
            l = l * ptx::ex2(m - m_new) + acc;
            m = m_new;
          }
        } else {
          // 4 blocks of 16 keys per thread; warp transpose-reduce: 6 shuffles
          // leave block (2*bit4 + bit3) of lane's warp sum in every lane
          float a[4];
#pragma unroll
          for (int bi = 0; bi < 4; ++bi) {
            float p4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int c = bi * 16 + i;
              p4[i & 3] += (c < valid && live) ? ptx::ex2(fmaf(s[c], scale_log2, -lse2)) : 0.f;
            }
            a[bi] = (p4[0] + p4[1]) + (p4[2] + p4[3]);
          }
          const bool b4 = lane & 16, b3 = lane & 8;
          const float r0 = __shfl_xor_sync(0xffffffffu, b4 ? a[0] : a[2], 16);
          const float r1 = __shfl_xor_sync(0xffffffffu, b4 ? a[1] : a[3], 16);
          const float c0 = (b4 ? a[2] : a[0]) + r0;
          const float c1 = (b4 ? a[3] : a[1]) + r1;
          const float rr = __shfl_xor_sync(0xffffffffu, b3 ? c0 : c1, 8);
          float v = (b3 ? c1 : c0) + rr;
          v += __shfl_xor_sync(0xffffffffu, v, 4);
          v += __shfl_xor_sync(0xffffffffu, v, 2);
          v += __shfl_xor_sync(0xffffffffu, v, 1);
          double* rb = red + (j & 1) * 32;  // [8 blocks][4 warps]
          if ((lane & 7) == 0) rb[(wg * 4 + (lane >> 3)) * 4 + wq] = (double)v;
          asm volatile("bar.sync 1, 256;" ::: "memory");
          if (wg == 0 && wq == 0 && lane < 8) {
            const int blk = lt * (BN / 16) + lane;
            if (blk < nb) {
              const double* x = rb + lane * 4;
              mass[(long long)g * nb + blk] = ((x[0] + x[1]) + x[2]) + x[3];
            }
          }
        }
      }
      t0 += n;
      if constexpr (!MASS) {
        // combine the two column halves of each row, then the split partials
        if (wg == 1) {
          xch[row] = m;
          xch[BM + row] = l;
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (wg == 0) {
          const float m1 = xch[row], l1 = xch[BM + row];
          const float mm = fmaxf(m, m1);
          const float lt = l * ptx::ex2(m - mm) + l1 * ptx::ex2(m1 - mm);
          const bool whole = sc.item_begin(item) >= t_begin && sc.item_end(item) <= t_end;
          const float lse = mm + log2f(lt);
          if (whole) {
            if (live) lse2_out[orow] = lse;
          } else {
            ws_l[sc.slot(blockIdx.x, item) * BM + row] = lse;
          }
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 256);
  }
}

// ---------------------------------------------------------------- fused K5
template <int D>
struct ScoreFusedCfg {
  static constexpr int STAGES = 5;
  static constexpr int NBOX = D / BOX_COLS;
  static constexpr uint32_t BOX_BYTES = BM * BOX_COLS * 2;
  static constexpr uint32_t TILE_BYTES = NBOX * BOX_BYTES;
  static constexpr uint32_t OFF_Q = 0;
  static constexpr uint32_t OFF_K = OFF_Q + TILE_BYTES;
  static constexpr uint32_t OFF_BAR = OFF_K + STAGES * TILE_BYTES;
  static constexpr uint32_t OFF_X = OFF_BAR + 512;  // [3 quarters][2: m, l][128] floats
  static constexpr uint32_t SMEM = OFF_X + 3 * 2 * BM * 4 + 1024;
};
static_assert(ScoreFusedCfg<128>::SMEM <= 232448, "fused K5 shared memory exceeds 227 KB");

struct ScoreFusedBars {
  uint64_t q_full, q_empty;
  uint64_t k_full[5], k_empty[5];
  uint64_t s_full[2], s_free[2];
  uint32_t tmem_base;
};

constexpr int SCORE_FUSED_THREADS = 640;  // 4 control warps + 4 score warpgroups
constexpr int K5_POLY_DEFAULT = 0;        // exp2 pairs of 8 per 16-key block on the FMA pipes
                                          // (2 / 4: no gain measured -- MUFU is not the binding unit here)

template <int D, int POLY>
__global__ void __launch_bounds__(SCORE_FUSED_THREADS, 1)
score_fused_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_ki, Paged pg, Sched sc, int q_rows, int n_ext,
                   int n_in, int ext_tiles, float scale_log2, float* __restrict__ lse2_out,
                   float* __restrict__ ws_l, float* __restrict__ ws_a, float* __restrict__ ws_m) {
  using C = ScoreFusedCfg<D>;
  constexpr int QC = BN / 4;  // columns per warpgroup
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  ScoreFusedBars* bar = reinterpret_cast<ScoreFusedBars*>(smem + C::OFF_BAR);
  float* xch = reinterpret_cast<float*>(smem + C::OFF_X);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long t_begin = sc.start(blockIdx.x), t_end = sc.start(blockIdx.x + 1);  // uniform items

  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::mbar_init(&bar->q_full, 1);
    ptx::mbar_init(&bar->q_empty, 1);
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&bar->k_full[s], 1);
      ptx::mbar_init(&bar->k_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&bar->s_full[b], 1);
      ptx::mbar_init(&bar->s_free[b], 512);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(&bar->tmem_base, 256);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = bar->tmem_base;
  ptx::pdl_wait();
  ptx::pdl_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t keep = ptx::policy_evict_last(), stream = ptx::policy_evict_first();
      int j = 0, seg = 0;
      for (long long t = t_begin; t < t_end; ++seg) {
        const int item = (int)(t / sc.tpi);
        const long long seg_end = min(t_end, (long long)(item + 1) * sc.tpi);
        const int g = sc.group_of(item), mt = sc.mtile_of(item);
        if (seg > 0) ptx::mbar_wait(&bar->q_empty, (seg - 1) & 1);
        ptx::mbar_expect_tx(&bar->q_full, C::TILE_BYTES);
        for (int b = 0; b < C::NBOX; ++b)
          ptx::tma_load_3d(smem + C::OFF_Q + b * C::BOX_BYTES, &tm_q, &bar->q_full, b * BOX_COLS,
                           mt * BM, g, keep);
        for (; t < seg_end; ++t, ++j) {
          const int s = j % C::STAGES;
          const int lt = (int)(t - (long long)item * sc.tpi);
          const bool ext = lt < ext_tiles;
          int row = ext ? lt * BN : (lt - ext_tiles) * BN;
          int slab = g;
          if (ext && pg.table != nullptr) {  // paged cache: the tile's page, row inside it
            slab = __ldg(pg.table + (long long)g * pg.max_pages + row / pg.page_rows);
            row %= pg.page_rows;
          }
          ptx::mbar_wait(&bar->k_empty[s], ((j / C::STAGES) & 1) ^ 1);
          ptx::mbar_expect_tx(&bar->k_full[s], C::TILE_BYTES);
          for (int b = 0; b < C::NBOX; ++b)
            ptx::tma_load_3d(smem + C::OFF_K + s * C::TILE_BYTES + b * C::BOX_BYTES,
                             ext ? &tm_k : &tm_ki, &bar->k_full[s], b * BOX_COLS, row, slab, stream);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t IDESC_S = ptx::idesc_bf16_f32(BM, BN, false);
      const uint32_t q_base = ptx::smem_u32(smem + C::OFF_Q);
      int j = 0, seg = 0;
      for (long long t0 = t_begin; t0 < t_end; ++seg) {
        const int item = (int)(t0 / sc.tpi);
        const int n = (int)(min(t_end, (long long)(item + 1) * sc.tpi) - t0);
        ptx::mbar_wait(&bar->q_full, seg & 1);
        ptx::tc_fence_after();
        for (int t = 0; t < n; ++t, ++j) {
          const int s = j % C::STAGES;
          ptx::mbar_wait(&bar->k_full[s], (j / C::STAGES) & 1);
          if (j >= 2) ptx::mbar_wait(&bar->s_free[j & 1], ((j >> 1) - 1) & 1);
          ptx::tc_fence_after();
          const uint32_t k_base = ptx::smem_u32(smem + C::OFF_K + s * C::TILE_BYTES);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk / 4) * C::BOX_BYTES + (kk % 4) * 32;
            ptx::mma_ss(tmem + (j & 1) * 128, ptx::sdesc_sw128(q_base + off, 16, 1024),
                        ptx::sdesc_sw128(k_base + off, 16, 1024), IDESC_S, kk > 0);
          }
          ptx::tc_commit(&bar->k_empty[s]);
          ptx::tc_commit(&bar->s_full[j & 1]);
          if (t == n - 1) ptx::tc_commit(&bar->q_empty);
        }
        t0 += n;
      }
    }
  } else if (warp >= 4) {
    // warpgroup w (warps 4+4w .. 7+4w): columns [32w, 32w+32) of every S tile
    const int wq = warp & 3;
    const int w = (warp - 4) >> 2;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const int row = wq * 32 + lane;
    float s[QC];
    int j = 0, seg = 0;
    const uint64_t c2 = ptx::f2_pack(scale_log2, scale_log2);
    for (long long t0 = t_begin; t0 < t_end; ++seg) {
      const int item = (int)(t0 / sc.tpi);
      const int lt0 = (int)(t0 - (long long)item * sc.tpi);
      const int n = (int)(min(t_end, (long long)(item + 1) * sc.tpi) - t0);
      const int g = sc.group_of(item), mt = sc.mtile_of(item);
      const int grow = mt * BM + row;
      const long long orow = (long long)g * q_rows + grow;
      float m = -INFINITY, l = 0.f;
      for (int t = 0; t < n; ++t, ++j) {
        const int lt = lt0 + t;
        ptx::mbar_wait(&bar->s_full[j & 1], (j >> 1) & 1);
        ptx::tc_fence_after();
        ptx::tmem_ld32(tmem + lane_off + (j & 1) * 128 + w * QC, reinterpret_cast<uint32_t*>(s));
        ptx::tmem_wait_ld();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&bar->s_free[j & 1]);
        const bool ext = lt < ext_tiles;
        const int valid = (ext ? n_ext - lt * BN : n_in - (lt - ext_tiles) * BN) - w * QC;
        float a[QC / 16];
        float tmax;
        if constexpr (POLY == -1) {  // diagnostics: the TMA + MMA pipeline alone (no score math)
          continue;
        }
        constexpr int NP = POLY < 0 ? 0 : POLY;  // -2: diagnostics, the math without the A / mt stores
        if (valid >= QC) {
          // full quarter tile (warp-uniform): no masking; per 16-key block,
          // pairs [0, 8 - POLY) on MUFU.EX2 and the rest on the FMA pipes
          float mx4[4] = {s[0], s[1], s[2], s[3]};
#pragma unroll
          for (int i = 4; i < QC; ++i) mx4[i & 3] = fmaxf(mx4[i & 3], s[i]);
          tmax = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * scale_log2;
          const uint64_t n2 = ptx::f2_pack(-tmax, -tmax);
#pragma unroll
          for (int bi = 0; bi < QC / 16; ++bi) {
            uint64_t acc0 = ptx::f2_pack(0.f, 0.f), acc1 = acc0;
#pragma unroll
            for (int pi = 0; pi < 8; ++pi) {
              const uint64_t x = ptx::f2_fma(ptx::f2_pack(s[bi * 16 + 2 * pi], s[bi * 16 + 2 * pi + 1]), c2, n2);
              uint64_t e;
              if (pi >= 8 - NP) {
                e = ptx::ex2_poly5x2(x);
              } else {
                float x0, x1;
                ptx::f2_unpack(x, x0, x1);
                e = ptx::f2_pack(ptx::ex2(x0), ptx::ex2(x1));
              }
              if (pi & 1) acc1 = ptx::f2_add(acc1, e); else acc0 = ptx::f2_add(acc0, e);
            }
            float u0, u1, u2, u3;
            ptx::f2_unpack(acc0, u0, u1);
            ptx::f2_unpack(acc1, u2, u3);
            a[bi] = (u0 + u1) + (u2 + u3);
          }
        } else {
          float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int i = 0; i < QC; ++i) {
            if (i >= valid) s[i] = -INFINITY;
            mx4[i & 3] = fmaxf(mx4[i & 3], s[i]);
          }
          tmax = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * scale_log2;
#pragma unroll
          for (int bi = 0; bi < QC / 16; ++bi) {
            float p4[4] = {0.f, 0.f, 0.f, 0.f};
            if (tmax != -INFINITY) {  // a quarter tile may be fully masked
#pragma unroll
              for (int i = 0; i < 16; ++i) p4[i & 3] += ptx::ex2(fmaf(s[bi * 16 + i], scale_log2, -tmax));
            }
            a[bi] = (p4[0] + p4[1]) + (p4[2] + p4[3]);
          }
        }
        if (tmax != -INFINITY) {
          const float m_new = fmaxf(m, tmax);
          l = l * ptx::ex2(m - m_new) + (a[0] + a[1]) * ptx::ex2(tmax - m_new);
          m = m_new;
        }
        if (ext && POLY != -2) {  // A [group][ext tile][8 blocks][128 rows], mt [group][ext tile][4 quarters][128 rows]
          const long long tb = (long long)g * ext_tiles + lt;
#pragma unroll
          for (int bi = 0; bi < QC / 16; ++bi) ws_a[(tb * 8 + w * (QC / 16) + bi) * BM + row] = a[bi];
          ws_m[(tb * 4 + w) * BM + row] = tmax;
        }
      }
      t0 += n;
      // combine the four column quarters of each row, then the split partials
      if (w > 0) {
        xch[((w - 1) * 2 + 0) * BM + row] = m;
        xch[((w - 1) * 2 + 1) * BM + row] = l;
      }
      asm volatile("bar.sync 1, 512;" ::: "memory");
      if (w == 0) {
        float mm = m;
#pragma unroll
        for (int k = 0; k < 3; ++k) mm = fmaxf(mm, xch[(k * 2) * BM + row]);
        float lt = mm == -INFINITY ? 0.f : l * ptx::ex2(m - mm);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const float mk = xch[(k * 2) * BM + row];
          if (mk != -INFINITY) lt += xch[(k * 2 + 1) * BM + row] * ptx::ex2(mk - mm);
        }
        const bool whole = sc.item_begin(item) >= t_begin && sc.item_end(item) <= t_end;
        const float lse = mm + log2f(lt);
        if (whole) {
          if (grow < q_rows) lse2_out[orow] = lse;
        } else {
          ws_l[sc.slot(blockIdx.x, item) * BM + row] = lse;
        }
      }
      asm volatile("bar.sync 1, 512;" ::: "memory");
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 256);
  }
}

__global__ void score_lse_merge_kernel(Sched sc, int q_rows, const float* __restrict__ ws_l,
                                       float* __restrict__ lse2_out) {
  ptx::pdl_wait();
  ptx::pdl_launch_dependents();
  const long long gr = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // item*BM + row
  const int item = (int)(gr / BM);
  const int row = (int)(gr % BM);
  if (item >= sc.items) return;
  const int c_first = sc.cta_of(sc.item_begin(item));
  const int c_last = sc.cta_of(sc.item_end(item) - 1);
  const int g = sc.group_of(item), mt = sc.mtile_of(item);
  const int grow = mt * BM + row;
  if (c_first == c_last || grow >= q_rows) return;
  float mx = -INFINITY;
  for (int c = c_first; c <= c_last; ++c) mx = fmaxf(mx, ws_l[sc.slot(c, item) * BM + row]);
  float z = 0.f;
  for (int c = c_first; c <= c_last; ++c) z += exp2f(ws_l[sc.slot(c, item) * BM + row] - mx);
  lse2_out[(long long)g * q_rows + grow] = mx + log2f(z);
}

// Fused K5, second half: mass[g][blk] = sum over the group's rows of
// A[g][tile][blk % 8][row] * exp2(mt[g][tile][quarter][row] - lse2[row]).  One
// CTA per (group, tiles_per_cta external tiles); the group's final row LSEs
// (the stream-K split partials merged here, as score_lse_merge_kernel does)
// sit in shared memory; a warp takes every 8th tile (its first tile's loads
// issued before the LSE merge), 4 CTAs per SM, lane = 4 rows, then a fixed-order double transpose-reduce over the
// lanes (equal inputs -> bit-equal masses).
__device__ __forceinline__ void mass_tile_reduce(const float4 (&mq)[4], const float4 (&a)[8], float4 ls,
                                                 int lane, int lt, int nb, double* __restrict__ mrow) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
  double v[8];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float w0 = ptx::ex2(mq[q].x - ls.x), w1 = ptx::ex2(mq[q].y - ls.y);
    const float w2 = ptx::ex2(mq[q].z - ls.z), w3 = ptx::ex2(mq[q].w - ls.w);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float4 x = a[2 * q + h];
      v[2 * q + h] = (double)(((x.x * w0) + (x.y * w1)) + ((x.z * w2) + (x.w * w3)));
    }
  }
  // transpose-reduce: 8 -> 4 -> 2 -> 1 values per lane, then the last two levels
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double r = __shfl_xor_sync(0xffffffffu, b4 ? v[k] : v[k + 4], 16);
    v[k] = (b4 ? v[k + 4] : v[k]) + r;
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double r = __shfl_xor_sync(0xffffffffu, b3 ? v[k] : v[k + 2], 8);
    v[k] = (b3 ? v[k + 2] : v[k]) + r;
  }
  {
    const double r = __shfl_xor_sync(0xffffffffu, b2 ? v[0] : v[1], 4);
    v[0] = (b2 ? v[1] : v[0]) + r;
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
  if ((lane & 3) == 0) {
    const int blk = lt * 8 + (b4 ? 4 : 0) + (b3 ? 2 : 0) + (b2 ? 1 : 0);
    if (blk < nb) mrow[blk] = v[0];
  }
}

__global__ void __launch_bounds__(256, 4)
score_mass_kernel(Sched sc, int q_rows, int ext_tiles, int nb, int tiles_per_cta,
                  const float* __restrict__ lse2_whole, const float* __restrict__ ws_l,
                  const float* __restrict__ ws_a, const float* __restrict__ ws_m, double* __restrict__ mass) {
  __shared__ __align__(16) float lse2[BM];
  const int g = blockIdx.y;  // q_rows <= BM: item == group
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lt_end = min(ext_tiles, (int)(blockIdx.x + 1) * tiles_per_cta);
  double* mrow = mass + (long long)g * nb;
  float4 mq[1][4], a[1][8];  // one tile in flight per warp: 4 CTAs (32 warps) per SM
  auto load = [&](int u, int lt) {
    const long long tb = (long long)g * ext_tiles + lt;
#pragma unroll
    for (int q = 0; q < 4; ++q) mq[u][q] = __ldcg(reinterpret_cast<const float4*>(ws_m + (tb * 4 + q) * BM) + lane);
#pragma unroll
    for (int b = 0; b < 8; ++b) a[u][b] = __ldcg(reinterpret_cast<const float4*>(ws_a + (tb * 8 + b) * BM) + lane);
  };
  ptx::pdl_wait();
  ptx::pdl_launch_dependents();
  int lt = blockIdx.x * tiles_per_cta + warp;
  if (lt < lt_end) load(0, lt);  // in flight while the row LSEs are merged
  if (threadIdx.x < BM) {
    const int row = threadIdx.x;
    float v = INFINITY;  // rows past q_rows weigh 0
    if (row < q_rows) {
      const int c_first = sc.cta_of(sc.item_begin(g));
      const int c_last = sc.cta_of(sc.item_end(g) - 1);
      if (c_first == c_last) {
        v = lse2_whole[(long long)g * q_rows + row];
      } else {
        float x[8];
        const int nc = min(c_last - c_first + 1, 8);
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = c < nc ? __ldcg(ws_l + sc.slot(c_first + c, g) * BM + row) : -INFINITY;
        float mx = -INFINITY;
        for (int c = c_first + 8; c <= c_last; ++c) mx = fmaxf(mx, __ldcg(ws_l + sc.slot(c, g) * BM + row));
#pragma unroll
        for (int c = 0; c < 8; ++c) mx = fmaxf(mx, x[c]);
        float z = 0.f;
#pragma unroll
        for (int c = 0; c < 8; ++c) z += c < nc ? exp2f(x[c] - mx) : 0.f;
        for (int c = c_first + 8; c <= c_last; ++c) z += exp2f(__ldcg(ws_l + sc.slot(c, g) * BM + row) - mx);
        v = mx + log2f(z);
      }
    }
    lse2[row] = v;
  }
  __syncthreads();
  const float4 ls = *reinterpret_cast<const float4*>(lse2 + 4 * lane);
  for (; lt < lt_end; lt += 8) {
    mass_tile_reduce(mq[0], a[0], ls, lane, lt, nb, mrow);
    if (lt + 8 < lt_end) load(0, lt + 8);
  }
}

// ---------------------------------------------------------------- host side

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

}  // namespace sm100

// 3-D view [dim2][dim1][inner] (element size 2 or 4 bytes) with a
// box_rows x box_inner 128B-swizzled box.  Rows >= dim1 read as zero (TMA
// out-of-bounds fill), so slab tails never leak uninitialised memory.
int make_tmap_3d(CUtensorMap* map, const void* base, int dtype_bytes, int64_t inner, int64_t dim1,
                 int64_t dim1_stride_elems, int64_t dim2, int box_inner, int box_rows) {
  auto enc = sm100::get_encode();
  if (!enc) return fail(FB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)dim1, (cuuint64_t)dim2};
  cuuint64_t strides[2] = {(cuuint64_t)(inner * dtype_bytes),
                           (cuuint64_t)(dim1_stride_elems * inner * dtype_bytes)};
  cuuint32_t box[3] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  const CUtensorMapDataType dt =
      dtype_bytes == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  CUresult r = enc(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(FB_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return FB_OK;
}

// N-D bf16 view (rank 2..5): dims[0] = contiguous elements, byte strides for
// dims 1..rank-1, 128B-swizzled box.  Out-of-bounds boxes read as zero.
int make_tmap_nd(CUtensorMap* map, const void* base, int rank, const int64_t* dims,
                 const int64_t* stride_bytes, const int* box) {
  auto enc = sm100::get_encode();
  if (!enc) return fail(FB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t d[5], st[4];
  cuuint32_t bx[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = (cuuint64_t)dims[i];
    bx[i] = (cuuint32_t)box[i];
    es[i] = 1;
    if (i > 0) st[i - 1] = (cuuint64_t)stride_bytes[i];
  }
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), d, st, bx, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(FB_ERR_CUDA, "cuTensorMapEncodeTiled (nd) failed: " + std::to_string((int)r));
  return FB_OK;
}

bool sm100_supported(int64_t head_dim) { return head_dim == 64 || head_dim == 128; }

// diagnostics: per-CTA globaltimer stamps (set through fb_debug_set_trace)
static unsigned long long* g_trace = nullptr;
static int g_k1_diag = 0;  // diagnostics: refresh_kernel<.., DIAG> variant
void set_k1_diag(int d) { g_k1_diag = d; }
static int g_trace_launch = 0;  // successive launches stamp successive 148x8 slabs

struct RefreshPlan {
  int ctas, tpi, m_tiles, items;
  long long T;
  size_t ws_bytes;
};

// Uniform items (every group has n_keys keys); ragged plans fill T on device.
static RefreshPlan plan_refresh(int64_t groups, int64_t q_rows, int64_t head_dim, int64_t n_keys) {
  RefreshPlan p{};
  p.m_tiles = (int)((q_rows + sm100::BM - 1) / sm100::BM);
  p.items = (int)(groups * p.m_tiles);
  p.tpi = (int)((n_keys + sm100::BN - 1) / sm100::BN);
  p.T = (long long)p.items * p.tpi;
  p.ctas = (int)std::max<long long>(1, std::min<long long>(num_sms(), p.T));
  // Small problems: a CTA count that is a multiple of the item count and cuts
  // every item into equal whole-tile ranges gives each CTA one segment (no
  // second epilogue / Q reload) at the price of fewer SMs.  Cost model in
  // tiles per CTA + SEG_COST per segment (measured at C2 shapes: b=2 / b=4
  // 62 / 99 us on 128 CTAs vs 70 / 106 us on 148; b >= 8 keeps 148).
  {
    constexpr long long SEG_COST = 10;
    const long long full = (p.T + p.ctas - 1) / p.ctas + 2 * SEG_COST;
    for (long long k = num_sms() / std::max(p.items, 1); k >= 1; --k) {
      if (p.tpi % k) continue;
      const long long c = (long long)p.items * k;
      if (c > num_sms() || c > p.T) continue;
      if (p.tpi / k + SEG_COST < full) p.ctas = (int)c;
      break;  // the largest aligned count is the only candidate worth trying
    }
  }
  if (const char* e = getenv("FB_REFRESH_CTAS")) {  // diagnostics: force the CTA count
    const long long want = atoll(e);
    if (want > 0) p.ctas = (int)std::max<long long>(1, std::min<long long>(want, p.T));
  }
  // two split-partial slots per CTA (its first and last segment)
  p.ws_bytes = (size_t)2 * p.ctas * sm100::BM * (head_dim + 1) * sizeof(float);
  return p;
}

void set_refresh_trace(void* p) {
  g_trace = reinterpret_cast<unsigned long long*>(p);
  g_trace_launch = 0;
}

static int pair_clusters();
static bool quad_enabled();

size_t refresh_sm100_workspace_bytes(int64_t groups, int64_t q_rows, int64_t head_dim, int64_t n_keys) {
  if (n_keys <= 0 || groups <= 0 || q_rows <= 0) return 0;
  size_t b = plan_refresh(groups, q_rows, head_dim, n_keys).ws_bytes;
  if (head_dim == 128 && q_rows > sm100::BM) {  // CTA-pair plan: 256-row split slots
    const long long T = groups * ((q_rows + sm100::pair::PM - 1) / sm100::pair::PM) *
                        ((n_keys + sm100::BN - 1) / sm100::BN);
    const long long pairs = std::min<long long>(pair_clusters(), T);
    b = std::max<size_t>(b, (size_t)2 * pairs * sm100::pair::PM * (head_dim + 1) * sizeof(float));
    if (quad_enabled()) {
      const long long qc = std::min<long long>(num_sms(), T);
      b = std::max<size_t>(b, (size_t)2 * qc * sm100::pair::PM * (head_dim + 1) * sizeof(float));
    }
  }
  return b;
}

// ragged: split slots for num_sms CTAs + the item offsets
size_t refresh_sm100_ragged_workspace_bytes(int64_t groups, int64_t q_rows, int64_t head_dim) {
  const int64_t items = groups * ((q_rows + sm100::BM - 1) / sm100::BM);
  return align_up((size_t)(items + 1) * sizeof(long long), 256) +
         (size_t)2 * num_sms() * sm100::BM * (head_dim + 1) * sizeof(float);
}

// Ragged contexts: item tile offsets prefix[items+1] from per-group key ends
// (one CTA, chunked serial sums + a warp scan of the chunk totals).
__global__ void ragged_prefix_kernel(const int* __restrict__ key_len, int items, int m_tiles,
                                     int key_begin, int key_cap, long long* __restrict__ prefix) {
  __shared__ long long part[1024];
  __shared__ long long warp_sum_sh[32];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = (items + nt - 1) / nt;
  const int i0 = min(items, tid * per), i1 = min(items, i0 + per);
  long long sum = 0;
  for (int i = i0; i < i1; ++i)
    sum += max(0, min(key_len[i / m_tiles], key_cap) - key_begin + sm100::BN - 1) / sm100::BN;
  part[tid] = sum;
  __syncthreads();
  if (tid < 32) {  // exclusive scan of the 1024 chunk sums, 32 per lane
    long long acc = 0;
    for (int k = 0; k < 32; ++k) acc += part[tid * 32 + k];
    long long inc = acc;
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, inc, o);
      if (tid >= o) inc += y;
    }
    warp_sum_sh[tid] = inc - acc;
  }
  __syncthreads();
  long long base = warp_sum_sh[tid / 32];
  for (int k = (tid / 32) * 32; k < tid; ++k) base += part[k];
  for (int i = i0; i < i1; ++i) {
    prefix[i] = base;
    base += max(0, min(key_len[i / m_tiles], key_cap) - key_begin + sm100::BN - 1) / sm100::BN;
  }
  if (i1 == items && i0 < i1) prefix[items] = base;
  if (items == 0 && tid == 0) prefix[0] = 0;
}

// Block-causal items: item i = (group, 128-row tile mt) streams keys
// [0, lim) with lim the largest row limit of the tile (its last row, or the
// head's full length when the tile straddles two heads); tile offsets as above.
__device__ __forceinline__ long long causal_item_tiles(int i, int items, int m_tiles, int q_rows,
                                                       sm100::Causal cz, int bm) {
  const int mt = i % m_tiles;
  const int r0 = mt * bm, r1 = min(r0 + bm, q_rows) - 1;
  const int lim = (r0 / cz.n_q != r1 / cz.n_q) ? cz.n_prefix + cz.n_q : cz.row_limit(r1);
  return (lim + sm100::BN - 1) / sm100::BN;
}

__global__ void causal_prefix_kernel(int items, int m_tiles, int q_rows, sm100::Causal cz,
                                     long long* __restrict__ prefix, int bm) {
  __shared__ long long part[1024];
  __shared__ long long warp_sum_sh[32];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = (items + nt - 1) / nt;
  const int i0 = min(items, tid * per), i1 = min(items, i0 + per);
  long long sum = 0;
  for (int i = i0; i < i1; ++i) sum += causal_item_tiles(i, items, m_tiles, q_rows, cz, bm);
  part[tid] = sum;
  __syncthreads();
  if (tid < 32) {
    long long acc = 0;
    for (int k = 0; k < 32; ++k) acc += part[tid * 32 + k];
    long long inc = acc;
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, inc, o);
      if (tid >= o) inc += y;
    }
    warp_sum_sh[tid] = inc - acc;
  }
  __syncthreads();
  long long base = warp_sum_sh[tid / 32];
  for (int k = (tid / 32) * 32; k < tid; ++k) base += part[k];
  for (int i = i0; i < i1; ++i) {
    prefix[i] = base;
    base += causal_item_tiles(i, items, m_tiles, q_rows, cz, bm);
  }
  if (i1 == items && i0 < i1) prefix[items] = base;
  if (items == 0 && tid == 0) prefix[0] = 0;
}

// CTA-pair K1 (fb_sm100_pair.cuh) for many query rows per group.  Default:
// block-causal prefill only, where it measured 1.09-1.17x faster than the
// single-CTA kernel (32K / 8K prompts at the C2 shapes); for the non-causal
// C5 refresh the single-CTA kernel stays faster (1.50 vs 1.65-1.70 ms at
// 56,160 keys; profiles/r01f_pair_notes.md).  Returns -1 when it does not
// apply (workspace too small), so the caller runs the single-CTA kernel.
// FB_PAIR=0 / 1: never / for every shape with > 128 query rows (diagnostics).
// K/V cache policy when several query tiles of a group stream the same keys
// (C5 chunks, prefill): evict_last keeps them in L2 for the other tiles;
// otherwise (C2: one tile per group) they stream evict_first.  FB_KV_KEEP=0
// disables it (diagnostics).
static bool kv_keep_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FB_KV_KEEP");
    on = (e != nullptr && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

static int pair_mode() {  // 0 never, 1 always, 2 block-causal only
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("FB_PAIR");
    m = e == nullptr ? 2 : (e[0] == '0' ? 0 : 1);
  }
  return m;
}
static thread_local bool t_partial_bf16 = false;
bool partial_out_bf16() { return t_partial_bf16; }
ScopedPartialBf16::ScopedPartialBf16(bool on) { t_partial_bf16 = on; }
ScopedPartialBf16::~ScopedPartialBf16() { t_partial_bf16 = false; }
static thread_local const PagingCtx* t_paging = nullptr;
const PagingCtx* current_paging() { return t_paging; }
ScopedPaging::ScopedPaging(const PagingCtx* p) { t_paging = p; }
ScopedPaging::~ScopedPaging() { t_paging = nullptr; }

static int g_pair_override = -1;
void set_pair_enabled(int on) { g_pair_override = on; }
static long long g_pair_launches = 0;
long long pair_launches() { return g_pair_launches; }

static int pair_clusters() {
  static int n = -1;
  if (n < 0) {
    auto kern = sm100::pair::pair_kernel<128>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sm100::pair::PCfg<128>::SMEM);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * (num_sms() / 2)));
    cfg.blockDim = dim3(sm100::THREADS);
    cfg.dynamicSmemBytes = sm100::pair::PCfg<128>::SMEM;
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, kern, &cfg) != cudaSuccess || c <= 0) {
      cudaGetLastError();
      c = num_sms() / 2;
    }
    n = c;
  }
  return n;
}

static int launch_pair_128(const __nv_bfloat16* k, const CUtensorMap& mq, const CUtensorMap& mv,
                           int64_t groups, int64_t q_rows, int64_t kv_rows_cap, int64_t key_begin,
                           int64_t key_end, double scale, float* o_out, float* lse_out, void* ws,
                           size_t ws_bytes, cudaStream_t st, const sm100::Causal* causal,
                           const int32_t* glist, int64_t n_list, const MergeFinal* fin = nullptr,
                           const sm100::Paged* paged = nullptr, int64_t num_pages = 0) {
  constexpr int D = 128;
  using P = sm100::pair::PCfg<D>;
  constexpr int PM = sm100::pair::PM;
  const int m_tiles = (int)((q_rows + PM - 1) / PM);
  const int items = (int)((glist ? n_list : groups) * m_tiles);
  const long long tpi = (key_end - key_begin + sm100::BN - 1) / sm100::BN;
  if (items <= 0 || tpi <= 0) return -1;
  CUtensorMap mk;
  int rc;
  if (paged != nullptr) {  // K halves over the page pool [num_pages, page_rows, D]
    if ((rc = make_tmap_3d(&mk, k, 2, D, paged->page_rows, paged->page_rows, num_pages, sm100::BOX_COLS,
                           sm100::pair::HN)))
      return rc;
  } else if ((rc = make_tmap_3d(&mk, k, 2, D, key_end, kv_rows_cap, groups, sm100::BOX_COLS,
                                sm100::pair::HN))) {
    return rc;
  }
  const sm100::Paged pgv = paged ? *paged : sm100::Paged{nullptr, 0, 1};
  sm100::Causal cz{1, 0, 0};
  if (causal) cz = *causal;
  const int maxp = pair_clusters();
  sm100::Sched sc{(long long)items * tpi, (int)tpi, m_tiles, items, 0, nullptr, glist};
  sc.kv_keep = m_tiles > 1 && kv_keep_enabled();
  {
    static int rot = -1;  // key-tile rotation for non-causal pair plans (FB_QUAD_ROT=0: off)
    if (rot < 0) {
      const char* e = getenv("FB_QUAD_ROT");
      rot = (e != nullptr && e[0] == '0') ? 0 : 1;
    }
    sc.rot = causal == nullptr ? rot : 0;
  }
  float* ws_o = nullptr;
  float* ws_l = nullptr;
  bool need_merge;
  if (causal && fin != nullptr) return -1;
  if (causal) {
    // whole items round-robin over the pairs (SegIter): no prefix scan, no
    // split partials, no merge kernel; all pairs on one group's K/V at a time
    sc.rr = 1;
    sc.tpi = 0;
    sc.ctas = std::min(maxp, items);
    need_merge = false;
  } else {
    sc.ctas = (int)std::min<long long>(maxp, sc.T);
    need_merge = !(sc.T % sc.ctas == 0 && (sc.T / sc.ctas) % tpi == 0);
    const bool split = need_merge;
    if (fin != nullptr) need_merge = true;  // the merge kernel writes the final output
    if (split) {
      const size_t need = (size_t)2 * sc.ctas * PM * (D + 1) * sizeof(float);
      if (ws == nullptr || ws_bytes < need) return -1;
      ws_o = reinterpret_cast<float*>(ws);
      ws_l = ws_o + (size_t)2 * sc.ctas * PM * D;
    }
  }
  static int poly = -1;
  if (poly < 0) {
    const char* e = getenv("FB_PAIR_POLY");  // diagnostics: MUFU offload share
    poly = e ? atoi(e) : 0;
  }
  if (poly < 0) {  // diagnostics: the pipeline without softmax math
    auto kd = sm100::pair::pair_kernel<D, -1>;
    cudaFuncSetAttribute(kd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM);
    const float sl = (float)(scale * 1.4426950408889634);
    launch_pdl(kd, dim3((unsigned)(2 * sc.ctas)), dim3(sm100::THREADS), P::SMEM, st, mq, mk, mv, pgv, cz, sc,
               (int)q_rows, (int)key_begin, (int)key_end, sl, o_out, lse_out, ws_o, ws_l);
    count_launch();
    if ((rc = check_launch("pair_kernel(diag)"))) return rc;
    if (!need_merge) return FB_OK;
    const long long warps = (long long)items * PM;
    launch_pdl(sm100::refresh_merge_kernel, dim3((unsigned)((warps + 7) / 8)), dim3(256), 0, st, sc,
               (int)q_rows, D, (const float*)ws_o, (const float*)ws_l, o_out, lse_out, PM, MergeFinal{});
    count_launch();
    return check_launch("refresh_merge_kernel(sm100, pair diag)");
  }
  auto kern = poly == 4 ? sm100::pair::pair_kernel<D, 4>
              : poly == 3 ? sm100::pair::pair_kernel<D, 3>
              : poly == 2 ? sm100::pair::pair_kernel<D, 2> : sm100::pair::pair_kernel<D, 0>;
  static bool attr[9] = {};
  if (!attr[poly & 7]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM);
    attr[poly & 7] = true;
  }
  const float scale_log2 = (float)(scale * 1.4426950408889634);
  launch_pdl(kern, dim3((unsigned)(2 * sc.ctas)), dim3(sm100::THREADS), P::SMEM, st, mq, mk, mv, pgv, cz, sc,
             (int)q_rows, (int)key_begin, (int)key_end, scale_log2, o_out, lse_out, ws_o, ws_l);
  count_launch();
  ++g_pair_launches;
  if ((rc = check_launch("pair_kernel(sm100)"))) return rc;
  if (!need_merge) return FB_OK;
  const long long warps = (long long)items * PM;
  launch_pdl(sm100::refresh_merge_kernel, dim3((unsigned)((warps + 7) / 8)), dim3(256), 0, st, sc,
             (int)q_rows, D, (const float*)ws_o, (const float*)ws_l, o_out, lse_out, PM,
             fin ? *fin : MergeFinal{});
  count_launch();
  return check_launch("refresh_merge_kernel(sm100, pair)");
}

// Two-query-tile K1 (fb_sm100_quad.cuh).  Default: block-causal prefill
// (32K prompt 7.72 ms vs 8.67 on CTA pairs and 9.5 single-CTA); the
// non-causal C5 refresh keeps the single-CTA kernel (1.65 vs 1.53 ms -- the
// 256-row stream-K ranges drift off the lock-step L2 reuse, as the pair's do).
// FB_K1_QUAD=0 / 1: never / every shape with > 128 query rows (diagnostics);
// fb_debug_set_quad overrides (tests).
static int g_quad_override = -1;
void set_quad_mode(int m) { g_quad_override = m; }
static long long g_quad_launches = 0;
long long quad_launches() { return g_quad_launches; }
static int quad_mode() {  // 0 never, 1 always, 2 block-causal only
  if (g_quad_override >= 0) return g_quad_override;
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("FB_K1_QUAD");
    m = e == nullptr ? 2 : (e[0] == '0' ? 0 : 1);
  }
  return m;
}
static bool quad_enabled() { return quad_mode() != 0; }

static int launch_quad_128(const __nv_bfloat16* k, const CUtensorMap& mq, const CUtensorMap& mk,
                           const CUtensorMap& mv, int64_t groups, int64_t q_rows, int64_t key_begin,
                           int64_t key_end, double scale, float* o_out, float* lse_out, void* ws,
                           size_t ws_bytes, cudaStream_t st, const sm100::Causal* causal,
                           const int32_t* glist, int64_t n_list, const MergeFinal* fin,
                           const sm100::Paged* paged) {
  constexpr int D = 128;
  using Q = sm100::quad::QCfg<D>;
  const sm100::Paged pgv = paged ? *paged : sm100::Paged{nullptr, 0, 1};
  constexpr int PM = sm100::pair::PM;
  const int m_tiles = (int)((q_rows + PM - 1) / PM);
  const int items = (int)((glist ? n_list : groups) * m_tiles);
  const long long tpi = (key_end - key_begin + sm100::BN - 1) / sm100::BN;
  if (items <= 0 || tpi <= 0) return -1;
  if (causal && fin != nullptr) return -1;
  sm100::Causal cz{1, 0, 0};
  if (causal) cz = *causal;
  sm100::Sched sc{(long long)items * tpi, (int)tpi, m_tiles, items, 0, nullptr, glist};
  sc.kv_keep = m_tiles > 1 && kv_keep_enabled();
  {
    static int rot = -1;  // FB_QUAD_ROT=0: no key-tile rotation (diagnostics)
    if (rot < 0) {
      const char* e = getenv("FB_QUAD_ROT");
      rot = (e != nullptr && e[0] == '0') ? 0 : 1;
    }
    sc.rot = causal == nullptr ? rot : 0;
  }
  float* ws_o = nullptr;
  float* ws_l = nullptr;
  bool need_merge;
  if (causal) {
    sc.rr = 1;
    sc.tpi = 0;
    sc.ctas = std::min(num_sms(), items);
    need_merge = false;
  } else {
    sc.ctas = (int)std::min<long long>(num_sms(), sc.T);
    need_merge = !(sc.T % sc.ctas == 0 && (sc.T / sc.ctas) % tpi == 0);
    const bool split = need_merge;
    if (fin != nullptr) need_merge = true;
    if (split) {
      const size_t need = (size_t)2 * sc.ctas * PM * (D + 1) * sizeof(float);
      if (ws == nullptr || ws_bytes < need) return -1;
      ws_o = reinterpret_cast<float*>(ws);
      ws_l = ws_o + (size_t)2 * sc.ctas * PM * D;
    }
  }
  auto kern = sm100::quad::quad_kernel<D, 0>;
  static int qpoly = -1;  // FB_QUAD_POLY=2 / 3 / 4: every n-th exp2 pair on the FMA pipes (diagnostics)
  if (qpoly < 0) {
    const char* e = getenv("FB_QUAD_POLY");
    qpoly = e ? atoi(e) : 0;
    cudaFuncSetAttribute(sm100::quad::quad_kernel<D, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Q::SMEM);
    cudaFuncSetAttribute(sm100::quad::quad_kernel<D, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Q::SMEM);
    cudaFuncSetAttribute(sm100::quad::quad_kernel<D, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Q::SMEM);
    cudaFuncSetAttribute(sm100::quad::quad_kernel<D, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Q::SMEM);
  }
  if (qpoly == 2) kern = sm100::quad::quad_kernel<D, 2>;
  if (qpoly == 3) kern = sm100::quad::quad_kernel<D, 3>;
  if (qpoly == 4) kern = sm100::quad::quad_kernel<D, 4>;
  if (qpoly == 9) {  // diagnostics: no softmax (TMA + MMA pipeline only)
    kern = sm100::quad::quad_kernel<D, -1>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Q::SMEM);
  }
  const int threads = sm100::THREADS;
  const float scale_log2 = (float)(scale * 1.4426950408889634);
  int rc;
  launch_pdl(kern, dim3((unsigned)sc.ctas), dim3(threads), Q::SMEM, st, mq, mk, mv, pgv, cz, sc,
             (int)q_rows, (int)key_begin, (int)key_end, scale_log2, o_out, lse_out, ws_o, ws_l);
  count_launch();
  ++g_quad_launches;
  if ((rc = check_launch("quad_kernel(sm100)"))) return rc;
  if (!need_merge) return FB_OK;
  const long long warps = (long long)items * PM;
  launch_pdl(sm100::refresh_merge_kernel, dim3((unsigned)((warps + 7) / 8)), dim3(256), 0, st, sc,
             (int)q_rows, D, (const float*)ws_o, (const float*)ws_l, o_out, lse_out, PM,
             fin ? *fin : MergeFinal{});
  count_launch();
  return check_launch("refresh_merge_kernel(sm100, quad)");
}

// Cluster split-K (few items, e.g. C3 b=1 shards, C2 b <= 4, C4 K8): every
// item runs on one cluster of CTAs that merge their partials through DSMEM at
// the end of the kernel (no split workspace, no merge kernel; a MergeFinal is
// applied in the same pass).  FB_K1_CLUSTER=0 never, 1 whenever feasible,
// default: when the stream-K plan would need the split-merge kernel.
static int g_cluster_override = -1;
void set_k1_cluster_mode(int m) { g_cluster_override = m; }
static int k1_cluster_mode() {
  if (g_cluster_override >= 0) return g_cluster_override;
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("FB_K1_CLUSTER");
    m = e == nullptr ? 2 : atoi(e);
  }
  return m;
}
static int g_fin_whole_override = -1;
void set_k1_fin_whole(int m) { g_fin_whole_override = m; }
static bool k1_fin_whole_enabled() {
  if (g_fin_whole_override >= 0) return g_fin_whole_override == 1;
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FB_K1_FIN_WHOLE");
    v = (e != nullptr && e[0] == '0') ? 0 : 1;
  }
  return v != 0;
}
// grid-barrier split-K: 0 off, 1 instead of the split-merge kernel (default),
// 2 also instead of the in-kernel owner merge (FB_K1_GBAR / fb_debug_set_k1_gbar)
static int g_gbar_override = -1;
void set_k1_gbar_mode(int m) { g_gbar_override = m; }
static int k1_gbar_mode() {
  if (g_gbar_override >= 0) return g_gbar_override;
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FB_K1_GBAR");
    v = e == nullptr ? 1 : atoi(e);
  }
  return v;
}
static long long g_cluster_launches = 0;
long long k1_cluster_launches() { return g_cluster_launches; }

// co-resident clusters of `cl` refresh-kernel CTAs (one CTA per SM)
template <int D, bool GATHER>
static int k1_max_clusters(int cl) {
  static int cache[17] = {};
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (cache[cl] == 0) {
    auto kern = sm100::refresh_kernel<D, GATHER, 0, sm100::K1_POLY, true, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm100::Cfg<D>::SMEM);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)cl);
    cfg.blockDim = dim3(sm100::THREADS);
    cfg.dynamicSmemBytes = sm100::Cfg<D>::SMEM;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = cl;
    a[0].val.clusterDim.y = 1;
    a[0].val.clusterDim.z = 1;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    cache[cl] = n > 0 ? n : -1;
  }
  return cache[cl] > 0 ? cache[cl] : 0;
}

// diagnostics: FB_K8_DIAG=2 skips the split-merge kernel after a gather launch
// (round 2 also measured gathering contiguous rows, FB_K8_DIAG=1: slower)
static int k8_diag() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FB_K8_DIAG");
    v = e ? atoi(e) : 0;
  }
  return v;
}

// Gather::atoms on / off (FB_GATHER_ATOMS=0: the two-box-per-block layout)
static int g_atoms_override = -1;
void set_gather_atoms(int m) { g_atoms_override = m; }
static bool gather_atoms_enabled() {
  if (g_atoms_override >= 0) return g_atoms_override != 0;
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FB_GATHER_ATOMS");
    v = (e != nullptr && e[0] == '0') ? 0 : 1;
  }
  return v != 0;
}

template <int D, bool GATHER>
static int launch_refresh_d(const __nv_bfloat16* q, const __nv_bfloat16* k, const __nv_bfloat16* v,
                            int64_t groups, int64_t q_rows, int64_t kv_rows_cap, int64_t key_begin,
                            int64_t key_end, double scale, float* o_out, float* lse_out, void* ws,
                            size_t ws_bytes, cudaStream_t st, const GatherSpec* gs = nullptr,
                            const int* key_len = nullptr, const sm100::Causal* causal = nullptr,
                            const int32_t* glist = nullptr, int64_t n_list = 0,
                            unsigned long long* sync_flags = nullptr, int64_t n_flags = 0,
                            const MergeFinal* fin = nullptr, const sm100::Paged* paged = nullptr,
                            int64_t num_pages = 0) {
  using C = sm100::Cfg<D>;
  CUtensorMap mq, mk, mv, mki, mvi;
  int rc;
  sm100::Gather ga{};
  int64_t tiles;
  if ((rc = make_tmap_3d(&mq, q, 2, D, q_rows, q_rows, groups, sm100::BOX_COLS, sm100::BM))) return rc;
  if constexpr (!GATHER) {
    // ragged: the whole slab is addressable; rows past each length are masked
    // (scores) and zeroed in smem (V) in the kernel
    const int64_t dim1 = (key_len && !causal) ? kv_rows_cap : key_end;
    if (paged != nullptr) {  // page pool [num_pages, page_rows, D]
      const int64_t pr = paged->page_rows;
      if ((rc = make_tmap_3d(&mk, k, 2, D, pr, pr, num_pages, sm100::BOX_COLS, sm100::BN))) return rc;
      if ((rc = make_tmap_3d(&mv, v, 2, D, pr, pr, num_pages, sm100::BOX_COLS, sm100::BN))) return rc;
    } else {
      if ((rc = make_tmap_3d(&mk, k, 2, D, dim1, kv_rows_cap, groups, sm100::BOX_COLS, sm100::BN))) return rc;
      if ((rc = make_tmap_3d(&mv, v, 2, D, dim1, kv_rows_cap, groups, sm100::BOX_COLS, sm100::BN))) return rc;
    }
    mki = mk;
    mvi = mv;
    tiles = (key_end - key_begin + sm100::BN - 1) / sm100::BN;
  } else if (D == 128 && gather_atoms_enabled() && gs->n_ext > 0 && gs->n_ext % 8 == 0 && gs->n_in > 0 &&
             gs->n_in % 8 == 0) {
    // atom layout (Gather::atoms): 5-D views {64 cols, 8 rows, 2 halves, atoms, slabs};
    // a 16-key block is one {64, 8, 2, 2, 1} box, a current-block tile one {64, 8, 2, 16, 1}
    const int box_blk[5] = {64, 8, 2, 2, 1}, box_tile[5] = {64, 8, 2, 16, 1};
    if (const PagingCtx* pc = current_paging()) {  // page pool [num_pages, page_rows, D]
      const int64_t dims[5] = {64, 8, 2, pc->page_rows / 8, pc->num_pages};
      const int64_t str[5] = {2, 256, 128, 2048, pc->page_rows * 256};
      if ((rc = make_tmap_nd(&mk, k, 5, dims, str, box_blk))) return rc;
      if ((rc = make_tmap_nd(&mv, v, 5, dims, str, box_blk))) return rc;
    } else {
      const int64_t dims[5] = {64, 8, 2, gs->n_ext / 8, groups};
      const int64_t str[5] = {2, 256, 128, 2048, kv_rows_cap * 256};
      if ((rc = make_tmap_nd(&mk, k, 5, dims, str, box_blk))) return rc;
      if ((rc = make_tmap_nd(&mv, v, 5, dims, str, box_blk))) return rc;
    }
    {
      const int64_t dims[5] = {64, 8, 2, gs->n_in / 8, groups};
      const int64_t str[5] = {2, 256, 128, 2048, gs->n_in * 256};
      if ((rc = make_tmap_nd(&mki, gs->k_in, 5, dims, str, box_tile))) return rc;
      if ((rc = make_tmap_nd(&mvi, gs->v_in, 5, dims, str, box_tile))) return rc;
    }
    ga.atoms = 1;
    ga.list = gs->list;
    ga.n_list = (int)gs->n_list;
    ga.n_ext = (int)gs->n_ext;
    ga.n_in = (int)gs->n_in;
    ga.sel_tiles = (int)((gs->n_list + 7) / 8);
    tiles = ga.sel_tiles + (gs->n_in + sm100::BN - 1) / sm100::BN;
  } else {
    // cache rows [0, n_ext) in 16-row boxes; current block [0, n_in) in 128-row boxes
    const int64_t n_ext_eff = gs->n_ext > 0 ? gs->n_ext : 1;
    if (const PagingCtx* pc = current_paging()) {  // page pool [num_pages, page_rows, D]
      if ((rc = make_tmap_3d(&mk, k, 2, D, pc->page_rows, pc->page_rows, pc->num_pages, sm100::BOX_COLS, 16)))
        return rc;
      if ((rc = make_tmap_3d(&mv, v, 2, D, pc->page_rows, pc->page_rows, pc->num_pages, sm100::BOX_COLS, 16)))
        return rc;
    } else {
      if ((rc = make_tmap_3d(&mk, k, 2, D, n_ext_eff, kv_rows_cap, groups, sm100::BOX_COLS, 16))) return rc;
      if ((rc = make_tmap_3d(&mv, v, 2, D, n_ext_eff, kv_rows_cap, groups, sm100::BOX_COLS, 16))) return rc;
    }
    if (gs->n_in > 0) {
      if ((rc = make_tmap_3d(&mki, gs->k_in, 2, D, gs->n_in, gs->n_in, groups, sm100::BOX_COLS, sm100::BN))) return rc;
      if ((rc = make_tmap_3d(&mvi, gs->v_in, 2, D, gs->n_in, gs->n_in, groups, sm100::BOX_COLS, sm100::BN))) return rc;
    } else {
      mki = mk;
      mvi = mv;
    }
    ga.list = gs->list;
    ga.n_list = (int)gs->n_list;
    ga.n_ext = (int)gs->n_ext;
    ga.n_in = (int)gs->n_in;
    ga.sel_tiles = (int)((gs->n_list + 7) / 8);
    tiles = ga.sel_tiles + (gs->n_in + sm100::BN - 1) / sm100::BN;
  }
  const bool o_bf16 = !GATHER && partial_out_bf16();
  if (o_bf16 && fin != nullptr) return fail(FB_ERR_UNSUPPORTED, "bf16 partial with a fused final merge");
  if constexpr (!GATHER && D == 128) {
    const int qm = quad_mode();
    const bool pair_forced = (g_pair_override >= 0 ? g_pair_override : pair_mode()) == 1;
    const bool quad_on = !pair_forced && (qm == 1 || (qm == 2 && causal != nullptr));
    if (quad_on && !o_bf16 && key_len == nullptr && q_rows > sm100::BM && g_k1_diag == 0) {
      const int qrc = launch_quad_128(k, mq, mk, mv, groups, q_rows, key_begin, key_end, scale, o_out, lse_out,
                                      ws, ws_bytes, st, causal, glist, n_list, fin, paged);
      if (qrc != -1) return qrc;
    }
  }
  if constexpr (!GATHER && D == 128) {
    const int pm = g_pair_override >= 0 ? g_pair_override : pair_mode();
    const bool pair_on = pm == 1 || (pm == 2 && causal != nullptr);
    if (pair_on && !o_bf16 && key_len == nullptr && q_rows > sm100::BM && g_k1_diag == 0) {
      const int prc = launch_pair_128(k, mq, mv, groups, q_rows, kv_rows_cap, key_begin, key_end, scale,
                                      o_out, lse_out, ws, ws_bytes, st, causal, glist, n_list, fin,
                                      paged, num_pages);
      if (prc != -1) return prc;
    }
  }
  auto kern = sm100::refresh_kernel<D, GATHER>;
  if constexpr (!GATHER && D == 128) {
    if (g_k1_diag == 1) kern = sm100::refresh_kernel<D, false, 1>;
    if (g_k1_diag == 2) kern = sm100::refresh_kernel<D, false, 2>;
    if (g_k1_diag == 3) kern = sm100::refresh_kernel<D, false, 0, 4>;  // 1/4 of the pairs on FMA
    if (g_k1_diag == 6) kern = sm100::refresh_kernel<D, false, 3>;     // no softmax, no P V
  }
  int ai = GATHER ? 0 : (g_k1_diag > 0 && g_k1_diag < 5 ? g_k1_diag : (g_k1_diag == 6 ? 5 : 0));
  if constexpr (!GATHER && D == 128) {
    static int poly = -1;
    if (poly < 0) {
      const char* e = getenv("FB_K1_POLY");  // diagnostics: MUFU offload share 1/POLY
      poly = e ? atoi(e) : 0;
    }
    if (g_k1_diag == 0 && poly >= 2 && poly <= 4) {
      kern = poly == 2 ? sm100::refresh_kernel<D, false, 0, 2>
             : poly == 3 ? sm100::refresh_kernel<D, false, 0, 3> : sm100::refresh_kernel<D, false, 0, 4>;
      ai = 5 + poly;
    }
  }
  // group subset: items over the listed groups only (tensor maps span all groups)
  RefreshPlan p = plan_refresh(glist ? n_list : groups, q_rows, D, std::max<int64_t>(tiles, 1) * sm100::BN);
  sm100::Sched sc{p.T, p.tpi, p.m_tiles, p.items, p.ctas, nullptr, glist};
  sc.kv_keep = p.m_tiles > 1 && kv_keep_enabled();
  sc.o_bf16 = o_bf16 ? 1 : 0;
  {
    // V from a second producer thread: measured on the gathered path (C4
    // cached sparse step, 16 small boxes per K / V tile) 11 % faster at 50 %
    // density, 4 % at 10 %; ~1 % slower on the dense streams (C2 / C3 / C5),
    // so dense keeps one producer.  FB_K1_VPROD=0 / 1 forces it (diagnostics).
    static int vp = -2;
    if (vp == -2) {
      const char* e = getenv("FB_K1_VPROD");
      vp = e == nullptr ? -1 : (e[0] == '0' ? 0 : 1);
    }
    sc.vprod = vp >= 0 ? vp : (GATHER ? 1 : 0);
  }
  float* ws_o = nullptr;
  float* ws_l = nullptr;
  unsigned long long* flags = nullptr;  // in-kernel split merge (uniform items only)
  MergeFinal kfin{};                    // final merge applied by the cluster reduction
  bool need_merge;
  sm100::Causal cz{1, 0, 0};
  if (causal) cz = *causal;
  if (key_len != nullptr || causal != nullptr) {
    const size_t pre = align_up((size_t)(p.items + 1) * sizeof(long long), 256);
    if (ws == nullptr || ws_bytes < refresh_sm100_ragged_workspace_bytes(groups, q_rows, D))
      return fail(FB_ERR_VALUE, "ragged / block-causal refresh needs its workspace");
    long long* prefix = reinterpret_cast<long long*>(ws);
    if (causal)
      causal_prefix_kernel<<<1, 1024, 0, st>>>(p.items, p.m_tiles, (int)q_rows, cz, prefix, (int)sm100::BM);
    else
      ragged_prefix_kernel<<<1, 1024, 0, st>>>(key_len, p.items, p.m_tiles, (int)key_begin,
                                               (int)key_end, prefix);
    count_launch();
    if ((rc = check_launch("prefix_kernel"))) return rc;
    sc.prefix = prefix;
    sc.tpi = 0;
    sc.ctas = num_sms();
    p.ctas = sc.ctas;
    ws_o = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + pre);
    ws_l = ws_o + (size_t)2 * sc.ctas * sm100::BM * D;
    need_merge = true;
  } else {
    if (ws == nullptr || ws_bytes < p.ws_bytes) {
      // no room for split partials: one CTA per whole item (no split, no workspace)
      p.ctas = p.items;
      sc.ctas = p.items;
    } else {
      ws_o = reinterpret_cast<float*>(ws);
      ws_l = ws_o + (size_t)2 * p.ctas * sm100::BM * D;
      if (sync_flags != nullptr && n_flags >= p.ctas) flags = sync_flags;
    }
    need_merge = !(p.T % p.ctas == 0 && (p.T / p.ctas) % p.tpi == 0);  // items never split
    // split items are merged inside the kernel when every CTA is resident at
    // once (one per SM: the waits always make progress) and an item spans at
    // most 3 CTAs (the owner merges <= 2 partials; measured at b = 1, where an
    // item spans ~19 CTAs, the parallel merge kernel is 2.6x faster)
    int max_span = 3;
    if (const char* e = getenv("FB_K1_MAXSPAN")) max_span = std::max(2, atoi(e));  // diagnostics
    const bool short_spans = (long long)(max_span - 1) * (p.T / p.ctas) >= p.tpi;
    if (need_merge && flags != nullptr && short_spans && p.ctas <= num_sms() && g_k1_diag != 5)
      need_merge = false;
    else
      flags = nullptr;
    // the merge kernel finishes every row (fused K3).  (Measured: the owner CTAs
    // doing this final merge themselves, C4 K8 at 10 % density with items over
    // ~5 CTAs, 64.5 vs 44.9 us -- the owners wait for CTAs that finish last.)
    if (fin != nullptr) {
      need_merge = true;
      flags = nullptr;
      // items one CTA finishes apply the final merge in their epilogue (the
      // merge kernel then only finishes split items): the C5 large-block
      // cached step wrote / re-read every row's fp32 partial (FB_K1_FIN_WHOLE=0: off)
      if (k1_fin_whole_enabled()) {
        sc.fin_whole = 1;
        kfin = *fin;
        // every item whole (C5: 444 items of 37 tiles = 3 per CTA): nothing left
        // for the merge kernel -- no launch
        if (p.T % p.ctas == 0 && (p.T / p.ctas) % p.tpi == 0) need_merge = false;
      }
    }
    // cluster split-K instead of the merge kernel: the largest cluster that
    // gives every item its own cluster in one wave, >= 2 tiles per CTA.  Auto
    // mode: clusters of <= 4 CTAs, and only while the CTAs' tile count stays
    // within 3 of the stream-K plan's (measured, scripts/ab_cluster.py: C2 b=4
    // 90 vs 97 us, C4 K8 at 10 % density 39 vs 45 us; clusters of 8 / 16 --
    // C2 b=2 / b=1, C3 b=1 shards -- 1.3-1.6x slower, their launch waits for
    // whole free GPC slices)
    const int cm = k1_cluster_mode();
    if (cm != 0 && g_k1_diag == 0 && (cm == 1 || need_merge)) {
      const long long per_streamk = (p.T + p.ctas - 1) / p.ctas;
      for (int cl = cm == 1 ? 16 : 4; cl >= 2; cl >>= 1) {
        if ((long long)p.items * cl > num_sms() || p.tpi < 2 * cl) continue;
        if (ws == nullptr || ws_bytes < (size_t)p.items * cl * sm100::BM * (D + 1) * sizeof(float)) continue;
        if (cm != 1 && (p.tpi + cl - 1) / cl > per_streamk + 3) continue;
        if (k1_max_clusters<D, GATHER>(cl) < p.items) continue;
        sc.clus = cl;
        p.ctas = sc.ctas = p.items * cl;
        ws_o = reinterpret_cast<float*>(ws);  // one partial slot per CTA
        ws_l = ws_o + (size_t)p.ctas * sm100::BM * D;
        need_merge = false;
        flags = nullptr;
        if (fin != nullptr) kfin = *fin;
        break;
      }
    }
    // grid-barrier split-K: the same per-item reduction for larger CTA groups
    // (C2 b=1 / 2, C3 b=1 shards: 8-16 CTAs per item), the item's CTAs meeting
    // at a counter in the caller's sync-flag buffer instead of a cluster
    // barrier -- co-resident by construction (one CTA per SM, ctas <= SMs) --
    // so no merge-kernel launch and no GPC-placement wait
    const int gm = k1_gbar_mode();
    const bool owner_path = flags != nullptr && !need_merge && !(p.T % p.ctas == 0 && (p.T / p.ctas) % p.tpi == 0);
    if (cm == 2 && (need_merge || (gm == 2 && owner_path)) && sc.clus == 0 && g_k1_diag == 0 && gm >= 1 &&
        sync_flags != nullptr && n_flags >= 512 + 2 * (int64_t)p.items) {
      const long long per_streamk = (p.T + p.ctas - 1) / p.ctas;
      for (int k = 16; k >= 2; k >>= 1) {
        if ((long long)p.items * k > num_sms() || p.tpi < 2 * k) continue;
        if (!need_merge && (p.tpi + k - 1) / k > per_streamk + per_streamk / 5) break;  // owner path: <= +20 % tiles
        // large items (C3 b >= 4, C2 b >= 4): the SMs a power-of-two CTA group
        // leaves idle cost more than the split-merge kernel (C3 b=4 P=1: 256 vs
        // 222 tiles per CTA, 0.81 vs 0.9 of peak) -- stay on stream-K
        if (need_merge && (p.tpi + k - 1) / k > per_streamk + 4) break;
        if (ws == nullptr || ws_bytes < (size_t)p.items * k * sm100::BM * (D + 1) * sizeof(float)) break;
        sc.clus = k;
        sc.gbar = 1;
        p.ctas = sc.ctas = p.items * k;
        ws_o = reinterpret_cast<float*>(ws);
        ws_l = ws_o + (size_t)p.ctas * sm100::BM * D;
        need_merge = false;
        flags = sync_flags;  // counters at flags + 512
        if (fin != nullptr) kfin = *fin;
        break;
      }
    }
  }
  const float scale_log2 = (float)(scale * 1.4426950408889634);
  sm100::Paged pgv = paged ? *paged : sm100::Paged{nullptr, 0, 1};
  if (GATHER && current_paging() != nullptr) {
    const PagingCtx* pc = current_paging();
    pgv = sm100::Paged{pc->table, (int)pc->max_pages, (int)pc->page_rows};
  }
  // lean variants: cluster split-K and / or the atom-layout gather (diagnostic
  // variants above are plain stream-K kernels)
  if (ai == 0 && (sc.clus > 0 || ga.atoms)) {
    constexpr int PL = sm100::K1_POLY;
    const bool cl = sc.clus > 0, at = GATHER && ga.atoms;
    if constexpr (GATHER) {
      kern = cl ? (at ? sm100::refresh_kernel<D, true, 0, PL, true, true>
                      : sm100::refresh_kernel<D, true, 0, PL, true, false>)
                : sm100::refresh_kernel<D, true, 0, PL, false, true>;
    } else {
      kern = sm100::refresh_kernel<D, false, 0, PL, true, false>;
    }
    ai = 10 + (cl ? 1 : 0) + (at ? 2 : 0);
  }
  static bool attr[14] = {};
  if (!attr[ai]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (ai >= 10) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr[ai] = true;
  }
  CUtensorMap mws{};  // cluster split-K: TMA-store view of the per-CTA partial slots
  if (sc.clus > 0) {
    ++g_cluster_launches;
    if ((rc = make_tmap_3d(&mws, ws_o, 4, D, sm100::BM, sm100::BM, p.ctas, 32, sm100::BM))) return rc;
  }
  launch_pdl_cluster(kern, dim3((unsigned)p.ctas), dim3(sm100::THREADS), C::SMEM, st, sc.gbar ? 0 : sc.clus, mq, mk, mv, mki,
                     mvi, ga, pgv, cz, sc, (int)q_rows, (int)key_begin, (int)key_end, key_len, scale_log2, o_out,
                     lse_out, ws_o, ws_l, g_trace ? g_trace + (size_t)(g_trace_launch++) * 148 * 8 : nullptr,
                     flags, kfin, mws);
  count_launch();
  if ((rc = check_launch("refresh_kernel(sm100)"))) return rc;
  if (!need_merge) return FB_OK;
  if (GATHER && k8_diag() == 2) return FB_OK;  // diagnostics: gather kernel alone
  const long long warps = (long long)p.items * sm100::BM;
  launch_pdl(sm100::refresh_merge_kernel, dim3((unsigned)((warps + 7) / 8)), dim3(256), 0, st, sc,
             (int)q_rows, D, (const float*)ws_o, (const float*)ws_l, o_out, lse_out, (int)sm100::BM,
             fin ? *fin : MergeFinal{});
  count_launch();
  return check_launch("refresh_merge_kernel(sm100)");
}

int launch_refresh_sm100(const __nv_bfloat16* q, const __nv_bfloat16* k, const __nv_bfloat16* v,
                         int64_t groups, int64_t q_rows, int64_t head_dim, int64_t kv_rows_cap,
                         int64_t key_begin, int64_t key_end, double scale, float* o_out,
                         float* lse_out, void* ws, size_t ws_bytes, cudaStream_t st,
                         unsigned long long* sync_flags, int64_t n_flags, const MergeFinal* fin) {
  if (head_dim == 128)
    return launch_refresh_d<128, false>(q, k, v, groups, q_rows, kv_rows_cap, key_begin, key_end,
                                        scale, o_out, lse_out, ws, ws_bytes, st, nullptr, nullptr,
                                        nullptr, nullptr, 0, sync_flags, n_flags, fin);
  if (head_dim == 64)
    return launch_refresh_d<64, false>(q, k, v, groups, q_rows, kv_rows_cap, key_begin, key_end,
                                       scale, o_out, lse_out, ws, ws_bytes, st, nullptr, nullptr,
                                       nullptr, nullptr, 0, sync_flags, n_flags, fin);
  return FB_ERR_UNSUPPORTED;
}

int launch_refresh_ragged_sm100(const __nv_bfloat16* q, const __nv_bfloat16* k,
                                const __nv_bfloat16* v, int64_t groups, int64_t q_rows,
                                int64_t head_dim, int64_t kv_rows_cap, int64_t key_begin,
                                const int32_t* key_end, double scale, float* o_out, float* lse_out,
                                void* ws, size_t ws_bytes, cudaStream_t st) {
  if (head_dim == 128)
    return launch_refresh_d<128, false>(q, k, v, groups, q_rows, kv_rows_cap, key_begin, kv_rows_cap,
                                        scale, o_out, lse_out, ws, ws_bytes, st, nullptr, key_end);
  if (head_dim == 64)
    return launch_refresh_d<64, false>(q, k, v, groups, q_rows, kv_rows_cap, key_begin, kv_rows_cap,
                                       scale, o_out, lse_out, ws, ws_bytes, st, nullptr, key_end);
  return FB_ERR_UNSUPPORTED;
}

// Block-causal (prefill / commit) attention reading the prompt's keys through
// a paged cache: same rows and limits as launch_block_causal_sm100.
int launch_block_causal_paged_sm100(const __nv_bfloat16* q, const __nv_bfloat16* k_pages,
                                    const __nv_bfloat16* v_pages, int64_t num_pages, int64_t page_rows,
                                    const int32_t* page_table, int64_t max_pages, int64_t groups,
                                    int64_t q_rows, int64_t head_dim, int64_t n_q, int64_t n_prefix,
                                    int64_t block, double scale, float* o_out, float* lse_out, void* ws,
                                    size_t ws_bytes, cudaStream_t st) {
  if (page_rows <= 0 || page_rows % sm100::BN != 0)
    return fail(FB_ERR_UNSUPPORTED, "page_rows must be a positive multiple of 128");
  const sm100::Paged pg{page_table, (int)max_pages, (int)page_rows};
  const sm100::Causal cz{(int)n_q, (int)block, (int)n_prefix};
  const int64_t cap = max_pages * page_rows, end = n_prefix + n_q;
  if (head_dim == 128)
    return launch_refresh_d<128, false>(q, k_pages, v_pages, groups, q_rows, cap, 0, end, scale, o_out,
                                        lse_out, ws, ws_bytes, st, nullptr, nullptr, &cz, nullptr, 0,
                                        nullptr, 0, nullptr, &pg, num_pages);
  if (head_dim == 64)
    return launch_refresh_d<64, false>(q, k_pages, v_pages, groups, q_rows, cap, 0, end, scale, o_out,
                                       lse_out, ws, ws_bytes, st, nullptr, nullptr, &cz, nullptr, 0,
                                       nullptr, 0, nullptr, &pg, num_pages);
  return FB_ERR_UNSUPPORTED;
}

// Paged KV cache: K1 over per-sequence lengths whose keys
// live in a shared page pool addressed through per-group page tables.
int launch_refresh_paged_sm100(const __nv_bfloat16* q, const __nv_bfloat16* k_pages,
                               const __nv_bfloat16* v_pages, int64_t num_pages, int64_t page_rows,
                               const int32_t* page_table, int64_t max_pages, int64_t groups,
                               int64_t q_rows, int64_t head_dim, const int32_t* key_len, double scale,
                               float* o_out, float* lse_out, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (page_rows <= 0 || page_rows % sm100::BN != 0)
    return fail(FB_ERR_UNSUPPORTED, "page_rows must be a positive multiple of 128");
  const sm100::Paged pg{page_table, (int)max_pages, (int)page_rows};
  const int64_t cap = max_pages * page_rows;
  if (head_dim == 128)
    return launch_refresh_d<128, false>(q, k_pages, v_pages, groups, q_rows, cap, 0, cap, scale, o_out,
                                        lse_out, ws, ws_bytes, st, nullptr, key_len, nullptr, nullptr, 0,
                                        nullptr, 0, nullptr, &pg, num_pages);
  if (head_dim == 64)
    return launch_refresh_d<64, false>(q, k_pages, v_pages, groups, q_rows, cap, 0, cap, scale, o_out,
                                       lse_out, ws, ws_bytes, st, nullptr, key_len, nullptr, nullptr, 0,
                                       nullptr, 0, nullptr, &pg, num_pages);
  return FB_ERR_UNSUPPORTED;
}

// Head-gated refresh: K1 over a device list of groups only;
// the other groups' outputs are left untouched.
int launch_refresh_groups_sm100(const __nv_bfloat16* q, const __nv_bfloat16* k, const __nv_bfloat16* v,
                                int64_t groups, int64_t q_rows, int64_t head_dim, int64_t kv_rows_cap,
                                int64_t key_begin, int64_t key_end, const int32_t* glist,
                                int64_t n_list, double scale, float* o_out, float* lse_out, void* ws,
                                size_t ws_bytes, cudaStream_t st) {
  if (head_dim == 128)
    return launch_refresh_d<128, false>(q, k, v, groups, q_rows, kv_rows_cap, key_begin, key_end,
                                        scale, o_out, lse_out, ws, ws_bytes, st, nullptr, nullptr,
                                        nullptr, glist, n_list);
  if (head_dim == 64)
    return launch_refresh_d<64, false>(q, k, v, groups, q_rows, kv_rows_cap, key_begin, key_end,
                                       scale, o_out, lse_out, ws, ws_bytes, st, nullptr, nullptr,
                                       nullptr, glist, n_list);
  return FB_ERR_UNSUPPORTED;
}

// Block-causal (prefill / commit) attention: keys [0, n_prefix + n_q) of every
// slab, per-row block-causal limits; writes the fp32 attention output + LSE.
int launch_block_causal_sm100(const __nv_bfloat16* q, const __nv_bfloat16* k, const __nv_bfloat16* v,
                              int64_t groups, int64_t q_rows, int64_t head_dim, int64_t kv_rows_cap,
                              int64_t n_q, int64_t n_prefix, int64_t block, double scale,
                              float* o_out, float* lse_out, void* ws, size_t ws_bytes,
                              cudaStream_t st) {
  const sm100::Causal cz{(int)n_q, (int)block, (int)n_prefix};
  const int64_t end = n_prefix + n_q;
  if (head_dim == 128)
    return launch_refresh_d<128, false>(q, k, v, groups, q_rows, kv_rows_cap, 0, end, scale, o_out,
                                        lse_out, ws, ws_bytes, st, nullptr, nullptr, &cz);
  if (head_dim == 64)
    return launch_refresh_d<64, false>(q, k, v, groups, q_rows, kv_rows_cap, 0, end, scale, o_out,
                                       lse_out, ws, ws_bytes, st, nullptr, nullptr, &cz);
  return FB_ERR_UNSUPPORTED;
}

size_t gather_sm100_workspace_bytes(int64_t groups, int64_t q_rows, int64_t head_dim,
                                    int64_t n_list, int64_t n_in) {
  const int64_t tiles = (n_list + 7) / 8 + (n_in + sm100::BN - 1) / sm100::BN;
  if (tiles <= 0 || groups <= 0 || q_rows <= 0) return 0;
  return plan_refresh(groups, q_rows, head_dim, tiles * sm100::BN).ws_bytes;
}

int launch_gather_sm100(const __nv_bfloat16* q, const __nv_bfloat16* k, const __nv_bfloat16* v,
                        int64_t groups, int64_t q_rows, int64_t head_dim, int64_t kv_rows_cap,
                        const GatherSpec& gs, double scale, float* o_out, float* lse_out, void* ws,
                        size_t ws_bytes, cudaStream_t st, const MergeFinal* fin) {
  const int64_t tiles = (gs.n_list + 7) / 8 + (gs.n_in + sm100::BN - 1) / sm100::BN;
  if (tiles == 0 && fin == nullptr)
    return launch_fill_sentinel<float, float>(o_out, lse_out, groups * q_rows, head_dim, st);
  if (tiles == 0) return FB_ERR_UNSUPPORTED;  // caller combines the sentinel itself
  if (head_dim == 128)
    return launch_refresh_d<128, true>(q, k, v, groups, q_rows, kv_rows_cap, 0, 0, scale, o_out,
                                       lse_out, ws, ws_bytes, st, &gs, nullptr, nullptr, nullptr, 0,
                                       nullptr, 0, fin);
  if (head_dim == 64)
    return launch_refresh_d<64, true>(q, k, v, groups, q_rows, kv_rows_cap, 0, 0, scale, o_out,
                                      lse_out, ws, ws_bytes, st, &gs, nullptr, nullptr, nullptr, 0,
                                      nullptr, 0, fin);
  return FB_ERR_UNSUPPORTED;
}


// K5 on sm_100a: q_rows <= 128 (one query tile per group), kbs == 16.
bool score_sm100_supported(int64_t head_dim, int64_t q_rows, int64_t kbs) {
  return (head_dim == 64 || head_dim == 128) && q_rows <= 128 && kbs == 16;
}

// FB_K5_TWO_PASS=1 / fb_debug_set_k5_mode(1): the LSE + MASS two-pass scoring
// (diagnostics / A-B); fb_debug_set_k5_mode(-1) returns to the environment
static int g_k5_mode = -1;
static long long g_k5_fused_launches = 0;
void set_k5_mode(int m) { g_k5_mode = m; }
long long k5_fused_launches() { return g_k5_fused_launches; }
static bool k5_two_pass() {
  if (g_k5_mode >= 0) return g_k5_mode == 1;
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FB_K5_TWO_PASS");
    v = (e != nullptr && e[0] == '1') ? 1 : 0;
  }
  return v != 0;
}

// two-pass workspace: row LSEs + split partials; the fused pass adds the
// per-(row, 16-key block) sums A and the per-(row, half tile) maxima
static size_t score_two_pass_bytes(int64_t groups, int64_t q_rows, int64_t n_ext, int64_t n_in) {
  const int64_t tiles = (n_ext + 127) / 128 + (n_in + 127) / 128;
  const RefreshPlan p = plan_refresh(groups, q_rows, 0, tiles * 128);
  return align_up((size_t)groups * q_rows * sizeof(float), 256) + align_up(p.ws_bytes, 256);
}
static size_t score_fused_extra_bytes(int64_t groups, int64_t n_ext) {
  return (size_t)groups * ((n_ext + 127) / 128) * 12 * sm100::BM * sizeof(float);  // A: 8, mt: 4 per row
}
// the fused pass's per-(row, block) sums are ~19 % of the K bytes; past 256 MB
// of them the workspace query reports the two-pass size instead (the launcher
// then takes the two-pass kernels: 2 x K bytes, no proportional scratch)
constexpr size_t SCORE_FUSED_MAX_EXTRA = size_t(256) << 20;
size_t score_sm100_workspace_bytes(int64_t groups, int64_t q_rows, int64_t n_ext, int64_t n_in) {
  const size_t extra = score_fused_extra_bytes(groups, n_ext);
  return score_two_pass_bytes(groups, q_rows, n_ext, n_in) + (extra <= SCORE_FUSED_MAX_EXTRA ? extra : 0);
}
size_t score_sm100_min_workspace_bytes(int64_t groups, int64_t q_rows, int64_t n_ext, int64_t n_in) {
  return score_two_pass_bytes(groups, q_rows, n_ext, n_in);
}

template <int D>
static int launch_score_d(const __nv_bfloat16* q, const __nv_bfloat16* k, const __nv_bfloat16* k_in,
                          int64_t groups, int64_t q_rows, int64_t cap, int64_t n_ext, int64_t n_in,
                          double scale, double* mass, void* ws, size_t ws_bytes, cudaStream_t st) {
  using C = sm100::ScoreCfg<D>;
  CUtensorMap mq, mk, mki;
  int rc;
  if ((rc = make_tmap_3d(&mq, q, 2, D, q_rows, q_rows, groups, sm100::BOX_COLS, sm100::BM))) return rc;
  const PagingCtx* pc = current_paging();
  if (pc != nullptr) {  // page pool [num_pages, page_rows, D]
    if ((rc = make_tmap_3d(&mk, k, 2, D, pc->page_rows, pc->page_rows, pc->num_pages, sm100::BOX_COLS,
                           sm100::BN)))
      return rc;
  } else if ((rc = make_tmap_3d(&mk, k, 2, D, n_ext, cap, groups, sm100::BOX_COLS, sm100::BN))) {
    return rc;
  }
  const sm100::Paged pgv = pc ? sm100::Paged{pc->table, (int)pc->max_pages, (int)pc->page_rows}
                              : sm100::Paged{nullptr, 0, 1};
  if (n_in > 0) {
    if ((rc = make_tmap_3d(&mki, k_in, 2, D, n_in, n_in, groups, sm100::BOX_COLS, sm100::BN))) return rc;
  } else {
    mki = mk;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sm100::score_kernel<D, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    cudaFuncSetAttribute(sm100::score_kernel<D, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    attr = true;
  }
  const int ext_tiles = (int)((n_ext + 127) / 128);
  const int in_tiles = (int)((n_in + 127) / 128);
  const float scale_log2 = (float)(scale * 1.4426950408889634);
  const int64_t nb = (n_ext + 15) / 16;
  float* lse2 = reinterpret_cast<float*>(ws);
  const size_t lse_bytes = align_up((size_t)groups * q_rows * sizeof(float), 256);
  float* ws_l = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + lse_bytes);
  // LSE (or fused) pass over ext + internal keys
  RefreshPlan p = plan_refresh(groups, q_rows, 0, (int64_t)(ext_tiles + in_tiles) * 128);
  const size_t two = score_two_pass_bytes(groups, q_rows, n_ext, n_in);
  if (ws_bytes < two) return fail(FB_ERR_VALUE, "score workspace too small");
  sm100::Sched sc{p.T, p.tpi, p.m_tiles, p.items, p.ctas, nullptr};
  if (!k5_two_pass() && score_fused_extra_bytes(groups, n_ext) <= SCORE_FUSED_MAX_EXTRA &&
      ws_bytes >= two + score_fused_extra_bytes(groups, n_ext)) {
    float* ws_a = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + two);
    float* ws_m = ws_a + (size_t)groups * ext_tiles * 8 * sm100::BM;
    using CF = sm100::ScoreFusedCfg<D>;
    auto kern = sm100::score_fused_kernel<D, sm100::K5_POLY_DEFAULT>;
    static int poly = -3;
    if (poly < -2) {  // diagnostics: FB_K5_POLY = 0 / 2 / 4 exp2 pairs of 8 on the FMA pipes;
                      // -1 the TMA + MMA pipeline alone, -2 the math without the A / mt stores
      const char* e = getenv("FB_K5_POLY");
      poly = e ? atoi(e) : sm100::K5_POLY_DEFAULT;
      cudaFuncSetAttribute(sm100::score_fused_kernel<D, sm100::K5_POLY_DEFAULT>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM);
      cudaFuncSetAttribute(sm100::score_fused_kernel<D, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM);
      cudaFuncSetAttribute(sm100::score_fused_kernel<D, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM);
      cudaFuncSetAttribute(sm100::score_fused_kernel<D, -1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM);
      cudaFuncSetAttribute(sm100::score_fused_kernel<D, -2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM);
    }
    if (poly == -1) kern = sm100::score_fused_kernel<D, -1>;
    if (poly == -2) kern = sm100::score_fused_kernel<D, -2>;
    if (poly == 2) kern = sm100::score_fused_kernel<D, 2>;
    if (poly == 4) kern = sm100::score_fused_kernel<D, 4>;
    launch_pdl(kern, dim3((unsigned)p.ctas), dim3(sm100::SCORE_FUSED_THREADS), CF::SMEM,
               st, mq, mk, mki, pgv, sc, (int)q_rows, (int)n_ext, (int)n_in, ext_tiles, scale_log2,
               lse2, ws_l, ws_a, ws_m);
    count_launch();
    ++g_k5_fused_launches;
    if ((rc = check_launch("score_kernel<fused>"))) return rc;
    // ~4 CTAs per SM in one wave, at least 8 tiles (one per warp) each
    const int64_t want = std::max<int64_t>(1, 4 * num_sms() / std::max<int64_t>(groups, 1));
    const int tpc = (int)std::max<int64_t>(8, (ext_tiles + want - 1) / want);
    const dim3 grid((unsigned)((ext_tiles + tpc - 1) / tpc), (unsigned)groups);
    launch_pdl(sm100::score_mass_kernel, grid, dim3(256), 0, st, sc, (int)q_rows, ext_tiles, (int)nb, tpc,
               (const float*)lse2, (const float*)ws_l, (const float*)ws_a, (const float*)ws_m, mass);
    count_launch();
    return check_launch("score_mass_kernel");
  }
  launch_pdl(sm100::score_kernel<D, 0>, dim3((unsigned)p.ctas), dim3(sm100::SCORE_THREADS), C::SMEM,
             st, mq, mk, mki, pgv, sc, (int)q_rows, (int)n_ext, (int)n_in, ext_tiles, scale_log2,
             (const float*)nullptr, lse2, ws_l, (double*)nullptr, (int)nb);
  count_launch();
  if ((rc = check_launch("score_kernel<lse>"))) return rc;
  if (!(p.T % p.ctas == 0 && (p.T / p.ctas) % p.tpi == 0)) {
    const long long rows = groups * p.m_tiles * (long long)sm100::BM;
    launch_pdl(sm100::score_lse_merge_kernel, dim3((unsigned)((rows + 255) / 256)), dim3(256), 0, st, sc,
               (int)q_rows, (const float*)ws_l, lse2);
    count_launch();
    if ((rc = check_launch("score_lse_merge_kernel"))) return rc;
  }
  // MASS pass over the external keys
  RefreshPlan pm = plan_refresh(groups, q_rows, 0, (int64_t)ext_tiles * 128);
  sm100::Sched sm{pm.T, pm.tpi, pm.m_tiles, pm.items, pm.ctas, nullptr};
  launch_pdl(sm100::score_kernel<D, 1>, dim3((unsigned)pm.ctas), dim3(sm100::SCORE_THREADS), C::SMEM,
             st, mq, mk, mki, pgv, sm, (int)q_rows, (int)n_ext, (int)n_in, ext_tiles, scale_log2,
             (const float*)lse2, (float*)nullptr, (float*)nullptr, mass, (int)nb);
  count_launch();
  return check_launch("score_kernel<mass>");
}

int launch_score_sm100(const __nv_bfloat16* q, const __nv_bfloat16* k, const __nv_bfloat16* k_in,
                       int64_t groups, int64_t q_rows, int64_t head_dim, int64_t cap, int64_t n_ext,
                       int64_t n_in, double scale, double* mass, void* ws, size_t ws_bytes,
                       cudaStream_t st) {
  if (head_dim == 128)
    return launch_score_d<128>(q, k, k_in, groups, q_rows, cap, n_ext, n_in, scale, mass, ws, ws_bytes, st);
  if (head_dim == 64)
    return launch_score_d<64>(q, k, k_in, groups, q_rows, cap, n_ext, n_in, scale, mass, ws, ws_bytes, st);
  return FB_ERR_UNSUPPORTED;
}

}  // namespace fb
