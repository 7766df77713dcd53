// K1 on a CTA pair (cta_group::2) -- the tensor-bound refresh / prefill path.
//
// Same contract as refresh_kernel (attention_partial over a key range,
// attention.py:136-182; block-causal rows for prefill, simulator.py:297-354),
// for problems with many query rows per kv group (video chunks, C5: 4680 rows
// per head; prefill: 4 * n_q rows per group), where the single-CTA kernel is
// bound by shared-memory bandwidth, not HBM: its SS QK^T reads 128 B/clk of
// A + B operands at the full MMA rate and TMA writes another 64 KB per tile.
//
// Here two CTAs of a cluster (one TPC) share one M = 256 MMA: CTA r holds
// query rows [256 mt + 128 r, +128) (A and D split by rows), K rows
// [64 r, +64) of each 128-key tile and V columns [64 r, +64) (B split by N).
// Per CTA and key tile: A 32 KB + B 16 KB for QK^T, 16 KB of V for P V, 32 KB
// of TMA fill -- 96 KB instead of 160 KB at the same MMA work.
//
//   warp 0      TMA producer (both CTAs; bytes land on the leader's barriers)
//   warp 1      MMA issuer (leader only): S_j = Q K_j^T (M=256, N=128) into
//               TMEM S[j&1] of both CTAs, O[w] += P_j V_j (TS, P from TMEM)
//   warp 2      TMEM allocator (cta_group::2, 512 columns: S0|S1|O0|O1)
//   warps 4-11  two softmax warpgroups on alternate key tiles (both CTAs, own
//               rows), as refresh_kernel: lazy rescale, exp2-domain, packed
//               fp32 pairs, exact two-warpgroup merge in the epilogue
// Pair-wide barriers: every MMA commit is multicast to both CTAs; P-ready and
// O-drained arrivals go to the leader (one per warp).  Split items write
// normalised partials to the workspace (slot = 2 pair + {first,last} segment,
// 256 rows) and refresh_merge_kernel merges them (bm = 256).
namespace pair {

constexpr int PM = 256;  // query rows per pair tile
constexpr int HN = 64;   // key rows (QK^T) / V columns (PV) per CTA and tile

template <int D>
struct PCfg {
  static_assert(D == 128, "pair kernel: head_dim 128");
  static constexpr int STAGES = 5;
  static constexpr uint32_t QBOX = BM * BOX_COLS * 2;        // 128 rows x 128 B = 16 KB
  static constexpr uint32_t KBOX = HN * BOX_COLS * 2;        // 64 rows x 128 B = 8 KB
  static constexpr uint32_t Q_BYTES = (D / BOX_COLS) * QBOX;  // 32 KB
  static constexpr uint32_t K_BYTES = (D / BOX_COLS) * KBOX;  // 16 KB (64 keys)
  static constexpr uint32_t V_BYTES = BN * BOX_COLS * 2;      // 16 KB (128 keys x 64 cols)
  static constexpr uint32_t OFF_Q = 0;
  static constexpr uint32_t OFF_K = OFF_Q + Q_BYTES;
  static constexpr uint32_t OFF_V = OFF_K + STAGES * K_BYTES;
  static constexpr uint32_t OFF_BAR = OFF_V + STAGES * V_BYTES;
  static constexpr uint32_t OFF_XCH = OFF_BAR + 512;
  static constexpr uint32_t SMEM = OFF_XCH + 3 * BM * 4 + 1024;
  static constexpr uint32_t COL_S0 = 0, COL_S1 = 128, COL_O0 = 256, COL_O1 = 384;
};

struct PBars {
  uint64_t q_full, q_empty;
  uint64_t k_full[8], k_empty[8], v_full[8], v_empty[8];
  uint64_t s_full[2], p_ready[2];
  uint64_t pv_done[2], o_full, o_empty;
  uint32_t tmem_base;
};
static_assert(sizeof(PBars) <= 512, "pair barrier block overflows its smem slot");
static_assert(PCfg<128>::SMEM <= 232448, "pair kernel shared memory exceeds 227 KB");

// A pair's work as a sequence of segments (part of one item each).
//  * stream-K (sc.rr == 0): the pair's contiguous tile range [t_begin, t_end);
//  * round-robin whole items (sc.rr == 1, block-causal prefill): pair p runs
//    items p, p + P, p + 2P, ... of one group after another, each in one
//    segment (no split partials, no merge kernel), so at any time all pairs
//    stream the same group's keys and its K/V (16.8 MB at a 32K prompt) stays
//    in L2.  Within a group the items go longest first (query positions
//    descending, heads interleaved) when 256-row tiles do not straddle heads.
struct Seg {
  int item;
  long long ib, t0;  // item's first tile, segment's first tile (same space)
  int n;             // tiles in the segment
  bool whole;
  int shift;         // key-tile rotation (Sched::rot): local tile lt reads key tile (lt + shift) % tpi
};
struct SegIter {
  long long t, t_begin, t_end;
  int item, k, pr, npairs;
  __device__ __forceinline__ bool next(const Sched& sc, const Causal& cz, int q_rows, Seg& s) {
    s.shift = 0;
    if (sc.rr) {
      const int idx = k * npairs + pr;
      if (idx >= sc.items) return false;
      ++k;
      const int gi = idx / sc.m_tiles, r = idx % sc.m_tiles;
      int mt = r;
      if (cz.n_q % PM == 0 && sc.m_tiles % (cz.n_q / PM) == 0) {
        const int tph = cz.n_q / PM, heads = sc.m_tiles / tph;
        mt = (r % heads) * tph + (tph - 1 - r / heads);
      }
      s.item = gi * sc.m_tiles + mt;
      const int r0 = mt * PM, r1 = min(r0 + PM, q_rows) - 1;
      const int lim = (r0 / cz.n_q != r1 / cz.n_q) ? cz.n_prefix + cz.n_q : cz.row_limit(r1);
      s.ib = 0;
      s.t0 = 0;
      s.n = (lim + BN - 1) / BN;
      s.whole = true;
      return true;
    }
    if (t >= t_end) return false;
    item = sc.item_next(t, item);
    s.item = item;
    s.ib = sc.item_begin(item);
    s.t0 = t;
    const long long ie = sc.item_end(item);
    s.n = (int)(min(t_end, ie) - t);
    s.whole = s.ib >= t_begin && ie <= t_end;
    // Key-tile rotation (attention over an item's keys is order-free): every
    // CTA starts streaming at key tile 0 of its first segment and whole items
    // start at the CTA's clock, so the CTAs sharing a head read the same K/V
    // tiles at about the same time (L2 reuse without lock-step items).  A
    // split item's part [x, y) reads key tiles [tpi - y, tpi - x): the parts
    // stay disjoint and cover the item.
    if (sc.rot && sc.prefix == nullptr) {
      const int tpi = sc.tpi;
      const int x = (int)(t - s.ib), y = x + s.n;
      s.shift = s.whole ? (int)((t - t_begin) % tpi) : (int)(((long long)2 * tpi - x - y) % tpi);
    }
    t += s.n;
    return true;
  }
};

template <int D, int POLY = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
pair_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
            const __grid_constant__ CUtensorMap tm_v, Paged pg, Causal cz, Sched sc, int q_rows, int key_begin,
            int key_end, float scale_log2, float* __restrict__ o_out, float* __restrict__ lse_out,
            float* __restrict__ ws_o, float* __restrict__ ws_l) {
  using C = PCfg<D>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  PBars* bar = reinterpret_cast<PBars*>(smem + C::OFF_BAR);
  float* xch = reinterpret_cast<float*>(smem + C::OFF_XCH);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int pr = blockIdx.x >> 1;  // pair index = stream-K "CTA"
  const int npairs = gridDim.x >> 1;
  if (!sc.rr) sc.resolve();
  const long long t_begin = sc.rr ? 0 : sc.start(pr);
  const long long t_end = sc.rr ? 0 : sc.start(pr + 1);

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
      ptx::mbar_init(&bar->p_ready[b], 8);   // 4 warps x 2 CTAs
      ptx::mbar_init(&bar->pv_done[b], 1);
    }
    ptx::mbar_init(&bar->o_full, 1);
    ptx::mbar_init(&bar->o_empty, 16);       // 8 softmax warps x 2 CTAs
    ptx::fence_barrier_init();
  }
  ptx::cluster_sync();  // both CTAs' barriers initialised before any remote arrive / TMA
  if (warp == 2) ptx::tmem_alloc2(&bar->tmem_base, TMEM_COLS);  // after the cluster barrier
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = bar->tmem_base;
  ptx::pdl_wait();
  ptx::pdl_launch_dependents();

  if (warp < 4) {
    ptx::setmaxnreg_dec<56>();
    if (warp == 0) {
      // ---------------------------------------------------------- TMA producer
      if (lane == 0) {
        const uint64_t keep = ptx::policy_evict_last();
        const uint64_t stream = (cz.blk > 0 || sc.kv_keep) ? ptx::policy_evict_last() : ptx::policy_evict_first();
        int j = 0, seg = 0;
        SegIter it{t_begin, t_begin, t_end, -1, 0, pr, npairs};
        Seg sg;
        for (; it.next(sc, cz, q_rows, sg); ++seg) {
          const long long ib = sg.ib;
          long long t = sg.t0;
          const long long seg_end = sg.t0 + sg.n;
          const int g = sc.group_of(sg.item), mt = sc.mtile_of(sg.item);
          if (seg > 0) ptx::mbar_wait(&bar->q_empty, (seg - 1) & 1);
          if (leader) ptx::mbar_expect_tx(&bar->q_full, 2 * C::Q_BYTES);
          const uint32_t qf = ptx::mapa(&bar->q_full, 0);
          for (int b = 0; b < D / BOX_COLS; ++b)
            ptx::tma_load_3d_pair(smem + C::OFF_Q + b * C::QBOX, &tm_q, qf, b * BOX_COLS,
                                  mt * PM + (int)rank * BM, g, keep);
          for (; t < seg_end; ++t, ++j) {
            const int s = j % C::STAGES;
            const uint32_t ph = (j / C::STAGES) & 1;
            int lt = (int)(t - ib);
            if (sg.shift) lt = (lt + sg.shift) % sc.tpi;  // key-tile rotation (Seg::shift)
            int row = key_begin + lt * BN;
            int slab = g;
            if (pg.table != nullptr) {  // paged cache: the tile's page, row inside it
              slab = __ldg(pg.table + (long long)g * pg.max_pages + row / pg.page_rows);
              row %= pg.page_rows;
            }
            ptx::mbar_wait(&bar->k_empty[s], ph ^ 1);
            if (leader) ptx::mbar_expect_tx(&bar->k_full[s], 2 * C::K_BYTES);
            const uint32_t kf = ptx::mapa(&bar->k_full[s], 0);
            for (int b = 0; b < D / BOX_COLS; ++b)
              ptx::tma_load_3d_pair(smem + C::OFF_K + s * C::K_BYTES + b * C::KBOX, &tm_k, kf,
                                    b * BOX_COLS, row + (int)rank * HN, slab, stream);
            ptx::mbar_wait(&bar->v_empty[s], ph ^ 1);
            if (leader) ptx::mbar_expect_tx(&bar->v_full[s], 2 * C::V_BYTES);
            ptx::tma_load_3d_pair(smem + C::OFF_V + s * C::V_BYTES, &tm_v, ptx::mapa(&bar->v_full[s], 0),
                                  (int)rank * HN, row, slab, stream);
          }
        }
      }
    } else if (warp == 1) {
      // ---------------------------------------------------------- MMA issuer (leader)
      if (leader && lane == 0) {
        constexpr uint32_t IDESC_S = ptx::idesc_bf16_f32(PM, BN, false);
        constexpr uint32_t IDESC_O = ptx::idesc_bf16_f32(PM, D, true);
        const uint32_t q_base = ptx::smem_u32(smem + C::OFF_Q);
        int jg = 0, seg = 0;
        SegIter it{t_begin, t_begin, t_end, -1, 0, pr, npairs};
        Seg sg;
        for (; it.next(sc, cz, q_rows, sg); ++seg) {
          const int n = sg.n;
          ptx::mbar_wait(&bar->q_full, seg & 1);
          ptx::tc_fence_after();
          for (int t = 0; t <= n; ++t) {
            if (t < n) {
              const int j = jg + t;
              const int s = j % C::STAGES;
              ptx::mbar_wait(&bar->k_full[s], (j / C::STAGES) & 1);
              ptx::tc_fence_after();
              const uint32_t k_base = ptx::smem_u32(smem + C::OFF_K + s * C::K_BYTES);
              const uint32_t d_s = tmem + ((j & 1) ? C::COL_S1 : C::COL_S0);
#pragma unroll
              for (int kk = 0; kk < D / 16; ++kk) {
                ptx::mma2_ss(d_s, ptx::sdesc_sw128(q_base + (kk / 4) * C::QBOX + (kk % 4) * 32, 16, 1024),
                             ptx::sdesc_sw128(k_base + (kk / 4) * C::KBOX + (kk % 4) * 32, 16, 1024),
                             IDESC_S, kk > 0);
              }
              ptx::tc_commit2(&bar->k_empty[s]);
              ptx::tc_commit2(&bar->s_full[j & 1]);
              if (t == n - 1) ptx::tc_commit2(&bar->q_empty);
            }
            if (t > 0) {
              const int jj = jg + t - 1;
              const int s = jj % C::STAGES;
              ptx::mbar_wait(&bar->p_ready[jj & 1], (jj >> 1) & 1);
              ptx::mbar_wait(&bar->v_full[s], (jj / C::STAGES) & 1);
              if (t == 1 && seg > 0) ptx::mbar_wait(&bar->o_empty, (seg - 1) & 1);
              ptx::tc_fence_after();
              const uint32_t v_base = ptx::smem_u32(smem + C::OFF_V + s * C::V_BYTES);
              const uint32_t p_tmem = tmem + ((jj & 1) ? C::COL_S1 : C::COL_S0);
              const uint32_t o_tmem = tmem + ((jj & 1) ? C::COL_O1 : C::COL_O0);
#pragma unroll
              for (int kk = 0; kk < BN / 16; ++kk)
                ptx::mma2_ts(o_tmem, p_tmem + kk * 8, ptx::sdesc_sw128(v_base + kk * 2048, C::V_BYTES, 1024),
                             IDESC_O, (t > 2 || kk > 0) ? 1u : 0u);
              ptx::tc_commit2(&bar->v_empty[s]);
              ptx::tc_commit2(&bar->pv_done[jj & 1]);
              if (t == n) ptx::tc_commit2(&bar->o_full);
            }
          }
          jg += n;
        }
      }
    }
  } else {
    ptx::setmaxnreg_inc<224>();
    // ------------------------------------------------------------ softmax
    const int wg = (warp - 4) >> 2;
    const int wq = warp & 3;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const int row = wq * 32 + lane;
    const uint32_t s_col = wg ? C::COL_S1 : C::COL_S0;
    const uint32_t o_col = wg ? C::COL_O1 : C::COL_O0;
    const uint32_t p_ready_l = ptx::mapa(&bar->p_ready[wg], 0);
    const uint32_t o_empty_l = ptx::mapa(&bar->o_empty, 0);
    uint32_t r[32];
    float s[BN];
    int jg = 0, seg = 0;
    SegIter it{t_begin, t_begin, t_end, -1, 0, pr, npairs};
    Seg sg;
    for (; it.next(sc, cz, q_rows, sg); ++seg) {
      const int item = sg.item;
      const long long ib = sg.ib;
      const int lt0 = (int)(sg.t0 - ib);
      const int n = sg.n;
      const int kb = key_begin + lt0 * BN;
      const int mt = sc.mtile_of(item);
      const int grow = mt * PM + (int)rank * BM + row;
      int ke = min(kb + n * BN, key_end);
      if (cz.blk > 0) ke = min(ke, cz.row_limit(grow));
      float m_used = -INFINITY;
      float l = 0.f;
      for (int t = ((jg & 1) == wg) ? 0 : 1; t < n; t += 2) {
        const int j = jg + t;
        ptx::mbar_wait(&bar->s_full[wg], (j >> 1) & 1);
        ptx::tc_fence_after();
        if constexpr (POLY == -1) {  // diagnostics (FB_PAIR_POLY=-1): no softmax, P = stale S
          m_used = 0.f;
          l += 1.f;
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive_cluster(p_ready_l);
          continue;
        }
#pragma unroll
        for (int c = 0; c < BN / 32; ++c)
          ptx::tmem_ld32(tmem + lane_off + s_col + c * 32, reinterpret_cast<uint32_t*>(s) + c * 32);
        ptx::tmem_wait_ld();
        {
          const int valid = sg.shift ? key_end - (key_begin + ((lt0 + t + sg.shift) % sc.tpi) * BN)
                                     : ke - (kb + t * BN);
          if (valid < BN) {
#pragma unroll
            for (int i = 0; i < BN; ++i)
              if (i >= valid) s[i] = -INFINITY;
          }
        }
        auto exp_tile = [&](float neg) -> float {
          const uint64_t sc2 = ptx::f2_pack(scale_log2, scale_log2), ng2 = ptx::f2_pack(neg, neg);
          uint64_t ls4[4] = {0, 0, 0, 0};
#pragma unroll
          for (int c = 0; c < BN / 64; ++c) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const uint64_t x2 = ptx::f2_fma(ptx::f2_pack(s[c * 64 + 2 * i], s[c * 64 + 2 * i + 1]), sc2, ng2);
              float x0, x1;
              ptx::f2_unpack(x2, x0, x1);
              float p0, p1;
              if (POLY > 0 && (i % (POLY > 0 ? POLY : 1)) == (POLY > 0 ? POLY : 1) - 1) {
                ptx::ex2_poly2(x2, p0, p1);  // every POLY-th pair on the FMA pipes (MUFU offload)
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
        float lt = 0.f;
        bool full = __any_sync(0xffffffffu, m_used == -INFINITY);
        if (!full) {
          lt = exp_tile(-m_used);
          full = __any_sync(0xffffffffu, !(lt <= 4294967296.f));
        }
        if (full) {
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
          lt = exp_tile(m_used == -INFINITY ? 0.f : -m_used);
        }
        l += lt;
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(p_ready_l);
      }
      jg += n;

      // ---------------------------------------------------------- segment epilogue
      const bool whole = sg.whole;
      const int g = sc.group_of(item);
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
        const float iz = z > 0.f ? 1.f / z : 0.f;
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
      const float c0 = wg == 0 ? c_own : c_oth;
      const float c1 = wg == 0 ? c_oth : c_own;
      float* dst;
      if (whole) {
        dst = live ? o_out + orow * D : nullptr;
      } else {
        const long long slot = sc.slot(pr, item) * PM + (int)rank * BM + row;
        dst = ws_o + slot * D;
        if (wg == 1) ws_l[slot] = lse;
      }
      ptx::mbar_wait(&bar->o_full, seg & 1);
      ptx::tc_fence_after();
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
          ptx::st_row32(dst + c * 32, v);
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_cluster(o_empty_l);  // MMA may overwrite O
      if (whole && live && wg == 1) lse_out[orow] = lse;
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();  // no CTA leaves while its peer may still signal it
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc2(tmem, TMEM_COLS);
  }
}

}  // namespace pair
