// K1 with two query tiles per CTA (experimental, FB_K1_QUAD=1): the
// tensor-bound shapes' alternative to the CTA pair.  One CTA owns a 256-row
// item (query tiles a and b of one group); every 128-key K / V tile is loaded
// once and used by both tiles, halving the TMA / L2 traffic per FLOP like the
// pair kernel, but without a cross-CTA hand-off:
//   warp 0      TMA producer (Qa, Qb per segment; K, V tiles, 2-stage ring)
//   warp 1      MMA issuer: per tile t  PV_a(t-1), S_a(t), PV_b(t-1), S_b(t)
//               (S_x(t) overwrites P_x(t-1) in TMEM only after PV_x(t-1) was
//               issued; the tensor pipe runs in order)
//   warp 2      TMEM allocator (512 columns: Sa | Sb | Oa | Ob)
//   warps 4-7   softmax of query tile a (every key tile), warps 8-11 of b;
//               each writes its own rows -- no cross-warpgroup merge.
// s_full_x(t) arrives after S_x(t), hence after PV_x(t-1): a warpgroup can
// rescale its O without waiting on a separate PV barrier.
namespace quad {

using pair::PM;
using pair::Seg;
using pair::SegIter;

template <int D>
struct QCfg {
  static_assert(D == 128, "quad kernel: head_dim 128");
  static constexpr int STAGES = 2;
  static constexpr uint32_t BOX_BYTES = BM * BOX_COLS * 2;   // 16 KB
  static constexpr uint32_t TILE_BYTES = (D / BOX_COLS) * BOX_BYTES;  // 32 KB
  static constexpr uint32_t OFF_QA = 0;
  static constexpr uint32_t OFF_QB = OFF_QA + TILE_BYTES;
  static constexpr uint32_t OFF_K = OFF_QB + TILE_BYTES;
  static constexpr uint32_t OFF_V = OFF_K + STAGES * TILE_BYTES;
  static constexpr uint32_t OFF_BAR = OFF_V + STAGES * TILE_BYTES;
  static constexpr uint32_t SMEM = OFF_BAR + 512 + 1024;
};
static_assert(QCfg<128>::SMEM <= 232448, "quad kernel shared memory exceeds 227 KB");

struct QBars {
  uint64_t q_full, q_empty;
  uint64_t k_full[2], k_empty[2], v_full[2], v_empty[2];
  uint64_t s_full[2], p_ready[2];
  uint64_t o_full, o_empty;
  uint32_t tmem_base;
};

template <int D, int POLY = 0>
__global__ void __launch_bounds__(THREADS, 1)
quad_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
            const __grid_constant__ CUtensorMap tm_v, Paged pg, Causal cz, Sched sc, int q_rows, int key_begin,
            int key_end, float scale_log2, float* __restrict__ o_out, float* __restrict__ lse_out,
            float* __restrict__ ws_o, float* __restrict__ ws_l) {
  using C = QCfg<D>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  QBars* bar = reinterpret_cast<QBars*>(smem + C::OFF_BAR);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  if (!sc.rr) sc.resolve();
  const long long t_begin = sc.rr ? 0 : sc.start(cta);
  const long long t_end = sc.rr ? 0 : sc.start(cta + 1);

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
    for (int x = 0; x < 2; ++x) {
      ptx::mbar_init(&bar->s_full[x], 1);
      ptx::mbar_init(&bar->p_ready[x], 4);  // the tile's softmax warps
    }
    ptx::mbar_init(&bar->o_full, 1);
    ptx::mbar_init(&bar->o_empty, 8);  // every softmax warp
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(&bar->tmem_base, TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = bar->tmem_base;
  ptx::pdl_wait();
  ptx::pdl_launch_dependents();

  if (warp < 4) {
    ptx::setmaxnreg_dec<56>();
    if (warp == 0 && lane == 0) {
      // ---------------------------------------------------------- TMA producer
      const uint64_t keep = ptx::policy_evict_last();
      const uint64_t stream = (cz.blk > 0 || sc.kv_keep) ? ptx::policy_evict_last() : ptx::policy_evict_first();
      int j = 0, seg = 0;
      SegIter it{t_begin, t_begin, t_end, -1, 0, cta, (int)gridDim.x};
      Seg sg;
      for (; it.next(sc, cz, q_rows, sg); ++seg) {
        const int g = sc.group_of(sg.item), mt = sc.mtile_of(sg.item);
        if (seg > 0) ptx::mbar_wait(&bar->q_empty, (seg - 1) & 1);
        ptx::mbar_expect_tx(&bar->q_full, 2 * C::TILE_BYTES);
        for (int x = 0; x < 2; ++x)
          for (int b = 0; b < D / BOX_COLS; ++b)
            ptx::tma_load_3d(smem + (x ? C::OFF_QB : C::OFF_QA) + b * C::BOX_BYTES, &tm_q, &bar->q_full,
                             b * BOX_COLS, mt * PM + x * BM, g, keep);
        for (long long t = sg.t0; t < sg.t0 + sg.n; ++t, ++j) {
          const int s = j % C::STAGES;
          const uint32_t ph = (j / C::STAGES) & 1;
          int lt = (int)(t - sg.ib);
          if (sg.shift) lt = (lt + sg.shift) % sc.tpi;
          int row = key_begin + lt * BN;
          int slab = g;
          if (pg.table != nullptr) {  // paged cache: the tile's page, row inside it
            slab = __ldg(pg.table + (long long)g * pg.max_pages + row / pg.page_rows);
            row %= pg.page_rows;
          }
          ptx::mbar_wait(&bar->k_empty[s], ph ^ 1);
          ptx::mbar_expect_tx(&bar->k_full[s], C::TILE_BYTES);
          for (int b = 0; b < D / BOX_COLS; ++b)
            ptx::tma_load_3d(smem + C::OFF_K + s * C::TILE_BYTES + b * C::BOX_BYTES, &tm_k, &bar->k_full[s],
                             b * BOX_COLS, row, slab, stream);
          ptx::mbar_wait(&bar->v_empty[s], ph ^ 1);
          ptx::mbar_expect_tx(&bar->v_full[s], C::TILE_BYTES);
          for (int b = 0; b < D / BOX_COLS; ++b)
            ptx::tma_load_3d(smem + C::OFF_V + s * C::TILE_BYTES + b * C::BOX_BYTES, &tm_v, &bar->v_full[s],
                             b * BOX_COLS, row, slab, stream);
        }
      }
    } else if (warp == 1 && lane == 0) {
      // ---------------------------------------------------------- MMA issuer
      constexpr uint32_t IDESC_S = ptx::idesc_bf16_f32(BM, BN, false);
      constexpr uint32_t IDESC_O = ptx::idesc_bf16_f32(BM, D, true);
      int jg = 0, seg = 0;
      SegIter it{t_begin, t_begin, t_end, -1, 0, cta, (int)gridDim.x};
      Seg sg;
      for (; it.next(sc, cz, q_rows, sg); ++seg) {
        const int n = sg.n;
        ptx::mbar_wait(&bar->q_full, seg & 1);
        ptx::tc_fence_after();
        for (int t = 0; t <= n; ++t) {
          for (int x = 0; x < 2; ++x) {
            if (t > 0) {  // PV_x(t-1): P_x from TMEM, V from smem
              const int jj = jg + t - 1;
              const int s = jj % C::STAGES;
              ptx::mbar_wait(&bar->p_ready[x], jj & 1);
              if (x == 0) ptx::mbar_wait(&bar->v_full[s], (jj / C::STAGES) & 1);
              if (t == 1 && seg > 0 && x == 0) ptx::mbar_wait(&bar->o_empty, (seg - 1) & 1);
              ptx::tc_fence_after();
              const uint32_t v_base = ptx::smem_u32(smem + C::OFF_V + s * C::TILE_BYTES);
#pragma unroll
              for (int kk = 0; kk < BN / 16; ++kk)
                ptx::mma_ts(tmem + (x ? 384u : 256u), tmem + (x ? 128u : 0u) + kk * 8,
                            ptx::sdesc_sw128(v_base + kk * 2048, C::BOX_BYTES, 1024), IDESC_O,
                            (t > 1 || kk > 0) ? 1u : 0u);
              if (x == 1) ptx::tc_commit(&bar->v_empty[s]);
              if (x == 1 && t == n) ptx::tc_commit(&bar->o_full);
            }
            if (t < n) {  // S_x(t) = Q_x K(t)^T
              const int j = jg + t;
              const int s = j % C::STAGES;
              if (x == 0) ptx::mbar_wait(&bar->k_full[s], (j / C::STAGES) & 1);
              ptx::tc_fence_after();
              const uint32_t q_base = ptx::smem_u32(smem + (x ? C::OFF_QB : C::OFF_QA));
              const uint32_t k_base = ptx::smem_u32(smem + C::OFF_K + s * C::TILE_BYTES);
#pragma unroll
              for (int kk = 0; kk < D / 16; ++kk) {
                const uint32_t off = (kk / 4) * C::BOX_BYTES + (kk % 4) * 32;
                ptx::mma_ss(tmem + (x ? 128u : 0u), ptx::sdesc_sw128(q_base + off, 16, 1024),
                            ptx::sdesc_sw128(k_base + off, 16, 1024), IDESC_S, kk > 0);
              }
              ptx::tc_commit(&bar->s_full[x]);
              if (x == 1) {
                ptx::tc_commit(&bar->k_empty[s]);
                if (t == n - 1) ptx::tc_commit(&bar->q_empty);
              }
            }
          }
        }
        jg += n;
      }
    }
  } else {
    ptx::setmaxnreg_inc<224>();
    // ------------------------------------------------------------ softmax
    const int x = (warp - 4) >> 2;  // query tile a (0) or b (1)
    const int wq = warp & 3;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const int row = wq * 32 + lane;
    const uint32_t s_col = x ? 128u : 0u, o_col = x ? 384u : 256u;
    uint32_t r[32];
    float s[BN];
    int jg = 0, seg = 0;
    SegIter it{t_begin, t_begin, t_end, -1, 0, cta, (int)gridDim.x};
    Seg sg;
    for (; it.next(sc, cz, q_rows, sg); ++seg) {
      const int item = sg.item;
      const int lt0 = (int)(sg.t0 - sg.ib);
      const int n = sg.n;
      const int kb = key_begin + lt0 * BN;
      const int mt = sc.mtile_of(item);
      const int grow = mt * PM + x * BM + row;
      int ke = min(kb + n * BN, key_end);
      if (cz.blk > 0) ke = min(ke, cz.row_limit(grow));
      float m_used = -INFINITY;
      float l = 0.f;
      for (int t = 0; t < n; ++t) {
        const int j = jg + t;
        ptx::mbar_wait(&bar->s_full[x], j & 1);
        ptx::tc_fence_after();
        if constexpr (POLY < 0) {  // diagnostics: the TMA + MMA pipeline without the softmax
          m_used = 0.f;
          l = 1.f;
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&bar->p_ready[x]);
          continue;
        }
#pragma unroll
        for (int c = 0; c < BN / 32; ++c)
          ptx::tmem_ld32(tmem + lane_off + s_col + c * 32, reinterpret_cast<uint32_t*>(s) + c * 32);
        ptx::tmem_wait_ld();
        {
          // (rotated: the tile's own key range, clipped at the range end)
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
            const float alpha = m_new == -INFINITY ? 1.f : ptx::ex2(m_used - m_new);
            if (t >= 1) {
              // s_full_x(t) arrived after S_x(t), which the MMA thread issued
              // after PV_x(t-1): O_x holds every P V so far
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
        if (lane == 0) ptx::mbar_arrive(&bar->p_ready[x]);
      }
      jg += n;

      // ---------------------------------------------------------- segment epilogue
      const bool whole = sg.whole;
      const int g = sc.group_of(item);
      const bool live = grow < q_rows;
      const long long orow = (long long)g * q_rows + grow;
      const float iz = l > 0.f ? 1.f / l : 0.f;
      const float lse = l > 0.f ? (m_used + log2f(l)) * 0.69314718055994530942f : -INFINITY;
      float* dst;
      if (whole) {
        dst = live ? o_out + orow * D : nullptr;
      } else {
        const long long slot = sc.slot(cta, item) * PM + x * BM + row;
        dst = ws_o + slot * D;
        ws_l[slot] = lse;
      }
      ptx::mbar_wait(&bar->o_full, seg & 1);
      ptx::tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        ptx::tmem_ld32(tmem + lane_off + o_col + c * 32, r);
        ptx::tmem_wait_ld();
        if (dst != nullptr) {
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * iz;
          ptx::st_row32(dst + c * 32, v);
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&bar->o_empty);
      if (whole && live) lse_out[orow] = lse;
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, TMEM_COLS);
  }
}

}  // namespace quad
