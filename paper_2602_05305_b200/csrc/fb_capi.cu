// extern "C" entry points (include/flashblock_b200.h): validation, precision
// dispatch, split-KV planning.  No host synchronisation, no allocation.
#include "fb_kernels.cuh"

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>

namespace fb {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}
int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return FB_OK;
}
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("FB_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------- split planning

struct SplitPlan {
  int splits;
  int64_t per_split;  // keys per split
};

// SIMT: aim for ~2 waves of 4-warp CTAs; at least 256 keys per split.
static SplitPlan plan_simt(int64_t groups, int64_t q_rows, int64_t n, size_t ws_bytes,
                           size_t bytes_per_split) {
  const int64_t ctas = groups * ((q_rows + 15) / 16);
  int64_t want = (2 * (int64_t)num_sms() * 4 + ctas - 1) / std::max<int64_t>(ctas, 1);
  want = std::min<int64_t>(want, (n + 255) / 256);
  want = std::min<int64_t>(want, 1024);
  if (bytes_per_split > 0) want = std::min<int64_t>(want, (int64_t)(ws_bytes / bytes_per_split));
  want = std::max<int64_t>(want, 1);
  int64_t per = (n + want - 1) / want;
  per = (per + 31) / 32 * 32;
  const int splits = (int)((n + per - 1) / per);
  return {splits, per};
}

template <typename Mode>
static size_t split_bytes(int64_t rows, int64_t d) {
  return (size_t)rows * (size_t)(d + 1) * sizeof(typename Mode::Ta) + 256;
}

template <typename Mode>
static CombineList strided_list(void* ws, int splits, int64_t rows, int64_t d) {
  CombineList L{};
  L.n = splits;
  L.strided = true;
  L.o[0] = ws;
  L.l[0] = reinterpret_cast<typename Mode::Ta*>(ws) + (size_t)splits * rows * d;
  L.o_stride = rows * d;
  L.l_stride = rows;
  return L;
}

// Partial over a key map into (o_out, lse_out) of the mode's partial types.
template <typename Mode, typename Map>
static int partial_any(const typename Mode::Tin* q, const Map& map, int64_t groups, int64_t q_rows,
                       int64_t d, int64_t n, double scale, typename Mode::To* o_out,
                       typename Mode::Tl* lse_out, void* ws, size_t ws_bytes, cudaStream_t st) {
  using Ta = typename Mode::Ta;
  const int64_t rows = groups * q_rows;
  const size_t per = split_bytes<Mode>(rows, d);
  SplitPlan p = plan_simt(groups, q_rows, n, ws ? ws_bytes : 0, per);
  constexpr bool direct_ok = std::is_same<Ta, typename Mode::To>::value &&
                             std::is_same<Ta, typename Mode::Tl>::value;
  MergeOut<Mode> none{};
  if (p.splits == 1 && direct_ok) {
    return launch_partial_simt<Mode, false, false>(q, map, groups, q_rows, d, p.per_split, 1, scale,
                                                   reinterpret_cast<Ta*>(o_out),
                                                   reinterpret_cast<typename Mode::Tl*>(lse_out),
                                                   none, st);
  }
  if (ws == nullptr || ws_bytes < per * p.splits)
    return fail(FB_ERR_VALUE, "workspace too small (query fb_partial_workspace_bytes)");
  Ta* wo = reinterpret_cast<Ta*>(ws);
  Ta* wl = wo + (size_t)p.splits * rows * d;
  int rc = launch_partial_simt<Mode, false, false>(q, map, groups, q_rows, d, p.per_split, p.splits,
                                                   scale, wo, reinterpret_cast<typename Mode::Tl*>(wl),
                                                   none, st);
  if (rc) return rc;
  return launch_combine<Ta, Ta, Ta, typename Mode::To, typename Mode::Tl>(
      strided_list<Mode>(ws, p.splits, rows, d), rows, d, o_out, lse_out, nullptr, st);
}

static int check_dtype(int dt) {
  if (dt != FB_F64 && dt != FB_F32 && dt != FB_BF16) return fail(FB_ERR_VALUE, "unknown dtype");
  return FB_OK;
}

static const char* const PB16_MSG =
    "FB_PARTIAL_BF16 needs the tcgen05 refresh path (head_dim 64 / 128, 16-byte aligned, non-empty range)";

// dtype with an optional FB_PARTIAL_BF16 bit (BF16 mode only): strips the bit
static int split_partial_bf16(int& dt, bool& pb) {
  pb = (dt & FB_PARTIAL_BF16) != 0;
  dt &= ~FB_PARTIAL_BF16;
  if (int rc = check_dtype(dt)) return rc;
  if (pb && dt != FB_BF16) return fail(FB_ERR_VALUE, "FB_PARTIAL_BF16 applies to FB_BF16 mode only");
  return FB_OK;
}

template <typename Mode>
static int attention_partial_t(const void* qv, const void* kv, const void* vv, int64_t groups,
                               int64_t q_rows, int64_t d, int64_t cap, int64_t kb, int64_t ke,
                               double scale, void* o_out, void* lse_out, void* ws, size_t ws_bytes,
                               cudaStream_t st, uint64_t* sync_flags = nullptr,
                               int64_t n_flags = 0) {
  using Tin = typename Mode::Tin;
  auto* q = reinterpret_cast<const Tin*>(qv);
  auto* k = reinterpret_cast<const Tin*>(kv);
  auto* v = reinterpret_cast<const Tin*>(vv);
  auto* o = reinterpret_cast<typename Mode::To*>(o_out);
  auto* l = reinterpret_cast<typename Mode::Tl*>(lse_out);
  const int64_t rows = groups * q_rows;
  const int64_t n = ke - kb;
  if constexpr (std::is_same<Mode, ModeBF16>::value) {
    if (n == 0 && partial_out_bf16())
      return launch_fill_sentinel<__nv_bfloat16, float>(reinterpret_cast<__nv_bfloat16*>(o_out), l, rows, d, st);
  }
  if (n == 0) return launch_fill_sentinel<typename Mode::To, typename Mode::Tl>(o, l, rows, d, st);
  if constexpr (std::is_same<Mode, ModeBF16>::value) {
    if (sm100_supported(d) && ke < (int64_t(1) << 31) && q_rows < (int64_t(1) << 31) &&
        (reinterpret_cast<uintptr_t>(q) % 16 == 0) && (reinterpret_cast<uintptr_t>(k) % 16 == 0) &&
        (reinterpret_cast<uintptr_t>(v) % 16 == 0) && groups < 65536) {
      return launch_refresh_sm100(q, k, v, groups, q_rows, d, cap, kb, ke, scale, o, l, ws, ws_bytes, st,
                                  reinterpret_cast<unsigned long long*>(sync_flags), n_flags);
    }
    if (partial_out_bf16()) return fail(FB_ERR_UNSUPPORTED, PB16_MSG);
  }
  RangeMap<Tin> map{k, v, cap * d, kb, ke, d};
  return partial_any<Mode>(q, map, groups, q_rows, d, n, scale, o, l, ws, ws_bytes, st);
}

template <typename Mode>
static int internal_merge_t(const void* qv, const void* kv, const void* vv, int64_t groups,
                            int64_t q_rows, int64_t d, int64_t n_in, double scale,
                            const void* o_ext, const void* lse_ext, void* out, bool out_bf16,
                            void* lse_merged, void* o_int, void* lse_int, int32_t* empty,
                            cudaStream_t st, bool ext_early = false, bool extb = false) {
  using Tin = typename Mode::Tin;
  if constexpr (std::is_same<Mode, ModeBF16>::value) {
    auto a16 = [](const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
    if (sm100_k2_supported(d, n_in) && o_ext != nullptr && lse_ext != nullptr && a16(qv) &&
        a16(kv) && a16(vv) && a16(o_ext) && a16(out) && a16(o_int) && groups * ((q_rows + 127) / 128) < (1LL << 31))
      return launch_internal_merge_sm100(
          reinterpret_cast<const __nv_bfloat16*>(qv), reinterpret_cast<const __nv_bfloat16*>(kv),
          reinterpret_cast<const __nv_bfloat16*>(vv), groups, q_rows, d, n_in, scale, o_ext,
          reinterpret_cast<const float*>(lse_ext), out, out_bf16, reinterpret_cast<float*>(lse_merged),
          reinterpret_cast<float*>(o_int), reinterpret_cast<float*>(lse_int), empty, ext_early, extb, st);
  }
  if (extb)  // the SIMT kernel reads the mode's fp32 partial
    return fail(FB_ERR_UNSUPPORTED, "FB_PARTIAL_BF16 cached step needs the tcgen05 kernel "
                                    "(head_dim 64 / 128, 1 <= n_in <= 128, 16-byte aligned rows)");
  MergeOut<Mode> mo{};
  mo.o_ext = reinterpret_cast<const typename Mode::To*>(o_ext);
  mo.lse_ext = reinterpret_cast<const typename Mode::Tl*>(lse_ext);
  mo.out = out;
  mo.out_bf16 = out_bf16;
  mo.lse_merged = reinterpret_cast<typename Mode::Tl*>(lse_merged);
  mo.o_int = reinterpret_cast<typename Mode::To*>(o_int);
  mo.lse_int = reinterpret_cast<typename Mode::Tl*>(lse_int);
  mo.empty_rows = empty;
  RangeMap<Tin> map{reinterpret_cast<const Tin*>(kv), reinterpret_cast<const Tin*>(vv), n_in * d, 0,
                    n_in, d};
  const int64_t per = std::max<int64_t>(n_in, 1);
  return launch_partial_simt<Mode, true, false>(reinterpret_cast<const Tin*>(qv), map, groups, q_rows,
                                                d, per, 1, scale, nullptr, nullptr, mo, st);
}

template <typename Mode>
static int combine_t(int n_parts, const void* const* o_parts, const void* const* lse_parts,
                     int64_t rows, int64_t d, void* o_out, bool out_bf16, void* lse_out,
                     int32_t* empty, cudaStream_t st) {
  CombineList L{};
  L.n = n_parts;
  L.strided = false;
  for (int i = 0; i < n_parts; ++i) {
    L.o[i] = o_parts[i];
    L.l[i] = lse_parts[i];
  }
  using To = typename Mode::To;
  using Tl = typename Mode::Tl;
  using Ta = typename Mode::Ta;
  if constexpr (std::is_same<Mode, ModeBF16>::value) {
    if (out_bf16)
      return launch_combine<float, float, float, __nv_bfloat16, float>(
          L, rows, d, reinterpret_cast<__nv_bfloat16*>(o_out), reinterpret_cast<float*>(lse_out),
          empty, st);
  }
  return launch_combine<To, Tl, Ta, To, Tl>(L, rows, d, reinterpret_cast<To*>(o_out),
                                            reinterpret_cast<Tl*>(lse_out), empty, st);
}

template <typename MaskMode>
static int block_mass_t(const void* qv, const void* kv, const void* kin, int64_t groups,
                        int64_t q_rows, int64_t d, int64_t cap, int64_t n_ext, int64_t n_in,
                        int64_t kbs, double scale, double* mass, void* ws, size_t ws_bytes,
                        cudaStream_t st) {
  using Tin = typename MaskMode::Tin;
  const int64_t rows = groups * q_rows;
  double* row_lse = reinterpret_cast<double*>(ws);
  void* rest = reinterpret_cast<char*>(ws) + align_up((size_t)rows * sizeof(double), 256);
  const size_t rest_bytes = ws_bytes - align_up((size_t)rows * sizeof(double), 256);
  ConcatMap<Tin> map{reinterpret_cast<const Tin*>(kv), nullptr, reinterpret_cast<const Tin*>(kin),
                     nullptr, cap * d, n_ext, n_in, d};
  const int64_t n = n_ext + n_in;
  const size_t per = (size_t)rows * sizeof(double) + 256;
  SplitPlan p = plan_simt(groups, q_rows, n, rest_bytes, per);
  MergeOut<MaskMode> none{};
  int rc;
  if (p.splits == 1) {
    rc = launch_partial_simt<MaskMode, false, true>(reinterpret_cast<const Tin*>(qv), map, groups,
                                                    q_rows, d, p.per_split, 1, scale, nullptr,
                                                    row_lse, none, st);
  } else {
    // lognorm-only split partials: [splits][rows] doubles, combined with d = 0 columns
    double* wl = reinterpret_cast<double*>(rest);
    rc = launch_partial_simt<MaskMode, false, true>(reinterpret_cast<const Tin*>(qv), map, groups,
                                                    q_rows, d, p.per_split, p.splits, scale, nullptr,
                                                    wl, none, st);
    if (rc) return rc;
    CombineList L{};
    L.n = p.splits;
    L.strided = true;
    L.o[0] = wl;  // never read with head_dim 0
    L.l[0] = wl;
    L.o_stride = 0;
    L.l_stride = rows;
    rc = launch_combine<double, double, double, double, double>(L, rows, 0, nullptr, row_lse, nullptr, st);
  }
  if (rc) return rc;
  return launch_block_mass<MaskMode>(reinterpret_cast<const Tin*>(qv), reinterpret_cast<const Tin*>(kv),
                                     row_lse, groups, q_rows, d, cap * d, n_ext, kbs, scale, mass, st);
}

template <typename Mode>
static int sparse_partitioned_t(const void* qv, const void* kv, const void* vv, const void* kin,
                                const void* vin, int64_t groups, int64_t q_rows, int64_t d,
                                int64_t cap, int64_t n_ext, int64_t n_in, const int32_t* sel,
                                int64_t n_sel, int64_t kbs, double scale, void* o_sel, void* l_sel,
                                void* o_res, void* l_res, void* out, bool out_bf16, int32_t* empty,
                                void* ws, size_t ws_bytes, cudaStream_t st) {
  using Tin = typename Mode::Tin;
  using To = typename Mode::To;
  using Tl = typename Mode::Tl;
  if constexpr (std::is_same<Mode, ModeBF16>::value) {
    if (sm100_supported(d) && kbs == 16 && n_ext < (int64_t(1) << 31) && ws != nullptr) {
      const int64_t nb = (n_ext + kbs - 1) / kbs;
      const int64_t n_res = nb - n_sel;
      const size_t list_bytes = align_up((size_t)groups * std::max<int64_t>(n_res, 1) * 4, 256);
      const size_t need = list_bytes + std::max(
          gather_sm100_workspace_bytes(groups, q_rows, d, n_sel, n_in),
          gather_sm100_workspace_bytes(groups, q_rows, d, n_res, 0));
      if (ws_bytes >= need) {
        int32_t* res_list = reinterpret_cast<int32_t*>(ws);
        void* gws = reinterpret_cast<char*>(ws) + list_bytes;
        int rc = launch_complement(sel, groups, n_sel, nb, res_list, st);
        if (rc) return rc;
        GatherSpec gsel{sel, n_sel, n_ext, n_in, reinterpret_cast<const __nv_bfloat16*>(kin),
                        reinterpret_cast<const __nv_bfloat16*>(vin)};
        rc = launch_gather_sm100(reinterpret_cast<const __nv_bfloat16*>(qv),
                                 reinterpret_cast<const __nv_bfloat16*>(kv),
                                 reinterpret_cast<const __nv_bfloat16*>(vv), groups, q_rows, d, cap,
                                 gsel, scale, reinterpret_cast<float*>(o_sel),
                                 reinterpret_cast<float*>(l_sel), gws, ws_bytes - list_bytes, st);
        if (rc) return rc;
        GatherSpec gres{res_list, n_res, n_ext, 0, nullptr, nullptr};
        // the residual pass's merge kernel also merges the selected partial and
        // writes the step's output (K3 fused), unless no output is wanted
        const MergeFinal fin{reinterpret_cast<const float*>(o_sel), reinterpret_cast<const float*>(l_sel),
                             out, out_bf16 ? 1 : 0, empty};
        const bool fuse = out != nullptr && n_res > 0;
        rc = launch_gather_sm100(reinterpret_cast<const __nv_bfloat16*>(qv),
                                 reinterpret_cast<const __nv_bfloat16*>(kv),
                                 reinterpret_cast<const __nv_bfloat16*>(vv), groups, q_rows, d, cap,
                                 gres, scale, reinterpret_cast<float*>(o_res),
                                 reinterpret_cast<float*>(l_res), gws, ws_bytes - list_bytes, st,
                                 fuse ? &fin : nullptr);
        if (rc) return rc;
        if (out == nullptr || fuse) return FB_OK;
        const void* op[2] = {o_sel, o_res};
        const void* lp[2] = {l_sel, l_res};
        return combine_t<Mode>(2, op, lp, groups * q_rows, d, out, out_bf16, nullptr, empty, st);
      }
    }
  }
  const Tin* q = reinterpret_cast<const Tin*>(qv);
  const Tin* k = reinterpret_cast<const Tin*>(kv);
  const Tin* v = reinterpret_cast<const Tin*>(vv);
  // selected external blocks + every current-block key, fused with nothing
  SelectedMap<Tin> smap{k, v, reinterpret_cast<const Tin*>(kin), reinterpret_cast<const Tin*>(vin),
                        sel, n_sel, kbs, n_ext, n_in, cap * d, d};
  MergeOut<Mode> mo{};
  mo.o_ext = nullptr;
  mo.lse_ext = nullptr;
  mo.out = o_sel;
  mo.out_bf16 = false;
  mo.lse_merged = reinterpret_cast<Tl*>(l_sel);
  int rc = launch_partial_simt<Mode, true, false>(q, smap, groups, q_rows, d, int64_t(1) << 40, 1,
                                                  scale, nullptr, nullptr, mo, st);
  if (rc) return rc;
  // residual: the unselected external keys (partial, unmerged)
  ResidualMap<Tin> rmap{k, v, sel, n_sel, kbs, n_ext, cap * d, d};
  MergeOut<Mode> mr{};
  mr.o_ext = nullptr;
  mr.lse_ext = nullptr;
  mr.out = o_res;
  mr.out_bf16 = false;
  mr.lse_merged = reinterpret_cast<Tl*>(l_res);
  rc = launch_partial_simt<Mode, true, false>(q, rmap, groups, q_rows, d, int64_t(1) << 40, 1, scale,
                                              nullptr, nullptr, mr, st);
  if (rc) return rc;
  if (out == nullptr) return FB_OK;
  const void* op[2] = {o_sel, o_res};
  const void* lp[2] = {l_sel, l_res};
  return combine_t<Mode>(2, op, lp, groups * q_rows, d, out, out_bf16, nullptr, empty, st);
}

template <typename Mode>
static int sparse_attend_t(const void* qv, const void* kv, const void* vv, const void* kin,
                           const void* vin, int64_t groups, int64_t q_rows, int64_t d, int64_t cap,
                           int64_t n_ext, int64_t n_in, const int32_t* sel, int64_t n_sel,
                           int64_t kbs, double scale, const void* o_res, const void* l_res,
                           void* out, bool out_bf16, int32_t* empty, void* ws, size_t ws_bytes,
                           cudaStream_t st) {
  using Tin = typename Mode::Tin;
  if constexpr (std::is_same<Mode, ModeBF16>::value) {
    const int64_t rows = groups * q_rows;
    const size_t tmp_bytes = align_up((size_t)rows * (d + 1) * sizeof(float), 256);
    if (sm100_supported(d) && kbs == 16 && n_ext < (int64_t(1) << 31) && ws != nullptr &&
        ws_bytes >= tmp_bytes + gather_sm100_workspace_bytes(groups, q_rows, d, n_sel, n_in)) {
      float* o_tmp = reinterpret_cast<float*>(ws);
      float* l_tmp = o_tmp + (size_t)rows * d;
      GatherSpec gsel{sel, n_sel, n_ext, n_in, reinterpret_cast<const __nv_bfloat16*>(kin),
                      reinterpret_cast<const __nv_bfloat16*>(vin)};
      // selected-blocks partial, merged with the cached residual and written as
      // the output inside K1's merge kernel (no separate K3 launch)
      // (the selected partial itself is scratch here: skip_partial)
      const MergeFinal fin{o_res, reinterpret_cast<const float*>(l_res), out, out_bf16 ? 1 : 0, empty, 0, 1};
      int rc = launch_gather_sm100(reinterpret_cast<const __nv_bfloat16*>(qv),
                                   reinterpret_cast<const __nv_bfloat16*>(kv),
                                   reinterpret_cast<const __nv_bfloat16*>(vv), groups, q_rows, d,
                                   cap, gsel, scale, o_tmp, l_tmp,
                                   reinterpret_cast<char*>(ws) + tmp_bytes, ws_bytes - tmp_bytes, st,
                                   n_sel + n_in > 0 ? &fin : nullptr);
      if (rc) return rc;
      if (n_sel + n_in > 0) return FB_OK;
      const void* op[2] = {o_tmp, o_res};
      const void* lp[2] = {l_tmp, l_res};
      return combine_t<Mode>(o_res ? 2 : 1, op, lp, rows, d, out, out_bf16, nullptr, empty, st);
    }
  }
  SelectedMap<Tin> smap{reinterpret_cast<const Tin*>(kv), reinterpret_cast<const Tin*>(vv),
                        reinterpret_cast<const Tin*>(kin), reinterpret_cast<const Tin*>(vin),
                        sel, n_sel, kbs, n_ext, n_in, cap * d, d};
  MergeOut<Mode> mo{};
  mo.o_ext = reinterpret_cast<const typename Mode::To*>(o_res);
  mo.lse_ext = reinterpret_cast<const typename Mode::Tl*>(l_res);
  mo.out = out;
  mo.out_bf16 = out_bf16;
  mo.empty_rows = empty;
  return launch_partial_simt<Mode, true, false>(reinterpret_cast<const Tin*>(qv), smap, groups, q_rows,
                                                d, int64_t(1) << 40, 1, scale, nullptr, nullptr, mo, st);
}

template <typename Mode>
static int attention_partial_ragged_t(const void* qv, const void* kv, const void* vv, int64_t groups,
                                      int64_t q_rows, int64_t d, int64_t cap, int64_t kb,
                                      const int32_t* ends, double scale, void* o_out, void* lse_out,
                                      void* ws, size_t ws_bytes, cudaStream_t st) {
  using Tin = typename Mode::Tin;
  auto* q = reinterpret_cast<const Tin*>(qv);
  auto* k = reinterpret_cast<const Tin*>(kv);
  auto* v = reinterpret_cast<const Tin*>(vv);
  auto* o = reinterpret_cast<typename Mode::To*>(o_out);
  auto* l = reinterpret_cast<typename Mode::Tl*>(lse_out);
  if constexpr (std::is_same<Mode, ModeBF16>::value) {
    if (sm100_supported(d) && cap < (int64_t(1) << 31) &&
        ws_bytes >= refresh_sm100_ragged_workspace_bytes(groups, q_rows, d))
      return launch_refresh_ragged_sm100(q, k, v, groups, q_rows, d, cap, kb, ends, scale, o, l, ws,
                                         ws_bytes, st);
    if (partial_out_bf16()) return fail(FB_ERR_UNSUPPORTED, PB16_MSG);
  }
  // SIMT: one split per group (lengths live on the device)
  RaggedMap<Tin> map{k, v, ends, cap * d, kb, cap, d};
  MergeOut<Mode> none{};
  using Ta = typename Mode::Ta;
  constexpr bool direct_ok = std::is_same<Ta, typename Mode::To>::value &&
                             std::is_same<Ta, typename Mode::Tl>::value;
  if constexpr (direct_ok) {
    return launch_partial_simt<Mode, false, false>(q, map, groups, q_rows, d, int64_t(1) << 40, 1,
                                                   scale, reinterpret_cast<Ta*>(o),
                                                   reinterpret_cast<typename Mode::Tl*>(l), none, st);
  } else {
    const int64_t rows = groups * q_rows;
    if (ws == nullptr || ws_bytes < split_bytes<Mode>(rows, d))
      return fail(FB_ERR_VALUE, "workspace too small (fb_ragged_workspace_bytes)");
    Ta* wo = reinterpret_cast<Ta*>(ws);
    int rc = launch_partial_simt<Mode, false, false>(q, map, groups, q_rows, d, int64_t(1) << 40, 1,
                                                     scale, wo,
                                                     reinterpret_cast<typename Mode::Tl*>(wo + rows * d),
                                                     none, st);
    if (rc) return rc;
    return launch_combine<Ta, Ta, Ta, typename Mode::To, typename Mode::Tl>(
        strided_list<Mode>(ws, 1, rows, d), rows, d, o, l, nullptr, st);
  }
}

}  // namespace fb

using namespace fb;

// Scores in the dense oracle's precision: float64 for F64 / F32 inputs
// (attention_dense, attention.py:113-133, used by the commit pass at
// simulator.py:318-320), fp32 from bf16 products in BF16 mode.
template <typename Mode> struct DenseMode { using type = Mode; };
template <> struct DenseMode<ModeF32> { using type = ModeMaskF32; };

template <typename Mode>
static int block_causal_t(const void* qv, const void* kv, const void* vv, int64_t groups,
                          int64_t q_rows, int64_t d, int64_t cap, int64_t n_q, int64_t n_prefix,
                          int64_t blk, double scale, void* o_out, void* lse_out, void* ws,
                          size_t ws_bytes, cudaStream_t st) {
  using Tin = typename Mode::Tin;
  using SM = typename DenseMode<Mode>::type;
  using Ta = typename SM::Ta;
  auto* q = reinterpret_cast<const Tin*>(qv);
  auto* k = reinterpret_cast<const Tin*>(kv);
  auto* v = reinterpret_cast<const Tin*>(vv);
  auto* o = reinterpret_cast<typename Mode::To*>(o_out);
  auto* l = reinterpret_cast<typename Mode::Tl*>(lse_out);
  if constexpr (std::is_same<Mode, ModeBF16>::value) {
    if (sm100_supported(d) && cap < (int64_t(1) << 31) && groups * q_rows < (int64_t(1) << 31) &&
        ws_bytes >= refresh_sm100_ragged_workspace_bytes(groups, q_rows, d))
      return launch_block_causal_sm100(q, k, v, groups, q_rows, d, cap, n_q, n_prefix, blk, scale,
                                       o, l, ws, ws_bytes, st);
  }
  CausalMap<Tin> map{k, v, cap * d, d, n_q, blk, n_prefix};
  MergeOut<SM> none{};
  constexpr bool direct_ok = std::is_same<Ta, typename Mode::To>::value &&
                             std::is_same<Ta, typename Mode::Tl>::value;
  if constexpr (direct_ok) {
    return launch_partial_simt<SM, false, false>(q, map, groups, q_rows, d, int64_t(1) << 40, 1,
                                                 scale, reinterpret_cast<Ta*>(o),
                                                 reinterpret_cast<typename SM::Tl*>(l), none, st);
  } else {
    const int64_t rows = groups * q_rows;
    if (ws == nullptr || ws_bytes < split_bytes<SM>(rows, d))
      return fail(FB_ERR_VALUE, "workspace too small (fb_block_causal_workspace_bytes)");
    Ta* wo = reinterpret_cast<Ta*>(ws);
    int rc = launch_partial_simt<SM, false, false>(q, map, groups, q_rows, d, int64_t(1) << 40, 1,
                                                   scale, wo,
                                                   reinterpret_cast<typename SM::Tl*>(wo + rows * d),
                                                   none, st);
    if (rc) return rc;
    return launch_combine<Ta, Ta, Ta, typename Mode::To, typename Mode::Tl>(
        strided_list<SM>(ws, 1, rows, d), rows, d, o, l, nullptr, st);
  }
}

// K1 over a device list of groups (head-gated refresh).  F64 / BF16 write
// directly (SIMT or tcgen05); F32 would need a scattered combine: unsupported.
template <typename Mode>
static int attention_partial_groups_t(const void* qv, const void* kv, const void* vv, int64_t groups,
                                      int64_t q_rows, int64_t d, int64_t cap, int64_t kb, int64_t ke,
                                      const int32_t* glist, int64_t n_list, double scale, void* o_out,
                                      void* lse_out, void* ws, size_t ws_bytes, cudaStream_t st) {
  using Tin = typename Mode::Tin;
  using Ta = typename Mode::Ta;
  auto* q = reinterpret_cast<const Tin*>(qv);
  auto* k = reinterpret_cast<const Tin*>(kv);
  auto* v = reinterpret_cast<const Tin*>(vv);
  auto* o = reinterpret_cast<typename Mode::To*>(o_out);
  auto* l = reinterpret_cast<typename Mode::Tl*>(lse_out);
  if constexpr (std::is_same<Mode, ModeBF16>::value) {
    if (ke > kb && sm100_supported(d) && ke < (int64_t(1) << 31) && q_rows < (int64_t(1) << 31) &&
        (reinterpret_cast<uintptr_t>(q) % 16 == 0) && (reinterpret_cast<uintptr_t>(k) % 16 == 0) &&
        (reinterpret_cast<uintptr_t>(v) % 16 == 0) && groups < 65536)
      return launch_refresh_groups_sm100(q, k, v, groups, q_rows, d, cap, kb, ke, glist, n_list,
                                         scale, o, l, ws, ws_bytes, st);
    if (partial_out_bf16()) return fail(FB_ERR_UNSUPPORTED, PB16_MSG);
  }
  constexpr bool direct_ok = std::is_same<Ta, typename Mode::To>::value &&
                             std::is_same<Ta, typename Mode::Tl>::value;
  if constexpr (direct_ok) {
    RangeMap<Tin> map{k, v, cap * d, kb, ke, d};
    MergeOut<Mode> none{};
    return launch_partial_simt<Mode, false, false>(q, map, n_list, q_rows, d, int64_t(1) << 40, 1,
                                                   scale, reinterpret_cast<Ta*>(o),
                                                   reinterpret_cast<typename Mode::Tl*>(l), none, st,
                                                   glist);
  } else {
    return fail(FB_ERR_UNSUPPORTED, "group-subset refresh is not built for F32 mode");
  }
}

extern "C" {

const char* fb_last_error(void) { return g_last_error.c_str(); }
const char* fb_version(void) { return "fb200 0.1.0 sm_100a"; }
// Diagnostics (not in the public header): per-CTA timestamps of the refresh kernel.
FB_API void fb_debug_set_trace(void* device_buffer) { set_refresh_trace(device_buffer); }
FB_API void fb_debug_set_k1_diag(int diag) { set_k1_diag(diag); }
FB_API void fb_debug_set_pair(int on) { set_pair_enabled(on); }
FB_API int64_t fb_debug_pair_launches(void) { return (int64_t)pair_launches(); }
FB_API void fb_debug_set_quad(int m) { set_quad_mode(m); }
FB_API int64_t fb_debug_quad_launches(void) { return (int64_t)quad_launches(); }
FB_API void fb_debug_set_k1_cluster(int m) { set_k1_cluster_mode(m); }
FB_API void fb_debug_set_k1_fin_whole(int m) { set_k1_fin_whole(m); }
FB_API void fb_debug_set_gather_atoms(int m) { set_gather_atoms(m); }
FB_API void fb_debug_set_k1_gbar(int m) { set_k1_gbar_mode(m); }
FB_API int64_t fb_debug_k1_cluster_launches(void) { return (int64_t)k1_cluster_launches(); }
FB_API void fb_debug_set_k2_variant(int v) { set_k2_v2(v); }
FB_API void fb_debug_set_k2_store(int v) { set_k2_store(v); }
FB_API void fb_debug_set_k2_vsplit(int v) { set_k2_vsplit(v); }
FB_API void fb_debug_set_k5_mode(int m) { set_k5_mode(m); }
FB_API int64_t fb_debug_k5_fused_launches(void) { return (int64_t)k5_fused_launches(); }
FB_API void fb_debug_set_k2_trace(void* p, int launches) { set_k2_trace(p, launches); }
int64_t fb_launch_count(void) { return g_launches.load(); }

size_t fb_partial_workspace_bytes(int dtype, int64_t groups, int64_t q_rows, int64_t head_dim,
                                  int64_t n_keys) {
  if (groups <= 0 || q_rows <= 0 || n_keys <= 0) return 0;
  const int64_t rows = groups * q_rows;
  if (dtype == FB_BF16 && sm100_supported(head_dim)) {
    const size_t per = (size_t)rows * (size_t)(head_dim + 1) * sizeof(float) + 256;
    SplitPlan s = plan_simt(groups, q_rows, n_keys, SIZE_MAX, per);
    return std::max(refresh_sm100_workspace_bytes(groups, q_rows, head_dim, n_keys),
                    per * (size_t)s.splits);
  }
  const size_t elem = dtype == FB_BF16 ? 4 : 8;
  const size_t per = (size_t)rows * (size_t)(head_dim + 1) * elem + 256;
  SplitPlan s = plan_simt(groups, q_rows, n_keys, SIZE_MAX, per);
  return per * (size_t)s.splits;
}

int fb_attention_partial(int dtype, const void* q, const void* k, const void* v, int64_t groups,
                         int64_t q_rows, int64_t head_dim, int64_t kv_rows_cap, int64_t key_begin,
                         int64_t key_end, double scale, void* o_out, void* lse_out, void* workspace,
                         size_t workspace_bytes, void* stream) {
  return fb_attention_partial_sync(dtype, q, k, v, groups, q_rows, head_dim, kv_rows_cap, key_begin,
                                   key_end, scale, o_out, lse_out, workspace, workspace_bytes,
                                   nullptr, 0, stream);
}

int64_t fb_sync_flags_count(void) { return 1024; }

int fb_attention_partial_sync(int dtype, const void* q, const void* k, const void* v,
                              int64_t groups, int64_t q_rows, int64_t head_dim,
                              int64_t kv_rows_cap, int64_t key_begin, int64_t key_end,
                              double scale, void* o_out, void* lse_out, void* workspace,
                              size_t workspace_bytes, uint64_t* sync_flags, int64_t n_flags,
                              void* stream) {
  bool pb = false;
  if (int rc = split_partial_bf16(dtype, pb)) return rc;
  ScopedPartialBf16 pb_scope(pb);
  if (sync_flags != nullptr && n_flags < 1) return fail(FB_ERR_VALUE, "sync_flags needs n_flags >= 1");
  if (groups < 0 || q_rows < 0 || head_dim < 1 || kv_rows_cap < 0)
    return fail(FB_ERR_SHAPE, "negative extent or head_dim < 1");
  if (!(0 <= key_begin && key_begin <= key_end && key_end <= kv_rows_cap))
    return fail(FB_ERR_BOUNDS, "key range [" + std::to_string(key_begin) + ", " +
                                   std::to_string(key_end) + ") outside [0, " +
                                   std::to_string(kv_rows_cap) + "]");
  if (groups == 0 || q_rows == 0) return FB_OK;
  cudaStream_t st = as_stream(stream);
  switch (dtype) {
    case FB_F64:
      return attention_partial_t<ModeF64>(q, k, v, groups, q_rows, head_dim, kv_rows_cap, key_begin,
                                          key_end, scale, o_out, lse_out, workspace, workspace_bytes, st);
    case FB_F32:
      return attention_partial_t<ModeF32>(q, k, v, groups, q_rows, head_dim, kv_rows_cap, key_begin,
                                          key_end, scale, o_out, lse_out, workspace, workspace_bytes, st);
    default:
      return attention_partial_t<ModeBF16>(q, k, v, groups, q_rows, head_dim, kv_rows_cap, key_begin,
                                           key_end, scale, o_out, lse_out, workspace, workspace_bytes, st,
                                           sync_flags, n_flags);
  }
}

int fb_commit_block(int dtype, void* k_cache, void* v_cache, int64_t groups, int64_t kv_rows_cap,
                    int64_t head_dim, const void* k_block, const void* v_block, int64_t block_rows,
                    int32_t* lengths, int32_t* overflow, void* stream) {
  if (int rc = check_dtype(dtype)) return rc;
  if (groups < 0 || kv_rows_cap < 0 || head_dim < 1 || block_rows < 0)
    return fail(FB_ERR_SHAPE, "bad extents");
  if (block_rows == 0) return fail(FB_ERR_SHAPE, "a block commit needs at least one row");
  if (lengths == nullptr) return fail(FB_ERR_VALUE, "lengths (device int32 [groups]) is required");
  return launch_commit_block(k_cache, v_cache, k_block, v_block, groups, kv_rows_cap,
                             head_dim * (int64_t)dtype_size(dtype), block_rows, lengths, overflow,
                             as_stream(stream));
}

size_t fb_paged_workspace_bytes(int dtype, int64_t groups, int64_t q_rows, int64_t head_dim) {
  if (dtype != FB_BF16 || !sm100_supported(head_dim) || groups <= 0 || q_rows <= 0) return 0;
  return refresh_sm100_ragged_workspace_bytes(groups, q_rows, head_dim);
}

int fb_attention_partial_paged(int dtype, const void* q, const void* k_pages, const void* v_pages,
                               int64_t num_pages, int64_t page_rows, const int32_t* page_table,
                               int64_t max_pages, int64_t groups, int64_t q_rows, int64_t head_dim,
                               const int32_t* key_len, double scale, void* o_out, void* lse_out,
                               void* workspace, size_t workspace_bytes, void* stream) {
  bool pb = false;
  if (int rc = split_partial_bf16(dtype, pb)) return rc;
  ScopedPartialBf16 pb_scope(pb);
  if (groups < 0 || q_rows < 0 || head_dim < 1 || num_pages < 0 || max_pages < 0)
    return fail(FB_ERR_SHAPE, "bad extents");
  if (page_table == nullptr || key_len == nullptr)
    return fail(FB_ERR_VALUE, "page_table and key_len (device int32) are required");
  if (dtype != FB_BF16 || !sm100_supported(head_dim))
    return fail(FB_ERR_UNSUPPORTED, "paged KV: bf16 with head_dim 64 or 128");
  if (page_rows <= 0 || page_rows % 128 != 0)
    return fail(FB_ERR_UNSUPPORTED, "page_rows must be a positive multiple of 128");
  if (max_pages * page_rows >= (int64_t(1) << 31)) return fail(FB_ERR_SHAPE, "logical capacity >= 2^31 rows");
  if (groups == 0 || q_rows == 0) return FB_OK;
  if (workspace == nullptr || workspace_bytes < fb_paged_workspace_bytes(dtype, groups, q_rows, head_dim))
    return fail(FB_ERR_VALUE, "workspace too small (fb_paged_workspace_bytes)");
  return launch_refresh_paged_sm100(
      reinterpret_cast<const __nv_bfloat16*>(q), reinterpret_cast<const __nv_bfloat16*>(k_pages),
      reinterpret_cast<const __nv_bfloat16*>(v_pages), num_pages, page_rows, page_table, max_pages,
      groups, q_rows, head_dim, key_len, scale, reinterpret_cast<float*>(o_out),
      reinterpret_cast<float*>(lse_out), workspace, workspace_bytes, as_stream(stream));
}

int fb_block_causal_attention_paged(int dtype, const void* q, const void* k_pages, const void* v_pages,
                                    int64_t num_pages, int64_t page_rows, const int32_t* page_table,
                                    int64_t max_pages, int64_t groups, int64_t q_rows, int64_t n_q,
                                    int64_t head_dim, int64_t n_prefix, int64_t block_size, double scale,
                                    void* o_out, void* lse_out, void* workspace, size_t workspace_bytes,
                                    void* stream) {
  if (int rc = check_dtype(dtype)) return rc;
  if (groups < 0 || q_rows < 0 || n_q < 1 || head_dim < 1 || n_prefix < 0 || block_size < 1 ||
      num_pages < 0 || max_pages < 0)
    return fail(FB_ERR_SHAPE, "bad extents");
  if (q_rows % n_q != 0) return fail(FB_ERR_SHAPE, "q_rows must be heads_per_group * n_q");
  if (page_table == nullptr) return fail(FB_ERR_VALUE, "page_table (device int32) is required");
  if (dtype != FB_BF16 || !sm100_supported(head_dim))
    return fail(FB_ERR_UNSUPPORTED, "paged KV: bf16 with head_dim 64 or 128");
  if (page_rows <= 0 || page_rows % 128 != 0)
    return fail(FB_ERR_UNSUPPORTED, "page_rows must be a positive multiple of 128");
  if (n_prefix + n_q > max_pages * page_rows) return fail(FB_ERR_BOUNDS, "prompt exceeds the pages");
  if (groups == 0 || q_rows == 0) return FB_OK;
  if (workspace == nullptr || workspace_bytes < fb_paged_workspace_bytes(dtype, groups, q_rows, head_dim))
    return fail(FB_ERR_VALUE, "workspace too small (fb_paged_workspace_bytes)");
  return launch_block_causal_paged_sm100(
      reinterpret_cast<const __nv_bfloat16*>(q), reinterpret_cast<const __nv_bfloat16*>(k_pages),
      reinterpret_cast<const __nv_bfloat16*>(v_pages), num_pages, page_rows, page_table, max_pages,
      groups, q_rows, head_dim, n_q, n_prefix, block_size, scale, reinterpret_cast<float*>(o_out),
      reinterpret_cast<float*>(lse_out), workspace, workspace_bytes, as_stream(stream));
}

// ---- sparse path over a paged cache: the bf16 tcgen05 kernels with the page
// translation (PagingCtx) active for the duration of the call
static int paged_sparse_check(int dtype, int64_t head_dim, int64_t kbs, int64_t page_rows,
                              const int32_t* table, int64_t max_pages, int64_t n_ext) {
  if (dtype != FB_BF16 || !sm100_supported(head_dim) || kbs != 16)
    return fail(FB_ERR_UNSUPPORTED, "paged sparse path: bf16, head_dim 64 / 128, key_block_size 16");
  if (page_rows <= 0 || page_rows % 128 != 0)
    return fail(FB_ERR_UNSUPPORTED, "page_rows must be a positive multiple of 128");
  if (table == nullptr) return fail(FB_ERR_VALUE, "page_table (device int32) is required");
  if (n_ext < 0 || n_ext > max_pages * page_rows) return fail(FB_ERR_SHAPE, "n_ext outside the pages");
  return FB_OK;
}

int fb_block_mass_paged(int dtype, const void* q, const void* k_pages, const void* k_in,
                        int64_t num_pages, int64_t page_rows, const int32_t* page_table,
                        int64_t max_pages, int64_t groups, int64_t q_rows, int64_t head_dim,
                        int64_t n_ext, int64_t n_in, int64_t key_block_size, double scale,
                        double* mass, void* workspace, size_t workspace_bytes, void* stream) {
  if (int rc = paged_sparse_check(dtype, head_dim, key_block_size, page_rows, page_table, max_pages, n_ext))
    return rc;
  if (!score_sm100_supported(head_dim, q_rows, key_block_size))
    return fail(FB_ERR_UNSUPPORTED, "paged block mass: q_rows <= 128");
  if (workspace_bytes < score_sm100_min_workspace_bytes(groups, q_rows, n_ext, n_in))
    return fail(FB_ERR_VALUE, "workspace too small (fb_block_mass_workspace_bytes_ex)");
  const PagingCtx pc{page_table, max_pages, page_rows, num_pages};
  ScopedPaging guard(&pc);
  return fb_block_mass(dtype, q, k_pages, k_in, groups, q_rows, head_dim, max_pages * page_rows, n_ext,
                       n_in, key_block_size, scale, mass, workspace, workspace_bytes, stream);
}

int fb_sparse_partitioned_paged(int dtype, const void* q, const void* k_pages, const void* v_pages,
                                const void* k_in, const void* v_in, int64_t num_pages,
                                int64_t page_rows, const int32_t* page_table, int64_t max_pages,
                                int64_t groups, int64_t q_rows, int64_t head_dim, int64_t n_ext,
                                int64_t n_in, const int32_t* selected, int64_t n_sel,
                                int64_t key_block_size, double scale, void* o_sel, void* lse_sel,
                                void* o_res, void* lse_res, void* out, int out_dtype,
                                int32_t* empty_rows, void* workspace, size_t workspace_bytes,
                                void* stream) {
  if (int rc = paged_sparse_check(dtype, head_dim, key_block_size, page_rows, page_table, max_pages, n_ext))
    return rc;
  if (workspace_bytes < fb_sparse_workspace_bytes(dtype, groups, q_rows, head_dim, n_ext, n_sel, n_in,
                                                  key_block_size))
    return fail(FB_ERR_VALUE, "workspace too small (fb_sparse_workspace_bytes)");
  const PagingCtx pc{page_table, max_pages, page_rows, num_pages};
  ScopedPaging guard(&pc);
  return fb_sparse_partitioned(dtype, q, k_pages, v_pages, k_in, v_in, groups, q_rows, head_dim,
                               max_pages * page_rows, n_ext, n_in, selected, n_sel, key_block_size,
                               scale, o_sel, lse_sel, o_res, lse_res, out, out_dtype, empty_rows,
                               workspace, workspace_bytes, stream);
}

int fb_sparse_attend_merge_paged(int dtype, const void* q, const void* k_pages, const void* v_pages,
                                 const void* k_in, const void* v_in, int64_t num_pages,
                                 int64_t page_rows, const int32_t* page_table, int64_t max_pages,
                                 int64_t groups, int64_t q_rows, int64_t head_dim, int64_t n_ext,
                                 int64_t n_in, const int32_t* selected, int64_t n_sel,
                                 int64_t key_block_size, double scale, const void* o_res,
                                 const void* lse_res, void* out, int out_dtype, int32_t* empty_rows,
                                 void* workspace, size_t workspace_bytes, void* stream) {
  if (int rc = paged_sparse_check(dtype, head_dim, key_block_size, page_rows, page_table, max_pages, n_ext))
    return rc;
  if (workspace_bytes < fb_sparse_workspace_bytes(dtype, groups, q_rows, head_dim, n_ext, n_sel, n_in,
                                                  key_block_size))
    return fail(FB_ERR_VALUE, "workspace too small (fb_sparse_workspace_bytes)");
  const PagingCtx pc{page_table, max_pages, page_rows, num_pages};
  ScopedPaging guard(&pc);
  return fb_sparse_attend_merge(dtype, q, k_pages, v_pages, k_in, v_in, groups, q_rows, head_dim,
                                max_pages * page_rows, n_ext, n_in, selected, n_sel, key_block_size,
                                scale, o_res, lse_res, out, out_dtype, empty_rows, workspace,
                                workspace_bytes, stream);
}

int fb_internal_merge_tok(int dtype, const void* q, int64_t q_token_stride, const void* k_in,
                          int64_t k_token_stride, const void* v_in, int64_t v_token_stride,
                          int64_t batch, int64_t block, int64_t num_q_heads, int64_t num_kv_heads,
                          int64_t head_dim, double scale, const void* o_ext, const void* lse_ext,
                          void* out, int out_dtype, int64_t out_token_stride, int flags, void* stream) {
  bool extb = false;
  if (int rc = split_partial_bf16(dtype, extb)) return rc;
  if (dtype != FB_BF16) return fail(FB_ERR_UNSUPPORTED, "token-major cached step: bf16");
  if (out_dtype != FB_BF16 && out_dtype != FB_F32) return fail(FB_ERR_VALUE, "BF16 mode writes F32 or BF16 output");
  if (flags & ~FB_EXT_STABLE) return fail(FB_ERR_VALUE, "unknown flags");
  if (batch < 0 || block < 1 || num_q_heads < 1 || num_kv_heads < 1) return fail(FB_ERR_SHAPE, "bad extents");
  if (num_q_heads % num_kv_heads) return fail(FB_ERR_SHAPE, "num_q_heads must be a multiple of num_kv_heads");
  if (head_dim != 128 || (num_q_heads / num_kv_heads) * block > 128 || block > 64)
    return fail(FB_ERR_UNSUPPORTED, "token-major cached step: d 128, (Hq/Hkv)*B <= 128, 1 <= B <= 64");
  if (batch == 0) return FB_OK;
  if (!q || !k_in || !v_in || !o_ext || !lse_ext || !out)
    return fail(FB_ERR_VALUE, "q, k_in, v_in, o_ext, lse_ext and out are required (device pointers)");
  // rows are read / written with >= 16-byte vector accesses (32-byte when aligned) and
  // mapped by TMA (16-byte strides)
  const int64_t osz = out_dtype == FB_BF16 ? 2 : 4;
  if ((reinterpret_cast<uintptr_t>(o_ext) & 15) || (reinterpret_cast<uintptr_t>(out) & 15) ||
      ((out_token_stride * osz) & 15) || (reinterpret_cast<uintptr_t>(q) & 15) ||
      (reinterpret_cast<uintptr_t>(k_in) & 15) || (reinterpret_cast<uintptr_t>(v_in) & 15) ||
      ((q_token_stride * 2) & 15) || ((k_token_stride * 2) & 15) || ((v_token_stride * 2) & 15))
    return fail(FB_ERR_VALUE, "o_ext, out, q, k_in and v_in need 16-byte aligned rows");
  return launch_internal_merge_tok_sm100(
      reinterpret_cast<const __nv_bfloat16*>(q), q_token_stride, reinterpret_cast<const __nv_bfloat16*>(k_in),
      k_token_stride, reinterpret_cast<const __nv_bfloat16*>(v_in), v_token_stride, batch, block, num_q_heads,
      num_kv_heads, head_dim, scale, o_ext, reinterpret_cast<const float*>(lse_ext), out, out_token_stride,
      out_dtype == FB_BF16, (flags & FB_EXT_STABLE) != 0, extb, as_stream(stream));
}

int fb_commit_block_paged(int dtype, void* k_pages, void* v_pages, int64_t page_rows,
                          const int32_t* page_table, int64_t max_pages, int64_t groups,
                          int64_t head_dim, const void* k_block, const void* v_block,
                          int64_t block_rows, int32_t* lengths, int32_t* overflow, void* stream) {
  if (int rc = check_dtype(dtype)) return rc;
  if (groups < 0 || head_dim < 1 || block_rows < 0 || page_rows < 1 || max_pages < 0)
    return fail(FB_ERR_SHAPE, "bad extents");
  if (block_rows == 0) return fail(FB_ERR_SHAPE, "a block commit needs at least one row");
  if (lengths == nullptr || page_table == nullptr)
    return fail(FB_ERR_VALUE, "lengths and page_table (device int32) are required");
  return launch_commit_block_paged(k_pages, v_pages, page_rows, page_table, max_pages, k_block, v_block,
                                   groups, head_dim * (int64_t)dtype_size(dtype), block_rows, lengths,
                                   overflow, as_stream(stream));
}

int fb_attention_partial_groups(int dtype, const void* q, const void* k, const void* v,
                                int64_t groups, int64_t q_rows, int64_t head_dim,
                                int64_t kv_rows_cap, int64_t key_begin, int64_t key_end,
                                const int32_t* group_list, int64_t n_list, double scale,
                                void* o_out, void* lse_out, void* workspace,
                                size_t workspace_bytes, void* stream) {
  bool pb = false;
  if (int rc = split_partial_bf16(dtype, pb)) return rc;
  ScopedPartialBf16 pb_scope(pb);
  if (groups < 0 || q_rows < 0 || head_dim < 1 || kv_rows_cap < 0 || n_list < 0)
    return fail(FB_ERR_SHAPE, "negative extent or head_dim < 1");
  if (n_list > groups) return fail(FB_ERR_SHAPE, "group list longer than the batch of groups");
  if (key_begin < 0 || key_end < key_begin || key_end > kv_rows_cap)
    return fail(FB_ERR_BOUNDS, "key range outside the slab");
  if (n_list == 0 || q_rows == 0) return FB_OK;
  if (group_list == nullptr) return fail(FB_ERR_VALUE, "group_list (device int32 [n_list]) is required");
  if (head_dim > 256) return fail(FB_ERR_UNSUPPORTED, "head_dim > 256");
  cudaStream_t st = as_stream(stream);
  switch (dtype) {
    case FB_F64:
      return attention_partial_groups_t<ModeF64>(q, k, v, groups, q_rows, head_dim, kv_rows_cap,
                                                 key_begin, key_end, group_list, n_list, scale, o_out,
                                                 lse_out, workspace, workspace_bytes, st);
    case FB_F32:
      return attention_partial_groups_t<ModeF32>(q, k, v, groups, q_rows, head_dim, kv_rows_cap,
                                                 key_begin, key_end, group_list, n_list, scale, o_out,
                                                 lse_out, workspace, workspace_bytes, st);
    default:
      return attention_partial_groups_t<ModeBF16>(q, k, v, groups, q_rows, head_dim, kv_rows_cap,
                                                  key_begin, key_end, group_list, n_list, scale,
                                                  o_out, lse_out, workspace, workspace_bytes, st);
  }
}

int fb_row_cosine(int dtype, const void* a, const void* b, int64_t heads, int64_t rows,
                  int64_t head_dim, double* row_cos, double* head_mean, void* stream) {
  if (int rc = check_dtype(dtype)) return rc;
  if (heads < 0 || rows < 0 || head_dim < 1) return fail(FB_ERR_SHAPE, "negative extent or head_dim < 1");
  if (heads == 0) return FB_OK;
  if (row_cos == nullptr) return fail(FB_ERR_VALUE, "row_cos ([heads*rows] float64) is required");
  cudaStream_t st = as_stream(stream);
  switch (dtype) {
    case FB_F64: return launch_row_cosine<double>(a, b, heads, rows, head_dim, row_cos, head_mean, st);
    case FB_F32: return launch_row_cosine<float>(a, b, heads, rows, head_dim, row_cos, head_mean, st);
    default: return launch_row_cosine<__nv_bfloat16>(a, b, heads, rows, head_dim, row_cos, head_mean, st);
  }
}

int fb_row_cosine_update(int dtype, const void* a, void* b, int64_t heads, int64_t rows, int64_t head_dim,
                         double* row_cos, double* head_mean, int32_t* nonzero, void* stream) {
  if (int rc = check_dtype(dtype)) return rc;
  if (heads < 0 || rows < 0 || head_dim < 1) return fail(FB_ERR_SHAPE, "negative extent or head_dim < 1");
  if (heads == 0) return FB_OK;
  if (row_cos == nullptr) return fail(FB_ERR_VALUE, "row_cos ([heads*rows] float64) is required");
  cudaStream_t st = as_stream(stream);
  switch (dtype) {
    case FB_F64: return launch_row_cosine<double>(a, b, heads, rows, head_dim, row_cos, head_mean, st, true, nonzero);
    case FB_F32: return launch_row_cosine<float>(a, b, heads, rows, head_dim, row_cos, head_mean, st, true, nonzero);
    default:
      return launch_row_cosine<__nv_bfloat16>(a, b, heads, rows, head_dim, row_cos, head_mean, st, true, nonzero);
  }
}

int fb_pairwise_cosine(int dtype, const void* later, const void* earlier, int64_t heads, int64_t rows,
                       int64_t head_dim, double* out, void* stream) {
  if (int rc = check_dtype(dtype)) return rc;
  if (heads < 0 || rows < 0 || head_dim < 1) return fail(FB_ERR_SHAPE, "negative extent or head_dim < 1");
  if (heads == 0 || rows == 0) return FB_OK;
  if (rows > 65535 * 16) return fail(FB_ERR_UNSUPPORTED, "too many rows for the all-pairs matrix");
  cudaStream_t st = as_stream(stream);
  switch (dtype) {
    case FB_F64: return launch_pairwise_cosine<double>(later, earlier, heads, rows, head_dim, out, st);
    case FB_F32: return launch_pairwise_cosine<float>(later, earlier, heads, rows, head_dim, out, st);
    default: return launch_pairwise_cosine<__nv_bfloat16>(later, earlier, heads, rows, head_dim, out, st);
  }
}

size_t fb_ragged_workspace_bytes(int dtype, int64_t groups, int64_t q_rows, int64_t head_dim,
                                 int64_t kv_rows_cap) {
  (void)kv_rows_cap;
  if (groups <= 0 || q_rows <= 0) return 0;
  const int64_t rows = groups * q_rows;
  size_t b = (size_t)rows * (head_dim + 1) * (dtype == FB_BF16 ? 4 : 8) + 256;
  if (dtype == FB_BF16 && sm100_supported(head_dim))
    b = std::max(b, refresh_sm100_ragged_workspace_bytes(groups, q_rows, head_dim));
  return b;
}

int fb_attention_partial_ragged(int dtype, const void* q, const void* k, const void* v,
                                int64_t groups, int64_t q_rows, int64_t head_dim,
                                int64_t kv_rows_cap, int64_t key_begin, const int32_t* key_end,
                                double scale, void* o_out, void* lse_out, void* workspace,
                                size_t workspace_bytes, void* stream) {
  bool pb = false;
  if (int rc = split_partial_bf16(dtype, pb)) return rc;
  ScopedPartialBf16 pb_scope(pb);
  if (groups < 0 || q_rows < 0 || head_dim < 1 || kv_rows_cap < 0)
    return fail(FB_ERR_SHAPE, "negative extent or head_dim < 1");
  if (key_begin < 0 || key_begin > kv_rows_cap) return fail(FB_ERR_BOUNDS, "key_begin outside the slab");
  if (groups == 0 || q_rows == 0) return FB_OK;
  if (key_end == nullptr) return fail(FB_ERR_VALUE, "key_end (device int32 [groups]) is required");
  if (head_dim > 256) return fail(FB_ERR_UNSUPPORTED, "head_dim > 256");
  cudaStream_t st = as_stream(stream);
  switch (dtype) {
    case FB_F64:
      return attention_partial_ragged_t<ModeF64>(q, k, v, groups, q_rows, head_dim, kv_rows_cap,
                                                 key_begin, key_end, scale, o_out, lse_out,
                                                 workspace, workspace_bytes, st);
    case FB_F32:
      return attention_partial_ragged_t<ModeF32>(q, k, v, groups, q_rows, head_dim, kv_rows_cap,
                                                 key_begin, key_end, scale, o_out, lse_out,
                                                 workspace, workspace_bytes, st);
    default:
      return attention_partial_ragged_t<ModeBF16>(q, k, v, groups, q_rows, head_dim, kv_rows_cap,
                                                  key_begin, key_end, scale, o_out, lse_out,
                                                  workspace, workspace_bytes, st);
  }
}

// ---------------------------------------------------------------- block-causal (prefill / commit)

size_t fb_block_causal_workspace_bytes(int dtype, int64_t groups, int64_t q_rows, int64_t head_dim) {
  const int64_t rows = groups * q_rows;
  switch (dtype) {
    case FB_F64: return 0;
    case FB_F32: return split_bytes<ModeMaskF32>(rows, head_dim);
    default:
      return sm100_supported(head_dim) ? refresh_sm100_ragged_workspace_bytes(groups, q_rows, head_dim) : 0;
  }
}

int fb_block_causal_attention(int dtype, const void* q, const void* k, const void* v,
                              int64_t groups, int64_t q_rows, int64_t n_q, int64_t head_dim,
                              int64_t kv_rows_cap, int64_t n_prefix, int64_t block_size,
                              double scale, void* o_out, void* lse_out, void* workspace,
                              size_t workspace_bytes, void* stream) {
  if (int rc = check_dtype(dtype)) return rc;
  if (groups < 0 || q_rows < 0 || n_q < 1 || head_dim < 1 || kv_rows_cap < 0 || n_prefix < 0)
    return fail(FB_ERR_SHAPE, "negative extent, n_q < 1 or head_dim < 1");
  if (q_rows % n_q != 0) return fail(FB_ERR_SHAPE, "q_rows must be heads_per_group * n_q");
  if (block_size < 1) return fail(FB_ERR_VALUE, "block_size must be >= 1");
  if (n_prefix + n_q > kv_rows_cap)
    return fail(FB_ERR_BOUNDS, "n_prefix + n_q exceeds the slab (commit the block's K/V first)");
  if (n_prefix + n_q >= (int64_t(1) << 31)) return fail(FB_ERR_UNSUPPORTED, "context >= 2^31 keys");
  if (groups == 0 || q_rows == 0) return FB_OK;
  if (head_dim > 256) return fail(FB_ERR_UNSUPPORTED, "head_dim > 256");
  cudaStream_t st = as_stream(stream);
  switch (dtype) {
    case FB_F64:
      return block_causal_t<ModeF64>(q, k, v, groups, q_rows, head_dim, kv_rows_cap, n_q, n_prefix,
                                     block_size, scale, o_out, lse_out, workspace, workspace_bytes, st);
    case FB_F32:
      return block_causal_t<ModeF32>(q, k, v, groups, q_rows, head_dim, kv_rows_cap, n_q, n_prefix,
                                     block_size, scale, o_out, lse_out, workspace, workspace_bytes, st);
    default:
      return block_causal_t<ModeBF16>(q, k, v, groups, q_rows, head_dim, kv_rows_cap, n_q, n_prefix,
                                      block_size, scale, o_out, lse_out, workspace, workspace_bytes, st);
  }
}

size_t fb_internal_merge_workspace_bytes(int dtype, int64_t groups, int64_t q_rows,
                                        int64_t head_dim, int64_t n_in) {
  if (dtype != FB_BF16 || !sm100_supported(head_dim) || sm100_k2_supported(head_dim, n_in) ||
      n_in <= 0)
    return 0;
  const int64_t rows = groups * q_rows;
  return align_up((size_t)rows * (head_dim + 1) * sizeof(float), 256) +
         refresh_sm100_workspace_bytes(groups, q_rows, head_dim, n_in);
}

int fb_internal_merge(int dtype, const void* q, const void* k_in, const void* v_in, int64_t groups,
                      int64_t q_rows, int64_t head_dim, int64_t n_in, double scale,
                      const void* o_ext, const void* lse_ext, void* out, int out_dtype,
                      void* lse_merged, void* o_int, void* lse_int, int32_t* empty_rows,
                      void* workspace, size_t workspace_bytes, void* stream) {
  return fb_internal_merge_ex(dtype, q, k_in, v_in, groups, q_rows, head_dim, n_in, scale, o_ext,
                              lse_ext, out, out_dtype, lse_merged, o_int, lse_int, empty_rows,
                              workspace, workspace_bytes, 0, stream);
}

// Per-thread (and per-device) staging for the host-buffer entries: a pinned
// host buffer and a device buffer, grown on demand.  Each call ends with a
// stream synchronisation, so the next call of the same thread may reuse both.
namespace {
struct HostStage {
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  void* dbuf = nullptr;
  size_t dbuf_bytes = 0;
};
constexpr int kMaxStageDevices = 16;
thread_local HostStage t_stage[kMaxStageDevices];

int stage_reserve(size_t host_bytes, size_t dev_bytes, HostStage*& out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxStageDevices)
    return fail(FB_ERR_CUDA, "no current CUDA device for the host staging");
  HostStage& s = t_stage[dev];
  if (s.pinned_bytes < host_bytes) {
    if (s.pinned) cudaFreeHost(s.pinned);
    s.pinned = nullptr;
    s.pinned_bytes = 0;
    const size_t want = std::max<size_t>(host_bytes * 2, 1 << 16);
    if (cudaMallocHost(&s.pinned, want) != cudaSuccess) return fail(FB_ERR_CUDA, "cudaMallocHost failed");
    s.pinned_bytes = want;
  }
  if (s.dbuf_bytes < dev_bytes) {
    if (s.dbuf) cudaFree(s.dbuf);
    s.dbuf = nullptr;
    s.dbuf_bytes = 0;
    const size_t want = std::max<size_t>(dev_bytes * 2, 1 << 16);
    if (cudaMalloc(&s.dbuf, want) != cudaSuccess) return fail(FB_ERR_CUDA, "cudaMalloc failed");
    s.dbuf_bytes = want;
  }
  out = &s;
  return FB_OK;
}
}  // namespace

int fb_internal_merge_host(int dtype, const void* q, const void* k_in, const void* v_in, int64_t groups,
                           int64_t q_rows, int64_t head_dim, int64_t n_in, double scale, const void* o_ext,
                           const void* lse_ext, void* out, void* o_int, double* lse_int,
                           int64_t* empty_rows, void* stream) {
  if (dtype != FB_F64 && dtype != FB_F32)
    return fail(FB_ERR_UNSUPPORTED, "fb_internal_merge_host: FB_F64 or FB_F32 host arrays");
  if (groups < 0 || q_rows < 0 || head_dim < 1 || n_in < 0)
    return fail(FB_ERR_SHAPE, "negative extent or head_dim < 1");
  if (empty_rows) *empty_rows = 0;
  if (groups == 0 || q_rows == 0) return FB_OK;
  if (q == nullptr || out == nullptr || o_ext == nullptr || lse_ext == nullptr ||
      (n_in > 0 && (k_in == nullptr || v_in == nullptr)))
    return fail(FB_ERR_VALUE, "fb_internal_merge_host: null pointer");
  const size_t E = dtype == FB_F64 ? sizeof(double) : sizeof(float);
  const size_t rows = (size_t)(groups * q_rows);
  const size_t qb = rows * head_dim * E, kb = (size_t)(groups * n_in) * head_dim * E;
  const size_t in_bytes = align_up(align_up(qb + 2 * kb, 16) + sizeof(int32_t), 256);
  // device / pinned layout: [q | k_in | v_in | empty counter] [out | o_int | lse_int]
  const size_t ob = align_up(rows * head_dim * E, 256), lb = align_up(rows * sizeof(double), 256);
  const size_t out_bytes = 2 * ob + lb;
  HostStage* s = nullptr;
  if (int rc = stage_reserve(in_bytes + out_bytes, in_bytes + out_bytes, s)) return rc;
  cudaStream_t st = as_stream(stream);
  char* hp = reinterpret_cast<char*>(s->pinned);
  char* dp = reinterpret_cast<char*>(s->dbuf);
  std::memcpy(hp, q, qb);
  if (kb) {
    std::memcpy(hp + qb, k_in, kb);
    std::memcpy(hp + qb + kb, v_in, kb);
  }
  // the empty-row counter travels with the inputs (zeroed in the same copy,
  // no memset launch): [q | k_in | v_in | counter]
  const size_t cnt_off = align_up(qb + 2 * kb, 16);
  std::memset(hp + cnt_off, 0, sizeof(int32_t));
  char* d_out = dp + in_bytes;
  char* d_oi = d_out + ob;
  char* d_li = d_oi + ob;
  int32_t* d_cnt = reinterpret_cast<int32_t*>(dp + cnt_off);
  if (cudaMemcpyAsync(dp, hp, cnt_off + sizeof(int32_t), cudaMemcpyHostToDevice, st) != cudaSuccess)
    return fail(FB_ERR_CUDA, "fb_internal_merge_host: staging copy failed");
  const bool want_int = o_int != nullptr || lse_int != nullptr;
  if (int rc = fb_internal_merge_ex(dtype, dp, dp + qb, dp + qb + kb, groups, q_rows, head_dim, n_in, scale,
                                    o_ext, lse_ext, d_out, dtype, nullptr, want_int ? d_oi : nullptr,
                                    want_int ? d_li : nullptr, d_cnt, nullptr, 0, FB_EXT_STABLE, stream))
    return rc;
  // one read-back: the counter and the outputs are contiguous from cnt_off
  // ([counter | pad | out | o_int | lse_int]); without the internal partial
  // only [counter .. out] is copied
  char* h_out = hp + in_bytes;
  const size_t back = (size_t)(d_out - (dp + cnt_off)) + (want_int ? 2 * ob + lb : ob);
  cudaError_t e = cudaMemcpyAsync(hp + cnt_off, dp + cnt_off, back, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return fail(FB_ERR_CUDA, cudaGetErrorString(e));
  std::memcpy(out, h_out, rows * head_dim * E);
  if (o_int) std::memcpy(o_int, h_out + ob, rows * head_dim * E);
  if (lse_int) std::memcpy(lse_int, h_out + 2 * ob, rows * sizeof(double));
  int32_t cnt = 0;
  std::memcpy(&cnt, hp + cnt_off, sizeof(int32_t));
  if (empty_rows) *empty_rows = cnt;
  return FB_OK;
}

int fb_internal_merge_ex(int dtype, const void* q, const void* k_in, const void* v_in,
                         int64_t groups, int64_t q_rows, int64_t head_dim, int64_t n_in,
                         double scale, const void* o_ext, const void* lse_ext, void* out,
                         int out_dtype, void* lse_merged, void* o_int, void* lse_int,
                         int32_t* empty_rows, void* workspace, size_t workspace_bytes, int flags,
                         void* stream) {
  bool extb = false;
  if (int rc = split_partial_bf16(dtype, extb)) return rc;
  if (flags & ~FB_EXT_STABLE) return fail(FB_ERR_VALUE, "unknown fb_internal_merge_ex flags");
  if (groups < 0 || q_rows < 0 || head_dim < 1 || n_in < 0)
    return fail(FB_ERR_SHAPE, "negative extent or head_dim < 1");
  if (groups == 0 || q_rows == 0) return FB_OK;
  if (head_dim > 256) return fail(FB_ERR_UNSUPPORTED, "head_dim > 256");
  cudaStream_t st = as_stream(stream);
  switch (dtype) {
    case FB_F64:
      if (out_dtype != FB_F64) return fail(FB_ERR_VALUE, "F64 mode writes F64 output");
      return internal_merge_t<ModeF64>(q, k_in, v_in, groups, q_rows, head_dim, n_in, scale, o_ext,
                                       lse_ext, out, false, lse_merged, o_int, lse_int, empty_rows, st);
    case FB_F32:
      if (out_dtype != FB_F32) return fail(FB_ERR_VALUE, "F32 mode writes F32 output");
      return internal_merge_t<ModeF32>(q, k_in, v_in, groups, q_rows, head_dim, n_in, scale, o_ext,
                                       lse_ext, out, false, lse_merged, o_int, lse_int, empty_rows, st);
    default:
      if (out_dtype != FB_F32 && out_dtype != FB_BF16)
        return fail(FB_ERR_VALUE, "BF16 mode writes F32 or BF16 output");
      if (extb && (o_int != nullptr || lse_int != nullptr))
        return fail(FB_ERR_UNSUPPORTED, "FB_PARTIAL_BF16 cached step: o_int / lse_int not supported");
      if (sm100_supported(head_dim) && !sm100_k2_supported(head_dim, n_in) && n_in > 0 &&
          n_in < (int64_t(1) << 31) && workspace != nullptr &&
          workspace_bytes >= fb_internal_merge_workspace_bytes(dtype, groups, q_rows, head_dim, n_in)) {
        // large current block (video chunks, C5): tensor-core internal partial over
        // the block's own keys (stream-K refresh kernel), then the K3 merge
        const int64_t rows = groups * q_rows;
        const size_t tmp = align_up((size_t)rows * (head_dim + 1) * sizeof(float), 256);
        float* oi = o_int ? reinterpret_cast<float*>(o_int) : reinterpret_cast<float*>(workspace);
        float* li = lse_int ? reinterpret_cast<float*>(lse_int)
                            : reinterpret_cast<float*>(workspace) + (size_t)rows * head_dim;
        // without an lse_merged output the K3 merge with the cached external
        // partial runs inside K1's split-merge kernel (MergeFinal): one launch
        // and one pass over the internal partial fewer
        // (the internal partial is scratch unless the caller asked for it)
        const MergeFinal fin{o_ext, reinterpret_cast<const float*>(lse_ext), out, out_dtype == FB_BF16 ? 1 : 0,
                             empty_rows, extb ? 1 : 0, (o_int == nullptr && lse_int == nullptr) ? 1 : 0};
        const bool fuse = lse_merged == nullptr;
        if (extb && !fuse)
          return fail(FB_ERR_UNSUPPORTED, "FB_PARTIAL_BF16 large-block cached step: lse_merged not supported");
        int rc = launch_refresh_sm100(reinterpret_cast<const __nv_bfloat16*>(q),
                                      reinterpret_cast<const __nv_bfloat16*>(k_in),
                                      reinterpret_cast<const __nv_bfloat16*>(v_in), groups, q_rows,
                                      head_dim, n_in, 0, n_in, scale, oi, li,
                                      reinterpret_cast<char*>(workspace) + tmp, workspace_bytes - tmp, st,
                                      nullptr, 0, fuse ? &fin : nullptr);
        if (rc) return rc;
        if (fuse) return FB_OK;
        const void* op[2] = {o_ext, oi};
        const void* lp[2] = {lse_ext, li};
        return combine_t<ModeBF16>(2, op, lp, rows, head_dim, out, out_dtype == FB_BF16, lse_merged,
                                   empty_rows, st);
      }
      return internal_merge_t<ModeBF16>(q, k_in, v_in, groups, q_rows, head_dim, n_in, scale, o_ext,
                                        lse_ext, out, out_dtype == FB_BF16, lse_merged, o_int,
                                        lse_int, empty_rows, st, (flags & FB_EXT_STABLE) != 0, extb);
  }
}

int fb_combine(int dtype, int n_parts, const void* const* o_parts, const void* const* lse_parts,
               int64_t rows, int64_t head_dim, void* o_out, int out_dtype, void* lse_out,
               int32_t* empty_rows, void* stream) {
  if (int rc = check_dtype(dtype)) return rc;
  if (n_parts < 1 || n_parts > FB_MAX_PARTS) return fail(FB_ERR_VALUE, "n_parts must be in [1, 16]");
  if (rows < 0 || head_dim < 1) return fail(FB_ERR_SHAPE, "negative rows or head_dim < 1");
  cudaStream_t st = as_stream(stream);
  switch (dtype) {
    case FB_F64:
      return combine_t<ModeF64>(n_parts, o_parts, lse_parts, rows, head_dim, o_out, false, lse_out,
                                empty_rows, st);
    case FB_F32:
      return combine_t<ModeF32>(n_parts, o_parts, lse_parts, rows, head_dim, o_out, false, lse_out,
                                empty_rows, st);
    default:
      return combine_t<ModeBF16>(n_parts, o_parts, lse_parts, rows, head_dim, o_out,
                                 out_dtype == FB_BF16, lse_out, empty_rows, st);
  }
}

int fb_full_attention(int dtype, const void* q, const void* k, const void* v, int64_t groups,
                      int64_t q_rows, int64_t head_dim, int64_t kv_rows_cap, int64_t n_ext,
                      const void* k_in, const void* v_in, int64_t n_in, double scale,
                      void* o_ext_scratch, void* lse_ext_scratch, void* out, int out_dtype,
                      int32_t* empty_rows, void* workspace, size_t workspace_bytes, void* stream) {
  int rc = fb_attention_partial(dtype, q, k, v, groups, q_rows, head_dim, kv_rows_cap, 0, n_ext,
                                scale, o_ext_scratch, lse_ext_scratch, workspace, workspace_bytes,
                                stream);
  if (rc) return rc;
  return fb_internal_merge(dtype, q, k_in, v_in, groups, q_rows, head_dim, n_in, scale,
                           o_ext_scratch, lse_ext_scratch, out, out_dtype, nullptr, nullptr, nullptr,
                           empty_rows, workspace, workspace_bytes, stream);
}

// ---------------------------------------------------------------- sparse

size_t fb_block_mass_workspace_bytes(int64_t groups, int64_t q_rows) {
  // row lognorms (double) + split scratch for the lognorm pass
  const int64_t rows = groups * q_rows;
  const size_t per = (size_t)rows * sizeof(double) * 2 + 256;
  return (size_t)rows * sizeof(double) + per * 1024;
}

size_t fb_block_mass_workspace_bytes_ex(int dtype, int64_t groups, int64_t q_rows, int64_t head_dim,
                                        int64_t n_ext, int64_t n_in, int64_t kbs) {
  size_t b = fb_block_mass_workspace_bytes(groups, q_rows);
  if (dtype == FB_BF16 && score_sm100_supported(head_dim, q_rows, kbs))
    b = std::max(b, score_sm100_workspace_bytes(groups, q_rows, n_ext, n_in));
  return b;
}

int64_t fb_mask_budget(int64_t n_ext, double density, int64_t key_block_size) {
  if (n_ext <= 0 || key_block_size < 1) return 0;
  const int64_t nb = (n_ext + key_block_size - 1) / key_block_size;
  const int64_t want = (int64_t)std::ceil(density * (double)n_ext / (double)key_block_size);
  return std::min<int64_t>(nb, std::max<int64_t>(1, want));
}

int fb_block_mass(int dtype, const void* q, const void* k, const void* k_in, int64_t groups,
                  int64_t q_rows, int64_t head_dim, int64_t kv_rows_cap, int64_t n_ext, int64_t n_in,
                  int64_t key_block_size, double scale, double* mass, void* workspace,
                  size_t workspace_bytes, void* stream) {
  if (int rc = check_dtype(dtype)) return rc;
  if (key_block_size < 1) return fail(FB_ERR_VALUE, "key_block_size must be >= 1");
  if (groups < 0 || q_rows < 0 || head_dim < 1 || n_in < 0) return fail(FB_ERR_SHAPE, "bad extents");
  if (n_ext < 0 || n_ext > kv_rows_cap) return fail(FB_ERR_VALUE, "n_ext outside [0, kv_rows_cap]");
  if (groups == 0 || n_ext == 0) return FB_OK;
  if (q_rows == 0) return fail(FB_ERR_SHAPE, "no query rows");
  if (head_dim > 256) return fail(FB_ERR_UNSUPPORTED, "head_dim > 256");
  if (workspace == nullptr || workspace_bytes < (size_t)groups * q_rows * sizeof(double) + 512)
    return fail(FB_ERR_VALUE, "workspace too small (fb_block_mass_workspace_bytes)");
  cudaStream_t st = as_stream(stream);
  if (dtype == FB_BF16 && score_sm100_supported(head_dim, q_rows, key_block_size) &&
      n_ext < (int64_t(1) << 31) &&
      workspace_bytes >= score_sm100_min_workspace_bytes(groups, q_rows, n_ext, n_in))
    return launch_score_sm100(reinterpret_cast<const __nv_bfloat16*>(q),
                              reinterpret_cast<const __nv_bfloat16*>(k),
                              reinterpret_cast<const __nv_bfloat16*>(k_in), groups, q_rows,
                              head_dim, kv_rows_cap, n_ext, n_in, scale, mass, workspace,
                              workspace_bytes, st);
  switch (dtype) {
    case FB_F64:
      return block_mass_t<ModeMaskF64>(q, k, k_in, groups, q_rows, head_dim, kv_rows_cap, n_ext, n_in,
                                       key_block_size, scale, mass, workspace, workspace_bytes, st);
    case FB_F32:
      return block_mass_t<ModeMaskF32>(q, k, k_in, groups, q_rows, head_dim, kv_rows_cap, n_ext, n_in,
                                       key_block_size, scale, mass, workspace, workspace_bytes, st);
    default:
      return block_mass_t<ModeMaskBF16>(q, k, k_in, groups, q_rows, head_dim, kv_rows_cap, n_ext,
                                        n_in, key_block_size, scale, mass, workspace, workspace_bytes, st);
  }
}

size_t fb_sparse_workspace_bytes(int dtype, int64_t groups, int64_t q_rows, int64_t head_dim,
                                 int64_t n_ext, int64_t n_sel, int64_t n_in, int64_t key_block_size) {
  if (dtype != FB_BF16 || !sm100_supported(head_dim) || key_block_size != 16) return 0;
  const int64_t nb = (n_ext + key_block_size - 1) / key_block_size;
  const int64_t rows = groups * q_rows;
  const size_t list_bytes = align_up((size_t)groups * std::max<int64_t>(nb - n_sel, 1) * 4, 256);
  const size_t tmp_bytes = align_up((size_t)rows * (head_dim + 1) * sizeof(float), 256);
  const size_t g1 = gather_sm100_workspace_bytes(groups, q_rows, head_dim, n_sel, n_in);
  const size_t g2 = gather_sm100_workspace_bytes(groups, q_rows, head_dim, nb - n_sel, 0);
  return std::max(list_bytes + std::max(g1, g2), tmp_bytes + g1) + 1024;
}

int fb_topk_blocks(const double* mass, int64_t groups, int64_t num_blocks, int64_t budget,
                   int32_t* selected, void* stream) {
  if (groups < 0 || num_blocks < 0 || budget < 0 || budget > num_blocks)
    return fail(FB_ERR_VALUE, "need 0 <= budget <= num_blocks");
  if (num_blocks > (int64_t(1) << 30)) return fail(FB_ERR_UNSUPPORTED, "too many blocks");
  return launch_topk(mass, groups, num_blocks, budget, selected, nullptr, 0, as_stream(stream));
}

int fb_sparse_partitioned(int dtype, const void* q, const void* k, const void* v, const void* k_in,
                          const void* v_in, int64_t groups, int64_t q_rows, int64_t head_dim,
                          int64_t kv_rows_cap, int64_t n_ext, int64_t n_in, const int32_t* selected,
                          int64_t n_sel, int64_t key_block_size, double scale, void* o_sel,
                          void* lse_sel, void* o_res, void* lse_res, void* out, int out_dtype,
                          int32_t* empty_rows, void* workspace, size_t workspace_bytes,
                          void* stream) {
  if (int rc = check_dtype(dtype)) return rc;
  if (key_block_size < 1) return fail(FB_ERR_VALUE, "key_block_size must be >= 1");
  if (groups < 0 || q_rows < 0 || head_dim < 1 || n_in < 0 || n_sel < 0)
    return fail(FB_ERR_SHAPE, "bad extents");
  if (n_ext < 0 || n_ext > kv_rows_cap) return fail(FB_ERR_SHAPE, "key set smaller than the mask");
  if (head_dim > 256) return fail(FB_ERR_UNSUPPORTED, "head_dim > 256");
  if (groups == 0 || q_rows == 0) return FB_OK;
  cudaStream_t st = as_stream(stream);
  switch (dtype) {
    case FB_F64:
      return sparse_partitioned_t<ModeF64>(q, k, v, k_in, v_in, groups, q_rows, head_dim, kv_rows_cap,
                                           n_ext, n_in, selected, n_sel, key_block_size, scale, o_sel,
                                           lse_sel, o_res, lse_res, out, false, empty_rows, workspace, workspace_bytes, st);
    case FB_F32:
      return sparse_partitioned_t<ModeF32>(q, k, v, k_in, v_in, groups, q_rows, head_dim, kv_rows_cap,
                                           n_ext, n_in, selected, n_sel, key_block_size, scale, o_sel,
                                           lse_sel, o_res, lse_res, out, false, empty_rows, workspace, workspace_bytes, st);
    default:
      return sparse_partitioned_t<ModeBF16>(q, k, v, k_in, v_in, groups, q_rows, head_dim,
                                            kv_rows_cap, n_ext, n_in, selected, n_sel, key_block_size,
                                            scale, o_sel, lse_sel, o_res, lse_res, out,
                                            out_dtype == FB_BF16, empty_rows, workspace,
                                            workspace_bytes, st);
  }
}

int fb_sparse_attend_merge(int dtype, const void* q, const void* k, const void* v, const void* k_in,
                           const void* v_in, int64_t groups, int64_t q_rows, int64_t head_dim,
                           int64_t kv_rows_cap, int64_t n_ext, int64_t n_in, const int32_t* selected,
                           int64_t n_sel, int64_t key_block_size, double scale, const void* o_res,
                           const void* lse_res, void* out, int out_dtype, int32_t* empty_rows,
                           void* workspace, size_t workspace_bytes, void* stream) {
  if (int rc = check_dtype(dtype)) return rc;
  if (key_block_size < 1) return fail(FB_ERR_VALUE, "key_block_size must be >= 1");
  if (groups < 0 || q_rows < 0 || head_dim < 1 || n_in < 0 || n_sel < 0)
    return fail(FB_ERR_SHAPE, "bad extents");
  if (n_ext < 0 || n_ext > kv_rows_cap) return fail(FB_ERR_SHAPE, "key set smaller than the mask");
  if (head_dim > 256) return fail(FB_ERR_UNSUPPORTED, "head_dim > 256");
  if ((o_res == nullptr) != (lse_res == nullptr)) return fail(FB_ERR_VALUE, "o_res/lse_res mismatch");
  if (groups == 0 || q_rows == 0) return FB_OK;
  cudaStream_t st = as_stream(stream);
  switch (dtype) {
    case FB_F64:
      if (out_dtype != FB_F64) return fail(FB_ERR_VALUE, "F64 mode writes F64 output");
      return sparse_attend_t<ModeF64>(q, k, v, k_in, v_in, groups, q_rows, head_dim, kv_rows_cap, n_ext,
                                      n_in, selected, n_sel, key_block_size, scale, o_res, lse_res,
                                      out, false, empty_rows, workspace, workspace_bytes, st);
    case FB_F32:
      if (out_dtype != FB_F32) return fail(FB_ERR_VALUE, "F32 mode writes F32 output");
      return sparse_attend_t<ModeF32>(q, k, v, k_in, v_in, groups, q_rows, head_dim, kv_rows_cap, n_ext,
                                      n_in, selected, n_sel, key_block_size, scale, o_res, lse_res,
                                      out, false, empty_rows, workspace, workspace_bytes, st);
    default:
      return sparse_attend_t<ModeBF16>(q, k, v, k_in, v_in, groups, q_rows, head_dim, kv_rows_cap,
                                       n_ext, n_in, selected, n_sel, key_block_size, scale, o_res,
                                       lse_res, out, out_dtype == FB_BF16, empty_rows, workspace,
                                       workspace_bytes, st);
  }
}

}  // extern "C"
