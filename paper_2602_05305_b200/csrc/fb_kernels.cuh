// Internal kernel-launch interface shared by the C-ABI layer and the kernels.
#pragma once

#include "fb_common.cuh"
#include "fb_keymap.cuh"

namespace fb {

constexpr int FB_MAX_PARTS = 16;

// Parts of a combine: a pointer list (API combine, split-KV shards) or a
// strided workspace (intra-GPU split partials).
struct CombineList {
  const void* o[FB_MAX_PARTS];
  const void* l[FB_MAX_PARTS];
  int n;
  bool strided;
  int64_t o_stride, l_stride;  // elements between parts when strided
};

// K2 merge-epilogue operands: the cached external partial and the outputs.
template <typename Mode>
struct MergeOut {
  const typename Mode::To* o_ext;  // [rows_total, d]
  const typename Mode::Tl* lse_ext;
  void* out;                       // To, or bf16 when out_bf16
  bool out_bf16;
  typename Mode::Tl* lse_merged;   // optional
  typename Mode::To* o_int;        // optional internal partial
  typename Mode::Tl* lse_int;
  int32_t* empty_rows;             // optional
};

template <typename Mode, bool MERGE, bool NO_V, typename Map>
int launch_partial_simt(const typename Mode::Tin* q, const Map& map, int64_t groups,
                        int64_t q_rows, int64_t head_dim, int64_t per_split, int splits,
                        double scale, typename Mode::Ta* po, typename Mode::Tl* pl,
                        const MergeOut<Mode>& mo, cudaStream_t st,
                        const int32_t* glist = nullptr);  // grid groups -> slabs (subset)

template <typename Tp, typename Tlp, typename Ta, typename To, typename Tlo>
int launch_combine(const CombineList& list, int64_t rows, int64_t head_dim, To* o_out, Tlo* l_out,
                   int32_t* empty_rows, cudaStream_t st);

template <typename Mode>
int launch_block_mass(const typename Mode::Tin* q, const typename Mode::Tin* k,
                      const double* row_lse, int64_t groups, int64_t q_rows, int64_t head_dim,
                      int64_t slab_stride, int64_t n_ext, int64_t kbs, double scale, double* mass,
                      cudaStream_t st);
int launch_commit_block(void* kc, void* vc, const void* kb, const void* vb, int64_t groups,
                        int64_t cap, int64_t row_bytes, int64_t blk_rows, int32_t* len,
                        int32_t* overflow, cudaStream_t st);
int launch_complement(const int32_t* sel, int64_t groups, int64_t n_sel, int64_t nb, int32_t* out,
                      cudaStream_t st);
int launch_topk(const double* mass, int64_t groups, int64_t nb, int64_t budget, int32_t* selected,
                void* scratch, size_t scratch_bytes, cudaStream_t st);

template <typename To, typename Tl>
int launch_fill_sentinel(To* o, Tl* l, int64_t rows, int64_t head_dim, cudaStream_t st);

// Optional final step fused into K1's split-merge kernel: merge every row's
// partial with a second fp32 partial (o2, l2; e.g. the cached residual) and
// write the attention output (bf16 or fp32) instead of a partial, counting
// rows empty on both sides -- K3 folded into the same launch.
struct MergeFinal {
  const void* o2;  // fp32, or bf16 when o2_bf16
  const float* l2;
  void* out;
  int out_bf16;
  int32_t* empty_rows;
  int o2_bf16;
  int skip_partial;  // the K1 partial itself is scratch: the cluster reduction does not store it (K8)
};

// tcgen05 / TMA refresh kernel (bf16, head_dim 64 or 128): normalised fp32
// partial + fp32 natural-log lse over keys [key_begin, key_end) of every
// group, written to (o_out, lse_out).  Stream-K over all SMs; split partials
// are merged in-kernel by the last CTA of each item (needs the workspace of
// refresh_sm100_workspace_bytes; with less it runs one CTA per item).
bool sm100_supported(int64_t head_dim);
void set_refresh_trace(void* p);
void set_k1_diag(int d);
void set_pair_enabled(int on);  // -1 default (env FB_PAIR; block-causal only), 0 off, 1 all shapes
long long pair_launches();       // CTA-pair K1 launches so far (diagnostics)
void set_quad_mode(int m);        // two-query-tile K1: -1 default (causal), 0 off, 1 all shapes
long long quad_launches();
void set_k1_cluster_mode(int m);  // cluster split-K K1: -1 default (auto), 0 off, 1 whenever feasible
void set_k1_fin_whole(int m);    // K1 epilogue final merge for whole items: -1 environment (default on), 0 off, 1 on
long long k1_cluster_launches();
void set_gather_atoms(int m);     // K7 / K8 atom layout: -1 default (on), 0 off, 1 on
void set_k1_gbar_mode(int m);     // grid-barrier split-K: -1 default, 0 off, 1 vs merge kernel, 2 also vs owner merge
void set_k2_trace(void* p, int launches);  // diagnostics: K2 v1 per-CTA stamps
void set_k5_mode(int m);         // K5 scoring: -1 environment (default fused), 0 fused, 1 two-pass
long long k5_fused_launches();
void set_k2_vsplit(int v);       // K2 v2: -1 default / 1 V_in on its own barrier, 0 one Q/K/V barrier
void set_k2_store(int v);        // K2 v2 output: -1 default (TMA store), 0 per-thread stores, 1 TMA store (diagnostics)
void set_k2_v2(int v);           // K2 variant: -1 by size (default), 0 v1, 1 v2 (diagnostics)
size_t refresh_sm100_workspace_bytes(int64_t groups, int64_t q_rows, int64_t head_dim, int64_t n_keys);
int launch_refresh_sm100(const __nv_bfloat16* q, const __nv_bfloat16* k, const __nv_bfloat16* v,
                         int64_t groups, int64_t q_rows, int64_t head_dim, int64_t kv_rows_cap,
                         int64_t key_begin, int64_t key_end, double scale, float* o_out,
                         float* lse_out, void* ws, size_t ws_bytes, cudaStream_t st,
                         unsigned long long* sync_flags = nullptr, int64_t n_flags = 0,
                         const MergeFinal* fin = nullptr);

// Ragged per-group key ends (device int32 [groups], clamped to kv_rows_cap).
size_t refresh_sm100_ragged_workspace_bytes(int64_t groups, int64_t q_rows, int64_t head_dim);
// Paging context for the sparse path (K5 / K7 / K8) over a paged cache: set
// for the duration of one fb_*_paged call on the calling thread (re-entrant
// across threads), read by launch_score_sm100 / launch_gather_sm100 to build
// tensor maps over the page pool and translate block rows through the table.
struct PagingCtx {
  const int32_t* table;
  int64_t max_pages, page_rows, num_pages;
};
const PagingCtx* current_paging();
struct ScopedPaging {
  explicit ScopedPaging(const PagingCtx* p);
  ~ScopedPaging();
};
// Partial-out context (FB_PARTIAL_BF16): set for the duration of one
// fb_attention_partial* call on the calling thread; the refresh launcher then
// writes the final partial O as bf16 (split workspace partials stay fp32).
struct ScopedPartialBf16 {
  explicit ScopedPartialBf16(bool on);
  ~ScopedPartialBf16();
};
bool partial_out_bf16();
int launch_refresh_paged_sm100(const __nv_bfloat16* q, const __nv_bfloat16* k_pages,
                               const __nv_bfloat16* v_pages, int64_t num_pages, int64_t page_rows,
                               const int32_t* page_table, int64_t max_pages, int64_t groups,
                               int64_t q_rows, int64_t head_dim, const int32_t* key_len, double scale,
                               float* o_out, float* lse_out, void* ws, size_t ws_bytes, cudaStream_t st);
int launch_block_causal_paged_sm100(const __nv_bfloat16* q, const __nv_bfloat16* k_pages,
                                    const __nv_bfloat16* v_pages, int64_t num_pages, int64_t page_rows,
                                    const int32_t* page_table, int64_t max_pages, int64_t groups,
                                    int64_t q_rows, int64_t head_dim, int64_t n_q, int64_t n_prefix,
                                    int64_t block, double scale, float* o_out, float* lse_out, void* ws,
                                    size_t ws_bytes, cudaStream_t st);
int launch_commit_block_paged(void* kp, void* vp, int64_t page_rows, const int32_t* table,
                              int64_t max_pages, const void* kb, const void* vb, int64_t groups,
                              int64_t row_bytes, int64_t blk_rows, int32_t* len, int32_t* overflow,
                              cudaStream_t st);
int launch_refresh_ragged_sm100(const __nv_bfloat16* q, const __nv_bfloat16* k,
                                const __nv_bfloat16* v, int64_t groups, int64_t q_rows,
                                int64_t head_dim, int64_t kv_rows_cap, int64_t key_begin,
                                const int32_t* key_end, double scale, float* o_out, float* lse_out,
                                void* ws, size_t ws_bytes, cudaStream_t st);
int launch_refresh_groups_sm100(const __nv_bfloat16* q, const __nv_bfloat16* k, const __nv_bfloat16* v,
                                int64_t groups, int64_t q_rows, int64_t head_dim, int64_t kv_rows_cap,
                                int64_t key_begin, int64_t key_end, const int32_t* glist,
                                int64_t n_list, double scale, float* o_out, float* lse_out, void* ws,
                                size_t ws_bytes, cudaStream_t st);
int launch_block_causal_sm100(const __nv_bfloat16* q, const __nv_bfloat16* k, const __nv_bfloat16* v,
                              int64_t groups, int64_t q_rows, int64_t head_dim, int64_t kv_rows_cap,
                              int64_t n_q, int64_t n_prefix, int64_t block, double scale,
                              float* o_out, float* lse_out, void* ws, size_t ws_bytes,
                              cudaStream_t st);

// Gathered variant (sparse K7/K8): keys = mask-selected 16-row blocks of the
// cache (list [groups, n_list] of ascending block ids, rows clipped at n_ext)
// followed by the n_in current-block rows of k_in / v_in ([groups, n_in, d]).
struct GatherSpec {
  const int32_t* list;
  int64_t n_list, n_ext, n_in;
  const __nv_bfloat16* k_in;
  const __nv_bfloat16* v_in;
};
size_t gather_sm100_workspace_bytes(int64_t groups, int64_t q_rows, int64_t head_dim,
                                    int64_t n_list, int64_t n_in);
int launch_gather_sm100(const __nv_bfloat16* q, const __nv_bfloat16* k, const __nv_bfloat16* v,
                        int64_t groups, int64_t q_rows, int64_t head_dim, int64_t kv_rows_cap,
                        const GatherSpec& gs, double scale, float* o_out, float* lse_out, void* ws,
                        size_t ws_bytes, cudaStream_t st, const MergeFinal* fin = nullptr);

// K5 on the tensor cores (bf16, q_rows <= 128, kbs == 16): float64 block masses.
bool score_sm100_supported(int64_t head_dim, int64_t q_rows, int64_t kbs);
size_t score_sm100_workspace_bytes(int64_t groups, int64_t q_rows, int64_t n_ext, int64_t n_in);
size_t score_sm100_min_workspace_bytes(int64_t groups, int64_t q_rows, int64_t n_ext, int64_t n_in);
int launch_score_sm100(const __nv_bfloat16* q, const __nv_bfloat16* k, const __nv_bfloat16* k_in,
                       int64_t groups, int64_t q_rows, int64_t head_dim, int64_t cap, int64_t n_ext,
                       int64_t n_in, double scale, double* mass, void* ws, size_t ws_bytes,
                       cudaStream_t st);

bool sm100_k2_supported(int64_t head_dim, int64_t n_in);
int launch_internal_merge_tok_sm100(const __nv_bfloat16* q, int64_t q_ts, const __nv_bfloat16* k,
                                    int64_t k_ts, const __nv_bfloat16* v, int64_t v_ts, int64_t batch,
                                    int64_t B, int64_t Hq, int64_t Hkv, int64_t d, double scale,
                                    const void* o_ext, const float* lse_ext, void* out, int64_t out_ts,
                                    bool out_bf16, bool ext_early, bool extb, cudaStream_t st);
int launch_internal_merge_sm100(const __nv_bfloat16* q, const __nv_bfloat16* k_in,
                                const __nv_bfloat16* v_in, int64_t groups, int64_t q_rows,
                                int64_t head_dim, int64_t n_in, double scale, const void* o_ext,
                                const float* lse_ext, void* out, bool out_bf16, float* lse_merged,
                                float* o_int, float* lse_int, int32_t* empty, bool ext_early,
                                bool extb, cudaStream_t st);

// cross-step similarity (fb_similarity.cu)
template <typename T>
int launch_row_cosine(const void* a, const void* b, int64_t heads, int64_t rows, int64_t d,
                      double* row_cos, double* head_mean, cudaStream_t st, bool update = false,
                      int* nonzero = nullptr);
template <typename T>
int launch_pairwise_cosine(const void* later, const void* earlier, int64_t heads, int64_t n,
                           int64_t d, double* out, cudaStream_t st);

}  // namespace fb
