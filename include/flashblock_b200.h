/*
 * flashblock_b200.h -- C ABI of the B200 (sm_100a) FlashBlock attention hot path.
 *
 * The reference (flashblock 0.1.0, /root/reference/pkg/src/flashblock) exposes
 * this path as synchronous numpy functions, one (layer, head) at a time.  This
 * library is the device-side replacement: every entry point below is
 * asynchronous on the given CUDA stream, takes caller-owned DEVICE pointers
 * with the layouts stated here, never synchronises the host, and returns an
 * fb_status.  fb_last_error() gives a human-readable message for the calling
 * thread.  Entry points are CUDA-graph capturable (no allocation, no sync).
 *
 * Layout model ("groups").  One call processes `groups` independent pairs of
 * (query block, key/value slab):
 *
 *   queries  q  + g * q_rows * head_dim            [q_rows, head_dim] row-major
 *   keys     k  + g * kv_rows_cap * head_dim       rows [key_begin, key_end)
 *   values   v  + g * kv_rows_cap * head_dim       same rows as keys
 *   partial  o  + g * q_rows * head_dim            [q_rows, head_dim]
 *   lognorm  lse+ g * q_rows                       [q_rows]
 *
 * GQA stacking: with Q laid out [batch, Hq, B, d] and the KV cache
 * [batch, Hkv, N_cap, d], groups = batch*Hkv and q_rows = (Hq/Hkv)*B -- the
 * G query heads sharing a kv head are one contiguous [G*B, d] matrix.  Every
 * hot-path function is row-independent, so this is exactly the reference
 * applied to the stacked query matrix ("GQA mapping").
 *
 * Precision modes (fb_dtype of the inputs):
 *   FB_F64  : q,k,v double; scores/statistics double; partial out double,
 *             lognorm double.                     (reference float64 path)
 *   FB_F32  : q,k,v float; scores float, statistics and accumulation double
 *             (attention.py:158-174); partial out float, lognorm double.
 *   FB_BF16 : q,k,v bf16; tcgen05 tensor cores, fp32 accumulate; partial out
 *             float, lognorm float (natural log).
 * The "partial types" of a mode are (out, lognorm) as listed.
 * An empty key group yields the sentinel out = 0, lognorm = -inf
 * (attention.py:77-82).
 */
#ifndef FLASHBLOCK_B200_H
#define FLASHBLOCK_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define FB_API __attribute__((visibility("default")))
#else
#define FB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum fb_status {
  FB_OK = 0,
  FB_ERR_SHAPE = 1,       /* -> ShapeError          (linalg.py:28)            */
  FB_ERR_BOUNDS = 2,      /* -> BoundsError         (kv_cache.py:26)          */
  FB_ERR_DEGENERATE = 3,  /* -> DegenerateInputError (attention.py:52)        */
  FB_ERR_REUSE = 4,       /* -> ReusePreconditionError (attention.py:56)      */
  FB_ERR_STALE = 5,       /* -> StalenessError      (sparse.py:43)            */
  FB_ERR_CUDA = 6,        /* CUDA runtime / launch failure                    */
  FB_ERR_VALUE = 7,       /* -> ValueError (bad density, tile, block size)    */
  FB_ERR_UNSUPPORTED = 8  /* shape/dtype combination not built                */
} fb_status;

typedef enum fb_dtype { FB_F64 = 0, FB_F32 = 1, FB_BF16 = 2 } fb_dtype;
/* OR'ed into dtype FB_BF16 where an entry point says so: the partial out of
 * the mode is stored as bf16 (the lognorm stays fp32).  The reference keeps a
 * partial's out in the tensor dtype (attention.py:70-71); for the cached
 * external partial this halves the bytes every cached step re-reads.
 * Accepted by fb_attention_partial(_sync/_ragged/_paged/_groups) (o_out
 * written bf16; the tcgen05 path only, else FB_ERR_UNSUPPORTED) and by
 * fb_internal_merge(_ex) / fb_internal_merge_tok (o_ext read as bf16; o_int /
 * lse_int not supported).  fb_combine already writes a bf16 o_out through
 * out_dtype FB_BF16 (its inputs stay fp32).  Other entry points reject the
 * bit (FB_ERR_VALUE: unknown dtype). */
#define FB_PARTIAL_BF16 0x100

/* Message for the last non-OK status returned on this host thread. */
FB_API const char* fb_last_error(void);
/* Library version string, e.g. "fb200 0.1.0 sm_100a". */
FB_API const char* fb_version(void);

/* Bytes of scratch fb_attention_partial may use for split-KV partials at this
 * shape (0 if it will not split).  Passing less makes it split less. */
FB_API size_t fb_partial_workspace_bytes(int dtype, int64_t groups, int64_t q_rows,
                                  int64_t head_dim, int64_t n_keys);

/* K1 -- block-external partial ("refresh").
 * Replaces attention_partial (attention.py:136-182) and the external half of
 * attention_streamed (attention.py:185-204, call at :202); batched over groups.
 * Streams keys [key_begin, key_end) of every slab once; writes the normalised
 * partial (o_out, lse_out) in the mode's partial types.  key_begin==key_end
 * writes the empty sentinel.  BF16 with head_dim in {64,128} runs the
 * TMA + tcgen05/TMEM kernel; other shapes run the SIMT kernel. */
FB_API int fb_attention_partial(int dtype, const void* q, const void* k, const void* v,
                         int64_t groups, int64_t q_rows, int64_t head_dim,
                         int64_t kv_rows_cap, int64_t key_begin, int64_t key_end,
                         double scale, void* o_out, void* lse_out,
                         void* workspace, size_t workspace_bytes, void* stream);

/* K1 with the in-kernel split merge (stream-K fix-up without a second kernel).
 * sync_flags: a DEVICE buffer of n_flags uint64 (>= fb_sync_flags_count()),
 * all zero before the first use and not shared by launches that may run
 * concurrently; every launch leaves it zero again.  Used when every split
 * item spans <= 3 CTAs (C2 b >= 16); otherwise -- and with sync_flags NULL,
 * which is fb_attention_partial -- split items are merged by a second kernel.
 * The merging CTA spin-waits (bounded, 4 s watchdog) on partials written by
 * other CTAs of the same launch: the grid is one CTA per SM, so the wait
 * makes progress when the launch owns the GPU; a kernel running concurrently
 * on another stream only delays it.  Keep one buffer per stream (the Python
 * layer keys it by stream).
 * Same arguments and results as fb_attention_partial otherwise. */
FB_API int fb_attention_partial_sync(int dtype, const void* q, const void* k, const void* v,
                                     int64_t groups, int64_t q_rows, int64_t head_dim,
                                     int64_t kv_rows_cap, int64_t key_begin, int64_t key_end,
                                     double scale, void* o_out, void* lse_out, void* workspace,
                                     size_t workspace_bytes, uint64_t* sync_flags, int64_t n_flags,
                                     void* stream);
/* Length of the sync_flags buffer fb_attention_partial_sync expects. */
FB_API int64_t fb_sync_flags_count(void);

/* K1 over per-sequence (ragged) context lengths -- the serving layout where
 * each sequence of the batch has its own committed length.
 * Group g streams rows [key_begin, min(key_end[g], kv_rows_cap)) of its slab;
 * key_end is a DEVICE int32 array [groups].  Rows past a group's end are never
 * used (scores masked, V rows zeroed in shared memory), even if the slab holds
 * uninitialised memory there; groups with no keys get the empty sentinel.
 * Same outputs and partial types as fb_attention_partial. */
FB_API int fb_attention_partial_ragged(int dtype, const void* q, const void* k, const void* v,
                                       int64_t groups, int64_t q_rows, int64_t head_dim,
                                       int64_t kv_rows_cap, int64_t key_begin,
                                       const int32_t* key_end, double scale, void* o_out,
                                       void* lse_out, void* workspace, size_t workspace_bytes,
                                       void* stream);
FB_API size_t fb_ragged_workspace_bytes(int dtype, int64_t groups, int64_t q_rows,
                                        int64_t head_dim, int64_t kv_rows_cap);

/* Block-causal attention: the prefill / commit pass.
 * Replaces the per-block attention_dense calls of the reference's commit pass
 * (_context_hidden, simulator.py:297-325) over a whole prompt (prefill,
 * simulator.py:343-354) in one launch.  q: [groups, q_rows, head_dim] with
 * q_rows = heads_per_group * n_q (the group's query heads stacked, each n_q
 * positions); k/v slabs hold the committed prefix in rows [0, n_prefix) and
 * the new positions' keys in rows [n_prefix, n_prefix + n_q) (commit them
 * with fb_commit_block first).  Query row r (position p = r % n_q) attends
 * rows [0, n_prefix + min(n_q, (p / block_size + 1) * block_size)): every
 * earlier block and its own block, bidirectionally.  Writes the attention
 * output and its log-sum-exp in the mode's partial types (F64: f64/f64;
 * F32: f32/f64, scores in float64 as attention_dense; BF16: f32/f32, the
 * TMA + tcgen05 kernel for head_dim in {64,128}). */
FB_API int fb_block_causal_attention(int dtype, const void* q, const void* k, const void* v,
                                     int64_t groups, int64_t q_rows, int64_t n_q, int64_t head_dim,
                                     int64_t kv_rows_cap, int64_t n_prefix, int64_t block_size,
                                     double scale, void* o_out, void* lse_out, void* workspace,
                                     size_t workspace_bytes, void* stream);
FB_API size_t fb_block_causal_workspace_bytes(int dtype, int64_t groups, int64_t q_rows,
                                              int64_t head_dim);

/* K1 over a subset of groups -- the head-gated refresh (policy.py:84-94 with
 * per-head gates, simulator.py:401-405): only the groups listed in
 * group_list (DEVICE int32 [n_list], distinct indices < groups) are refreshed;
 * every other group's rows of o_out / lse_out are left untouched.  Same
 * arguments and partial types as fb_attention_partial otherwise; scratch from
 * fb_partial_workspace_bytes(dtype, n_list, ...).  F64 and BF16 modes (F32:
 * FB_ERR_UNSUPPORTED). */
FB_API int fb_attention_partial_groups(int dtype, const void* q, const void* k, const void* v,
                                       int64_t groups, int64_t q_rows, int64_t head_dim,
                                       int64_t kv_rows_cap, int64_t key_begin, int64_t key_end,
                                       const int32_t* group_list, int64_t n_list, double scale,
                                       void* o_out, void* lse_out, void* workspace,
                                       size_t workspace_bytes, void* stream);

/* Cross-step similarity (head-gate calibration, policy.py:188-246; stability
 * study, analysis.py:28-148).  a, b: [heads, rows, head_dim] partial outputs
 * of the same rows at two steps, dtype FB_F64 / FB_F32 / FB_BF16 (the array
 * type).  row_cos[heads*rows] (required): cosine of row r of a and b, 0 when
 * either norm < 1e-12 (linalg.py:68-80); head_mean[heads] (optional): its
 * mean over the rows.  Float64 accumulation, fixed reduction order. */
FB_API int fb_row_cosine(int dtype, const void* a, const void* b, int64_t heads, int64_t rows,
                         int64_t head_dim, double* row_cos, double* head_mean, void* stream);
/* fb_row_cosine for the calibrator's step (policy.py:232-240 per adjacent step
 * pair): the same statistics of a against b, then b <- a (b is the previous
 * step's copy, in place), and *nonzero (optional int32) set to 1 if any row of
 * a is nonzero (the all-zero-partials CalibrationError check).  One pass:
 * 2 reads + 1 write per element. */
FB_API int fb_row_cosine_update(int dtype, const void* a, void* b, int64_t heads, int64_t rows,
                                int64_t head_dim, double* row_cos, double* head_mean, int32_t* nonzero,
                                void* stream);
/* All-pairs cosine between the rows of a later and an earlier step, per head:
 * out[heads, rows, rows], entry (i, j) = cos(later_i, earlier_j); rows with
 * norm < 1e-12 give 0 (pairwise_step_similarity, analysis.py:28-51). */
FB_API int fb_pairwise_cosine(int dtype, const void* later, const void* earlier, int64_t heads,
                              int64_t rows, int64_t head_dim, double* out, void* stream);

/* Device-side block commit (kv_cache.py:121-144; simulator.py:327-333):
 * append a finished block's K/V rows ([groups, block_rows, head_dim]) to each
 * group's slab at row lengths[g] (device int32 [groups]), then advance
 * lengths[g] by block_rows.  Rows past kv_rows_cap are dropped and counted in
 * *overflow (device int32, optional).  The caller invalidates its cached
 * external partials afterwards (attention.py:287-289). */
FB_API int fb_commit_block(int dtype, void* k_cache, void* v_cache, int64_t groups,
                           int64_t kv_rows_cap, int64_t head_dim, const void* k_block,
                           const void* v_block, int64_t block_rows, int32_t* lengths,
                           int32_t* overflow, void* stream);

/* Paged KV cache (the serving layout): K and V of every
 * group live in a shared page pool [num_pages, page_rows, head_dim]; group
 * g's logical row r is row r % page_rows of page page_table[g * max_pages +
 * r / page_rows] (device int32).  K1 over rows [0, key_len[g]) of each group
 * (device int32 [groups]) -- same outputs as fb_attention_partial_ragged on
 * the equivalent contiguous slabs.  Page-table entries covering rows below
 * key_len[g] must be valid pages.  BF16 with head_dim 64 / 128 and page_rows a
 * multiple of 128 (one TMA box per 128-key tile); FB_ERR_UNSUPPORTED
 * otherwise. */
FB_API int fb_attention_partial_paged(int dtype, const void* q, const void* k_pages,
                                      const void* v_pages, int64_t num_pages, int64_t page_rows,
                                      const int32_t* page_table, int64_t max_pages, int64_t groups,
                                      int64_t q_rows, int64_t head_dim, const int32_t* key_len,
                                      double scale, void* o_out, void* lse_out, void* workspace,
                                      size_t workspace_bytes, void* stream);
FB_API size_t fb_paged_workspace_bytes(int dtype, int64_t groups, int64_t q_rows, int64_t head_dim);
/* Block-causal (prefill / commit) attention over a paged cache: the same
 * rows and limits as fb_block_causal_attention, keys [0, n_prefix + n_q) of
 * group g read through its page table (the prompt committed into the pages
 * first).  BF16, head_dim 64 / 128, page_rows a multiple of 128; workspace
 * fb_paged_workspace_bytes. */
FB_API int fb_block_causal_attention_paged(int dtype, const void* q, const void* k_pages,
                                           const void* v_pages, int64_t num_pages, int64_t page_rows,
                                           const int32_t* page_table, int64_t max_pages,
                                           int64_t groups, int64_t q_rows, int64_t n_q,
                                           int64_t head_dim, int64_t n_prefix, int64_t block_size,
                                           double scale, void* o_out, void* lse_out,
                                           void* workspace, size_t workspace_bytes, void* stream);
/* Sparse path (K5 block mass, K7 first step, K8 cached step) over a paged
 * cache: the same semantics as fb_block_mass / fb_sparse_partitioned /
 * fb_sparse_attend_merge, with group g's cache row r read from row
 * r % page_rows of page page_table[g * max_pages + r / page_rows] of the
 * pools [num_pages, page_rows, head_dim].  BF16, head_dim 64 / 128,
 * key_block_size 16, page_rows a multiple of 128 (fb_block_mass_paged: q_rows
 * <= 128); rows of the last page past n_ext must hold finite values.
 * Workspace: fb_block_mass_workspace_bytes_ex / fb_sparse_workspace_bytes. */
FB_API int fb_block_mass_paged(int dtype, const void* q, const void* k_pages, const void* k_in,
                               int64_t num_pages, int64_t page_rows, const int32_t* page_table,
                               int64_t max_pages, int64_t groups, int64_t q_rows, int64_t head_dim,
                               int64_t n_ext, int64_t n_in, int64_t key_block_size, double scale,
                               double* mass, void* workspace, size_t workspace_bytes, void* stream);
FB_API int fb_sparse_partitioned_paged(int dtype, const void* q, const void* k_pages,
                                       const void* v_pages, const void* k_in, const void* v_in,
                                       int64_t num_pages, int64_t page_rows,
                                       const int32_t* page_table, int64_t max_pages, int64_t groups,
                                       int64_t q_rows, int64_t head_dim, int64_t n_ext, int64_t n_in,
                                       const int32_t* selected, int64_t n_sel,
                                       int64_t key_block_size, double scale, void* o_sel,
                                       void* lse_sel, void* o_res, void* lse_res, void* out,
                                       int out_dtype, int32_t* empty_rows, void* workspace,
                                       size_t workspace_bytes, void* stream);
FB_API int fb_sparse_attend_merge_paged(int dtype, const void* q, const void* k_pages,
                                        const void* v_pages, const void* k_in, const void* v_in,
                                        int64_t num_pages, int64_t page_rows,
                                        const int32_t* page_table, int64_t max_pages, int64_t groups,
                                        int64_t q_rows, int64_t head_dim, int64_t n_ext, int64_t n_in,
                                        const int32_t* selected, int64_t n_sel,
                                        int64_t key_block_size, double scale, const void* o_res,
                                        const void* lse_res, void* out, int out_dtype,
                                        int32_t* empty_rows, void* workspace,
                                        size_t workspace_bytes, void* stream);
/* Cached step (K2) on token-major tensors: q [batch, block, num_q_heads,
 * head_dim], k_in / v_in [batch, block, num_kv_heads, head_dim] given by their
 * token strides in elements (e.g. views into one fused QKV projection output
 * [batch * block, (Hq + 2 Hkv) * d]), output written token-major with
 * out_token_stride (the O projection's input [batch * block, Hq * d]); the
 * cached external partial keeps the stacked [batch * Hkv, G * block, d]
 * layout.  Same arithmetic as fb_internal_merge_ex; bf16, head_dim 128,
 * G * block <= 128, block <= 64. */
FB_API int fb_internal_merge_tok(int dtype, const void* q, int64_t q_token_stride, const void* k_in,
                                 int64_t k_token_stride, const void* v_in, int64_t v_token_stride,
                                 int64_t batch, int64_t block, int64_t num_q_heads,
                                 int64_t num_kv_heads, int64_t head_dim, double scale,
                                 const void* o_ext, const void* lse_ext, void* out, int out_dtype,
                                 int64_t out_token_stride, int flags, void* stream);
/* Paged block commit: rows lengths[g] .. lengths[g] + block_rows - 1 of group
 * g go to their pages (rows past the table or onto a negative page id are
 * dropped and counted in *overflow); lengths advance by block_rows. */
FB_API int fb_commit_block_paged(int dtype, void* k_pages, void* v_pages, int64_t page_rows,
                                 const int32_t* page_table, int64_t max_pages, int64_t groups,
                                 int64_t head_dim, const void* k_block, const void* v_block,
                                 int64_t block_rows, int32_t* lengths, int32_t* overflow,
                                 void* stream);

/* K2 -- cached step: block-internal partial fused with the log-space merge
 * against the cached external partial.
 * Replaces attention_with_reuse (attention.py:295-321) = attention_partial on
 * the internal keys (:320) + merge_partials (:321, :236-245).  Never receives
 * the KV cache.  k_in/v_in: [groups, n_in, head_dim] (slab stride n_in).
 * o_ext/lse_ext: partial types of the mode.  out: out_dtype (FB_F64 for F64,
 * FB_F32 for F32; FB_F32 or FB_BF16 for BF16).  Optional (NULL to skip):
 * lse_merged (lognorm type), o_int/lse_int (the internal partial, partial
 * types), empty_rows (device int32 counter incremented once per row with no
 * keys on either side; the caller raises DegenerateInputError if > 0). */
FB_API int fb_internal_merge(int dtype, const void* q, const void* k_in, const void* v_in,
                      int64_t groups, int64_t q_rows, int64_t head_dim, int64_t n_in,
                      double scale, const void* o_ext, const void* lse_ext,
                      void* out, int out_dtype, void* lse_merged,
                      void* o_int, void* lse_int, int32_t* empty_rows,
                      void* workspace, size_t workspace_bytes, void* stream);
/* fb_internal_merge with flags.  FB_EXT_STABLE: o_ext / lse_ext were not
 * written by the kernel immediately preceding this call on the stream (true
 * for every cached step: the external partial is produced at the last
 * refresh), so the kernel may read them before its programmatic-dependent-
 * launch wait and overlap those loads with the predecessor's tail. */
#define FB_EXT_STABLE 1
FB_API int fb_internal_merge_ex(int dtype, const void* q, const void* k_in, const void* v_in,
                                int64_t groups, int64_t q_rows, int64_t head_dim, int64_t n_in,
                                double scale, const void* o_ext, const void* lse_ext, void* out,
                                int out_dtype, void* lse_merged, void* o_int, void* lse_int,
                                int32_t* empty_rows, void* workspace, size_t workspace_bytes,
                                int flags, void* stream);
/* Scratch fb_internal_merge needs at this shape: 0 for blocks of <= 128 keys
 * (one fused tcgen05 kernel); large blocks (video chunks) run the stream-K
 * tensor-core partial over the block's keys plus a K3 merge and need this
 * much (without it they fall back to the SIMT kernel). */
/* Host-buffer cached step: attention_with_reuse (attention.py:295-321) for
 * the reference's synchronous numpy signature in ONE call.  q [groups,
 * q_rows, d], k_in / v_in [groups, n_in, d] and the outputs are HOST arrays
 * in the mode's element type (FB_F64: double, FB_F32: float; lognorms are
 * double in both); o_ext / lse_ext are the DEVICE cached external partial
 * (the partial types of the mode).  The inputs are packed into a per-thread
 * pinned staging buffer and uploaded with one copy, the cached step runs on
 * `stream`, and out / o_int / lse_int (o_int, lse_int optional: NULL skips)
 * come back with one copy and one stream synchronisation.  *empty_rows (may
 * be NULL) receives the number of rows with no keys on either side; the
 * caller raises DegenerateInputError if it is > 0, as the reference does.
 * Only FB_F64 / FB_F32 (numpy has no bf16). */
FB_API int fb_internal_merge_host(int dtype, const void* q, const void* k_in, const void* v_in,
                                  int64_t groups, int64_t q_rows, int64_t head_dim, int64_t n_in,
                                  double scale, const void* o_ext, const void* lse_ext, void* out,
                                  void* o_int, double* lse_int, int64_t* empty_rows, void* stream);
FB_API size_t fb_internal_merge_workspace_bytes(int dtype, int64_t groups, int64_t q_rows,
                                                int64_t head_dim, int64_t n_in);

/* K3 -- P-way log-space combine of partials over disjoint key groups.
 * Replaces combine_partials (attention.py:207-233) / merge_partials (:236-245)
 * and is the split-KV merge (one partial per shard).  o_parts[p], lse_parts[p]
 * are host arrays of device pointers (partial types of the mode), each
 * [rows, head_dim] / [rows].  Rows empty on one side pass through bitwise;
 * rows empty everywhere stay empty and bump *empty_rows when given.
 * Outputs: o_out in out_dtype (partial out type, or FB_BF16 in BF16 mode),
 * lse_out (lognorm type, may be NULL).  1 <= n_parts <= 16. */
FB_API int fb_combine(int dtype, int n_parts, const void* const* o_parts,
               const void* const* lse_parts, int64_t rows, int64_t head_dim,
               void* o_out, int out_dtype, void* lse_out, int32_t* empty_rows,
               void* stream);

/* K4 -- full recompute over [committed | current block] keys, normalised
 * output.  Replaces attention_streamed(boundary=committed) + merge_partials
 * (simulator.py:424-429) and attention_dense for the GPU baseline.  Runs K1
 * over the cache into (o_ext_scratch, lse_ext_scratch) then K2; those scratch
 * buffers (partial types, [groups, q_rows, (head_dim)]) also receive the
 * refreshed external partial, so a refresh step is exactly this call. */
FB_API int fb_full_attention(int dtype, const void* q, const void* k, const void* v,
                      int64_t groups, int64_t q_rows, int64_t head_dim,
                      int64_t kv_rows_cap, int64_t n_ext,
                      const void* k_in, const void* v_in, int64_t n_in, double scale,
                      void* o_ext_scratch, void* lse_ext_scratch,
                      void* out, int out_dtype, int32_t* empty_rows,
                      void* workspace, size_t workspace_bytes, void* stream);

/* K5 -- sparse block scoring.  Replaces the score/softmax/mass stage of
 * build_sparse_mask (sparse.py:117-125): softmax over ALL keys (external
 * [0,n_ext) from the cache plus the n_in current-block keys), probability
 * mass per external key block of key_block_size rows summed over the q_rows
 * rows of the group.  mass: double [groups, ceil(n_ext/kbs)].  Scores are
 * formed in double for FB_F64/FB_F32 (as the reference) and in float from
 * bf16 products for FB_BF16; masses always accumulate in double. */
FB_API int fb_block_mass(int dtype, const void* q, const void* k, const void* k_in,
                  int64_t groups, int64_t q_rows, int64_t head_dim,
                  int64_t kv_rows_cap, int64_t n_ext, int64_t n_in,
                  int64_t key_block_size, double scale, double* mass,
                  void* workspace, size_t workspace_bytes, void* stream);
FB_API size_t fb_block_mass_workspace_bytes(int64_t groups, int64_t q_rows);
/* Workspace for fb_block_mass at this exact shape (covers the tcgen05 path
 * taken for BF16, head_dim 64/128, q_rows <= 128, key_block_size 16). */
FB_API size_t fb_block_mass_workspace_bytes_ex(int dtype, int64_t groups, int64_t q_rows,
                                               int64_t head_dim, int64_t n_ext, int64_t n_in,
                                               int64_t key_block_size);

/* K6 -- stable top-k block selection.  Replaces sparse.py:126-128: order by
 * (mass desc, index asc), keep `budget`, emit ascending.  selected: int32
 * [groups, budget].  budget must be min(nb, max(1, ceil(density*n_ext/kbs)))
 * (fb_mask_budget computes it exactly as the reference, in double). */
FB_API int fb_topk_blocks(const double* mass, int64_t groups, int64_t num_blocks,
                   int64_t budget, int32_t* selected, void* stream);
FB_API int64_t fb_mask_budget(int64_t n_ext, double density, int64_t key_block_size);

/* K7 -- sparse first step, exact partition (sparse.py:166-175): selected
 * partial over the selected external blocks PLUS all n_in current-block keys,
 * residual partial over the unselected external keys; both written (partial
 * types), plus the merged output (out_dtype).  selected: int32 [groups, n_sel]
 * ascending block ids of key_block_size rows (tail block clipped at n_ext). */
FB_API int fb_sparse_partitioned(int dtype, const void* q, const void* k, const void* v,
                          const void* k_in, const void* v_in,
                          int64_t groups, int64_t q_rows, int64_t head_dim,
                          int64_t kv_rows_cap, int64_t n_ext, int64_t n_in,
                          const int32_t* selected, int64_t n_sel,
                          int64_t key_block_size, double scale,
                          void* o_sel, void* lse_sel, void* o_res, void* lse_res,
                          void* out, int out_dtype, int32_t* empty_rows,
                          void* workspace, size_t workspace_bytes, void* stream);

/* K8 -- later sparse steps (sparse.py:177-183): attend the selected external
 * blocks (gathered straight from the cache by block index, no copy) plus the
 * current block, and merge the cached residual in the epilogue.  o_res may be
 * NULL for the renormalised sparse-only baseline (sparse.py:317-322). */
FB_API int fb_sparse_attend_merge(int dtype, const void* q, const void* k, const void* v,
                           const void* k_in, const void* v_in,
                           int64_t groups, int64_t q_rows, int64_t head_dim,
                           int64_t kv_rows_cap, int64_t n_ext, int64_t n_in,
                           const int32_t* selected, int64_t n_sel,
                           int64_t key_block_size, double scale,
                           const void* o_res, const void* lse_res,
                           void* out, int out_dtype, int32_t* empty_rows,
                           void* workspace, size_t workspace_bytes, void* stream);

/* Scratch for fb_sparse_partitioned / fb_sparse_attend_merge (BF16 tcgen05
 * gather path: split partials, the residual block list, the temporary
 * selected partial).  Other modes need none. */
FB_API size_t fb_sparse_workspace_bytes(int dtype, int64_t groups, int64_t q_rows,
                                        int64_t head_dim, int64_t n_ext, int64_t n_sel,
                                        int64_t n_in, int64_t key_block_size);

/* Count of kernel launches issued by this library since load (for bench). */
FB_API int64_t fb_launch_count(void);

/* ---------------------------------------------------------------- peer memory
 * Split-KV exchange over peer memory: the ranks of one node map
 * each other's packed partial buffers with CUDA IPC; a refresh then signals
 * its peers after K1, waits for theirs, and runs the K3 merge (fb_combine)
 * straight on the peers' mapped partials -- no collective, no staging copy.
 * Replaces the NCCL exchange of the reference-side split (there is none in
 * the single-process reference: simulator.py runs one sequence on one CPU;
 * the merge itself is combine_partials, attention.py:207-233). */
#define FB_P2P_HANDLE_BYTES 64
/* cudaMalloc'ed, zeroed device memory and its 64-byte IPC handle. */
FB_API int fb_p2p_alloc(size_t bytes, void** ptr, void* handle);
FB_API int fb_p2p_free(void* ptr);
/* Map a peer process's buffer (its fb_p2p_alloc handle) into this process. */
FB_API int fb_p2p_open(const void* handle, void** ptr);
FB_API int fb_p2p_close(void* ptr);
/* On `stream`, after everything queued before it: a system-scope fence, then
 * flags[p][slot] = value (release) for each of the n DEVICE pointers in the
 * DEVICE array peer_flags (typically every rank's flag array, own included). */
FB_API int fb_p2p_signal(uint64_t* const* peer_flags, int n, int slot, uint64_t value, void* stream);
/* On `stream`: block until flags[i] >= value for every i < n (n <= 32;
 * acquire, system scope).  Watchdog: traps after ~4 s without progress. */
FB_API int fb_p2p_wait(const uint64_t* flags, int n, uint64_t value, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FLASHBLOCK_B200_H */
