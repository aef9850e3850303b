/*
 * adakv_b200.h -- C ABI of the B200-native Ada-KV compression + compressed-decode path.
 *
 * This is the drop-in boundary.  The reference is a header-only
 * C++20 library (namespace adakv, /root/reference/proj/include/adakv/); its hot
 * path is evict_layer() and the decode math applied to the retained cache.  Each
 * entry point below names the reference function(s) it replaces (file:line).  The
 * C++ wrappers in include/adakv_b200/adakv.hpp keep the reference's exact
 * signatures on top of these calls; performance callers use this ABI directly.
 *
 * Conventions
 *   - Device pointers, stream-ordered, caller-owned buffers and workspace; the
 *     library allocates nothing on the hot path.  Entry points return an
 *     adakv_status; adakv_last_error() holds the message (thread-local).
 *   - Status codes map one-to-one onto the reference's exception vocabulary:
 *     std::invalid_argument, std::out_of_range, adakv::FormatError (serde.hpp:18-21),
 *     adakv::IoError (serde.hpp:24-27).
 *   - Shapes are validated on the host before anything is launched, reproducing
 *     the reference's throw sites (policies.hpp:65-72, 208-237; budget.hpp:48-59,
 *     121, 130-131, 148-152; flat_cache.hpp:94-101; attention.hpp:128-131, 170-172).
 *     Data-dependent violations detected on the device (e.g. a non-finite key)
 *     latch into the workspace error word; adakv_workspace_status() reads it.
 *   - A "problem" is one independent (request, layer) unit; P problems of equal
 *     shape are processed by one call (batch and layer batching).
 *   - Prompt K/V layout: [P, G, n, d] row-major, n = n_o + m; the observation
 *     window is the last m rows (the reference passes them separately as
 *     cache_outside / window_cache, policies.hpp:204-206).  Each KV group is
 *     stored once (the reference keeps g identical copies, policies.hpp:276).
 *   - Queries: [P, H, m, d] for scoring, [P, H, d] for decode; head i reads KV
 *     group i / (H / G) (policies.hpp:244).
 *   - Compressed cache: two planes K,V of [rows, d]; segment (p, g) occupies rows
 *     [seg_start[p*G+g], seg_start + capacity), holds seqlens[p*G+g] valid rows:
 *     the kept outside rows in original order, then the m window rows
 *     (policies.hpp:273-290).  With reserve = 0, seg_start is exactly the
 *     flattened layout's offsets (flat_cache.hpp:24-36, SPEC "offsets count rows").
 */
#ifndef ADAKV_B200_H
#define ADAKV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADAKV_B200_ABI_VERSION 2

typedef struct CUstream_st* adakv_stream_t; /* == cudaStream_t */

typedef enum adakv_status {
    ADAKV_OK = 0,
    ADAKV_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    ADAKV_OUT_OF_RANGE = 2,     /* std::out_of_range */
    ADAKV_FORMAT_ERROR = 3,     /* adakv::FormatError */
    ADAKV_IO_ERROR = 4,         /* adakv::IoError */
    ADAKV_CUDA_ERROR = 5,
    ADAKV_UNSUPPORTED = 6,
    ADAKV_WORKSPACE_TOO_SMALL = 7
} adakv_status;

typedef enum adakv_dtype {
    ADAKV_F32 = 0,  /* fp32 storage, fp32 math (SIMT) */
    ADAKV_F64 = 1,  /* fp64 storage, fp64 math (SIMT; the reference-typed wrappers) */
    ADAKV_BF16 = 2  /* bf16 storage, fp32 accumulate; tcgen05 tensor cores when d == 128 */
} adakv_dtype;

/* PolicyKind, policies.hpp:20-26 (same numeric order). */
typedef enum adakv_policy_kind {
    ADAKV_SNAPKV = 0,
    ADAKV_PYRAMID = 1,
    ADAKV_ADA_SNAPKV = 2,
    ADAKV_ADA_PYRAMID = 3,
    ADAKV_STREAMING_LLM = 4
} adakv_policy_kind;

/* PolicyConfig, policies.hpp:56-73 (POD mirror). */
typedef struct adakv_policy_config {
    int32_t kind;           /* adakv_policy_kind */
    int32_t scale;          /* 1: logits * 1/sqrt(d) (attention.hpp:159-163) */
    int64_t window_size;    /* validated only (policies.hpp:58, 218) */
    int64_t pool_kernel;    /* odd */
    double alpha;           /* safeguard blend, [0,1] */
    int64_t sink_tokens;    /* streaming_llm */
    int64_t gqa_group_size; /* g = H / G */
} adakv_policy_config;

typedef struct adakv_layer_shape {
    int64_t problems;  /* P */
    int64_t q_heads;   /* H */
    int64_t kv_groups; /* G */
    int64_t window;    /* m */
    int64_t outside;   /* n_o: positions before the window */
    int64_t head_dim;  /* d */
} adakv_layer_shape;

const char* adakv_last_error(void);
int adakv_abi_version(void);
/* Selects the scoring kernel for eligible shapes (bf16, d == 128, m == 32, g*m <= 128):
 * 1 = tcgen05 tensor-core kernel (default), 0 = the generic SIMT kernel.  Returns the
 * previous setting.  Both compute the same function; this exists for A/B checks. */
int adakv_set_tensor_core_scoring(int enabled);
/* Device address of a pinned (page-locked) host buffer, for the arguments documented as
 * accepting one (adakv_compress's v).  ADAKV_INVALID_ARGUMENT if `host` is not pinned host
 * memory mapped into the device's address space. */
adakv_status adakv_host_device_pointer(const void* host, void** device_ptr);
/* Reads back (synchronously) the device error word latched in a workspace and maps it onto
 * the reference's exception (message included):
 *   non-finite K/V               -> ADAKV_INVALID_ARGUMENT "LayerCache: non-finite entry"
 *                                   (LayerCache::validate, attention.hpp:76-83)
 *   budget outside floor/capacity -> ADAKV_INVALID_ARGUMENT (policies.hpp:229-231, budget.hpp:48-59)
 *   append past a segment's capacity -> ADAKV_INVALID_ARGUMENT "append_kv: capacity exhausted"
 * Every workspace starts with this 256-byte error header; it is cleared by the entry points
 * that take the workspace as their first stage (compress, window_scores, segmented_select)
 * and accumulates otherwise (decode, append), so one read after a decode loop reports any
 * step that overflowed.  adakv_clear_workspace_status() resets it. */
adakv_status adakv_workspace_status(const void* workspace, adakv_stream_t stream);
adakv_status adakv_clear_workspace_status(void* workspace, adakv_stream_t stream);

/* LayerCache::validate (attention.hpp:76-83) on the device: latches ERR_NONFINITE in the
 * workspace error word if any of the n elements at `data` (dtype) is NaN or +-Inf.  The
 * compress path checks, for free, every K entry that reaches a window row's softmax
 * statistics (a NaN or +Inf logit) and every K/V row the gather copies (retained + window
 * rows); a caller that needs the reference's full check of the prompt cache (every K and V
 * entry, including evicted rows) runs this over k and v first: one extra HBM read. */
adakv_status adakv_validate_finite(adakv_dtype dtype, const void* data, int64_t n, void* workspace,
                                   adakv_stream_t stream);

/* ----------------------------------------------------------------------------
 * Full single-layer eviction pass for P problems:
 *   replaces evict_layer (policies.hpp:204-293): window_scores (119-132) for every
 *   head, group_mean_scores (136-156), adaptive_allocation (budget.hpp:118-140) +
 *   safeguard_blend (145-158) + repair_zero_budgets (policies.hpp:178-196) or
 *   uniform_allocation (budget.hpp:103-113), topk_decision (policies.hpp:80-93) or
 *   streaming_llm_decision (159-165), and the compaction loop (273-290) ==
 *   select_and_compact (flat_cache.hpp:92-120).
 *
 *   layer_budget     unique KV entries per problem incl. the window (policies.hpp:229-231)
 *   layer_budgets    optional DEVICE int64 [P] per-problem budgets (pyramid kinds); NULL = uniform
 *   reserve          extra rows per segment for decode appends (capacity = budget_g + m + reserve)
 *   k_cache,v_cache  output planes, adakv_cache_rows() rows of d elements (same dtype as k)
 *   seg_start,seqlens  DEVICE int32 [P*G]
 *   seg_cap          DEVICE int32 [P*G] or NULL: each segment's capacity in rows
 *                    (budget_g + m + reserve); decode / append refuse to write past it
 *   budgets          DEVICE int32 [P*G] outside budget per group (EvictLayerResult::allocation)
 *   group_scores     DEVICE [P*G*n_o] f32 (f64 for ADAKV_F64) or NULL (EvictLayerResult::scores)
 *   keep             DEVICE uint8 [P*G*n_o] or NULL (EvictLayerResult::decision, group leaders)
 *   v                may also be a device-accessible address of pinned HOST memory (see
 *                    adakv_host_device_pointer): V is read only by the final gather, for the
 *                    retained and window rows (layer_budget rows per problem), so a prompt
 *                    whose V lives on the host crosses the host link for those rows only
 *                    (k and q are read in full by the scoring and must be in device memory)
 * ------------------------------------------------------------------------- */
adakv_status adakv_compress(adakv_dtype dtype, const adakv_layer_shape* shape,
                            const adakv_policy_config* cfg, int64_t layer_budget,
                            const int64_t* layer_budgets, const void* q, const void* k,
                            const void* v, int64_t reserve, void* k_cache, void* v_cache,
                            int32_t* seg_start, int32_t* seqlens, int32_t* seg_cap, int32_t* budgets,
                            void* group_scores, uint8_t* keep, void* workspace,
                            size_t workspace_bytes, adakv_stream_t stream);
/* adakv_compress with the final gather (the copy of the retained K/V rows into the cache
 * planes) enqueued on `gather_stream` instead of `stream`, after an event recorded on
 * `stream` once the selection and the layout are written; `stream` does not wait for it.
 * For a model compressed in layer chunks as its prompt arrives, chunk i's gather -- bound by
 * the host link when V is in pinned host memory -- then overlaps chunk i+1's scoring.  The
 * gather reads this call's workspace (kept positions) and writes its error word, so:
 *   - k_cache / v_cache (and the workspace status) are complete only once the caller has
 *     made its next reader wait for gather_stream (cudaStreamWaitEvent);
 *   - the workspace must not be reused on `stream` before that wait.
 * gather_stream == NULL or == stream is adakv_compress exactly.  (No reference counterpart:
 * evict_layer is one synchronous call, policies.hpp:204-293.) */
adakv_status adakv_compress_split(adakv_dtype dtype, const adakv_layer_shape* shape,
                                  const adakv_policy_config* cfg, int64_t layer_budget,
                                  const int64_t* layer_budgets, const void* q, const void* k,
                                  const void* v, int64_t reserve, void* k_cache, void* v_cache,
                                  int32_t* seg_start, int32_t* seqlens, int32_t* seg_cap,
                                  int32_t* budgets, void* group_scores, uint8_t* keep, void* workspace,
                                  size_t workspace_bytes, adakv_stream_t stream,
                                  adakv_stream_t gather_stream);
adakv_status adakv_compress_workspace(adakv_dtype dtype, const adakv_layer_shape* shape,
                                      const adakv_policy_config* cfg, size_t* bytes);
/* Rows of each output plane: P * (layer_budget + G * reserve), or the sum over
 * problems when per-problem budgets are used (pass their host copy). */
int64_t adakv_cache_rows(const adakv_layer_shape* shape, int64_t layer_budget,
                         const int64_t* layer_budgets_host, int64_t reserve);

/* ----------------------------------------------------------------------------
 * Stage 1 -- observation-window scoring (K1).
 *   replaces window_scores (policies.hpp:119-132) over attention_weights
 *   (attention.hpp:169-179) and maxpool_same (99-112), for every head, and
 *   group_mean_scores (136-156).
 *   head_scores   DEVICE [P, H, n_o] or NULL (per-head window_scores output)
 *   group_scores  DEVICE [P, G, n_o] (f32; f64 for ADAKV_F64)
 * ------------------------------------------------------------------------- */
adakv_status adakv_window_scores(adakv_dtype dtype, const adakv_layer_shape* shape,
                                 int64_t pool_kernel, int32_t scale, const void* q,
                                 const void* k, void* head_scores, void* group_scores,
                                 void* workspace, size_t workspace_bytes, adakv_stream_t stream);
adakv_status adakv_window_scores_workspace(adakv_dtype dtype, const adakv_layer_shape* shape,
                                           size_t* bytes);

/* ----------------------------------------------------------------------------
 * Stage 2 -- segmented selection (K2 layer-wide radix select + allocation, K3
 * per-segment select).  S segments per problem, ragged: segment s is
 * scores[p*off[S] + off[s] .. + off[s+1]).  Keys are f32 or f64 (exact order,
 * -0 == +0; NaN not allowed).  Order (score desc, segment asc, position asc).
 * S (<= 64: KV groups, for adakv_compress) is held in one CTA's shared memory as
 * per-segment histograms; beyond ~39 segments on B200 a leaner layout with one
 * more cluster barrier per radix pass is used.
 * ------------------------------------------------------------------------- */
typedef enum adakv_alloc_mode {
    ADAKV_ALLOC_ADAPTIVE = 0, /* adaptive_allocation (budget.hpp:118-140) [+ safeguard_blend] */
    ADAKV_ALLOC_UNIFORM = 1,  /* uniform_allocation (budget.hpp:103-113) */
    ADAKV_ALLOC_GIVEN = 2     /* budgets supplied in `budgets` (topk_decision per segment) */
} adakv_alloc_mode;

typedef struct adakv_select_config {
    int32_t alloc_mode;  /* adakv_alloc_mode */
    int32_t blend;       /* apply safeguard_blend(alpha) after adaptive allocation */
    int32_t repair;      /* apply repair_zero_budgets (policies.hpp:178-196) */
    int32_t streaming;   /* decision = streaming_llm_decision(sink, b - sink) instead of top-k */
    double alpha;
    int64_t sink_tokens;
} adakv_select_config;

/*   seg_off       HOST int64 [S+1], seg_off[0] == 0
 *   total         outside budget per problem (ignored for GIVEN); totals: optional DEVICE int64 [P]
 *   raw_counts    DEVICE int32 [P*S] adaptive counts before blending, or NULL
 *   budgets       DEVICE int32 [P*S]: out (in for GIVEN)
 *   keep          DEVICE uint8 [P*off[S]] or NULL
 *   kept_pos      DEVICE int32 [P*kept_stride] or NULL: kept positions (within segment),
 *                 segment-major, ascending; problem p's list starts at p*kept_stride */
adakv_status adakv_segmented_select(adakv_dtype key_dtype, int64_t problems, int64_t segments,
                                    const int64_t* seg_off, const void* scores, int64_t total,
                                    const int64_t* totals, const adakv_select_config* cfg,
                                    int32_t* raw_counts, int32_t* budgets, uint8_t* keep,
                                    int32_t* kept_pos, int64_t kept_stride, void* workspace,
                                    size_t workspace_bytes, adakv_stream_t stream);
adakv_status adakv_segmented_select_workspace(int64_t problems, int64_t segments,
                                              size_t* bytes);

/* ----------------------------------------------------------------------------
 * Stage 3 -- compaction gather (K3 copy half): for every (p, g) copy the kept
 * outside rows (kept_pos from adakv_segmented_select) then the m window rows into
 * the output planes; writes seg_start / seqlens (and seg_cap if not NULL).  Bit-exact copy,
 * 16-byte vectors; the copied rows are checked for non-finite entries (ERR_NONFINITE in the
 * error word at `workspace`, which may be NULL to skip the latch).
 * layer_budget / layer_budgets as for adakv_compress (they fix each problem's row base).
 * ------------------------------------------------------------------------- */
adakv_status adakv_gather(adakv_dtype dtype, const adakv_layer_shape* shape, int64_t layer_budget,
                          const int64_t* layer_budgets, const void* k, const void* v,
                          const int32_t* budgets, const int32_t* kept_pos, int64_t kept_stride,
                          int64_t reserve, void* k_cache, void* v_cache, int32_t* seg_start,
                          int32_t* seqlens, int32_t* seg_cap, void* workspace, adakv_stream_t stream);

/* ----------------------------------------------------------------------------
 * Decode (K4 split-K varlen flash-decoding + K5 append):
 *   replaces attention_weights (attention.hpp:169-179) + row_times(a, V) (the context
 *   part of attention_output, 182-196) for one new token per problem, applied to the
 *   retained cache as in report.hpp:133-144; and append_kv (attention.hpp:126-134).
 *   q          DEVICE [P, H, d]
 *   k_cache, v_cache  the planes (cache_rows rows of d elements each; the segments'
 *              seg_start offsets index into them)
 *   seg_cap    DEVICE int32 [P*G]: capacity of each segment in rows (from adakv_compress)
 *   k_new,v_new  DEVICE [P, G, d] or NULL: appended at row seqlens (the new token's
 *              own K/V, attended in the same step); seqlens is then incremented on the
 *              device.  A segment already at capacity is not written: its attention runs
 *              over the existing rows and ERR_CAPACITY is latched in the workspace error
 *              word (append_kv's std::invalid_argument through adakv_workspace_status).
 *   out        DEVICE [P, H, d] (same dtype as q)
 *   flags      ADAKV_DECODE_CHAINED: the caller guarantees that the kernel enqueued directly
 *              before this call on `stream` is an adakv_decode of OTHER segments and writes
 *              nothing this call reads (its cache rows, seg_start, seg_cap, seqlens, q, k_new,
 *              v_new) -- the layers of one decode step, enqueued back to back.  The call
 *              then overlaps its predecessor through programmatic dependent launch (its
 *              cache rows stream in while the previous layer finishes; q is still read only
 *              after the predecessor has completed).  0: plain stream order.
 * ------------------------------------------------------------------------- */
#define ADAKV_DECODE_CHAINED 1u
adakv_status adakv_decode(adakv_dtype dtype, int64_t problems, int64_t q_heads,
                          int64_t kv_groups, int64_t head_dim, int32_t scale, const void* q,
                          void* k_cache, void* v_cache, int64_t cache_rows, const int32_t* seg_start,
                          const int32_t* seg_cap, int32_t* seqlens, int64_t max_rows, const void* k_new,
                          const void* v_new, void* out, void* workspace, size_t workspace_bytes,
                          uint32_t flags, adakv_stream_t stream);
/* max_rows: upper bound of any segment length during this call (grid sizing; the
 * launch covers ceil(max_rows / chunk) splits so the call can live in a CUDA graph).
 * The workspace must be zero-initialised before its first decode; the split-K kernels re-arm
 * the per-segment tickets they keep in it, so it stays valid for further calls of the SAME
 * (problems, q_heads, kv_groups, head_dim, max_rows) -- a call of another layout needs its own
 * (or a re-zeroed) workspace. */
adakv_status adakv_decode_workspace(int64_t problems, int64_t q_heads, int64_t kv_groups,
                                    int64_t head_dim, int64_t max_rows, size_t* bytes);

/* Disables (0) the overlap of ADAKV_DECODE_CHAINED calls (they then run in plain stream
 * order; for A/B measurements); returns the previous setting (default 1). */
int adakv_set_decode_overlap(int enabled);

/* append_kv (attention.hpp:126-134) alone: one row per segment listed.  A segment at
 * capacity (seg_cap) is left untouched and ERR_CAPACITY is latched in `workspace`'s error
 * word (>= 256 bytes). */
adakv_status adakv_append_kv(adakv_dtype dtype, int64_t segments, int64_t head_dim,
                             void* k_cache, void* v_cache, const int32_t* seg_start,
                             const int32_t* seg_cap, int32_t* seqlens, const void* k_new,
                             const void* v_new, void* workspace, adakv_stream_t stream);
/* append_kv (attention.hpp:126-134) repeated `rows` times per segment (e.g. the question
 * tokens appended after a question-agnostic compression): k_new / v_new DEVICE
 * [segments, rows, d]; seqlens[s] += rows.  A segment without `rows` free rows is left
 * untouched and ERR_CAPACITY is latched, as for adakv_append_kv. */
adakv_status adakv_append_rows(adakv_dtype dtype, int64_t segments, int64_t rows, int64_t head_dim,
                               void* k_cache, void* v_cache, const int32_t* seg_start,
                               const int32_t* seg_cap, int32_t* seqlens, const void* k_new,
                               const void* v_new, void* workspace, adakv_stream_t stream);

/* ----------------------------------------------------------------------------
 * Budget integerisation on the device (bit-exact fp64, no FMA contraction).
 * HOST arrays in/out; each call runs one single-thread kernel and synchronises.
 * ------------------------------------------------------------------------- */
/* detail::apportion, budget.hpp:45-93 (caps NULL = ample_caps, 95-97) */
adakv_status adakv_apportion(const double* quotas, int64_t h, int64_t total,
                             const int64_t* caps, int64_t* out);
/* uniform_allocation, budget.hpp:103-113 */
adakv_status adakv_uniform_allocation(int64_t total, int64_t h, const int64_t* caps,
                                      int64_t* out);
/* safeguard_blend, budget.hpp:145-164 */
adakv_status adakv_safeguard_blend(const int64_t* adaptive, int64_t adaptive_total,
                                   int64_t total, int64_t h, double alpha, const int64_t* caps,
                                   int64_t* out);
/* detail::repair_zero_budgets, policies.hpp:178-196 (in place) */
adakv_status adakv_repair_zero_budgets(int64_t* counts, const int64_t* caps, int64_t h);
/* pyramid_layer_budgets, budget.hpp:169-191 */
adakv_status adakv_pyramid_layer_budgets(int64_t per_layer_avg, int64_t num_layers,
                                         double beta_max, double beta_min, int64_t* out);

/* ----------------------------------------------------------------------------
 * fp64 device kernels behind the reference-typed C++ API (include/adakv_b200/adakv.hpp).
 * All pointers DEVICE, stream-ordered; loop orders follow the reference without FMA.
 * ------------------------------------------------------------------------- */
/* matmul (matrix.hpp:91-102) for every head: q[h] = x * w[h]; x [m, D], w [H, D, d], q [H, m, d] */
adakv_status adakv_project_queries_f64(const double* x, const double* w, int64_t H, int64_t m, int64_t D,
                                       int64_t d, double* q, adakv_stream_t stream);
/* group_mean_scores (policies.hpp:136-156): scores [h, n] -> out [h/g, n] */
adakv_status adakv_group_mean_scores_f64(const double* scores, int64_t h, int64_t n, int64_t g, double* out,
                                         adakv_stream_t stream);
/* attention_weights (attention.hpp:169-179): q [m, d], k [n, d] -> out [m, n] */
adakv_status adakv_attention_weights_f64(const double* q, int64_t m, const double* k, int64_t n, int64_t d,
                                         int32_t scale, double* out, adakv_stream_t stream);
/* attention_output (attention.hpp:182-196): ragged weight rows w (woff[H+1]), values v (voff[H+1]
 * rows of dh), wo [H, dh, D] -> y [D]; ctx_ws holds H*dh doubles */
adakv_status adakv_attention_output_f64(const double* w, const int64_t* woff, const double* v,
                                        const int64_t* voff, int64_t H, int64_t dh, const double* wo, int64_t D,
                                        double* ctx_ws, double* y, adakv_stream_t stream);
/* select_and_compact (flat_cache.hpp:92-120): rows with mask != 0 of each segment, in order.
 * off / out_off: DEVICE int64 [segments + 1] */
adakv_status adakv_compact_rows_f64(int64_t segments, const uint8_t* mask, const int64_t* off, const double* src_k,
                                    const double* src_v, int64_t d, const int64_t* out_off, double* dst_k,
                                    double* dst_v, adakv_stream_t stream);

/* ----------------------------------------------------------------------------
 * KV-group sharding glue (sharding.py; no single reference counterpart: the
 * layer-wide top-B of adaptive_allocation, budget.hpp:118-140, with the KV
 * groups of a layer spread over ranks).
 * adakv_shard_pack_candidates: this rank's ONE all-gather payload, int32
 *   [local_groups + 2k] = [counts | f32 bits of the k candidate scores | positions],
 *   from scores [local_groups, outside] f32 and the local top-k (counts per group,
 *   positions segment-major ascending), all DEVICE.
 * adakv_shard_build_union: gathered [world, local_groups + 2k] -> union [world *
 *   local_groups, slots] f32: each group's candidate scores in position order, -1
 *   (below every score) in the empty slots.
 * ------------------------------------------------------------------------- */
adakv_status adakv_shard_pack_candidates(const float* scores, const int32_t* counts, const int32_t* pos,
                                         int64_t local_groups, int64_t outside, int64_t k, int32_t* payload,
                                         adakv_stream_t stream);
adakv_status adakv_shard_build_union(const int32_t* gathered, int64_t world, int64_t local_groups, int64_t k,
                                     int64_t slots, float* out, adakv_stream_t stream);

/* Device memory helpers so C/C++ callers need nothing but this header (synchronous). */
adakv_status adakv_device_malloc(void** ptr, size_t bytes);
adakv_status adakv_device_free(void* ptr);
adakv_status adakv_memcpy_to_device(void* dst, const void* src, size_t bytes);
adakv_status adakv_memcpy_to_host(void* dst, const void* src, size_t bytes);
adakv_status adakv_device_synchronize(void);

#ifdef __cplusplus
}
#endif
#endif /* ADAKV_B200_H */
