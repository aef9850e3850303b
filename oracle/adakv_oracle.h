/*
 * adakv_oracle.h -- CPU restatement of the Ada-KV reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * B200 kernels in paper_2407_11550_b200/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path never links, imports or calls anything under oracle/.
 *
 * Every function restates one reference function in plain C99 with the same
 * fp64 operation order (compiled with -ffp-contract=off, no -march), citing
 * the reference file:line under /root/reference/proj/include/adakv/.
 *
 * Layout conventions (shared with the device path):
 *   - a "segment" is one KV group (or one head in the weights-only API);
 *     segment s owns rows [off[s], off[s+1]) of a flat array;
 *   - K/V are stored ONCE per KV group ([rows, d] row-major), not once per
 *     query head as in the reference's LayerCache;
 *   - queries are [H, m, d]; head i belongs to group i / g.
 *
 * Status: 0 = ok, 1 = std::invalid_argument, 2 = std::out_of_range.
 * orc_last_error() returns the message of the last failure (thread-local).
 */
#ifndef ADAKV_ORACLE_H
#define ADAKV_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_INVALID_ARGUMENT = 1, ORC_OUT_OF_RANGE = 2 };

/* PolicyKind, policies.hpp:20-26 (same numeric order). */
enum { ORC_SNAPKV = 0, ORC_PYRAMID = 1, ORC_ADA_SNAPKV = 2, ORC_ADA_PYRAMID = 3,
       ORC_STREAMING_LLM = 4 };

const char* orc_last_error(void);

/* policies.hpp:80-93 */
int orc_topk_decision(const double* a, int64_t n, int64_t k, uint8_t* keep);

/* policies.hpp:99-112 */
int orc_maxpool_same(const double* row, int64_t n, int64_t kernel, double* out);

/* attention.hpp:169-179 (softmax rows of q·Kᵀ, optional 1/√d scale). out [m, n]. */
int orc_attention_weights(const double* q, int64_t m, const double* keys, int64_t n, int64_t d,
                          int scale, double* out);

/* policies.hpp:119-132.  out [n]. */
int orc_window_scores(const double* q, int64_t m, const double* keys, int64_t n, int64_t d,
                      int64_t pool_kernel, int scale, double* out);

/* policies.hpp:136-156.  scores [h, n] -> out [h/g, n]. */
int orc_group_mean_scores(const double* scores, int64_t h, int64_t n, int64_t g, double* out);

/* budget.hpp:45-93.  caps may be NULL (ample caps, budget.hpp:95-97). */
int orc_apportion(const double* quotas, int64_t h, int64_t total, const int64_t* caps,
                  int64_t* out);

/* budget.hpp:103-113 */
int orc_uniform_allocation(int64_t total, int64_t h, const int64_t* caps, int64_t* out);

/* budget.hpp:118-140.  Ragged rows: row i is a[off[i] .. off[i+1]). */
int orc_adaptive_allocation(const double* a, const int64_t* off, int64_t h, int64_t total,
                            int64_t* out);

/* budget.hpp:145-164 */
int orc_safeguard_blend(const int64_t* adaptive, int64_t adaptive_total, int64_t total,
                        int64_t h, double alpha, const int64_t* caps, int64_t* out);

/* budget.hpp:169-191 */
int orc_pyramid_layer_budgets(int64_t per_layer_avg, int64_t num_layers, double beta_max,
                              double beta_min, int64_t* out);

/* policies.hpp:178-196 (in place). */
int orc_repair_zero_budgets(int64_t* counts, const int64_t* caps, int64_t h);

/* policies.hpp:159-165 */
int orc_streaming_llm_decision(int64_t n, int64_t sink, int64_t recent, uint8_t* keep);

/* policies.hpp:298-323 (weights-only theory mode).  Ragged rows via off[h+1]. */
int orc_evict_rows(const double* w, const int64_t* off, int64_t h, int64_t total_budget,
                   int adaptive, double alpha, int64_t* alloc, uint8_t* keep);

typedef struct {
    int kind;              /* ORC_SNAPKV ... ORC_STREAMING_LLM */
    int64_t window_size;   /* validated only, policies.hpp:58, 218 */
    int64_t pool_kernel;
    double alpha;
    int64_t sink_tokens;
    int64_t gqa_group_size;
    int scale;
} orc_policy_config;

/*
 * policies.hpp:204-293 with the query projection already applied (Q = X·W_q
 * is model-side).
 *   q        [H, m, d]
 *   k_out,v_out  per-group outside rows, flat [off[G], d]; off has G+1 entries
 *   k_win,v_win  [G, m, d]
 * Outputs (caller-allocated):
 *   head_scores  [off[G] per head] -> laid out [H][n_g of its group] flat by head: may be NULL
 *   group_scores [off[G]]            pooled group-mean scores (EvictLayerResult::scores)
 *   alloc        [G]                 outside budget per group
 *   keep         [off[G]]            decision per group (members share it)
 *   k_ret,v_ret  [layer_budget, d]   retained rows, group-major, kept outside rows in
 *                                     order then the m window rows (policies.hpp:273-290)
 *   ret_len      [G]                 alloc[g] + m
 */
int orc_evict_layer(const double* q, const double* k_out, const double* v_out,
                    const int64_t* off, const double* k_win, const double* v_win, int64_t H,
                    int64_t G, int64_t m, int64_t d, int64_t layer_budget,
                    const orc_policy_config* cfg, double* head_scores, double* group_scores,
                    int64_t* alloc, uint8_t* keep, double* k_ret, double* v_ret,
                    int64_t* ret_len);

/*
 * Compressed decode for one token (report.hpp:133-144 pattern):
 * per head i: a_i = attention_weights(q_i, K_{group(i)}) (attention.hpp:169-179),
 * ctx_i = row_times(a_i, V_{group(i)}) (attention.hpp:191, matrix.hpp:79-89).
 * The W_o projection of attention_output is model-side and omitted.
 *   q [H, d]; k, v flat [off[G], d]; out [H, d]
 */
int orc_decode_attention(const double* q, const double* k, const double* v, const int64_t* off,
                         int64_t H, int64_t G, int64_t d, int scale, double* out);

/* flat_cache.hpp:44-66 / 92-120 on the reference's interleaved layout:
 * per head [K rows][V rows]; offsets count rows. */
int orc_flatten(const double* k, const double* v, const int64_t* len, int64_t h, int64_t d,
                double* data, int64_t* offsets);
int orc_select_and_compact(const double* data, const int64_t* offsets, const int64_t* lengths,
                           int64_t h, int64_t d, const uint8_t* keep /* flat by head */,
                           double* out_data, int64_t* out_offsets, int64_t* out_lengths);

/* attention.hpp:126-134 on a per-group row buffer with capacity: writes the row
 * at seg_start + len and increments len. */
int orc_append_kv(double* k_cache, double* v_cache, const int64_t* seg_start, int64_t* len,
                  const int64_t* cap, int64_t n_seg, int64_t seg, const double* k,
                  const double* v, int64_t d);

#ifdef __cplusplus
}
#endif
#endif /* ADAKV_ORACLE_H */
