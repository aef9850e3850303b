/*
 * adakv_oracle.c -- plain-C fp64 restatement of the Ada-KV reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see adakv_oracle.h).  Compile with
 *   gcc -std=c99 -O2 -ffp-contract=off -fPIC -shared
 * so that every a*b+c stays two roundings, exactly as the reference's
 * Release build (-O3, no -march => no FMA on x86-64) evaluates it.
 *
 * Citations are /root/reference/proj/include/adakv/<file>:<line>.
 */
#include "adakv_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

const char* orc_last_error(void) { return g_err; }

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

/* std::max(a, b) == (a < b) ? b : a */
static double dmax(double a, double b) { return (a < b) ? b : a; }

/* ------------------------------------------------------------------------ */
/* Sorting helpers: a stable merge sort of index arrays under a strict weak
 * order.  The reference's orders are total (value, then index), so any
 * correct sort reproduces std::sort's permutation.                          */

typedef int (*less_fn)(int64_t x, int64_t y, const void* ctx);

static void merge_sort(int64_t* idx, int64_t* tmp, int64_t n, less_fn less, const void* ctx) {
    if (n < 2) return;
    int64_t h = n / 2;
    merge_sort(idx, tmp, h, less, ctx);
    merge_sort(idx + h, tmp, n - h, less, ctx);
    int64_t i = 0, j = h, o = 0;
    while (i < h && j < n) {
        if (less(idx[j], idx[i], ctx)) tmp[o++] = idx[j++];
        else tmp[o++] = idx[i++];
    }
    while (i < h) tmp[o++] = idx[i++];
    while (j < n) tmp[o++] = idx[j++];
    memcpy(idx, tmp, (size_t)n * sizeof(int64_t));
}

/* policies.hpp:86-89: a[x] != a[y] ? a[x] > a[y] : x < y */
static int less_value_desc_pos_asc(int64_t x, int64_t y, const void* ctx) {
    const double* a = (const double*)ctx;
    if (a[x] != a[y]) return a[x] > a[y];
    return x < y;
}

/* ------------------------------------------------------------------------ */

int orc_topk_decision(const double* a, int64_t n, int64_t k, uint8_t* keep) {
    /* policies.hpp:80-93 */
    if (k > n) return fail(ORC_INVALID_ARGUMENT, "topk_decision: k exceeds length");
    int64_t* order = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    int64_t* tmp = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) order[i] = i;
    merge_sort(order, tmp, n, less_value_desc_pos_asc, a);
    memset(keep, 0, (size_t)n);
    for (int64_t r = 0; r < k; ++r) keep[order[r]] = 1;
    free(order);
    free(tmp);
    return ORC_OK;
}

int orc_maxpool_same(const double* row, int64_t n, int64_t kernel, double* out) {
    /* policies.hpp:99-112: stride 1, pad (k-1)/2, padded cells excluded */
    if (kernel % 2 == 0 || kernel == 0)
        return fail(ORC_INVALID_ARGUMENT, "maxpool: kernel must be odd");
    const int64_t pad = (kernel - 1) / 2;
    for (int64_t j = 0; j < n; ++j) {
        const int64_t lo = j >= pad ? j - pad : 0;
        const int64_t hi = (n < j + pad + 1) ? n : j + pad + 1;
        double m = row[lo];
        for (int64_t t = lo + 1; t < hi; ++t) m = dmax(m, row[t]);
        out[j] = m;
    }
    return ORC_OK;
}

/* matrix.hpp:111-116 */
static double dot(const double* a, const double* b, int64_t n) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* attention.hpp:141-157 with an empty mask */
static int softmax_inplace(double* logits, int64_t n) {
    double maxv = -INFINITY;
    for (int64_t j = 0; j < n; ++j) maxv = dmax(maxv, logits[j]);
    if (!isfinite(maxv)) return fail(ORC_INVALID_ARGUMENT, "softmax: no retained position");
    double denom = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        logits[j] = exp(logits[j] - maxv);
        denom += logits[j];
    }
    for (int64_t j = 0; j < n; ++j) logits[j] /= denom;
    return ORC_OK;
}

int orc_attention_weights(const double* q, int64_t m, const double* keys, int64_t n, int64_t d,
                          int scale, double* out) {
    /* attention.hpp:169-179; scores_row 159-163 */
    if (n == 0) return fail(ORC_INVALID_ARGUMENT, "attention_weights: empty key set");
    const double inv = scale ? 1.0 / sqrt((double)d) : 1.0;
    for (int64_t r = 0; r < m; ++r) {
        double* row = out + r * n;
        for (int64_t j = 0; j < n; ++j) row[j] = dot(q + r * d, keys + j * d, d) * inv;
        int st = softmax_inplace(row, n);
        if (st) return st;
    }
    return ORC_OK;
}

int orc_window_scores(const double* q, int64_t m, const double* keys, int64_t n, int64_t d,
                      int64_t pool_kernel, int scale, double* out) {
    /* policies.hpp:119-132 */
    if (m == 0) return fail(ORC_INVALID_ARGUMENT, "window_scores: empty window");
    double* a = (double*)malloc((size_t)(m * n > 0 ? m * n : 1) * sizeof(double));
    double* pooled = (double*)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    int st = orc_attention_weights(q, m, keys, n, d, scale, a);
    if (st) goto done;
    for (int64_t j = 0; j < n; ++j) out[j] = 0.0;
    for (int64_t r = 0; r < m; ++r) {
        st = orc_maxpool_same(a + r * n, n, pool_kernel, pooled);
        if (st) goto done;
        for (int64_t j = 0; j < n; ++j) out[j] += pooled[j];
    }
    for (int64_t j = 0; j < n; ++j) out[j] /= (double)m;
done:
    free(a);
    free(pooled);
    return st;
}

int orc_group_mean_scores(const double* scores, int64_t h, int64_t n, int64_t g, double* out) {
    /* policies.hpp:136-156 (uniform member length) */
    if (g == 0) return fail(ORC_INVALID_ARGUMENT, "group_mean_scores: zero group size");
    if (h % g != 0)
        return fail(ORC_INVALID_ARGUMENT,
                    "group_mean_scores: head count not divisible by group size");
    for (int64_t gi = 0; gi < h / g; ++gi) {
        double* acc = out + gi * n;
        for (int64_t j = 0; j < n; ++j) acc[j] = 0.0;
        for (int64_t k = 0; k < g; ++k) {
            const double* s = scores + (gi * g + k) * n;
            for (int64_t j = 0; j < n; ++j) acc[j] += s[j];
        }
        for (int64_t j = 0; j < n; ++j) acc[j] /= (double)g;
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* budget.hpp */

static const uint64_t kAmpleCap = UINT64_MAX / 2; /* budget.hpp:95-97 */

static int apportion_u(const double* quotas, int64_t h, uint64_t total, const uint64_t* caps,
                       uint64_t* out) {
    /* budget.hpp:45-93 */
    uint64_t cap_sum = 0;
    for (int64_t i = 0; i < h; ++i)
        cap_sum = (cap_sum > UINT64_MAX - caps[i]) ? UINT64_MAX : cap_sum + caps[i];
    if (total > cap_sum) return fail(ORC_INVALID_ARGUMENT, "apportion: total exceeds capacity");
    uint64_t assigned = 0;
    for (int64_t i = 0; i < h; ++i) {
        if (!(quotas[i] >= 0.0)) return fail(ORC_INVALID_ARGUMENT, "apportion: negative quota");
        const uint64_t base = (uint64_t)floor(quotas[i]);
        out[i] = base < caps[i] ? base : caps[i];
        assigned += out[i];
    }
    while (assigned < total) {
        int64_t pick = h;
        double best = -INFINITY;
        for (int64_t i = 0; i < h; ++i) {
            if (out[i] >= caps[i]) continue;
            const double deficit = quotas[i] - (double)out[i];
            if (deficit > best) {
                best = deficit;
                pick = i;
            }
        }
        ++out[pick];
        ++assigned;
    }
    while (assigned > total) {
        int64_t pick = h;
        double best = -INFINITY;
        for (int64_t i = 0; i < h; ++i) {
            if (out[i] == 0) continue;
            const double surplus = (double)out[i] - quotas[i];
            if (surplus > best) {
                best = surplus;
                pick = i;
            }
        }
        --out[pick];
        --assigned;
    }
    return ORC_OK;
}

static uint64_t* caps_or_ample(const int64_t* caps, int64_t h) {
    uint64_t* c = (uint64_t*)malloc((size_t)(h > 0 ? h : 1) * sizeof(uint64_t));
    for (int64_t i = 0; i < h; ++i) c[i] = caps ? (uint64_t)caps[i] : kAmpleCap;
    return c;
}

int orc_apportion(const double* quotas, int64_t h, int64_t total, const int64_t* caps,
                  int64_t* out) {
    uint64_t* c = caps_or_ample(caps, h);
    uint64_t* o = (uint64_t*)malloc((size_t)(h > 0 ? h : 1) * sizeof(uint64_t));
    int st = apportion_u(quotas, h, (uint64_t)total, c, o);
    if (!st)
        for (int64_t i = 0; i < h; ++i) out[i] = (int64_t)o[i];
    free(c);
    free(o);
    return st;
}

int orc_uniform_allocation(int64_t total, int64_t h, const int64_t* caps, int64_t* out) {
    /* budget.hpp:103-113 */
    if (h == 0) return fail(ORC_INVALID_ARGUMENT, "uniform_allocation: no heads");
    double* quotas = (double*)malloc((size_t)h * sizeof(double));
    for (int64_t i = 0; i < h; ++i) quotas[i] = (double)total / (double)h;
    int st = orc_apportion(quotas, h, total, caps, out);
    free(quotas);
    return st;
}

typedef struct {
    const double* a;
    const int64_t* head;
    const int64_t* pos;
} entry_ctx;

/* budget.hpp:132-136: w desc, head asc, pos asc */
static int less_entry(int64_t x, int64_t y, const void* vctx) {
    const entry_ctx* c = (const entry_ctx*)vctx;
    if (c->a[x] != c->a[y]) return c->a[x] > c->a[y];
    if (c->head[x] != c->head[y]) return c->head[x] < c->head[y];
    return c->pos[x] < c->pos[y];
}

int orc_adaptive_allocation(const double* a, const int64_t* off, int64_t h, int64_t total,
                            int64_t* out) {
    /* budget.hpp:118-140 */
    if (h == 0) return fail(ORC_INVALID_ARGUMENT, "adaptive_allocation: no heads");
    const int64_t n = off[h] - off[0];
    if (total > n)
        return fail(ORC_INVALID_ARGUMENT, "adaptive_allocation: total exceeds element count");
    int64_t* head = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    int64_t* pos = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    int64_t* order = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    int64_t* tmp = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    for (int64_t i = 0; i < h; ++i)
        for (int64_t j = off[i]; j < off[i + 1]; ++j) {
            head[j - off[0]] = i;
            pos[j - off[0]] = j - off[i];
        }
    for (int64_t e = 0; e < n; ++e) order[e] = e;
    entry_ctx ctx = {a + off[0], head, pos};
    merge_sort(order, tmp, n, less_entry, &ctx);
    for (int64_t i = 0; i < h; ++i) out[i] = 0;
    for (int64_t r = 0; r < total; ++r) ++out[head[order[r]]];
    free(head);
    free(pos);
    free(order);
    free(tmp);
    return ORC_OK;
}

int orc_safeguard_blend(const int64_t* adaptive, int64_t adaptive_total, int64_t total,
                        int64_t h, double alpha, const int64_t* caps, int64_t* out) {
    /* budget.hpp:145-158 */
    if (adaptive_total != total)
        return fail(ORC_INVALID_ARGUMENT, "safeguard_blend: total mismatch");
    if (!(alpha >= 0.0 && alpha <= 1.0))
        return fail(ORC_INVALID_ARGUMENT, "safeguard_blend: alpha outside [0,1]");
    const double share = (double)total / (double)h;
    double* quotas = (double*)malloc((size_t)(h > 0 ? h : 1) * sizeof(double));
    for (int64_t i = 0; i < h; ++i)
        quotas[i] = alpha * (double)(uint64_t)adaptive[i] + (1.0 - alpha) * share;
    int st = orc_apportion(quotas, h, total, caps, out);
    free(quotas);
    return st;
}

int orc_pyramid_layer_budgets(int64_t per_layer_avg, int64_t num_layers, double beta_max,
                              double beta_min, int64_t* out) {
    /* budget.hpp:169-191 */
    if (num_layers == 0) return fail(ORC_INVALID_ARGUMENT, "pyramid_layer_budgets: zero layers");
    if (!(beta_min > 0.0) || beta_max < beta_min)
        return fail(ORC_INVALID_ARGUMENT, "pyramid_layer_budgets: invalid betas");
    if (num_layers == 1) {
        out[0] = per_layer_avg;
        return ORC_OK;
    }
    double* quotas = (double*)malloc((size_t)num_layers * sizeof(double));
    const double avg = (double)per_layer_avg;
    double quota_sum = 0.0;
    for (int64_t l = 0; l < num_layers; ++l) {
        const double t = (double)l / (double)(num_layers - 1);
        quotas[l] = avg * (beta_max - (beta_max - beta_min) * t);
        quota_sum += quotas[l];
    }
    const int64_t total = per_layer_avg * num_layers;
    if (quota_sum > 0.0) {
        const double sc = (double)total / quota_sum;
        for (int64_t l = 0; l < num_layers; ++l) quotas[l] *= sc;
    }
    int st = orc_apportion(quotas, num_layers, total, NULL, out);
    free(quotas);
    return st;
}

int orc_repair_zero_budgets(int64_t* counts, const int64_t* caps, int64_t h) {
    /* policies.hpp:178-196 */
    for (int64_t gi = 0; gi < h; ++gi) {
        while (counts[gi] == 0) {
            int64_t donor = h;
            int64_t best = 1;
            for (int64_t k = 0; k < h; ++k)
                if (counts[k] > best) {
                    best = counts[k];
                    donor = k;
                }
            if (donor == h || caps[gi] == 0)
                return fail(ORC_INVALID_ARGUMENT,
                            "evict_layer: cannot guarantee one element per head");
            --counts[donor];
            ++counts[gi];
        }
    }
    return ORC_OK;
}

int orc_streaming_llm_decision(int64_t n, int64_t sink, int64_t recent, uint8_t* keep) {
    /* policies.hpp:159-165 */
    memset(keep, 0, (size_t)n);
    for (int64_t j = 0; j < (sink < n ? sink : n); ++j) keep[j] = 1;
    for (int64_t j = n > recent ? n - recent : 0; j < n; ++j) keep[j] = 1;
    return ORC_OK;
}

int orc_evict_rows(const double* w, const int64_t* off, int64_t h, int64_t total_budget,
                   int adaptive, double alpha, int64_t* alloc, uint8_t* keep) {
    /* policies.hpp:298-323 */
    if (h == 0) return fail(ORC_INVALID_ARGUMENT, "evict_rows: no heads");
    int64_t* caps = (int64_t*)malloc((size_t)h * sizeof(int64_t));
    int st = ORC_OK;
    for (int64_t i = 0; i < h; ++i) {
        caps[i] = off[i + 1] - off[i];
        if (caps[i] == 0) {
            st = fail(ORC_INVALID_ARGUMENT, "evict_rows: empty head");
            goto done;
        }
    }
    if (total_budget < h) {
        st = fail(ORC_INVALID_ARGUMENT, "evict_rows: budget below one per head");
        goto done;
    }
    if (adaptive) {
        int64_t* raw = (int64_t*)malloc((size_t)h * sizeof(int64_t));
        st = orc_adaptive_allocation(w, off, h, total_budget, raw);
        if (!st) st = orc_safeguard_blend(raw, total_budget, total_budget, h, alpha, caps, alloc);
        free(raw);
    } else {
        st = orc_uniform_allocation(total_budget, h, caps, alloc);
    }
    if (st) goto done;
    st = orc_repair_zero_budgets(alloc, caps, h);
    if (st) goto done;
    for (int64_t i = 0; i < h; ++i) {
        st = orc_topk_decision(w + off[i], caps[i], alloc[i], keep + (off[i] - off[0]));
        if (st) goto done;
    }
done:
    free(caps);
    return st;
}

static int all_finite(const double* x, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        if (!isfinite(x[i])) return 0;
    return 1;
}

int orc_evict_layer(const double* q, const double* k_out, const double* v_out,
                    const int64_t* off, const double* k_win, const double* v_win, int64_t H,
                    int64_t G, int64_t m, int64_t d, int64_t layer_budget,
                    const orc_policy_config* cfg, double* head_scores, double* group_scores,
                    int64_t* alloc, uint8_t* keep, double* k_ret, double* v_ret,
                    int64_t* ret_len) {
    /* policies.hpp:204-293 */
    /* config.validate(): policies.hpp:65-72 */
    if (cfg->window_size < 1) return fail(ORC_INVALID_ARGUMENT, "PolicyConfig: window_size < 1");
    if (cfg->pool_kernel % 2 == 0 || cfg->pool_kernel == 0)
        return fail(ORC_INVALID_ARGUMENT, "PolicyConfig: pool_kernel must be odd");
    if (!(cfg->alpha >= 0.0 && cfg->alpha <= 1.0))
        return fail(ORC_INVALID_ARGUMENT, "PolicyConfig: alpha outside [0,1]");
    if (cfg->gqa_group_size == 0) return fail(ORC_INVALID_ARGUMENT, "PolicyConfig: zero group size");
    /* cache.validate(): attention.hpp:76-83 */
    const int64_t n_all = off[G] - off[0];
    if (!all_finite(k_out, n_all * d) || !all_finite(v_out, n_all * d) ||
        !all_finite(k_win, G * m * d) || !all_finite(v_win, G * m * d))
        return fail(ORC_INVALID_ARGUMENT, "LayerCache: non-finite entry");
    const int64_t g = cfg->gqa_group_size;
    if (H % g != 0) return fail(ORC_INVALID_ARGUMENT, "evict_layer: head count not divisible by group");
    if (H / g != G) return fail(ORC_INVALID_ARGUMENT, "evict_layer: head count mismatch");
    if (m == 0) return fail(ORC_INVALID_ARGUMENT, "evict_layer: empty window");
    /* policies.hpp:229-231 */
    if (layer_budget < m * G + G)
        return fail(ORC_INVALID_ARGUMENT, "evict_layer: budget below the window-plus-one floor");
    const int64_t outside_budget = layer_budget - m * G;
    int64_t* caps = (int64_t*)malloc((size_t)G * sizeof(int64_t));
    double* per_head = NULL;
    int st = ORC_OK;
    for (int64_t gi = 0; gi < G; ++gi) {
        caps[gi] = off[gi + 1] - off[gi];
        if (caps[gi] == 0) {
            st = fail(ORC_INVALID_ARGUMENT, "evict_layer: empty outside cache head");
            goto done;
        }
    }
    /* policies.hpp:241-247: per-head scores with the group leader's keys, then group mean */
    {
        int64_t nmax = 0;
        for (int64_t gi = 0; gi < G; ++gi) nmax = caps[gi] > nmax ? caps[gi] : nmax;
        per_head = (double*)malloc((size_t)(g * nmax) * sizeof(double));
        for (int64_t gi = 0; gi < G; ++gi) {
            const int64_t n = caps[gi];
            for (int64_t k = 0; k < g; ++k) {
                const int64_t i = gi * g + k;
                st = orc_window_scores(q + i * m * d, m, k_out + (off[gi] - off[0]) * d, n, d,
                                       cfg->pool_kernel, cfg->scale, per_head + k * n);
                if (st) goto done;
            }
            if (head_scores) {
                /* head i's scores land at head_scores[(off[gi]-off[0])*g + k*n ...] */
                memcpy(head_scores + (off[gi] - off[0]) * g, per_head,
                       (size_t)(g * n) * sizeof(double));
            }
            /* group_mean_scores, policies.hpp:143-154 */
            double* acc = group_scores + (off[gi] - off[0]);
            for (int64_t j = 0; j < n; ++j) acc[j] = 0.0;
            for (int64_t k = 0; k < g; ++k)
                for (int64_t j = 0; j < n; ++j) acc[j] += per_head[k * n + j];
            for (int64_t j = 0; j < n; ++j) acc[j] /= (double)g;
        }
    }
    /* policies.hpp:249-257 */
    if (cfg->kind == ORC_ADA_SNAPKV || cfg->kind == ORC_ADA_PYRAMID) {
        int64_t* raw = (int64_t*)malloc((size_t)G * sizeof(int64_t));
        int64_t* soff = (int64_t*)malloc((size_t)(G + 1) * sizeof(int64_t));
        for (int64_t gi = 0; gi <= G; ++gi) soff[gi] = off[gi] - off[0];
        st = orc_adaptive_allocation(group_scores, soff, G, outside_budget, raw);
        if (!st) st = orc_safeguard_blend(raw, outside_budget, outside_budget, G, cfg->alpha, caps, alloc);
        free(raw);
        free(soff);
    } else {
        st = orc_uniform_allocation(outside_budget, G, caps, alloc);
    }
    if (st) goto done;
    st = orc_repair_zero_budgets(alloc, caps, G);
    if (st) goto done;
    /* policies.hpp:259-271 */
    for (int64_t gi = 0; gi < G; ++gi) {
        uint8_t* kp = keep + (off[gi] - off[0]);
        if (cfg->kind == ORC_STREAMING_LLM) {
            const int64_t b = alloc[gi];
            const int64_t sink = cfg->sink_tokens < b ? cfg->sink_tokens : b;
            orc_streaming_llm_decision(caps[gi], sink, b - sink, kp);
        } else {
            st = orc_topk_decision(group_scores + (off[gi] - off[0]), caps[gi], alloc[gi], kp);
            if (st) goto done;
        }
    }
    /* policies.hpp:273-290: kept outside rows in order, then the window rows */
    {
        int64_t row = 0;
        for (int64_t gi = 0; gi < G; ++gi) {
            const int64_t base = off[gi] - off[0];
            int64_t len = 0;
            for (int64_t j = 0; j < caps[gi]; ++j) {
                if (!keep[base + j]) continue;
                memcpy(k_ret + (row + len) * d, k_out + (base + j) * d, (size_t)d * sizeof(double));
                memcpy(v_ret + (row + len) * d, v_out + (base + j) * d, (size_t)d * sizeof(double));
                ++len;
            }
            memcpy(k_ret + (row + len) * d, k_win + gi * m * d, (size_t)(m * d) * sizeof(double));
            memcpy(v_ret + (row + len) * d, v_win + gi * m * d, (size_t)(m * d) * sizeof(double));
            len += m;
            ret_len[gi] = len;
            row += len;
        }
    }
done:
    free(caps);
    free(per_head);
    return st;
}

int orc_decode_attention(const double* q, const double* k, const double* v, const int64_t* off,
                         int64_t H, int64_t G, int64_t d, int scale, double* out) {
    /* report.hpp:133-144: attention_weights over the retained keys, then
     * row_times(a, V) (attention.hpp:191; matrix.hpp:79-89). */
    if (G == 0 || H % G != 0) return fail(ORC_INVALID_ARGUMENT, "attention_output: head count mismatch");
    const int64_t g = H / G;
    int64_t nmax = 1;
    for (int64_t gi = 0; gi < G; ++gi)
        if (off[gi + 1] - off[gi] > nmax) nmax = off[gi + 1] - off[gi];
    double* a = (double*)malloc((size_t)nmax * sizeof(double));
    int st = ORC_OK;
    for (int64_t i = 0; i < H; ++i) {
        const int64_t gi = i / g;
        const int64_t n = off[gi + 1] - off[gi];
        const double* kk = k + (off[gi] - off[0]) * d;
        const double* vv = v + (off[gi] - off[0]) * d;
        st = orc_attention_weights(q + i * d, 1, kk, n, d, scale, a);
        if (st) break;
        double* o = out + i * d;
        for (int64_t c = 0; c < d; ++c) o[c] = 0.0;
        for (int64_t r = 0; r < n; ++r) {
            const double xr = a[r];
            if (xr == 0.0) continue;
            for (int64_t c = 0; c < d; ++c) o[c] += xr * vv[r * d + c];
        }
    }
    free(a);
    return st;
}

int orc_flatten(const double* k, const double* v, const int64_t* len, int64_t h, int64_t d,
                double* data, int64_t* offsets) {
    /* flat_cache.hpp:44-66: per head [K rows][V rows], offsets in rows */
    int64_t offset = 0, src = 0;
    double* o = data;
    for (int64_t i = 0; i < h; ++i) {
        offsets[i] = offset;
        offset += len[i];
    }
    for (int64_t i = 0; i < h; ++i) {
        memcpy(o, k + src * d, (size_t)(len[i] * d) * sizeof(double));
        o += len[i] * d;
        memcpy(o, v + src * d, (size_t)(len[i] * d) * sizeof(double));
        o += len[i] * d;
        src += len[i];
    }
    return ORC_OK;
}

int orc_select_and_compact(const double* data, const int64_t* offsets, const int64_t* lengths,
                           int64_t h, int64_t d, const uint8_t* keep, double* out_data,
                           int64_t* out_offsets, int64_t* out_lengths) {
    /* flat_cache.hpp:92-120 */
    int64_t offset = 0, kbase = 0;
    for (int64_t i = 0; i < h; ++i) {
        out_offsets[i] = offset;
        int64_t kept = 0;
        for (int64_t r = 0; r < lengths[i]; ++r) kept += keep[kbase + r] ? 1 : 0;
        out_lengths[i] = kept;
        offset += kept;
        kbase += lengths[i];
    }
    double* o = out_data;
    kbase = 0;
    for (int64_t i = 0; i < h; ++i) {
        const int64_t base = offsets[i] * 2 * d;
        const int64_t n = lengths[i];
        for (int pass = 0; pass < 2; ++pass)
            for (int64_t r = 0; r < n; ++r) {
                if (!keep[kbase + r]) continue;
                memcpy(o, data + base + (pass * n + r) * d, (size_t)d * sizeof(double));
                o += d;
            }
        kbase += n;
    }
    return ORC_OK;
}

int orc_append_kv(double* k_cache, double* v_cache, const int64_t* seg_start, int64_t* len,
                  const int64_t* cap, int64_t n_seg, int64_t seg, const double* k,
                  const double* v, int64_t d) {
    /* attention.hpp:126-134 */
    if (seg < 0 || seg >= n_seg) return fail(ORC_OUT_OF_RANGE, "append_kv: head index out of range");
    if (cap && len[seg] >= cap[seg]) return fail(ORC_INVALID_ARGUMENT, "append_kv: capacity exhausted");
    const int64_t row = seg_start[seg] + len[seg];
    memcpy(k_cache + row * d, k, (size_t)d * sizeof(double));
    memcpy(v_cache + row * d, v, (size_t)d * sizeof(double));
    ++len[seg];
    return ORC_OK;
}
