// ref_driver.cpp -- extern "C" shim over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile with
//   -I/root/reference/proj/include -O3 -DNDEBUG -ffp-contract=off
// (the reference's Release flags, CMakeLists.txt:5-7, plus no FMA contraction)
// into oracle/_ref/libadakv_ref.so.  It is used to (1) pin the C restatement in
// oracle/adakv_oracle.c bit-for-bit and (2) time the reference CPU path for
// bench.py's cpu_baseline / --impl reference legs.  Nothing from the reference
// is copied here: this file only marshals flat arrays into the reference's own
// types and calls its own functions.
//
// Marshalling conventions follow oracle/adakv_oracle.h (per-group K/V, queries
// [H, m, d]).  The reference stores one cache copy per query head
// (policies.hpp:276), so the shim expands each group to its g members and feeds
// the precomputed Q through block-selector W_q projections (trace.hpp:199-204
// pattern), which reproduces Q exactly.

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "adakv/attention.hpp"
#include "adakv/budget.hpp"
#include "adakv/flat_cache.hpp"
#include "adakv/matrix.hpp"
#include "adakv/policies.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 2;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

adakv::Matrix to_matrix(const double* p, std::size_t rows, std::size_t cols) {
    adakv::Matrix m(rows, cols);
    if (rows != 0 && cols != 0) std::memcpy(m.values().data(), p, rows * cols * sizeof(double));
    return m;
}

std::vector<std::size_t> to_sizes(const int64_t* p, std::size_t n) {
    std::vector<std::size_t> v(n);
    for (std::size_t i = 0; i < n; ++i) v[i] = static_cast<std::size_t>(p[i]);
    return v;
}

adakv::WeightRows to_rows(const double* a, const int64_t* off, int64_t h) {
    adakv::WeightRows rows(static_cast<std::size_t>(h));
    for (int64_t i = 0; i < h; ++i) rows[i].assign(a + off[i], a + off[i + 1]);
    return rows;
}

adakv::Matrix block_selector(std::size_t d, std::size_t d_h, std::size_t block) {
    adakv::Matrix m(d, d_h);
    for (std::size_t c = 0; c < d_h; ++c) m(block * d_h + c, c) = 1.0;
    return m;
}

struct RefLayer {
    adakv::LayerCache outside, window;
    adakv::Matrix x;  // window embeddings = concat of per-head queries
    adakv::LayerParams params;
};

RefLayer build_layer(const double* q, const double* k_out, const double* v_out,
                     const int64_t* off, const double* k_win, const double* v_win, int64_t H,
                     int64_t G, int64_t m, int64_t d) {
    RefLayer L;
    const std::size_t g = static_cast<std::size_t>(H / G);
    const std::size_t embed = static_cast<std::size_t>(H * d);
    L.x = adakv::Matrix(m, embed);
    for (int64_t i = 0; i < H; ++i)
        for (int64_t r = 0; r < m; ++r)
            for (int64_t c = 0; c < d; ++c) L.x(r, i * d + c) = q[(i * m + r) * d + c];
    L.params.heads.resize(H);
    for (int64_t i = 0; i < H; ++i) {
        auto& hp = L.params.heads[i];
        hp.wq = block_selector(embed, d, i);
        hp.wk = adakv::Matrix(embed, d);
        hp.wv = adakv::Matrix(embed, d);
        hp.wo = adakv::Matrix(d, embed);
    }
    L.outside.heads.resize(H);
    L.window.heads.resize(H);
    for (int64_t i = 0; i < H; ++i) {
        const int64_t gi = i / static_cast<int64_t>(g);
        const int64_t n = off[gi + 1] - off[gi];
        L.outside.heads[i] = {to_matrix(k_out + (off[gi] - off[0]) * d, n, d),
                              to_matrix(v_out + (off[gi] - off[0]) * d, n, d)};
        L.window.heads[i] = {to_matrix(k_win + gi * m * d, m, d), to_matrix(v_win + gi * m * d, m, d)};
    }
    return L;
}

adakv::PolicyConfig to_config(int kind, int64_t window, int64_t pool, double alpha, int64_t sink,
                              int64_t group, int scale) {
    adakv::PolicyConfig c;
    c.kind = static_cast<adakv::PolicyKind>(kind);
    c.window_size = static_cast<std::size_t>(window);
    c.pool_kernel = static_cast<std::size_t>(pool);
    c.alpha = alpha;
    c.sink_tokens = static_cast<std::size_t>(sink);
    c.gqa_group_size = static_cast<std::size_t>(group);
    c.scale = scale != 0;
    return c;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_topk_decision(const double* a, int64_t n, int64_t k, uint8_t* keep) {
    return guard([&] {
        const auto v = adakv::topk_decision(std::span<const double>(a, n), k);
        std::memcpy(keep, v.data(), v.size());
    });
}

int ref_window_scores(const double* q, int64_t m, const double* keys, int64_t n, int64_t d,
                      int64_t pool, int scale, double* out) {
    return guard([&] {
        const auto s = adakv::window_scores(to_matrix(q, m, d), to_matrix(keys, n, d), pool, scale);
        std::memcpy(out, s.data(), s.size() * sizeof(double));
    });
}

int ref_attention_weights(const double* q, int64_t m, const double* keys, int64_t n, int64_t d,
                          int scale, double* out) {
    return guard([&] {
        const auto a = adakv::attention_weights(to_matrix(q, m, d), to_matrix(keys, n, d), scale);
        std::memcpy(out, a.values().data(), a.values().size() * sizeof(double));
    });
}

int ref_group_mean_scores(const double* s, int64_t h, int64_t n, int64_t g, double* out) {
    return guard([&] {
        adakv::ObservationScores in(h);
        for (int64_t i = 0; i < h; ++i) in[i].assign(s + i * n, s + (i + 1) * n);
        const auto r = adakv::group_mean_scores(in, g);
        for (std::size_t gi = 0; gi < r.size(); ++gi)
            std::memcpy(out + gi * n, r[gi].data(), n * sizeof(double));
    });
}

int ref_apportion(const double* quotas, int64_t h, int64_t total, const int64_t* caps, int64_t* out) {
    return guard([&] {
        const std::vector<double> qv(quotas, quotas + h);
        const auto cv = caps ? to_sizes(caps, h) : adakv::detail::ample_caps(h);
        const auto r = adakv::detail::apportion(qv, total, cv);
        for (int64_t i = 0; i < h; ++i) out[i] = static_cast<int64_t>(r[i]);
    });
}

int ref_uniform_allocation(int64_t total, int64_t h, const int64_t* caps, int64_t* out) {
    return guard([&] {
        const auto r = caps ? adakv::uniform_allocation(total, h, to_sizes(caps, h))
                            : adakv::uniform_allocation(total, h);
        for (int64_t i = 0; i < h; ++i) out[i] = static_cast<int64_t>(r.per_head[i]);
    });
}

int ref_adaptive_allocation(const double* a, const int64_t* off, int64_t h, int64_t total,
                            int64_t* out) {
    return guard([&] {
        const auto r = adakv::adaptive_allocation(to_rows(a, off, h), total);
        for (int64_t i = 0; i < h; ++i) out[i] = static_cast<int64_t>(r.per_head[i]);
    });
}

int ref_safeguard_blend(const int64_t* adaptive, int64_t adaptive_total, int64_t total, int64_t h,
                        double alpha, const int64_t* caps, int64_t* out) {
    return guard([&] {
        adakv::BudgetAllocation in{to_sizes(adaptive, h), static_cast<std::size_t>(adaptive_total)};
        const auto r = caps ? adakv::safeguard_blend(in, total, h, alpha, to_sizes(caps, h))
                            : adakv::safeguard_blend(in, total, h, alpha);
        for (int64_t i = 0; i < h; ++i) out[i] = static_cast<int64_t>(r.per_head[i]);
    });
}

int ref_pyramid_layer_budgets(int64_t avg, int64_t layers, double bmax, double bmin, int64_t* out) {
    return guard([&] {
        const auto r = adakv::pyramid_layer_budgets(avg, layers, bmax, bmin);
        for (std::size_t i = 0; i < r.size(); ++i) out[i] = static_cast<int64_t>(r[i]);
    });
}

int ref_repair_zero_budgets(int64_t* counts, const int64_t* caps, int64_t h) {
    return guard([&] {
        auto c = to_sizes(counts, h);
        const auto cp = to_sizes(caps, h);
        adakv::detail::repair_zero_budgets(c, cp);
        for (int64_t i = 0; i < h; ++i) counts[i] = static_cast<int64_t>(c[i]);
    });
}

int ref_streaming_llm_decision(int64_t n, int64_t sink, int64_t recent, uint8_t* keep) {
    return guard([&] {
        const auto v = adakv::streaming_llm_decision(n, sink, recent);
        std::memcpy(keep, v.data(), v.size());
    });
}

int ref_evict_rows(const double* w, const int64_t* off, int64_t h, int64_t total, int adaptive,
                   double alpha, int64_t* alloc, uint8_t* keep) {
    return guard([&] {
        const auto [dec, al] = adakv::evict_rows(to_rows(w, off, h), total, adaptive != 0, alpha);
        for (int64_t i = 0; i < h; ++i) {
            alloc[i] = static_cast<int64_t>(al.per_head[i]);
            std::memcpy(keep + (off[i] - off[0]), dec.retain[i].data(), dec.retain[i].size());
        }
    });
}

// Same contract as orc_evict_layer (oracle/adakv_oracle.h).  Additionally
// checks the reference's per-head outputs are identical within each group.
int ref_evict_layer(const double* q, const double* k_out, const double* v_out, const int64_t* off,
                    const double* k_win, const double* v_win, int64_t H, int64_t G, int64_t m,
                    int64_t d, int64_t layer_budget, int kind, int64_t window_size, int64_t pool,
                    double alpha, int64_t sink, int scale, double* group_scores, int64_t* alloc,
                    uint8_t* keep, double* k_ret, double* v_ret, int64_t* ret_len) {
    return guard([&] {
        const int64_t g = H / G;
        const RefLayer L = build_layer(q, k_out, v_out, off, k_win, v_win, H, G, m, d);
        const auto cfg = to_config(kind, window_size, pool, alpha, sink, g, scale);
        const auto res = adakv::evict_layer(L.outside, L.window, L.x, L.params, layer_budget, cfg);
        int64_t row = 0;
        for (int64_t gi = 0; gi < G; ++gi) {
            const int64_t n = off[gi + 1] - off[gi];
            std::memcpy(group_scores + (off[gi] - off[0]), res.scores[gi].data(), n * sizeof(double));
            alloc[gi] = static_cast<int64_t>(res.allocation.per_head[gi]);
            std::memcpy(keep + (off[gi] - off[0]), res.decision.retain[gi * g].data(), n);
            const auto& hk = res.retained.heads[gi * g];
            const int64_t len = static_cast<int64_t>(hk.length());
            ret_len[gi] = len;
            std::memcpy(k_ret + row * d, hk.keys.values().data(), len * d * sizeof(double));
            std::memcpy(v_ret + row * d, hk.values.values().data(), len * d * sizeof(double));
            row += len;
        }
    });
}

int ref_decode_attention(const double* q, const double* k, const double* v, const int64_t* off,
                         int64_t H, int64_t G, int64_t d, int scale, double* out) {
    // report.hpp:133-144 without the model-side W_o: attention_weights then row_times(a, V).
    return guard([&] {
        const int64_t g = H / G;
        for (int64_t i = 0; i < H; ++i) {
            const int64_t gi = i / g;
            const int64_t n = off[gi + 1] - off[gi];
            const auto keys = to_matrix(k + (off[gi] - off[0]) * d, n, d);
            const auto vals = to_matrix(v + (off[gi] - off[0]) * d, n, d);
            const auto a = adakv::attention_weights(to_matrix(q + i * d, 1, d), keys, scale);
            const auto ctx = adakv::row_times(a.row(0), vals);
            std::memcpy(out + i * d, ctx.data(), d * sizeof(double));
        }
    });
}

int ref_select_and_compact(const double* k, const double* v, const int64_t* len, int64_t h,
                           int64_t d, const uint8_t* keep, double* out_data, int64_t* out_offsets,
                           int64_t* out_lengths) {
    return guard([&] {
        adakv::LayerCache cache;
        int64_t src = 0;
        adakv::EvictionDecision dec;
        for (int64_t i = 0; i < h; ++i) {
            cache.heads.push_back({to_matrix(k + src * d, len[i], d), to_matrix(v + src * d, len[i], d)});
            dec.retain.emplace_back(keep + src, keep + src + len[i]);
            src += len[i];
        }
        const auto out = adakv::select_and_compact(adakv::flatten(cache), dec);
        std::memcpy(out_data, out.data.data(), out.data.size() * sizeof(double));
        for (int64_t i = 0; i < h; ++i) {
            out_offsets[i] = static_cast<int64_t>(out.offsets[i]);
            out_lengths[i] = static_cast<int64_t>(out.lengths[i]);
        }
    });
}

// ---------------------------------------------------------------------------
// CPU baseline timing.  Runs `units` independent evict_layer calls on one shared
// input layer across `threads` std::thread workers pulling from an atomic
// counter -- the reference's own worker model (report.hpp:297-311).  Returns the
// wall seconds of the whole batch (input construction excluded).
int ref_bench_evict_layer(const double* q, const double* k_out, const double* v_out,
                          const int64_t* off, const double* k_win, const double* v_win, int64_t H,
                          int64_t G, int64_t m, int64_t d, int64_t layer_budget, int kind,
                          int64_t pool, double alpha, int threads, int units, double* seconds,
                          int64_t* alloc_out) {
    return guard([&] {
        const RefLayer L = build_layer(q, k_out, v_out, off, k_win, v_win, H, G, m, d);
        const auto cfg = to_config(kind, m, pool, alpha, 4, H / G, 1);
        std::atomic<int> next{0};
        std::vector<std::vector<std::size_t>> allocs(units);
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool_threads;
        for (int t = 0; t < threads; ++t)
            pool_threads.emplace_back([&] {
                for (int u = next++; u < units; u = next++) {
                    const auto res = adakv::evict_layer(L.outside, L.window, L.x, L.params,
                                                        layer_budget, cfg);
                    allocs[u] = res.allocation.per_head;
                }
            });
        for (auto& th : pool_threads) th.join();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (int64_t gi = 0; gi < G; ++gi) alloc_out[gi] = static_cast<int64_t>(allocs[0][gi]);
    });
}

// Decode baseline: `units` single-token decode steps (attention_weights +
// row_times over every head's retained cache) spread over `threads` workers.
int ref_bench_decode(const double* q, const double* k, const double* v, const int64_t* off,
                     int64_t H, int64_t G, int64_t d, int threads, int units, double* seconds) {
    return guard([&] {
        const int64_t g = H / G;
        std::vector<adakv::Matrix> keys(G), vals(G);
        for (int64_t gi = 0; gi < G; ++gi) {
            const int64_t n = off[gi + 1] - off[gi];
            keys[gi] = to_matrix(k + (off[gi] - off[0]) * d, n, d);
            vals[gi] = to_matrix(v + (off[gi] - off[0]) * d, n, d);
        }
        std::atomic<int> next{0};
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> ts;
        for (int t = 0; t < threads; ++t)
            ts.emplace_back([&] {
                for (int u = next++; u < units; u = next++)
                    for (int64_t i = 0; i < H; ++i) {
                        const auto a = adakv::attention_weights(to_matrix(q + i * d, 1, d),
                                                                keys[i / g], true);
                        volatile double sink = adakv::row_times(a.row(0), vals[i / g])[0];
                        (void)sink;
                    }
            });
        for (auto& th : ts) th.join();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

}  // extern "C"
