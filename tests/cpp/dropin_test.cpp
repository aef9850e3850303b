// dropin_test.cpp -- the reference-signature C++ API (include/adakv_b200/adakv.hpp) on the GPU.
//
// Known answers transcribed from the reference's gtest suites (file:line cited), then seeded
// random evict_layer / evict_rows / window_scores instances compared against the C oracle
// (oracle/adakv_oracle.c, linked as test infrastructure).  Exit code = number of failures.
#include <cmath>
#include <cstdio>
#include <random>
#include <sstream>
#include <vector>

#include "adakv_b200/adakv.hpp"

extern "C" {
#include "adakv_oracle.h"
}

namespace adakv = adakv_b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                          \
    do {                                                                     \
        ++g_checks;                                                          \
        if (!(cond)) {                                                       \
            ++g_fail;                                                        \
            std::fprintf(stderr, "FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond); \
        }                                                                    \
    } while (0)
#define CHECK_THROWS(expr, Ex)                 \
    do {                                       \
        bool thrown = false;                   \
        try {                                  \
            (void)(expr);                      \
        } catch (const Ex&) {                  \
            thrown = true;                     \
        }                                      \
        CHECK(thrown && #Ex);                  \
    } while (0)

using V = std::vector<std::size_t>;
using U8 = std::vector<std::uint8_t>;

static void kats() {
    // policies_test.cpp:56-73
    CHECK(adakv::topk_decision(std::vector<double>{0.5, 0.3, 0.2}, 2) == (U8{1, 1, 0}));
    CHECK(adakv::topk_decision(std::vector<double>{0.25, 0.25, 0.25, 0.25}, 2) == (U8{1, 1, 0, 0}));
    CHECK(adakv::topk_decision(std::vector<double>{0.1, 0.9}, 2) == (U8{1, 1}));
    CHECK_THROWS(adakv::topk_decision(std::vector<double>{1.0}, 2), std::invalid_argument);
    // policies_test.cpp:162-173
    CHECK(adakv::streaming_llm_decision(10, 4, 3) == (U8{1, 1, 1, 1, 0, 0, 0, 1, 1, 1}));
    CHECK(adakv::streaming_llm_decision(5, 4, 3) == (U8{1, 1, 1, 1, 1}));
    CHECK(adakv::streaming_llm_decision(4, 0, 0) == (U8{0, 0, 0, 0}));
    // budget_test.cpp:19-54
    CHECK(adakv::detail::apportion({1.2, 0.9, 0.9}, 3, V{10, 10, 10}) == (V{1, 1, 1}));
    CHECK(adakv::detail::apportion({3.5, 3.5, 3.0}, 8, V{10, 10, 10}) == (V{3, 3, 2}));
    CHECK(adakv::detail::apportion({5.0, 0.2}, 4, V{10, 10}) == (V{4, 0}));
    CHECK(adakv::uniform_allocation(10, 3).per_head == (V{4, 3, 3}));
    CHECK(adakv::uniform_allocation(4, 2, V{1, 10}).per_head == (V{1, 3}));
    CHECK_THROWS(adakv::uniform_allocation(3, 2, V{1, 1}), std::invalid_argument);
    // budget_test.cpp:79-108 (tie rule -> {3,0})
    const adakv::WeightRows two{{0.4, 0.3, 0.3}, {0.98, 0.01, 0.01}};
    CHECK(adakv::adaptive_allocation(two, 4).per_head == (V{3, 1}));
    CHECK(adakv::adaptive_allocation(two, 6).per_head == (V{3, 3}));
    CHECK(adakv::adaptive_allocation(two, 0).per_head == (V{0, 0}));
    CHECK(adakv::adaptive_allocation({{0.25, 0.25, 0.25, 0.25}, {0.25, 0.25, 0.25, 0.25}}, 3).per_head == (V{3, 0}));
    CHECK_THROWS(adakv::adaptive_allocation({{0.5, 0.5}}, 3), std::invalid_argument);
    // budget_test.cpp:157-185
    CHECK(adakv::safeguard_blend({{9, 1}, 10}, 10, 2, 0.2).per_head == (V{6, 4}));
    CHECK(adakv::safeguard_blend({{9, 1}, 10}, 10, 2, 1.0).per_head == (V{9, 1}));
    CHECK_THROWS(adakv::safeguard_blend({{5, 5}, 10}, 10, 2, 1.5), std::invalid_argument);
    CHECK_THROWS(adakv::safeguard_blend({{5, 5}, 10}, 10, 2, 0.5, V{4, 4}), std::invalid_argument);
    // budget_test.cpp:228-250
    CHECK(adakv::pyramid_layer_budgets(100, 3, 1.5, 0.5) == (V{150, 100, 50}));
    CHECK_THROWS(adakv::pyramid_layer_budgets(100, 0, 1.5, 0.5), std::invalid_argument);
    // policies_test.cpp:117-124: k=3 spreads the 0.7 peak
    const auto ws = adakv::window_scores(adakv::Matrix::from_rows({{1.0}}),
                                         adakv::Matrix::from_rows({{std::log(0.1)}, {std::log(0.7)}, {std::log(0.2)}}), 3);
    for (double s : ws) CHECK(std::fabs(s - 0.7) < 1e-12);
    // policies_test.cpp:141-147
    const auto gm = adakv::group_mean_scores({{0.2, 0.8}, {0.4, 0.6}}, 2);
    CHECK(gm.size() == 1 && std::fabs(gm[0][0] - 0.3) < 1e-15 && std::fabs(gm[0][1] - 0.7) < 1e-15);
    // attention_test.cpp:100-108 hand softmax
    adakv::Matrix q(1, 2);
    q(0, 0) = 1.0;
    const auto w = adakv::attention_weights(q, adakv::Matrix::from_rows({{1.0, 0.0}, {0.0, 1.0}}), false);
    const double e = std::exp(1.0);
    CHECK(std::fabs(w(0, 0) - e / (e + 1)) < 1e-12 && std::fabs(w(0, 1) - 1 / (e + 1)) < 1e-12);
    // attention_test.cpp:163-169 hand average
    adakv::LayerParams p1{{{adakv::Matrix::identity(2), adakv::Matrix::identity(2), adakv::Matrix::identity(2),
                            adakv::Matrix::identity(2)}}};
    adakv::LayerCache c1;
    c1.heads.push_back({adakv::Matrix::from_rows({{0.0, 0.0}, {0.0, 0.0}}), adakv::Matrix::from_rows({{2.0, 0.0}, {0.0, 2.0}})});
    CHECK(adakv::attention_output({{0.5, 0.5}}, c1, p1) == (std::vector<double>{1.0, 1.0}));
    // flat_cache_test.cpp:103-110, 182-198
    adakv::LayerCache fc1;
    fc1.heads.push_back({adakv::Matrix::from_rows({{1.0, 2.0}, {3.0, 4.0}, {5.0, 6.0}}),
                         adakv::Matrix::from_rows({{7.0, 8.0}, {9.0, 10.0}, {11.0, 12.0}})});
    const auto comp = adakv::select_and_compact(adakv::flatten(fc1), {{{1, 0, 1}}});
    CHECK(comp.lengths == (V{2}));
    CHECK(comp.data == (std::vector<double>{1.0, 2.0, 5.0, 6.0, 7.0, 8.0, 11.0, 12.0}));
    adakv::LayerCache g1;
    g1.heads.push_back({adakv::Matrix::from_rows({{1.5}}), adakv::Matrix::from_rows({{-2.0}})});
    std::stringstream ss;
    adakv::save_flattened(adakv::flatten(g1), ss);
    const std::string bytes = ss.str();
    CHECK(bytes.size() == 40u && bytes.substr(0, 4) == "AKVC" && (unsigned char)bytes[24 + 7] == 0x3F);
    std::stringstream in(bytes.substr(0, 10));
    CHECK_THROWS(adakv::load_flattened(in), adakv::FormatError);
    // policies_test.cpp:185-195: ScriptedLayer, Algorithm 1
    adakv::LayerParams sp;
    adakv::LayerCache so, sw;
    for (const auto& row : {std::vector<double>{0.4, 0.3, 0.3}, std::vector<double>{0.98, 0.01, 0.01}}) {
        const auto one = adakv::Matrix::from_rows({{1.0}});
        sp.heads.push_back({one, one, one, one});
        adakv::Matrix k(3, 1), v(3, 1);
        for (int j = 0; j < 3; ++j) {
            k(j, 0) = std::log(row[j]);
            v(j, 0) = j + 1;
        }
        so.heads.push_back({k, v});
        sw.heads.push_back({adakv::Matrix::from_rows({{0.0}}), adakv::Matrix::from_rows({{-1.0}})});
    }
    adakv::PolicyConfig cfg;
    cfg.window_size = 1;
    cfg.pool_kernel = 1;
    cfg.alpha = 1.0;
    const auto res = adakv::evict_layer(so, sw, adakv::Matrix::from_rows({{1.0}}), sp, 6, cfg);
    CHECK(res.allocation.per_head == (V{3, 1}));
    CHECK(res.decision.retain[1] == (U8{1, 0, 0}));
    CHECK(res.retained.heads[1].length() == 2 && res.retained.heads[1].values(1, 0) == -1.0);
    CHECK_THROWS(adakv::evict_layer(so, sw, adakv::Matrix::from_rows({{1.0}}), sp, 3, cfg), std::invalid_argument);
    cfg.kind = adakv::PolicyKind::snapkv;
    CHECK(adakv::evict_layer(so, sw, adakv::Matrix::from_rows({{1.0}}), sp, 6, cfg).allocation.per_head == (V{2, 2}));
}

// Random instances vs the C oracle (same marshalling as oracle/oracle.py).
static void random_parity() {
    std::mt19937_64 gen(2024);
    std::normal_distribution<double> nd;
    std::uniform_int_distribution<int> ui(0, 1 << 20);
    for (int trial = 0; trial < 20; ++trial) {
        const std::size_t G = 1 + ui(gen) % 3, g = 1 + ui(gen) % 4, H = G * g, m = 1 + ui(gen) % 4;
        const std::size_t n = 8 + ui(gen) % 40, d = 1 + ui(gen) % 8, D = H * d;
        const std::size_t LB = m * G + G + ui(gen) % (G * (n - 1) + 1);
        adakv::LayerParams params;
        adakv::LayerCache out, win;
        adakv::Matrix x(m, D);
        for (double& v : x.values()) v = nd(gen);
        std::vector<double> q(H * m * d), ko(G * n * d), vo(G * n * d), kw(G * m * d), vw(G * m * d);
        for (auto* vec : {&ko, &vo, &kw, &vw})
            for (double& v : *vec) v = nd(gen);
        for (std::size_t i = 0; i < H; ++i) {
            adakv::Matrix wq(D, d);
            for (std::size_t c = 0; c < d; ++c) wq(i * d + c, c) = 1.0;  // block selector: Q_i = X[:, i]
            params.heads.push_back({wq, adakv::Matrix(D, d), adakv::Matrix(D, d), adakv::Matrix(d, D)});
            for (std::size_t r = 0; r < m; ++r)
                for (std::size_t c = 0; c < d; ++c) q[(i * m + r) * d + c] = x(r, i * d + c);
            const std::size_t gi = i / g;
            adakv::Matrix K(n, d), Vv(n, d), KW(m, d), VW(m, d);
            std::copy(ko.begin() + gi * n * d, ko.begin() + (gi + 1) * n * d, K.values().begin());
            std::copy(vo.begin() + gi * n * d, vo.begin() + (gi + 1) * n * d, Vv.values().begin());
            std::copy(kw.begin() + gi * m * d, kw.begin() + (gi + 1) * m * d, KW.values().begin());
            std::copy(vw.begin() + gi * m * d, vw.begin() + (gi + 1) * m * d, VW.values().begin());
            out.heads.push_back({K, Vv});
            win.heads.push_back({KW, VW});
        }
        for (int kind = 0; kind < 5; ++kind) {
            adakv::PolicyConfig cfg;
            cfg.kind = static_cast<adakv::PolicyKind>(kind);
            cfg.window_size = m;
            cfg.pool_kernel = 1 + 2 * (ui(gen) % 4);
            cfg.alpha = (ui(gen) % 1000) / 1000.0;
            cfg.gqa_group_size = g;
            const auto r = adakv::evict_layer(out, win, x, params, LB, cfg);
            // oracle
            std::vector<int64_t> off(G + 1);
            for (std::size_t i = 0; i <= G; ++i) off[i] = int64_t(i * n);
            orc_policy_config oc{kind, int64_t(m), int64_t(cfg.pool_kernel), cfg.alpha, 4, int64_t(g), 1};
            std::vector<double> gs(G * n), hs(G * n * g), kr(LB * d), vr(LB * d);
            std::vector<int64_t> alloc(G), rl(G);
            std::vector<std::uint8_t> keep(G * n);
            const int st = orc_evict_layer(q.data(), ko.data(), vo.data(), off.data(), kw.data(), vw.data(), int64_t(H),
                                           int64_t(G), int64_t(m), int64_t(d), int64_t(LB), &oc, hs.data(), gs.data(),
                                           alloc.data(), keep.data(), kr.data(), vr.data(), rl.data());
            CHECK(st == 0);
            std::size_t row = 0;
            for (std::size_t gi = 0; gi < G; ++gi) {
                CHECK(r.allocation.per_head[gi] == std::size_t(alloc[gi]));
                double mx = 0;
                for (std::size_t j = 0; j < n; ++j) mx = std::max(mx, std::fabs(gs[gi * n + j]));
                for (std::size_t j = 0; j < n; ++j) CHECK(std::fabs(r.scores[gi][j] - gs[gi * n + j]) <= 1e-12 * mx);
                CHECK(r.decision.retain[gi * g] == U8(keep.begin() + gi * n, keep.begin() + (gi + 1) * n));
                const auto& hk = r.retained.heads[gi * g];
                CHECK(hk.length() == std::size_t(rl[gi]));
                for (std::size_t rr = 0; rr < hk.length(); ++rr)
                    for (std::size_t c = 0; c < d; ++c) CHECK(hk.keys(rr, c) == kr[(row + rr) * d + c]);
                row += hk.length();
            }
        }
    }
}

// evict_rows on ragged rows with ties, both modes, vs orc_evict_rows.
static void random_rows() {
    std::mt19937_64 gen(77);
    std::uniform_int_distribution<int> ui(0, 1 << 20);
    for (int trial = 0; trial < 40; ++trial) {
        const std::size_t h = 1 + ui(gen) % 6;
        adakv::WeightRows rows(h);
        std::vector<double> flat;
        std::vector<int64_t> off{0};
        for (auto& r : rows) {
            const std::size_t n = 1 + ui(gen) % 50;
            for (std::size_t j = 0; j < n; ++j) r.push_back((ui(gen) % 8) / 8.0);  // heavy ties
            flat.insert(flat.end(), r.begin(), r.end());
            off.push_back(int64_t(flat.size()));
        }
        const std::size_t total = h + ui(gen) % (flat.size() - h + 1);
        const bool adaptive = trial % 2 == 0;
        const double alpha = (ui(gen) % 11) / 10.0;
        const auto [dec, alloc] = adakv::evict_rows(rows, total, adaptive, alpha);
        std::vector<int64_t> oa(h);
        std::vector<std::uint8_t> ok(flat.size());
        CHECK(orc_evict_rows(flat.data(), off.data(), int64_t(h), int64_t(total), adaptive, alpha, oa.data(),
                             ok.data()) == 0);
        for (std::size_t i = 0; i < h; ++i) {
            CHECK(alloc.per_head[i] == std::size_t(oa[i]));
            CHECK(dec.retain[i] == U8(ok.begin() + off[i], ok.begin() + off[i + 1]));
        }
    }
}

int main() {
    try {
        kats();
        random_parity();
        random_rows();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "exception: %s\n", e.what());
        return 100;
    }
    std::printf("dropin_test: %d checks, %d failures\n", g_checks, g_fail);
    return g_fail;
}
