// ref_fig3.cpp -- the reference's own policy comparison, for golden vectors.
//
// TEST INFRASTRUCTURE ONLY.  Built by `make -C oracle fig3` (needs /root/reference and
// nlohmann/json, which trace.hpp:15 includes) and run by tests/golden/make_golden.py.
//
//   ref_fig3 accept <out.txt>
//       acceptance check #7 verbatim (acceptance_test.cpp:134-163): full trace h=8, n=512,
//       d_h=8, 1 layer, 200 samples, window 32, seed 71; ada_snapkv vs snapkv (window 32,
//       pool 7, alpha 0.2) at budget fractions 0.2 / 0.4 through run_comparison
//       (report.hpp:161-345).  Writes one line per row:
//         sample fraction policy budget loss epsilon epsilon_star epsilon_double_star mass alloc...
//       then "agg fraction adaptive_wins samples win_fraction" lines.
//   ref_fig3 dump <dir>
//       a small trace (h=8, n=256, d_h=4, 1 layer, 6 samples, window 32, seed 5) as raw
//       little-endian f64 arrays -- per sample the outside / window K and V of every head,
//       the window queries Q_i = window_embeddings * W_q,i (exactly as evict_layer forms
//       them, policies.hpp:243), the decode query of make_sample_context (report.hpp:104-127)
//       -- plus W_o and the run_comparison rows of this trace at fractions 0.2 / 0.4
//       (rows.txt, same format), so a restatement can be checked against the reference row
//       by row on identical inputs.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <vector>

#include "adakv/adakv.hpp"

namespace {

adakv::PolicyConfig policy(adakv::PolicyKind kind) {
    adakv::PolicyConfig c;
    c.kind = kind;
    c.window_size = 32;
    c.pool_kernel = 7;
    c.alpha = 0.2;
    return c;
}

void write_rows(const adakv::ComparisonReport& rep, const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "w");
    for (const auto& r : rep.rows) {
        std::fprintf(f, "%zu %.17g %s %zu %.17g %.17g %.17g %.17g %.17g", r.sample, r.budget_fraction,
                     r.policy.c_str(), r.budget, r.loss ? *r.loss : -1.0, r.epsilon, r.epsilon_star,
                     r.epsilon_double_star, r.retained_mass);
        for (auto a : r.allocation) std::fprintf(f, " %zu", a);
        std::fprintf(f, "\n");
    }
    for (const auto& a : rep.aggregates)
        std::fprintf(f, "agg %.17g %zu %zu %.17g\n", a.budget_fraction, a.adaptive_wins, a.samples, a.win_fraction);
    std::fclose(f);
}

void put(std::ofstream& o, const adakv::Matrix& m) {
    o.write(reinterpret_cast<const char*>(m.values().data()), std::streamsize(m.values().size() * sizeof(double)));
}

}  // namespace

int main(int argc, char** argv) {
    if (argc != 3) {
        std::fprintf(stderr, "usage: %s accept <out.txt> | dump <dir>\n", argv[0]);
        return 2;
    }
    const std::string mode = argv[1], out = argv[2];
    const std::vector<adakv::PolicyConfig> pols{policy(adakv::PolicyKind::ada_snapkv),
                                                policy(adakv::PolicyKind::snapkv)};
    adakv::GeneratorProfile p;
    p.kind = adakv::TraceKind::full;
    p.layers = 1;
    p.window_size = 32;
    p.fraction_sparse_heads = 0.75;
    p.sparse_top_mass = 0.95;
    if (mode == "accept") {
        p.h = 8;
        p.n = 512;
        p.d_h = 8;
        p.samples = 200;
        const auto trace = adakv::generate_synthetic_trace(p, 71);
        write_rows(adakv::run_comparison(trace, {0.2, 0.4}, pols), out);
        return 0;
    }
    p.h = 8;
    p.n = 256;
    p.d_h = 4;
    p.samples = 6;
    const auto trace = adakv::generate_synthetic_trace(p, 5);
    const auto& params = trace.params[0];
    {
        std::ofstream o(out + "/wo.f64", std::ios::binary);
        for (const auto& hp : params.heads) put(o, hp.wo);
    }
    for (std::size_t s = 0; s < p.samples; ++s) {
        const auto dl = adakv::derive_layer(trace, s, 0);
        const auto ctx = adakv::detail::make_sample_context(dl, params);
        std::ofstream o(out + "/s" + std::to_string(s) + ".f64", std::ios::binary);
        for (const auto& h : dl.outside.heads) put(o, h.keys);
        for (const auto& h : dl.outside.heads) put(o, h.values);
        for (const auto& h : dl.window.heads) put(o, h.keys);
        for (const auto& h : dl.window.heads) put(o, h.values);
        for (const auto& hp : params.heads) put(o, adakv::matmul(dl.window_embeddings, hp.wq));
        for (const auto& q : ctx.queries) o.write(reinterpret_cast<const char*>(q.data()), std::streamsize(q.size() * 8));
    }
    write_rows(adakv::run_comparison(trace, {0.2, 0.4}, pols), out + "/rows.txt");
    return 0;
}
