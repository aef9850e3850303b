// ref_golden.cpp -- golden-vector generator over the UNMODIFIED reference.
//
// TEST INFRASTRUCTURE ONLY.  Built by `make -C oracle golden` (needs
// /root/reference and nlohmann/json, which trace.hpp:15 includes) and run by
// tests/golden/make_golden.py.  It drives the reference's own synthetic trace
// generator (trace.hpp:277-305, derive_layer 315-350) and evict_layer
// (policies.hpp:204-293) and dumps raw little-endian arrays:
//
//   <out>/<name>.scores.f64   group scores   [G * n]
//   <out>/<name>.alloc.i64    allocation     [G]
//   <out>/<name>.keep.u8      decision       [G * n] (group leaders)
//   <out>/<name>.meta.txt     "G n" and the joined allocation
//
// usage: ref_golden <out_dir> <name> <h> <gqa> <n> <d_h> <window> <seed>
//                   <layer_budget> <kind> <alpha> <pool>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>

#include "adakv/adakv.hpp"

int main(int argc, char** argv) {
    if (argc != 13) {
        std::fprintf(stderr, "usage: %s out name h gqa n d_h window seed LB kind alpha pool\n", argv[0]);
        return 2;
    }
    const std::string out = argv[1], name = argv[2];
    adakv::GeneratorProfile p;
    p.h = std::strtoul(argv[3], nullptr, 10);
    p.gqa_group_size = std::strtoul(argv[4], nullptr, 10);
    p.n = std::strtoul(argv[5], nullptr, 10);
    p.d_h = std::strtoul(argv[6], nullptr, 10);
    p.window_size = std::strtoul(argv[7], nullptr, 10);
    p.samples = 1;
    p.layers = 1;
    const auto seed = std::strtoull(argv[8], nullptr, 10);
    const std::size_t budget = std::strtoul(argv[9], nullptr, 10);
    adakv::PolicyConfig cfg;
    cfg.kind = adakv::policy_kind_from_string(argv[10]);
    cfg.alpha = std::strtod(argv[11], nullptr);
    cfg.pool_kernel = std::strtoul(argv[12], nullptr, 10);
    cfg.window_size = p.window_size;
    cfg.gqa_group_size = p.gqa_group_size;

    const auto trace = adakv::generate_synthetic_trace(p, seed);
    const auto dl = adakv::derive_layer(trace, 0, 0);
    const auto res = adakv::evict_layer(dl.outside, dl.window, dl.window_embeddings,
                                        trace.params[0], budget, cfg);
    const std::size_t G = p.h / p.gqa_group_size;
    std::ofstream fs(out + "/" + name + ".scores.f64", std::ios::binary);
    std::ofstream fa(out + "/" + name + ".alloc.i64", std::ios::binary);
    std::ofstream fk(out + "/" + name + ".keep.u8", std::ios::binary);
    std::ofstream fm(out + "/" + name + ".meta.txt");
    fm << G << " " << p.n << "\n";
    for (std::size_t gi = 0; gi < G; ++gi) {
        fs.write(reinterpret_cast<const char*>(res.scores[gi].data()),
                 static_cast<std::streamsize>(res.scores[gi].size() * sizeof(double)));
        const auto a = static_cast<long long>(res.allocation.per_head[gi]);
        fa.write(reinterpret_cast<const char*>(&a), sizeof a);
        const auto& keep = res.decision.retain[gi * p.gqa_group_size];
        fk.write(reinterpret_cast<const char*>(keep.data()), static_cast<std::streamsize>(keep.size()));
        fm << (gi ? "|" : "") << a;
    }
    fm << "\n";
    return 0;
}
