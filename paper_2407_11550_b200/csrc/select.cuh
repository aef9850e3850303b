// select.cuh -- parameters of the cluster selection kernel (select.cu).
#pragma once

#include "budget_dev.cuh"

namespace adakv_b200 {

struct SelParams {
    int64_t off[kMaxSeg + 1];  // segment offsets within a problem (S + 1 entries)
    int S;
    int64_t N;                 // elements per problem (off[S])
    int alloc_mode, blend, repair, streaming;
    double alpha;
    int64_t sink;
    int64_t total;             // outside budget (uniform over problems) ...
    const int64_t* totals;     // ... or per problem (device), overrides total
    const void* scores;
    int32_t* raw_counts;
    int32_t* budgets;
    uint8_t* keep;
    int32_t* kept_pos;
    int64_t kept_stride;
    uint32_t* err;
    int cache_keys;            // set by launch_select: each CTA's key slice lives in shared memory
    int lean;                  // set by launch_select for many segments: one histogram buffer (an
                               // extra cluster barrier per pass) and no kept first-digit histogram
    int nonneg;                // every score is +0 or positive (adakv_compress's window scores):
                               // the bit patterns order as the values, no key transform needed
};

adakv_status launch_select(bool key64, int64_t P, const SelParams& prm, cudaStream_t stream);

}  // namespace adakv_b200
