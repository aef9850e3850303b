// shard.cu -- the device glue of KV-group-sharded allocation (sharding.py): the candidate
// payload a rank contributes to the one all-gather, and the candidate union every rank
// rebuilds from the gathered payloads.  Pure data movement; the selection itself is
// select.cu.  Replaces the torch glue (repeat_interleave / gather / cat / cumsum / where)
// around Algorithm 1's layer-wide top-B (budget.hpp:118-140) when the KV groups of a layer
// are spread over ranks.
#include "common.cuh"

namespace adakv_b200 {

namespace {

constexpr int kShardThreads = 256;

// payload = [counts (G_local) | scores of the k kept candidates as f32 bits | their positions]
// kept positions pos[k] are segment-major, ascending within a segment; segment g holds
// counts[g] of them; scores [G_local, n_o] f32.
__global__ void pack_kernel(const float* __restrict__ scores, const int32_t* __restrict__ counts,
                            const int32_t* __restrict__ pos, int G_local, int64_t n_o, int64_t k,
                            int32_t* __restrict__ payload) {
    __shared__ int64_t start[64 + 1];
    if (threadIdx.x == 0) {
        int64_t s = 0;
        for (int g = 0; g < G_local; ++g) {
            start[g] = s;
            s += counts[g];
        }
        start[G_local] = s;
    }
    __syncthreads();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < G_local + k;
         i += int64_t(gridDim.x) * blockDim.x) {
        if (i < G_local) {
            payload[i] = counts[i];
            continue;
        }
        const int64_t c = i - G_local;
        int g = 0;
        while (g + 1 < G_local && start[g + 1] <= c) ++g;
        const int32_t p = pos[c];
        payload[i] = __float_as_int(scores[int64_t(g) * n_o + p]);
        payload[G_local + k + c] = p;
    }
}

// union [G, S] f32: row g = global group (rank g / G_local, local g % G_local) holds that
// group's candidate scores in position order, then -1 (below every score) in empty slots
__global__ void union_kernel(const int32_t* __restrict__ gathered, int world, int G_local, int64_t k,
                             int64_t S, float* __restrict__ out) {
    const int64_t stride = G_local + 2 * k;
    const int64_t total = int64_t(world) * G_local * S;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t g = i / S, j = i - g * S;
        const int r = int(g / G_local), gl = int(g - int64_t(r) * G_local);
        const int32_t* row = gathered + r * stride;
        int64_t start = 0;
        for (int t = 0; t < gl; ++t) start += row[t];
        out[i] = j < row[gl] ? __int_as_float(row[G_local + start + j]) : -1.f;
    }
}

unsigned grid_for(int64_t n) {
    const int64_t b = (n + kShardThreads - 1) / kShardThreads;
    return unsigned(b < 1 ? 1 : (b > 4 * 148 ? 4 * 148 : b));
}

}  // namespace

}  // namespace adakv_b200

using namespace adakv_b200;

extern "C" adakv_status adakv_shard_pack_candidates(const float* scores, const int32_t* counts, const int32_t* pos,
                                                    int64_t local_groups, int64_t outside, int64_t k,
                                                    int32_t* payload, adakv_stream_t stream) {
    if (local_groups < 1 || local_groups > 64 || outside < 1 || k < 0)
        return fail(ADAKV_INVALID_ARGUMENT, "shard_pack_candidates: bad shape");
    if (!scores || !counts || !payload || (k > 0 && !pos))
        return fail(ADAKV_INVALID_ARGUMENT, "shard_pack_candidates: null argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    pack_kernel<<<grid_for(local_groups + k), kShardThreads, 0, st>>>(scores, counts, pos, int(local_groups), outside,
                                                                     k, payload);
    ADAKV_CUDA_TRY(cudaGetLastError());
    return ADAKV_OK;
}

extern "C" adakv_status adakv_shard_build_union(const int32_t* gathered, int64_t world, int64_t local_groups, int64_t k,
                                                int64_t slots, float* out, adakv_stream_t stream) {
    if (world < 1 || local_groups < 1 || k < 0 || slots < 1)
        return fail(ADAKV_INVALID_ARGUMENT, "shard_build_union: bad shape");
    if (!gathered || !out) return fail(ADAKV_INVALID_ARGUMENT, "shard_build_union: null argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    union_kernel<<<grid_for(world * local_groups * slots), kShardThreads, 0, st>>>(gathered, int(world),
                                                                                  int(local_groups), k, slots, out);
    ADAKV_CUDA_TRY(cudaGetLastError());
    return ADAKV_OK;
}
