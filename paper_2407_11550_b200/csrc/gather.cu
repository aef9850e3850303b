// gather.cu -- K3 copy half: pack kept K/V rows into the flattened varlen cache.
//
// Replaces the compaction loop of evict_layer (policies.hpp:273-290: kept outside
// rows in original order, then the m window rows) and select_and_compact
// (flat_cache.hpp:92-120: drop evicted rows, preserve order, offsets = prefix sums).
// Output planes K,V [rows, d]; segment (p, g) starts at seg_start[p*G+g] with
// capacity budget_g + m + reserve (reserve = decode appends, SPEC.md:454 notes the
// reference layout has no slack).  Copies are bit-exact, 16-byte vectorised and
// coalesced (one row = d*esize bytes = 16 x 16 B for bf16 d=128).
#include "budget_dev.cuh"
#include "common.cuh"

namespace adakv_b200 {

namespace {

constexpr int kGatherThreads = 256;
constexpr int kRowsPerBlock = 64;

// seg_start / seqlens for every (p, g).  Problem bases: uniform budgets give a
// closed form; per-problem budgets (pyramid kinds) need a prefix over problems,
// done by one block with a sequential carry over 1024-problem tiles.
__global__ void layout_kernel(const int32_t* __restrict__ budgets, int64_t P, int64_t G, int64_t m,
                              int64_t reserve, int64_t layer_budget,
                              const int64_t* __restrict__ layer_budgets, int32_t* __restrict__ seg_start,
                              int32_t* __restrict__ seqlens, int32_t* __restrict__ seg_cap) {
    __shared__ int64_t carry;
    __shared__ int64_t tile_sum[1024];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t t0 = 0; t0 < P; t0 += blockDim.x) {
        const int64_t p = t0 + threadIdx.x;
        int64_t rows = 0;
        if (p < P) rows = (layer_budgets ? layer_budgets[p] : layer_budget) + G * reserve;
        tile_sum[threadIdx.x] = rows;
        __syncthreads();
        // inclusive Hillis-Steele scan over the tile
        for (int o = 1; o < int(blockDim.x); o <<= 1) {
            const int64_t v = threadIdx.x >= unsigned(o) ? tile_sum[threadIdx.x - o] : 0;
            __syncthreads();
            tile_sum[threadIdx.x] += v;
            __syncthreads();
        }
        if (p < P) {
            int64_t base = carry + tile_sum[threadIdx.x] - rows;
            for (int64_t g = 0; g < G; ++g) {
                const int64_t len = budgets[p * G + g] + m;
                seg_start[p * G + g] = int32_t(base);
                seqlens[p * G + g] = int32_t(len);
                if (seg_cap) seg_cap[p * G + g] = int32_t(len + reserve);
                base += len + reserve;
            }
        }
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry += tile_sum[threadIdx.x];
        __syncthreads();
    }
}

// Non-finite test over the 32-bit words of a vector (LayerCache::validate, attention.hpp:76-83):
// mode 1 bf16 (two values per word), 2 f32, 3 f64 (the exponent lives in the odd words).
template <class V>
__device__ __forceinline__ bool nonfinite_vec(const V& x, int mode) {
    constexpr int NW = sizeof(V) / 4;
    if constexpr (NW == 0) {
        const uint32_t h = *reinterpret_cast<const uint16_t*>(&x);
        return mode == 1 && (h & 0x7f80u) == 0x7f80u;
    } else {
        const uint32_t* w = reinterpret_cast<const uint32_t*>(&x);
        bool bad = false;
#pragma unroll
        for (int i = 0; i < NW; ++i) {
            if (mode == 1) bad |= (w[i] & 0x7f80u) == 0x7f80u || (w[i] & 0x7f800000u) == 0x7f800000u;
            else if (mode == 2) bad |= (w[i] & 0x7f800000u) == 0x7f800000u;
            else if (mode == 3 && (i & 1)) bad |= (w[i] & 0x7ff00000u) == 0x7ff00000u;
        }
        return bad;
    }
}

template <class V>
__global__ void __launch_bounds__(kGatherThreads)
gather_kernel(const V* __restrict__ k, const V* __restrict__ v, int64_t G, int64_t n_rows,
              int64_t n_o, int64_t m, int64_t vec_per_row, const int32_t* __restrict__ budgets,
              const int32_t* __restrict__ kept_pos, int64_t kept_stride,
              const int32_t* __restrict__ seg_start, V* __restrict__ k_cache,
              V* __restrict__ v_cache, int fin_mode, uint32_t* __restrict__ err) {
    __shared__ int64_t cum[kMaxSeg + 1];   // cumulative (budget + m) per group
    __shared__ int64_t bcum[kMaxSeg + 1];  // cumulative budget per group (kept_pos offset)
    const int64_t p = blockIdx.y;
    if (threadIdx.x == 0) {
        cum[0] = 0;
        bcum[0] = 0;
        for (int64_t g = 0; g < G; ++g) {
            const int64_t b = budgets[p * G + g];
            cum[g + 1] = cum[g] + b + m;
            bcum[g + 1] = bcum[g] + b;
        }
    }
    __syncthreads();
    const int64_t total = cum[G];
    const int64_t r0 = int64_t(blockIdx.x) * kRowsPerBlock;
    const int64_t r1 = min(r0 + int64_t(kRowsPerBlock), total);
    const int nrow = int(r1 - r0), vpr = int(vec_per_row);
    // vec_per_row is a power of two for every supported row size (d * esize / sizeof(V)):
    // row and column of an item by shift and mask, in 32 bits (no 64-bit division per item)
    const int vshift = __ffs(vpr) - 1;
    const bool pow2 = (vpr & (vpr - 1)) == 0;
    const int items = nrow * vpr;
    bool bad = false;
    for (int it = threadIdx.x; it < items; it += kGatherThreads) {
        const int rr = pow2 ? (it >> vshift) : it / vpr;
        const int c = pow2 ? (it & (vpr - 1)) : it % vpr;
        const int64_t r = r0 + rr;
        int64_t g = 0;
        while (cum[g + 1] <= r) ++g;
        const int64_t rin = r - cum[g];
        const int64_t b = bcum[g + 1] - bcum[g];
        ADAKV_DCHECK(g < G && rin >= 0 && (rin >= b || bcum[g] + rin < kept_stride));
        const int64_t src_row = rin < b ? int64_t(kept_pos[p * kept_stride + bcum[g] + rin]) : n_o + (rin - b);
        ADAKV_DCHECK(src_row >= 0 && src_row < n_rows && (rin >= b ? true : src_row < n_o));
        const int64_t src = ((p * G + g) * n_rows + src_row) * vec_per_row + c;
        const int64_t dst = (int64_t(seg_start[p * G + g]) + rin) * vec_per_row + c;
        const V kx = k[src], vx = v[src];
        k_cache[dst] = kx;
        v_cache[dst] = vx;
        if (fin_mode) bad |= nonfinite_vec(kx, fin_mode) || nonfinite_vec(vx, fin_mode);
    }
    // the retained and window rows are checked as they are copied (one warp vote, one atomic)
    if (err && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, ERR_NONFINITE);
}

template <class V>
__global__ void validate_kernel(const V* __restrict__ x, int64_t nvec, int mode, uint32_t* __restrict__ err) {
    bool bad = false;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nvec; i += int64_t(gridDim.x) * blockDim.x)
        bad |= nonfinite_vec(x[i], mode);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, ERR_NONFINITE);
}

}  // namespace

adakv_status launch_layout(const int32_t* budgets, int64_t P, int64_t G, int64_t m, int64_t reserve,
                           int64_t layer_budget, const int64_t* layer_budgets, int32_t* seg_start,
                           int32_t* seqlens, int32_t* seg_cap, cudaStream_t stream) {
    if (G > kMaxSeg) return fail(ADAKV_UNSUPPORTED, "gather: more than 64 KV groups");
    layout_kernel<<<1, 1024, 0, stream>>>(budgets, P, G, m, reserve, layer_budget, layer_budgets,
                                          seg_start, seqlens, seg_cap);
    ADAKV_CUDA_TRY(cudaGetLastError());
    return ADAKV_OK;
}

adakv_status launch_gather(adakv_dtype dt, const adakv_layer_shape& s, int64_t max_rows,
                           const void* k, const void* v, const int32_t* budgets,
                           const int32_t* kept_pos, int64_t kept_stride, const int32_t* seg_start,
                           void* k_cache, void* v_cache, uint32_t* err, cudaStream_t stream) {
    const int fm = err ? (dt == ADAKV_BF16 ? 1 : dt == ADAKV_F32 ? 2 : 3) : 0;
    const int64_t P = s.problems, G = s.kv_groups, d = s.head_dim;
    const int64_t row_bytes = d * int64_t(dtype_size(dt));
    const dim3 grid(unsigned(ceil_div(max_rows, kRowsPerBlock)), unsigned(P));
    if (grid.x == 0 || P == 0) return ADAKV_OK;
    const bool aligned16 = row_bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(k) % 16 == 0) &&
                           (reinterpret_cast<uintptr_t>(v) % 16 == 0) &&
                           (reinterpret_cast<uintptr_t>(k_cache) % 16 == 0) &&
                           (reinterpret_cast<uintptr_t>(v_cache) % 16 == 0);
    const int64_t n_rows = s.outside + s.window;
    if (aligned16) {
        gather_kernel<int4><<<grid, kGatherThreads, 0, stream>>>(
            static_cast<const int4*>(k), static_cast<const int4*>(v), G, n_rows, s.outside, s.window,
            row_bytes / 16, budgets, kept_pos, kept_stride, seg_start, static_cast<int4*>(k_cache),
            static_cast<int4*>(v_cache), fm, err);
    } else if (row_bytes % 8 == 0) {
        gather_kernel<int2><<<grid, kGatherThreads, 0, stream>>>(
            static_cast<const int2*>(k), static_cast<const int2*>(v), G, n_rows, s.outside, s.window,
            row_bytes / 8, budgets, kept_pos, kept_stride, seg_start, static_cast<int2*>(k_cache),
            static_cast<int2*>(v_cache), fm, err);
    } else if (row_bytes % 4 == 0) {
        gather_kernel<int><<<grid, kGatherThreads, 0, stream>>>(
            static_cast<const int*>(k), static_cast<const int*>(v), G, n_rows, s.outside, s.window,
            row_bytes / 4, budgets, kept_pos, kept_stride, seg_start, static_cast<int*>(k_cache),
            static_cast<int*>(v_cache), fm, err);
    } else {
        gather_kernel<uint16_t><<<grid, kGatherThreads, 0, stream>>>(
            static_cast<const uint16_t*>(k), static_cast<const uint16_t*>(v), G, n_rows, s.outside,
            s.window, row_bytes / 2, budgets, kept_pos, kept_stride, seg_start,
            static_cast<uint16_t*>(k_cache), static_cast<uint16_t*>(v_cache), fm, err);
    }
    ADAKV_CUDA_TRY(cudaGetLastError());
    return ADAKV_OK;
}

}  // namespace adakv_b200

namespace adakv_b200 {
adakv_status launch_validate(adakv_dtype dt, const void* data, int64_t n, uint32_t* err, cudaStream_t stream) {
    const int mode = dt == ADAKV_BF16 ? 1 : dt == ADAKV_F32 ? 2 : 3;
    const int64_t bytes = n * int64_t(dtype_size(dt));
    const int grid = device_sm_count() * 4;
    if (reinterpret_cast<uintptr_t>(data) % 16 == 0 && bytes % 16 == 0)
        validate_kernel<int4><<<grid, 256, 0, stream>>>(static_cast<const int4*>(data), bytes / 16, mode, err);
    else if (dt == ADAKV_BF16)
        validate_kernel<uint16_t><<<grid, 256, 0, stream>>>(static_cast<const uint16_t*>(data), n, mode, err);
    else if (dt == ADAKV_F32)
        validate_kernel<int><<<grid, 256, 0, stream>>>(static_cast<const int*>(data), n, mode, err);
    else
        validate_kernel<int2><<<grid, 256, 0, stream>>>(static_cast<const int2*>(data), n, mode, err);
    ADAKV_CUDA_TRY(cudaGetLastError());
    return ADAKV_OK;
}
}  // namespace adakv_b200
