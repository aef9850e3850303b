// score_window_tc.cu -- K1 on the 5th-generation tensor cores (bf16, d == 128, m == 32,
// g*m <= 128): observation-window scoring fused into two persistent passes.
//
// Reference semantics (see score_window.cu for the file:line list): per KV group, the
// g*m window rows (g heads x m rows) are softmaxed over the OUTSIDE keys, max-pooled
// along keys (k odd, stride 1, padded cells excluded), averaged over rows (/m) and
// heads (/g).
//
// B200 mapping.  The g*m <= 128 query rows of a KV group are exactly one UMMA M=128
// tile; each 128-key K tile is the N=128 operand; d = 128 is the K extent (8 MMAs of
// K=16).  Per CTA (1 per SM, persistent over (group, key-chunk) items):
//   warp 0        TMA producer: Q tile (per item, double-buffered) and a 4-stage ring of
//                 K tiles, 128B-swizzled [128 x 64] halves, 3-D tensor maps so rows
//                 outside a group are zero-filled by the hardware;
//   warp 1        TMEM owner + single-thread tcgen05.mma issuer, fp32 accumulators in
//                 TMEM (2 x 128 columns, double-buffered);
//   warps 2..5    epilogue: thread r <-> TMEM lane r <-> window row r; with m == 32 each
//                 warp is exactly one query head.
// Pass 1 (row statistics): online max / sum of exp2 over the tile's logits, per item a
//   partial (max, sum) per row; the last CTA of a group (atomic ticket) folds them into
//   (M_r, Lw_r = M_r + log2(S_r * m)).
// Pass 2 (scores): tiles advance by 128 - 2*pad keys so every output key has its full
//   pooling halo inside the tile; pooling is done on LOGITS in registers (exp2 is
//   monotone), e = exp2(pool*c - Lw_r) = pooled_prob / m, then a 32-lane butterfly
//   reduce-scatter sums the warp's 32 rows (= its head) per key in fp32, heads are summed
//   through shared memory and divided by g.
// The two passes run back to back over a slice of problems small enough (~48 MB of K) to
// stay resident in the 126 MB L2, so pass 2 re-reads K from L2, not HBM (pass 1 loads
// with evict_last, pass 2 with evict_first).
#include <cuda.h>

#include <mutex>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace adakv_b200 {

namespace {

using namespace ptx;

constexpr int kThreads = 192;
constexpr int kStages = 4;
constexpr int kTile = 128;
constexpr uint32_t kTmemCols = 256;
constexpr uint32_t kHalfBytes = 128 * 128;  // [128 rows][64 bf16]
constexpr uint32_t kTileBytes = 2 * kHalfBytes;

struct __align__(1024) Smem {
    uint8_t q[2][2][kHalfBytes];
    uint8_t k[kStages][2][kHalfBytes];
    float head_part[2][4][kTile];
    uint64_t full[kStages], empty[kStages];
    uint64_t q_full[2], q_empty[2];
    uint64_t acc_full[2], acc_empty[2];
    uint32_t tmem_base;
    uint32_t is_last;
};

struct TcParams {
    int pass;
    int G, H, gs, m, n_o, step, pad;
    int tiles_per_pg, tiles_per_item, chunks_per_pg, n_items;
    int pg_base;  // first problem*group of this slice (for outputs / stats)
    float scale_log2;
    float log2_m;
    float inv_g;
    float* partial;      // [pg][chunk][128][2]
    float* final_stats;  // [pg][128][2]
    unsigned* tickets;   // [pg]
    float* head_scores;  // [P][H][n_o] or null
    float* group_scores; // [P][G][n_o]
};

// ------------------------------------------------------------------ epilogue helpers
template <int BASE, int NV>
__device__ __forceinline__ float butterfly32(float (&e)[NV], int lane) {
    // reduce-scatter over the 32 lanes: afterwards lane l holds sum_lanes e[BASE + l]
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const float lo = e[BASE + i], hi = e[BASE + i + o];
            const float send = up ? lo : hi;
            const float keep = up ? hi : lo;
            e[BASE + i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return e[BASE];
}

template <int PAD>
__device__ __forceinline__ void pool_exp(float (&v)[kTile], float sl, float lw) {
    // v: raw logits of 128 loaded keys (masked keys = -inf).  Output column c in
    // [PAD, PAD + STEP) is written to v[c - PAD] as exp2(max(v[c-PAD..c+PAD]) * sl - lw).
    constexpr int STEP = kTile - 2 * PAD;
    if constexpr (PAD == 0) {
#pragma unroll
        for (int c = 0; c < STEP; ++c) v[c] = ex2(fmaf(v[c], sl, -lw));
    } else if constexpr (PAD == 1) {
#pragma unroll
        for (int c = 0; c < STEP; ++c) v[c] = ex2(fmaf(max3(v[c], v[c + 1], v[c + 2]), sl, -lw));
    } else {
        // b[j] = max(v[j], v[j+1], v[j+2]) in place (v[j] is dead once b[j] exists)
#pragma unroll
        for (int j = 0; j < kTile - 2; ++j) v[j] = max3(v[j], v[j + 1], v[j + 2]);
        if constexpr (PAD == 2) {
            // window [c-2, c+2] = b[c-2] | b[c]
#pragma unroll
            for (int c = 2; c < 2 + STEP; ++c) v[c - 2] = ex2(fmaf(fmaxf(v[c - 2], v[c]), sl, -lw));
        } else {
            // PAD == 3: window [c-3, c+3] = b[c-3] | b[c] | b[c+1]; b[c-3] is dead after use
#pragma unroll
            for (int c = 3; c < 3 + STEP; ++c) v[c - 3] = ex2(fmaf(max3(v[c - 3], v[c], v[c + 1]), sl, -lw));
        }
    }
}

template <int PAD>
__global__ void __launch_bounds__(kThreads, 1)
score_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                const TcParams prm) {
    extern __shared__ uint8_t smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tm_q);
        prefetch_tmap(&tm_k);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&S.full[s], 1);
            mbar_init(&S.empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&S.q_full[b], 1);
            mbar_init(&S.q_empty[b], 1);
            mbar_init(&S.acc_full[b], 1);
            mbar_init(&S.acc_empty[b], 4);
        }
        mbar_fence_init();
    }
    if (warp == 1) tmem_alloc<kTmemCols>(&S.tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem_base;

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            const uint64_t pol = prm.pass == 1 ? policy_evict_last() : policy_evict_first();
            const uint64_t pol_q = policy_evict_last();
            uint32_t stage = 0, sphase = 0, qb = 0, qphase = 0;
            for (int item = blockIdx.x; item < prm.n_items; item += gridDim.x) {
                const int pg = item / prm.chunks_per_pg, chunk = item % prm.chunks_per_pg;
                const int t0 = chunk * prm.tiles_per_item;
                const int t1 = min(t0 + prm.tiles_per_item, prm.tiles_per_pg);
                mbar_wait(&S.q_empty[qb], qphase ^ 1);
                mbar_arrive_expect_tx(&S.q_full[qb], kTileBytes);
                tma_load_3d(S.q[qb][0], &tm_q, 0, 0, pg, &S.q_full[qb], pol_q);
                tma_load_3d(S.q[qb][1], &tm_q, 64, 0, pg, &S.q_full[qb], pol_q);
                for (int t = t0; t < t1; ++t) {
                    mbar_wait(&S.empty[stage], sphase ^ 1);
                    mbar_arrive_expect_tx(&S.full[stage], kTileBytes);
                    const int row = t * prm.step - prm.pad;
                    tma_load_3d(S.k[stage][0], &tm_k, 0, row, pg, &S.full[stage], pol);
                    tma_load_3d(S.k[stage][1], &tm_k, 64, row, pg, &S.full[stage], pol);
                    if (++stage == kStages) {
                        stage = 0;
                        sphase ^= 1;
                    }
                }
                if (++qb == 2) {
                    qb = 0;
                    qphase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // ===================== tcgen05 MMA issuer =====================
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_bf16_f32(128, kTile);
            uint32_t stage = 0, sphase = 0, qb = 0, qphase = 0, ab = 0, aphase = 0;
            for (int item = blockIdx.x; item < prm.n_items; item += gridDim.x) {
                const int chunk = item % prm.chunks_per_pg;
                const int t0 = chunk * prm.tiles_per_item;
                const int t1 = min(t0 + prm.tiles_per_item, prm.tiles_per_pg);
                mbar_wait(&S.q_full[qb], qphase);
                for (int t = t0; t < t1; ++t) {
                    mbar_wait(&S.acc_empty[ab], aphase ^ 1);
                    mbar_wait(&S.full[stage], sphase);
                    tc_fence_after();
                    const uint32_t d = tmem + ab * kTile;
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint32_t off = (kk & 3) * 32;
                        const uint64_t ad = desc_kmajor_sw128(smem_u32(S.q[qb][kk >> 2]) + off);
                        const uint64_t bd = desc_kmajor_sw128(smem_u32(S.k[stage][kk >> 2]) + off);
                        mma_bf16(d, ad, bd, idesc, kk > 0 ? 1u : 0u);
                    }
                    mma_commit(&S.empty[stage]);
                    mma_commit(&S.acc_full[ab]);
                    if (++stage == kStages) {
                        stage = 0;
                        sphase ^= 1;
                    }
                    if (++ab == 2) {
                        ab = 0;
                        aphase ^= 1;
                    }
                }
                mma_commit(&S.q_empty[qb]);
                if (++qb == 2) {
                    qb = 0;
                    qphase ^= 1;
                }
            }
        }
    } else {
        // ===================== epilogue (warps 2..5) =====================
        const int quarter = warp & 3;               // TMEM lane quarter this warp may access
        const int r = quarter * 32 + lane;          // window row == TMEM lane
        const int R = prm.gs * prm.m;
        const bool active = r < R;
        const int et = (warp - 2) * 32 + lane;      // 0..127 epilogue thread id
        const float sl = prm.scale_log2;
        uint32_t ab = 0, aphase = 0, hb = 0;
        for (int item = blockIdx.x; item < prm.n_items; item += gridDim.x) {
            const int pg = item / prm.chunks_per_pg, chunk = item % prm.chunks_per_pg;
            const int t0 = chunk * prm.tiles_per_item;
            const int t1 = min(t0 + prm.tiles_per_item, prm.tiles_per_pg);
            const int gpg = prm.pg_base + pg;
            float run_m = -INFINITY, run_s = 0.f, lw = INFINITY;
            if (prm.pass == 2 && active) lw = prm.final_stats[(size_t(gpg) * 128 + r) * 2 + 1];
            for (int t = t0; t < t1; ++t) {
                mbar_wait(&S.acc_full[ab], aphase);
                tc_fence_after();
                float v[kTile];
                const uint32_t taddr = tmem + ab * kTile + (uint32_t(quarter * 32) << 16);
                tmem_ld_x32<0>(taddr + 0, v);
                tmem_ld_x32<32>(taddr + 32, v);
                tmem_ld_x32<64>(taddr + 64, v);
                tmem_ld_x32<96>(taddr + 96, v);
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&S.acc_empty[ab]);
                if (++ab == 2) {
                    ab = 0;
                    aphase ^= 1;
                }
                const int key0 = t * prm.step - prm.pad;
                if (prm.pass == 1) {
                    const int nvalid = min(kTile, prm.n_o - key0);
                    if (nvalid < kTile) {
#pragma unroll
                        for (int j = 0; j < kTile; ++j)
                            if (j >= nvalid) v[j] = -INFINITY;
                    }
                    float tm = v[0];
#pragma unroll
                    for (int j = 1; j + 1 < kTile; j += 2) tm = max3(tm, v[j], v[j + 1]);
                    tm = fmaxf(tm, v[kTile - 1]);
                    const float nm = fmaxf(run_m, tm * sl);
                    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
                    for (int j = 0; j < kTile; j += 4) {
                        s0 += ex2(fmaf(v[j + 0], sl, -nm));
                        s1 += ex2(fmaf(v[j + 1], sl, -nm));
                        s2 += ex2(fmaf(v[j + 2], sl, -nm));
                        s3 += ex2(fmaf(v[j + 3], sl, -nm));
                    }
                    run_s = run_s * ex2(run_m - nm) + ((s0 + s1) + (s2 + s3));
                    run_m = nm;
                } else {
                    if (key0 < 0 || key0 + kTile > prm.n_o) {
#pragma unroll
                        for (int j = 0; j < kTile; ++j)
                            if (key0 + j < 0 || key0 + j >= prm.n_o) v[j] = -INFINITY;
                    }
                    pool_exp<PAD>(v, sl, active ? lw : INFINITY);
                    constexpr int STEP = kTile - 2 * PAD;
#pragma unroll
                    for (int c = STEP; c < kTile; ++c) v[c] = 0.f;
                    float* hp = S.head_part[hb][quarter];
                    hp[0 + lane] = butterfly32<0>(v, lane);
                    hp[32 + lane] = butterfly32<32>(v, lane);
                    hp[64 + lane] = butterfly32<64>(v, lane);
                    hp[96 + lane] = butterfly32<96>(v, lane);
                    named_bar(1, 128);
                    // heads -> group mean; one key per epilogue thread, coalesced stores
                    const int key = t * prm.step + et;
                    if (et < STEP && key < prm.n_o) {
                        const int p = gpg / prm.G, g = gpg % prm.G;
                        float gsum = 0.f;
                        for (int h = 0; h < prm.gs; ++h) {
                            const float hv = S.head_part[hb][h][et];
                            gsum += hv;
                            if (prm.head_scores)
                                prm.head_scores[(size_t(p) * prm.H + g * prm.gs + h) * prm.n_o + key] = hv;
                        }
                        prm.group_scores[size_t(gpg) * prm.n_o + key] = gsum * prm.inv_g;
                    }
                    hb ^= 1;
                }
            }
            if (prm.pass == 1) {
                float* pp = prm.partial + ((size_t(pg) * prm.chunks_per_pg + chunk) * 128 + r) * 2;
                pp[0] = active ? run_m : -INFINITY;
                pp[1] = active ? run_s : 0.f;
                __threadfence();
                named_bar(1, 128);
                if (et == 0) S.is_last = atomicAdd(&prm.tickets[pg], 1u) == unsigned(prm.chunks_per_pg - 1);
                named_bar(1, 128);
                if (S.is_last) {
                    __threadfence();
                    const float* base = prm.partial + size_t(pg) * prm.chunks_per_pg * 256;
                    float M = -INFINITY;
                    for (int c = 0; c < prm.chunks_per_pg; ++c) M = fmaxf(M, __ldcg(base + (c * 128 + r) * 2));
                    float Ssum = 0.f;
                    for (int c = 0; c < prm.chunks_per_pg; ++c) {
                        const float mc = __ldcg(base + (c * 128 + r) * 2);
                        if (mc != -INFINITY) Ssum += __ldcg(base + (c * 128 + r) * 2 + 1) * ex2(mc - M);
                    }
                    float* fs = prm.final_stats + (size_t(gpg) * 128 + r) * 2;
                    fs[0] = M;
                    fs[1] = active ? M + __log2f(Ssum) + prm.log2_m : INFINITY;
                    if (et == 0) prm.tickets[pg] = 0u;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc<kTmemCols>(tmem);
}

// ------------------------------------------------------------------ host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

// 3-D bf16 tensor [outer][rows][128] with a {64, 128, 1} box, 128-byte swizzle.
adakv_status make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t outer) {
    EncodeFn enc = get_encode();
    if (!enc) return fail(ADAKV_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[3] = {128, rows, outer};
    const cuuint64_t strides[2] = {128 * 2, rows * 128 * 2};
    const cuuint32_t box[3] = {64, 128, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(ADAKV_CUDA_ERROR, "cuTensorMapEncodeTiled failed");
    return ADAKV_OK;
}

size_t smem_bytes() { return sizeof(Smem) + 1024; }

struct Plan {
    int64_t slice;       // problems per slice (L2-resident pass pair)
    int chunks1, tpi1;   // pass 1 decomposition per (p, g)
    int chunks2, tpi2;
};

Plan make_plan(const adakv_layer_shape& s, int pad) {
    Plan pl{};
    const int64_t k_bytes = s.kv_groups * (s.outside + s.window) * s.head_dim * 2;
    pl.slice = std::max<int64_t>(1, std::min<int64_t>(s.problems, (48ll << 20) / std::max<int64_t>(k_bytes, 1)));
    const int sms = device_sm_count();
    const int step2 = kTile - 2 * pad;
    const int64_t tiles1 = ceil_div(s.outside, kTile), tiles2 = ceil_div(s.outside, step2);
    const int64_t pgs = pl.slice * s.kv_groups;
    // aim for ~4 items per CTA so the persistent grid balances
    pl.tpi1 = int(std::max<int64_t>(1, (pgs * tiles1) / (int64_t(sms) * 4)));
    pl.tpi2 = int(std::max<int64_t>(1, (pgs * tiles2) / (int64_t(sms) * 4)));
    pl.chunks1 = int(ceil_div(tiles1, pl.tpi1));
    pl.chunks2 = int(ceil_div(tiles2, pl.tpi2));
    return pl;
}

}  // namespace

bool score_window_tc_supported(adakv_dtype dt, const adakv_layer_shape& s, int64_t pool_kernel) {
    const int64_t gs = s.kv_groups > 0 ? s.q_heads / s.kv_groups : 0;
    return dt == ADAKV_BF16 && s.head_dim == 128 && s.window == 32 && gs >= 1 && gs * s.window <= 128 &&
           (pool_kernel == 1 || pool_kernel == 3 || pool_kernel == 5 || pool_kernel == 7) && s.outside >= 1 &&
           s.outside + s.window < (int64_t(1) << 31) && get_encode() != nullptr;
}

size_t score_window_tc_workspace(const adakv_layer_shape& s) {
    const Plan pl = make_plan(s, 3);
    const int64_t pgs_slice = pl.slice * s.kv_groups;
    const int64_t chunks = std::max(pl.chunks1, make_plan(s, 0).chunks1);
    return 3 * 256 + size_t(pgs_slice) * chunks * 128 * 2 * 4 + size_t(s.problems * s.kv_groups) * 128 * 2 * 4 +
           size_t(pgs_slice) * 4;
}

adakv_status score_window_tc(const adakv_layer_shape& s, int64_t pool_kernel, int32_t scale, const void* q,
                             const void* k, void* head_scores, void* group_scores, void* ws, cudaStream_t stream) {
    const int pad = int((pool_kernel - 1) / 2);
    const Plan pl = make_plan(s, pad);
    const int64_t G = s.kv_groups, H = s.q_heads, gs = H / G, m = s.window, n = s.outside + s.window;
    const int64_t d = s.head_dim;
    Arena ar(ws);
    const Plan pl0 = make_plan(s, 0);
    const int64_t chunks_max = std::max(pl.chunks1, pl0.chunks1);
    float* partial = ar.take<float>(size_t(pl.slice * G * chunks_max * 256));
    float* fstats = ar.take<float>(size_t(s.problems * G * 256));
    unsigned* tickets = ar.take<unsigned>(size_t(pl.slice * G));
    ADAKV_CUDA_TRY(cudaMemsetAsync(tickets, 0, size_t(pl.slice * G) * 4, stream));
    const size_t smem = smem_bytes();
    const int sms = device_sm_count();
    auto kfn = pad == 0 ? score_tc_kernel<0> : pad == 1 ? score_tc_kernel<1> : pad == 2 ? score_tc_kernel<2>
                                                                                        : score_tc_kernel<3>;
    ADAKV_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    ADAKV_CUDA_TRY(cudaFuncSetAttribute(score_tc_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const float sc = scale ? 1.0f / sqrtf(float(d)) : 1.0f;
    for (int64_t p0 = 0; p0 < s.problems; p0 += pl.slice) {
        const int64_t np = std::min(pl.slice, s.problems - p0);
        CUtensorMap tq, tk;
        const auto* qb = static_cast<const __nv_bfloat16*>(q) + p0 * H * m * d;
        const auto* kb = static_cast<const __nv_bfloat16*>(k) + p0 * G * n * d;
        ADAKV_TRY(make_map(&tq, qb, uint64_t(gs * m), uint64_t(np * G)));
        ADAKV_TRY(make_map(&tk, kb, uint64_t(n), uint64_t(np * G)));
        TcParams prm{};
        prm.G = int(G);
        prm.H = int(H);
        prm.gs = int(gs);
        prm.m = int(m);
        prm.n_o = int(s.outside);
        prm.pg_base = int(p0 * G);
        prm.scale_log2 = sc * 1.4426950408889634f;
        prm.log2_m = log2f(float(m));
        prm.inv_g = 1.0f / float(gs);
        prm.partial = partial;
        prm.final_stats = fstats;
        prm.tickets = tickets;
        prm.head_scores = static_cast<float*>(head_scores);
        prm.group_scores = static_cast<float*>(group_scores);
        // pass 1: row statistics over 128-key tiles
        prm.pass = 1;
        prm.step = kTile;
        prm.pad = 0;
        prm.tiles_per_pg = int(ceil_div(s.outside, kTile));
        prm.tiles_per_item = pl0.tpi1;
        prm.chunks_per_pg = pl0.chunks1;
        prm.n_items = int(np * G * prm.chunks_per_pg);
        int grid = std::min(prm.n_items, sms);
        score_tc_kernel<0><<<grid, kThreads, smem, stream>>>(tq, tk, prm);
        ADAKV_CUDA_TRY(cudaGetLastError());
        // pass 2: pooled scores over (128 - 2 pad)-key output tiles
        prm.pass = 2;
        prm.pad = pad;
        prm.step = kTile - 2 * pad;
        prm.tiles_per_pg = int(ceil_div(s.outside, prm.step));
        prm.tiles_per_item = pl.tpi2;
        prm.chunks_per_pg = pl.chunks2;
        prm.n_items = int(np * G * prm.chunks_per_pg);
        grid = std::min(prm.n_items, sms);
        kfn<<<grid, kThreads, smem, stream>>>(tq, tk, prm);
        ADAKV_CUDA_TRY(cudaGetLastError());
    }
    return ADAKV_OK;
}

}  // namespace adakv_b200
