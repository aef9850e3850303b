// decode_umma.cu -- K4 on the 5th-generation tensor cores (bf16, d == 128, g <= 8).
//
// Same contract as decode_tc.cu (attention_weights + row_times(a, V) per head over the
// retained cache, attention.hpp:169-196 / report.hpp:133-144, append_kv fused), different
// machine mapping: each CTA of a (problem, KV group) cluster takes a contiguous key range and
// turns it into T <= 31 tiles of 128 keys.
//   phase A  S^T[key, head] = K_tile . Q^T     tcgen05.mma, M = 128 keys, N = 16 (heads,
//            zero-padded), K = 128 = d; one TMEM accumulator per tile (16 columns each);
//   softmax  the 128 threads (thread = key row = TMEM lane) take the CTA-wide max per head
//            over every tile, then P = exp2(S c - M) is written as the bf16 B operand;
//   phase B  O^T[d, head] += V_tile^T . P^T     tcgen05.mma with V read MN-major straight
//            from its TMA tile (M = 128 = d, K = 128 keys), accumulated in TMEM.
// The CTA therefore produces ONE split-K partial (max, sum, O) -- no per-warp partials and
// no CTA-level merge -- which goes to the owning ranks with DSMEM st.async as in decode_tc.
// K and V tiles stream through a 4-slot TMA ring; the first four loads are issued before
// griddepcontrol.wait (programmatic dependent launch), exactly like decode_tc.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <mutex>
#include <utility>

#include <cooperative_groups.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace cg = cooperative_groups;

namespace adakv_b200 {

unsigned long long* dbg_buf();

namespace {

using namespace ptx;

constexpr int kT = 128;            // keys per tile
constexpr int kThreadsU = 128;     // 4 warps; warp w reads TMEM lanes 32w .. 32w + 31
constexpr int kNS = 4;             // TMA tile slots
constexpr int kHalfU = 128 * 128;  // one [128 rows][64 bf16] half tile, 128B-swizzled
constexpr int kMaxTU = 31;         // S tiles held in TMEM (16 columns each) besides O
constexpr int kMaxCSU = 16;
constexpr int kOCol = 0;           // TMEM columns: O^T at 0..15, S^T of tile t at 16 + 16 t

__host__ __device__ constexpr int chunk_floats_u(int cs) { return 16 + ((128 + cs - 1) / cs) * 8; }

struct USmem {
    uint8_t slot[kNS][2][kHalfU];        // K or V tiles: [half of d][128 rows][128 B]
    uint8_t qb[2][16 * 128];             // Q^T operand: [half of d][16 heads][128 B], K-major SW128
    uint8_t pb[2][2][16 * 128];          // P^T operand, double buffered: [buf][64-key block][16 heads][128 B]
    uint64_t full[kNS], freeb[kNS];      // slot loaded / the MMA reading the slot finished
    uint64_t s_done, o_done, pv_done[2];
    uint64_t rbar;                       // combine receive barrier (st.async complete_tx)
    uint32_t tmem;
    float red[4][16];                    // cross-warp reductions (max, then sum)
    alignas(16) float recv[kMaxCSU * 16 + 1024 + kMaxCSU * 8];
};
constexpr size_t kUSmemBytes = sizeof(USmem) + 1024;

__device__ __forceinline__ void sts128u(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void sts16u(uint32_t addr, uint16_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}
__device__ __forceinline__ uint32_t mapa_u(uint32_t addr, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_v2u(uint32_t addr, float x, float y, uint32_t bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1,%2}, [%3];" ::"r"(addr),
                 "f"(x), "f"(y), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void st_async_v4u(uint32_t addr, float4 v, uint32_t bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1,%2,%3,%4}, [%5];" ::"r"(addr),
                 "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ float ex2u(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// byte offset of 16-byte chunk c (0..15) of row r inside a [half][128 rows][128 B] SW128 tile
__device__ __forceinline__ uint32_t tile_off(int r, int c) {
    return uint32_t((c >> 3) * kHalfU + r * 128 + ((((c & 7) ^ (r & 7))) << 4));
}

// kind::f16, BF16 A/B, F32 D, A MN-major (bit 15), B K-major
__host__ __device__ constexpr uint32_t idesc_bf16_f32_amn(uint32_t M, uint32_t N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

template <int CS>
__global__ void __launch_bounds__(kThreadsU, 1)
decode_umma_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                   const __nv_bfloat16* __restrict__ q, __nv_bfloat16* __restrict__ k_cache,
                   __nv_bfloat16* __restrict__ v_cache, const int32_t* __restrict__ seg_start,
                   int32_t* __restrict__ seqlens, const __nv_bfloat16* __restrict__ k_new,
                   const __nv_bfloat16* __restrict__ v_new, __nv_bfloat16* __restrict__ out, int H, int G,
                   float scale_log2, unsigned long long* __restrict__ dbg) {
    constexpr int d = 128;
    auto stamp = [&](int k) {  // (debug) per-CTA phase timestamps, 32 slots per CTA
        if (dbg && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            dbg[blockIdx.x * 32 + k] = t;
        }
    };
    stamp(0);
    extern __shared__ uint8_t smem_raw[];
    USmem& S = *reinterpret_cast<USmem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = int(cluster.block_rank());
    const int pg = blockIdx.x / CS;
    const int p = pg / G, g = pg % G;
    const int gs = H / G;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool append = k_new != nullptr;

    const int L_old = __ldcg(seqlens + pg);
    const int base = seg_start[pg];
    const int L = L_old + (append ? 1 : 0);
    const int k_lo = int((int64_t(L) * rank) / CS), k_hi = int((int64_t(L) * (rank + 1)) / CS);
    const int nk = k_hi - k_lo;
    const int T = (nk + kT - 1) / kT;  // host guarantees T <= kMaxTU
    const int np = (gs + 1) >> 1;      // head pairs in the combine
    constexpr int chunk = chunk_floats_u(CS);
    const int col_lo = (d * rank) / CS, ncols = (d * (rank + 1)) / CS - col_lo;

    // loads: item i < T is K tile i, item T + i is V tile i; item i lives in slot i % kNS
    auto issue = [&](int i) {
        const int sl = i % kNS;
        const bool isk = i < T;
        const int row = base + k_lo + (isk ? i : i - T) * kT;
        mbar_arrive_expect_tx(&S.full[sl], 2 * kHalfU);
        const uint64_t pol = policy_evict_first();
        tma_load_3d(S.slot[sl][0], isk ? &tm_k : &tm_v, 0, row, 0, &S.full[sl], pol);
        tma_load_3d(S.slot[sl][1], isk ? &tm_k : &tm_v, 64, row, 0, &S.full[sl], pol);
    };
    if (tid == 0) {
        for (int i = 0; i < kNS; ++i) {
            mbar_init(&S.full[i], 1);
            mbar_init(&S.freeb[i], 1);
        }
        mbar_init(&S.s_done, 1);
        mbar_init(&S.o_done, 1);
        mbar_init(&S.pv_done[0], 1);
        mbar_init(&S.pv_done[1], 1);
        mbar_init(&S.rbar, 1);
        mbar_fence_init();
        mbar_arrive_expect_tx(&S.rbar, uint32_t(CS * np * (16 + 8 * ncols)));
        for (int i = 0; i < (2 * T < kNS ? 2 * T : kNS); ++i) issue(i);
    }
    if (warp == 1) tmem_alloc<512>(&S.tmem);
    // P^T rows of padded heads stay zero
    for (int i = tid; i < int(sizeof(S.pb) / 16); i += kThreadsU)
        sts128u(smem_u32(&S.pb[0][0][0]) + 16 * i, make_uint4(0, 0, 0, 0));
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem;
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    stamp(1);

    // Q^T operand (produced upstream): 16 rows (heads, zero beyond g) x 16 chunks of 16 B
    for (int i = tid; i < 256; i += kThreadsU) {
        const int n = i >> 4, c = i & 15;
        uint4 val = make_uint4(0, 0, 0, 0);
        if (n < gs) val = reinterpret_cast<const uint4*>(q + (int64_t(p) * H + g * gs + n) * d)[c];
        sts128u(smem_u32(S.qb[c >> 3]) + uint32_t(n * 128 + ((((c & 7) ^ (n & 7))) << 4)), val);
    }
    // the appended row (if this CTA holds it): tile / row, and this thread's 16-byte chunk of it
    const int rel_new = (append && L_old >= k_lo && L_old < k_hi) ? L_old - k_lo : -1;
    uint4 new_k = make_uint4(0, 0, 0, 0), new_v = make_uint4(0, 0, 0, 0);
    if (rel_new >= 0 && tid < 16) {
        new_k = reinterpret_cast<const uint4*>(k_new + int64_t(pg) * d)[tid];
        new_v = reinterpret_cast<const uint4*>(v_new + int64_t(pg) * d)[tid];
    }
    fence_async_smem();
    __syncthreads();
    stamp(2);

    // ---- phase A: S^T tiles
    constexpr uint32_t idS = idesc_bf16_f32(128, 16);
    for (int t = 0; t < T; ++t) {
        const int sl = t % kNS;
        mbar_wait(&S.full[sl], uint32_t((t / kNS) & 1));
        if (rel_new >= 0 && rel_new / kT == t && tid < 16) {
            sts128u(smem_u32(S.slot[sl][0]) + tile_off(rel_new % kT, tid), new_k);
            fence_async_smem();
        }
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint32_t off = (kk & 3) * 32;
                mma_bf16(tmem + 16 + 16 * t, desc_kmajor_sw128(smem_u32(S.slot[sl][kk >> 2]) + off),
                         desc_kmajor_sw128(smem_u32(S.qb[kk >> 2]) + off), idS, kk > 0 ? 1u : 0u);
            }
            mma_commit(&S.freeb[sl]);
            if (t == T - 1) mma_commit(&S.s_done);
            if (t + kNS < 2 * T) {
                mbar_wait(&S.freeb[sl], uint32_t((t / kNS) & 1));
                issue(t + kNS);
            }
        }
    }
    // ---- softmax statistics: CTA-wide max per head (log2 units)
    const int r = tid;  // this thread's key row within every tile (TMEM lane)
    float Mh[8];
#pragma unroll
    for (int h = 0; h < 8; ++h) Mh[h] = -INFINITY;
    if (T > 0) {
        mbar_wait(&S.s_done, 0);
        stamp(3);
        tc_fence_after();
        for (int t = 0; t < T; ++t) {
            float sv[16];
            tmem_ld_x16<0>(tmem + 16 + 16 * t + (uint32_t(warp * 32) << 16), sv);
            tmem_ld_wait();
            if (t * kT + r < nk) {
#pragma unroll
                for (int h = 0; h < 8; ++h) Mh[h] = fmaxf(Mh[h], sv[h] * scale_log2);
            }
        }
    }
#pragma unroll
    for (int h = 0; h < 8; ++h) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) Mh[h] = fmaxf(Mh[h], __shfl_xor_sync(0xffffffffu, Mh[h], o));
    }
    if (lane == 0)
#pragma unroll
        for (int h = 0; h < 8; ++h) S.red[warp][h] = Mh[h];
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 8; ++h) Mh[h] = fmaxf(fmaxf(S.red[0][h], S.red[1][h]), fmaxf(S.red[2][h], S.red[3][h]));

    stamp(4);
    // ---- phase B: P^T and O^T += V^T P^T per tile
    constexpr uint32_t idO = idesc_bf16_f32_amn(128, 16);
    float lh[8];
#pragma unroll
    for (int h = 0; h < 8; ++h) lh[h] = 0.f;
    for (int t = 0; t < T; ++t) {
        const int item = T + t, sl = item % kNS, b = t & 1;
        float sv[16];
        tmem_ld_x16<0>(tmem + 16 + 16 * t + (uint32_t(warp * 32) << 16), sv);
        tmem_ld_wait();
        const bool valid = t * kT + r < nk;
        if (t >= 2) mbar_wait(&S.pv_done[b], uint32_t(((t - 2) >> 1) & 1));  // P buffer free again
        const uint32_t pbase = smem_u32(S.pb[b][r >> 6]);
        const int kk = r & 63;
#pragma unroll
        for (int h = 0; h < 8; ++h) {
            if (h < gs) {
                const float pv = (valid && Mh[h] != -INFINITY) ? ex2u(fmaf(sv[h], scale_log2, -Mh[h])) : 0.f;
                lh[h] += pv;
                const __nv_bfloat16 pb16 = __float2bfloat16_rn(pv);
                sts16u(pbase + uint32_t(h * 128 + (((kk >> 3) ^ (h & 7)) << 4) + (kk & 7) * 2),
                       *reinterpret_cast<const uint16_t*>(&pb16));
            }
        }
        // V rows past the segment end must be finite (they meet p = 0); the appended row
        mbar_wait(&S.full[sl], uint32_t((item / kNS) & 1));
        const int grow = k_lo + t * kT + r;  // key index of this row within the segment
        if (grow >= L) {
#pragma unroll
            for (int c = 0; c < 16; ++c) sts128u(smem_u32(S.slot[sl][0]) + tile_off(r, c), make_uint4(0, 0, 0, 0));
        }
        if (rel_new >= 0 && rel_new / kT == t && tid < 16)
            sts128u(smem_u32(S.slot[sl][0]) + tile_off(rel_new % kT, tid), new_v);
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                // A = V^T (M = d, K = keys), MN-major: d halves 16 KB apart, 8-key atoms 1 KB apart
                const uint64_t ad = desc_mnmajor_sw128(smem_u32(S.slot[sl][0]) + ks * 2048, kHalfU, 1024);
                const uint64_t bd = desc_kmajor_sw128(smem_u32(S.pb[b][ks >> 2]) + (ks & 3) * 32);
                mma_bf16(tmem + kOCol, ad, bd, idO, (t > 0 || ks > 0) ? 1u : 0u);
            }
            mma_commit(&S.pv_done[b]);
            mma_commit(&S.freeb[sl]);
            if (t == T - 1) mma_commit(&S.o_done);
            if (item + kNS < 2 * T) {
                mbar_wait(&S.freeb[sl], uint32_t((item / kNS) & 1));
                issue(item + kNS);
            }
        }
    }
    // ---- the CTA partial: O^T row d = tid, (max, sum) per head
    float ov[16];
#pragma unroll
    for (int h = 0; h < 16; ++h) ov[h] = 0.f;
    stamp(5);
    if (T > 0) {
        mbar_wait(&S.o_done, 0);
        stamp(6);
        tc_fence_after();
        tmem_ld_x16<0>(tmem + kOCol + (uint32_t(warp * 32) << 16), ov);
        tmem_ld_wait();
    }
#pragma unroll
    for (int h = 0; h < 8; ++h) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lh[h] += __shfl_xor_sync(0xffffffffu, lh[h], o);
    }
    __syncthreads();  // S.red reused
    if (lane == 0)
#pragma unroll
        for (int h = 0; h < 8; ++h) S.red[warp][h] = lh[h];
    tc_fence_before();
    __syncthreads();
    float Lsum[8];
#pragma unroll
    for (int h = 0; h < 8; ++h) Lsum[h] = (S.red[0][h] + S.red[1][h]) + (S.red[2][h] + S.red[3][h]);
    if (warp == 1) tmem_dealloc<512>(tmem);
    // ---- push to the rank that finishes column c = tid (DSMEM st.async)
    {
        const int c = tid;
        const int owner = ((c + 1) * CS - 1) / d, cl = c - (d * owner) / CS;
        const uint32_t dst = smem_u32(S.recv + rank * chunk), bar = mapa_u(smem_u32(&S.rbar), owner);
#pragma unroll
        for (int hp = 0; hp < 4; ++hp) {
            if (hp >= np) break;
            st_async_v2u(mapa_u(dst + 4u * uint32_t(16 + cl * 8 + 2 * hp), owner), ov[2 * hp], ov[2 * hp + 1], bar);
            if (cl == 0)
                st_async_v4u(mapa_u(dst + 4u * uint32_t(4 * hp), owner),
                             make_float4(Mh[2 * hp], Lsum[2 * hp], Mh[2 * hp + 1], Lsum[2 * hp + 1]), bar);
        }
    }
    stamp(7);
    mbar_wait(&S.rbar, 0);
    stamp(8);
    // ---- this rank's columns: merge the CS chunks
    for (int t = tid; t < ncols * gs; t += kThreadsU) {
        const int cl = t / gs, h = t % gs;
        float M = -INFINITY;
#pragma unroll
        for (int rr = 0; rr < CS; ++rr) M = fmaxf(M, S.recv[rr * chunk + 2 * h]);
        float Ls = 0.f, Os = 0.f;
#pragma unroll
        for (int rr = 0; rr < CS; ++rr) {
            const float* ch = S.recv + rr * chunk;
            const float mr = ch[2 * h];
            const float f = mr == -INFINITY ? 0.f : ex2u(mr - M);
            Ls += ch[2 * h + 1] * f;
            Os += ch[16 + cl * 8 + h] * f;
        }
        out[(int64_t(p) * H + g * gs + h) * d + col_lo + cl] = __float2bfloat16_rn(Os / Ls);
    }
    if (rank == 0 && append) {
        if (tid < 32) {
            const __nv_bfloat16* kn = k_new + int64_t(pg) * d;
            const __nv_bfloat16* vn = v_new + int64_t(pg) * d;
            reinterpret_cast<uint2*>(k_cache + (int64_t(base) + L_old) * d)[tid] = reinterpret_cast<const uint2*>(kn)[tid];
            reinterpret_cast<uint2*>(v_cache + (int64_t(base) + L_old) * d)[tid] = reinterpret_cast<const uint2*>(vn)[tid];
        }
        if (tid == 0) seqlens[pg] = L;
    }
    stamp(9);
}

// 3-D view [1][rows][128] of a cache plane with a {64, 128, 1} box (one half of a 128-key tile)
adakv_status make_plane_map(CUtensorMap* m, const void* plane, int64_t rows) {
    EncodeFn enc = get_encode();
    if (!enc) return fail(ADAKV_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[3] = {128, cuuint64_t(rows), 1};
    const cuuint64_t strides[2] = {256, cuuint64_t(rows) * 256};
    const cuuint32_t box[3] = {64, 128, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(plane), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(ADAKV_CUDA_ERROR, "cuTensorMapEncodeTiled failed (decode plane)");
    return ADAKV_OK;
}

using UKernel = decltype(&decode_umma_kernel<1>);
template <int... CS>
UKernel ukernel_impl(int64_t cs, std::integer_sequence<int, CS...>) {
    UKernel k = nullptr;
    ((cs == CS + 1 ? (k = decode_umma_kernel<CS + 1>, 0) : 0), ...);
    return k;
}
UKernel ukernel_for(int64_t cs) { return ukernel_impl(cs, std::make_integer_sequence<int, kMaxCSU>{}); }

}  // namespace

// Opt-in (ADAKV_DECODE_UMMA=1 or adakv_debug_decode_umma(1)): correct, but on Llama-3.1-8B
// decode it measures 6.97 us per step-layer against 4.78 for decode_tc -- with N = 16 heads
// each tile's S and PV phases cost ~0.5 us of MMA / TMEM / barrier latency (scripts/dec_ts3.py).
static std::atomic<int> g_umma{-1};
bool decode_umma_enabled() {
    int v = g_umma.load();
    if (v < 0) {
        const char* e = std::getenv("ADAKV_DECODE_UMMA");
        v = (e && std::atoi(e) != 0) ? 1 : 0;
        g_umma.store(v);
    }
    return v != 0;
}

// CTAs per cluster: the largest size <= 10 whose clusters are all co-resident
static int64_t umma_cluster(int64_t segs) {
    static std::mutex mu;
    static int64_t c_segs = -1, c_cs = 1;
    static int c_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    if (segs == c_segs && dev == c_dev) return c_cs;
    int64_t best = 1;
    for (int64_t cs = 10; cs >= 2 && best == 1; --cs) {
        cudaFuncSetAttribute(ukernel_for(cs), cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(ukernel_for(cs), cudaFuncAttributeMaxDynamicSharedMemorySize, int(kUSmemBytes));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(segs * cs));
        cfg.blockDim = dim3(kThreadsU);
        cfg.dynamicSmemBytes = kUSmemBytes;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = unsigned(cs);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, ukernel_for(cs), &cfg) == cudaSuccess && n >= segs) best = cs;
        cudaGetLastError();
    }
    c_segs = segs;
    c_cs = best;
    c_dev = dev;
    return best;
}

bool decode_umma_supported(adakv_dtype dt, int64_t P, int64_t H, int64_t G, int64_t d, int64_t max_rows,
                           int64_t cache_rows) {
    if (!(dt == ADAKV_BF16 && d == 128 && G > 0 && H % G == 0 && H / G <= 8 && cache_rows < (int64_t(1) << 31) &&
          get_encode() != nullptr))
        return false;
    const int64_t cs = umma_cluster(P * G);
    return ceil_div(max_rows, cs) <= int64_t(kMaxTU) * kT - 1;
}

adakv_status launch_decode_umma(int64_t P, int64_t H, int64_t G, int32_t scale, const void* q, void* kc, void* vc,
                                int64_t cache_rows, const int32_t* ss, int32_t* sl, const void* kn, const void* vn,
                                void* out, bool overlap_prev, cudaStream_t stream) {
    static std::mutex mu;
    static const void* c_k = nullptr;
    static const void* c_v = nullptr;
    static int64_t c_rows = -1;
    static CUtensorMap c_tk, c_tv;
    CUtensorMap tk, tv;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (kc != c_k || vc != c_v || cache_rows != c_rows) {
            ADAKV_TRY(make_plane_map(&c_tk, kc, cache_rows));
            ADAKV_TRY(make_plane_map(&c_tv, vc, cache_rows));
            c_k = kc;
            c_v = vc;
            c_rows = cache_rows;
        }
        tk = c_tk;
        tv = c_tv;
    }
    const int64_t cs = umma_cluster(P * G);
    ADAKV_CUDA_TRY(cudaFuncSetAttribute(ukernel_for(cs), cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    ADAKV_CUDA_TRY(cudaFuncSetAttribute(ukernel_for(cs), cudaFuncAttributeMaxDynamicSharedMemorySize, int(kUSmemBytes)));
    const float sc = (scale ? 1.0f / sqrtf(128.f) : 1.0f) * 1.4426950408889634f;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(P * G * cs));
    cfg.blockDim = dim3(kThreadsU);
    cfg.dynamicSmemBytes = kUSmemBytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(cs);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = overlap_prev ? 2 : 1;
    ADAKV_CUDA_TRY(cudaLaunchKernelEx(&cfg, ukernel_for(cs), tk, tv, static_cast<const __nv_bfloat16*>(q),
                                      static_cast<__nv_bfloat16*>(kc), static_cast<__nv_bfloat16*>(vc), ss, sl,
                                      static_cast<const __nv_bfloat16*>(kn), static_cast<const __nv_bfloat16*>(vn),
                                      static_cast<__nv_bfloat16*>(out), int(H), int(G), sc, dbg_buf()));
    return ADAKV_OK;
}

}  // namespace adakv_b200

extern "C" int adakv_debug_decode_umma(int enable) {
    const int prev = adakv_b200::decode_umma_enabled() ? 1 : 0;
    adakv_b200::g_umma.store(enable ? 1 : 0);
    return prev;
}
