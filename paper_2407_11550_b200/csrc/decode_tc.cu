// decode_tc.cu -- K4 fast path: split-K varlen flash-decoding for bf16, d == 128,
// g = H/G <= 8 query heads per KV group, on warp-level tensor-core MMA (m16n8k16).
//
// Same contract as decode.cu (attention_weights + row_times(a, V) per head over the
// retained cache, attention.hpp:169-196 / report.hpp:133-144, with append_kv fused).
//
// Per warp, keys are consumed in blocks of 16:
//   S  = Q K^T      two m16n8k16 n8 tiles x 8 k-steps; rows = the g heads (padded to 16);
//   P  = exp2(S*c - m)  online softmax (block max over the 4 lanes of a row);
//   O^T += V^T P^T  eight m16n8k16 m-tiles over d.
// The dot products are invariant to a consistent permutation of d, so Q's and K's
// d-columns are permuted such that each lane's B-fragment words are exactly the
// 16-byte vectors it loads (K rows: lanes of a row read 64 contiguous bytes); V's d
// (the MMA M dimension) is permuted so each lane loads 2 x 16 B of a row (8 lanes cover
// 128 contiguous bytes) and un-permuted when O is written.  The S accumulator fragment
// (row = head, cols = keys 2t, 2t+1) is exactly the P^T B-fragment of the PV MMA, so P
// never leaves registers.  K/V are streamed once from HBM for all g heads.
#include <algorithm>

#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace adakv_b200 {

unsigned long long* dbg_buf();

namespace {

constexpr int kBlk = 16;
constexpr int kMaxSplitsB = 160;   // CTAs per problem (>= SM count)
constexpr int kMaxSegDec = 64;

__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

__device__ __forceinline__ float ex2f(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// d column held by (m-tile i, fragment row r) of the PV MMA
__device__ __forceinline__ int v_col(int i, int r) { return (i < 4 ? 0 : 64) + 8 * (r & 7) + 2 * (i & 3) + (r >> 3); }

// One thread-block cluster of CS CTAs per (problem, KV group): CTA rank r streams blocks
// [nblk r / CS, nblk (r+1) / CS) of the group's 16-row blocks, split again over its 8 warps.
// Warp partials (m, l, O) merge in shared memory; the CS CTA partials merge through
// distributed shared memory (each rank finishes 1/CS of the (head, column) pairs), so the
// split-K combine needs no global round trips, fences or atomics.  Launched with
// programmatic dependent launch: this layer's cache streams in before griddepcontrol.wait,
// q / k_new / v_new (produced upstream) are read after it.
constexpr int kWarpsB = 8;
constexpr int kThreadsB = 32 * kWarpsB;

__global__ void __launch_bounds__(kThreadsB, 1)
decode_tc_kernel(const __nv_bfloat16* __restrict__ q, __nv_bfloat16* __restrict__ k_cache,
                 __nv_bfloat16* __restrict__ v_cache, const int32_t* __restrict__ seg_start,
                 int32_t* __restrict__ seqlens, const __nv_bfloat16* __restrict__ k_new,
                 const __nv_bfloat16* __restrict__ v_new, __nv_bfloat16* __restrict__ out, int H, int G,
                 float scale_log2, unsigned long long* __restrict__ dbg) {
    constexpr int d = 128;
    cg::cluster_group cluster = cg::this_cluster();
    const int CS = int(cluster.num_blocks());
    const int rank = int(cluster.block_rank());
    const int pg = blockIdx.x / CS;
    const int p = pg / G, g = pg % G;
    const int gs = H / G;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const bool append = k_new != nullptr;
    const bool head_ok = gid < gs;
    auto stamp = [&](int k) {
        if (dbg && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            dbg[blockIdx.x * 8 + k] = t;
        }
    };
    stamp(0);

    __shared__ float s_m[kWarpsB][8], s_l[kWarpsB][8];
    __shared__ float s_o[kWarpsB][8][d];
    __shared__ float c_m[8], c_l[8];
    __shared__ float c_o[8][d];

    // this layer's own cache state (written by its previous decode step, long complete)
    const int L_old = __ldcg(seqlens + pg);
    const int L = L_old + (append ? 1 : 0);
    const int64_t base = seg_start[pg];
    const __nv_bfloat16* kn = append ? k_new + int64_t(pg) * d : nullptr;
    const __nv_bfloat16* vn = append ? v_new + int64_t(pg) * d : nullptr;
    const int nblk = (L + kBlk - 1) / kBlk;
    const int c_lo = (nblk * rank) / CS, c_hi = (nblk * (rank + 1)) / CS;
    const int w_lo = c_lo + ((c_hi - c_lo) * warp) / kWarpsB, w_hi = c_lo + ((c_hi - c_lo) * (warp + 1)) / kWarpsB;

    // K/V loads of one 16-row block: K rows blk+gid, blk+8+gid (4 x 16 B each), V rows
    // blk + {2t, 2t+1, 2t+8, 2t+9} (2 x 16 B each).  The appended row (r == L_old) comes from
    // k_new / v_new, produced upstream, so it is only read when `fresh`.
    auto load_block = [&](int blk, bool fresh, uint4 (&kv)[2][4], uint4 (&vv)[4][2]) {
#pragma unroll
        for (int tl = 0; tl < 2; ++tl) {
            const int r = blk + tl * 8 + gid;
            const bool isnew = append && r == L_old;
            const bool ok = r < L && (!isnew || fresh);
            const __nv_bfloat16* row = isnew ? kn : k_cache + (base + r) * d;
#pragma unroll
            for (int i = 0; i < 4; ++i)
                kv[tl][i] = ok ? __ldg(reinterpret_cast<const uint4*>(row) + i * 4 + tig) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int jv = 0; jv < 4; ++jv) {
            const int r = blk + 2 * tig + (jv & 1) + (jv >> 1) * 8;
            const bool isnew = append && r == L_old;
            const bool ok = r < L && (!isnew || fresh);
            const __nv_bfloat16* row = isnew ? vn : v_cache + (base + r) * d;
            vv[jv][0] = ok ? __ldg(reinterpret_cast<const uint4*>(row) + gid) : make_uint4(0, 0, 0, 0);
            vv[jv][1] = ok ? __ldg(reinterpret_cast<const uint4*>(row) + 8 + gid) : make_uint4(0, 0, 0, 0);
        }
    };
    uint4 pkv[2][4], pvv[4][2];
    const bool pre = w_lo < w_hi;
    if (pre) load_block(w_lo * kBlk, false, pkv, pvv);
    stamp(1);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    stamp(2);
    if (pre && append && L_old >= w_lo * kBlk && L_old < (w_lo + 1) * kBlk)
        load_block(w_lo * kBlk, true, pkv, pvv);  // the block holding the new row

    // Q A-fragments for this group's heads (rows 8..15 padding)
    uint32_t qa0[8], qa2[8];
    {
        uint4 qv[4] = {};
        if (head_ok) {
            const uint4* qrow = reinterpret_cast<const uint4*>(q + (int64_t(p) * H + g * gs + gid) * d);
#pragma unroll
            for (int i = 0; i < 4; ++i) qv[i] = qrow[i * 4 + tig];
        }
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const uint4 w = qv[s >> 1];
            qa0[s] = (s & 1) ? w.z : w.x;
            qa2[s] = (s & 1) ? w.w : w.y;
        }
    }
    float m_run = -INFINITY, l_run = 0.f;
    float acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;

    for (int bi = w_lo; bi < w_hi; ++bi) {
        const int blk = bi * kBlk;
        uint4 kv[2][4];
        uint4 vv[4][2];
        if (bi == w_lo) {
#pragma unroll
            for (int tl = 0; tl < 2; ++tl)
#pragma unroll
                for (int i = 0; i < 4; ++i) kv[tl][i] = pkv[tl][i];
#pragma unroll
            for (int jv = 0; jv < 4; ++jv) {
                vv[jv][0] = pvv[jv][0];
                vv[jv][1] = pvv[jv][1];
            }
        } else {
            load_block(blk, true, kv, vv);
        }
        float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const uint4 w0v = kv[0][s >> 1], w1v = kv[1][s >> 1];
            mma16816(s0, qa0[s], 0u, qa2[s], 0u, (s & 1) ? w0v.z : w0v.x, (s & 1) ? w0v.w : w0v.y);
            mma16816(s1, qa0[s], 0u, qa2[s], 0u, (s & 1) ? w1v.z : w1v.x, (s & 1) ? w1v.w : w1v.y);
        }
        const int kb = blk + 2 * tig;
        const float x0 = kb < L ? s0[0] : -INFINITY, x1 = kb + 1 < L ? s0[1] : -INFINITY;
        const float x2 = kb + 8 < L ? s1[0] : -INFINITY, x3 = kb + 9 < L ? s1[1] : -INFINITY;
        float bm = fmaxf(fmaxf(x0, x1), fmaxf(x2, x3));
        bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 1));
        bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 2));
        const float m_new = fmaxf(m_run, bm * scale_log2);
        const float corr = ex2f(m_run - m_new);
        float p0 = ex2f(fmaf(x0, scale_log2, -m_new)), p1 = ex2f(fmaf(x1, scale_log2, -m_new));
        float p2 = ex2f(fmaf(x2, scale_log2, -m_new)), p3 = ex2f(fmaf(x3, scale_log2, -m_new));
        if (!head_ok) p0 = p1 = p2 = p3 = 0.f;
        l_run = l_run * corr + ((p0 + p1) + (p2 + p3));
        m_run = m_new;
        if (__any_sync(0xffffffffu, head_ok && corr != 1.f)) {
            const float ca = __shfl_sync(0xffffffffu, corr, 8 * tig);
            const float cb = __shfl_sync(0xffffffffu, corr, 8 * tig + 4);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                acc[i][0] *= ca;
                acc[i][1] *= cb;
                acc[i][2] *= ca;
                acc[i][3] *= cb;
            }
        }
        const uint32_t b0 = pack_bf16(p0, p1), b1 = pack_bf16(p2, p3);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int h = i >> 2, wd = i & 3;
            const uint32_t* r0w = reinterpret_cast<const uint32_t*>(&vv[0][h]);
            const uint32_t* r1w = reinterpret_cast<const uint32_t*>(&vv[1][h]);
            const uint32_t* r8w = reinterpret_cast<const uint32_t*>(&vv[2][h]);
            const uint32_t* r9w = reinterpret_cast<const uint32_t*>(&vv[3][h]);
            mma16816(acc[i], __byte_perm(r0w[wd], r1w[wd], 0x5410), __byte_perm(r0w[wd], r1w[wd], 0x7632),
                     __byte_perm(r8w[wd], r9w[wd], 0x5410), __byte_perm(r8w[wd], r9w[wd], 0x7632), b0, b1);
        }
    }
    stamp(3);
    // ---- warps -> CTA partial (shared memory)
    {
        float lsum = l_run + __shfl_xor_sync(0xffffffffu, l_run, 1);
        lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
        if (tig == 0) {
            s_m[warp][gid] = m_run;
            s_l[warp][gid] = lsum;
        }
        const int ha = 2 * tig, hb = 2 * tig + 1;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int c0 = v_col(i, gid), c1 = v_col(i, gid + 8);
            s_o[warp][ha][c0] = acc[i][0];
            s_o[warp][hb][c0] = acc[i][1];
            s_o[warp][ha][c1] = acc[i][2];
            s_o[warp][hb][c1] = acc[i][3];
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < gs * d; i += kThreadsB) {
        const int h = i / d, c = i % d;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kWarpsB; ++w) M = fmaxf(M, s_m[w][h]);
        float Ls = 0.f, Os = 0.f;
#pragma unroll
        for (int w = 0; w < kWarpsB; ++w) {
            if (s_m[w][h] == -INFINITY) continue;
            const float f = ex2f(s_m[w][h] - M);
            Ls += s_l[w][h] * f;
            Os += s_o[w][h][c] * f;
        }
        c_o[h][c] = Os;
        if (c == 0) {
            c_m[h] = M;
            c_l[h] = Ls;
        }
    }
    cluster.sync();
    stamp(4);
    // ---- CTA partials -> output through DSMEM; rank r finishes pairs [512 r / CS, 512 (r+1) / CS)
    {
        const int npairs = gs * d;
        const int i0 = (npairs * rank) / CS, i1 = (npairs * (rank + 1)) / CS;
        for (int i = i0 + int(threadIdx.x); i < i1; i += kThreadsB) {
            const int h = i / d, c = i % d;
            float M = -INFINITY;
            for (int r = 0; r < CS; ++r) M = fmaxf(M, *cluster.map_shared_rank(&c_m[h], r));
            float Ls = 0.f, Os = 0.f;
            for (int r = 0; r < CS; ++r) {
                const float mr = *cluster.map_shared_rank(&c_m[h], r);
                if (mr == -INFINITY) continue;
                const float f = ex2f(mr - M);
                Ls += *cluster.map_shared_rank(&c_l[h], r) * f;
                Os += *cluster.map_shared_rank(&c_o[h][c], r) * f;
            }
            out[(int64_t(p) * H + g * gs + h) * d + c] = __float2bfloat16_rn(Os / Ls);
        }
    }
    if (rank == 0) {
        if (append && threadIdx.x < 32) {  // K5 append: the new row lands after the window rows
            reinterpret_cast<uint2*>(k_cache + (base + L_old) * d)[threadIdx.x] = reinterpret_cast<const uint2*>(kn)[threadIdx.x];
            reinterpret_cast<uint2*>(v_cache + (base + L_old) * d)[threadIdx.x] = reinterpret_cast<const uint2*>(vn)[threadIdx.x];
        }
    }
    cluster.sync();  // every rank has read its peers' partials and seqlens
    if (rank == 0 && threadIdx.x == 0 && append) seqlens[pg] = L;
    stamp(7);
}

}  // namespace

// debug: per-CTA phase timestamps (ADAKV_DECODE_DEBUG=1), exported for scripts/dec_ts.py
static unsigned long long* g_dbg = nullptr;
unsigned long long* dbg_buf() { return g_dbg; }
extern "C" void adakv_debug_set_decode_timestamps(void* buf) { g_dbg = static_cast<unsigned long long*>(buf); }

bool decode_tc_supported(adakv_dtype dt, int64_t H, int64_t G, int64_t d, int64_t /*nsplit*/) {
    return dt == ADAKV_BF16 && d == 128 && G > 0 && H % G == 0 && H / G <= 8;
}

// CTAs per cluster (one cluster per (problem, group)): the largest power of two <= 16 for
// which every cluster of the launch is co-resident (cudaOccupancyMaxActiveClusters), so no
// cluster waits for another to drain.
int64_t decode_tc_cluster(int64_t P, int64_t G) {
    static int64_t cached_segs = -1, cached_cs = 1;
    const int64_t segs = std::max<int64_t>(1, P * G);
    if (segs == cached_segs) return cached_cs;
    cudaFuncSetAttribute(decode_tc_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int64_t best = 1;
    for (int64_t cs = 16; cs >= 2; cs /= 2) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(segs * cs));
        cfg.blockDim = dim3(kThreadsB);
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = unsigned(cs);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, decode_tc_kernel, &cfg) == cudaSuccess && n >= segs) {
            best = cs;
            break;
        }
        cudaGetLastError();
    }
    cached_segs = segs;
    cached_cs = best;
    return best;
}

size_t decode_tc_workspace(int64_t, int64_t, int64_t, int64_t) { return 256; }

extern "C" int adakv_debug_decode_cluster(int64_t P, int64_t G) { return int(decode_tc_cluster(P, G)); }

adakv_status launch_decode_tc(int64_t P, int64_t H, int64_t G, int32_t scale, const void* q, void* kc, void* vc,
                              const int32_t* ss, int32_t* sl, const void* kn, const void* vn, void* out, void*,
                              cudaStream_t stream) {
    const float sc = (scale ? 1.0f / sqrtf(128.f) : 1.0f) * 1.4426950408889634f;
    const int64_t cs = decode_tc_cluster(P, G);
    static bool attr_set = false;
    if (!attr_set) {
        ADAKV_CUDA_TRY(cudaFuncSetAttribute(decode_tc_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        attr_set = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(P * G * cs));
    cfg.blockDim = dim3(kThreadsB);
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(cs);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    ADAKV_CUDA_TRY(cudaLaunchKernelEx(&cfg, decode_tc_kernel, static_cast<const __nv_bfloat16*>(q),
                                      static_cast<__nv_bfloat16*>(kc), static_cast<__nv_bfloat16*>(vc), ss, sl,
                                      static_cast<const __nv_bfloat16*>(kn), static_cast<const __nv_bfloat16*>(vn),
                                      static_cast<__nv_bfloat16*>(out), int(H), int(G), sc, dbg_buf()));
    return ADAKV_OK;
}

}  // namespace adakv_b200
