// score_window_tc.cu -- K1 on the 5th-generation tensor cores (bf16, d == 128, m == 32,
// g*m <= 128): observation-window scoring in two persistent passes.
//
// Reference semantics (file:line list in score_window.cu): per KV group, the g*m window
// rows (g heads x m rows) are softmaxed over the OUTSIDE keys, max-pooled along keys
// (k odd, stride 1, padded cells excluded), averaged over rows (/m) and heads (/g).
//
// B200 mapping.  The g*m <= 128 query rows of a KV group are one UMMA M=128 tile; each
// 128-key K tile is the N=128 operand; d = 128 is the K extent (8 MMAs of K=16).  One CTA
// per SM, persistent over balanced (group, key-chunk) items, 18 warps:
//   warp 0      TMA producer: the group's Q tile and a 3-stage ring of K tiles (128B-
//               swizzled [128 x 64] halves; 3-D tensor maps zero-fill rows outside a group);
//   warp 1      TMEM owner + single-thread tcgen05.mma issuer;
//   warps 2..17 epilogue, four warps per scheduler: warp (quarter q, group c) owns TMEM lanes
//               32q..32q+31 (= window rows, i.e. head q since m == 32) and columns 32c..32c+31.
// Pass 1 (row statistics): online max / sum of exp2 of the fp32 logits; per item a
//   partial (max, sum) per (row, column group); the last CTA of a group (atomic ticket)
//   folds them into Lw_r = M_r + log2(S_r * m).
// Pass 2 (scores): tiles advance by 128 - 2*pad keys so each output key's pooling halo is
//   inside the tile; pooling is done on LOGITS in registers (exp2 monotone), then
//   E = exp2(pool*c - Lw_r + 16) = 2^16 * pooled_prob / m is written as fp16 into an
//   MN-major shared tile and the per-head row sums are a second tcgen05 MMA:
//   D2[key][head] = E^T[key][row] * Hd[row][head] (Hd = head indicator), fp32 accumulate in
//   TMEM.  Scores = D2 * 2^-16, group score = sum over heads / g.
// The two passes run over ALL problems of a call (one pass-1 launch, one pass-2 launch).
// Slicing the call into L2-sized runs of groups (so pass 2 would re-read K from L2) was
// measured and dropped: ncu with --cache-control none shows pass 2 reading its whole slice from
// DRAM even at 42 MB slices (L2 hit rate 28%), and every slice boundary costs a grid tail --
// 32 layers of config 2 take 62 / 44 / 39 / 30 us per layer at 24 / 48 / 64 MB / unsliced
// (scripts/score_l2.sh).  ADAKV_SCORE_SLICE_MB still caps a slice for such experiments.
#include <cuda.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace adakv_b200 {

namespace {

using namespace ptx;

constexpr int kEpiWarps = 16;  // 4 per scheduler; warp = (lane quarter, 32-column group)
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kStages = 3;
constexpr int kTile = 128;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kD2Col = 256;
constexpr uint32_t kHalfBytes = 128 * 128;        // [128 rows][64 bf16]
constexpr uint32_t kTileBytes = 2 * kHalfBytes;   // a [128 x 128] bf16 tile
constexpr uint32_t kA2Bytes = 128 * 128 * 2;      // E^T tile, fp16
constexpr float kEScaleLog2 = 16.f;               // E carries a 2^16 scale (fp16 range)
#ifndef ADAKV_PASS2_POLY
#define ADAKV_PASS2_POLY 0
#endif
#ifndef ADAKV_PASS1_POLY
#define ADAKV_PASS1_POLY 2
#endif
constexpr int kPass1Poly = ADAKV_PASS1_POLY;      // pass-1 exp2 split (see exp2_mixed)
constexpr int kPass2Poly = ADAKV_PASS2_POLY;      // pass-2 exp2 split (see exp2_mixed)

struct __align__(1024) Smem {
    uint8_t q[2][kHalfBytes];
    uint8_t k[kStages][2][kHalfBytes];
    uint8_t a2[2][kA2Bytes];
    uint8_t b2[2][16 * 128];
    uint64_t full[kStages], empty[kStages];
    uint64_t q_full, q_empty;
    uint64_t acc_full[2], acc_empty[2];
    uint64_t e_full[2], e_empty[2];
    uint64_t d2_full[2], d2_empty[2];
    uint32_t tmem_base;
    uint32_t is_last;
};


struct TcParams {
    int pass;
    // a group of g*m > 128 window rows (Llama-70B: 8 x 32) is scored as vsplit UMMA tiles of
    // gs = g / vsplit heads each over the same K ("virtual groups": pg counts them); their
    // group-score halves are added into the zeroed output (two addends: order-independent)
    int G, H, gs, vsplit, m, n_o, step, pad;
    int tiles_per_pg, tiles_per_item, chunks_per_pg, n_items;
    int pg_base;
    int debug;  // (experiments) 1: pass 1 only; 4/8/16: skip ticket / fences / fold; 64: MUFU-only exp2 in pass 1
    float scale_log2;
    float log2_m;
    float inv_g;
    float* partial;      // pass 1: [pg][chunk][column group][128][2]
    float* final_stats;  // [pg][128][2]: (M_r, Lw_r)
    unsigned* tickets;   // [pg]
    float* head_scores;  // [P][H][n_o] or null
    float* group_scores; // [P][G][n_o]
    long long* dbg;      // (debug) per-CTA role wait counters, 16 per CTA per pass, or null
    uint32_t* err;       // error word (ERR_NONFINITE) or null
};

// ------------------------------------------------------------------ epilogue helpers
// exp2 of x[off .. off+count) in place; of every 8 elements, POLY go through the FMA-pipe
// polynomial (exp2_poly2), the rest through MUFU.EX2.
template <int N, int POLY>
__device__ __forceinline__ void exp2_mixed(float (&x)[N], int count) {
    static_assert(POLY % 2 == 0 && POLY <= 8, "pairs");
#pragma unroll
    for (int j = 0; j < N; j += 8) {
        if (j >= count) break;
#pragma unroll
        for (int u = 0; u < 8 - POLY; ++u)
            if (j + u < N && j + u < count) x[j + u] = ex2(x[j + u]);
#pragma unroll
        for (int u = 8 - POLY; u < 8; u += 2) {
            if (j + u + 1 < N && j + u + 1 < count) exp2_poly2(x[j + u], x[j + u + 1]);
            else if (j + u < N && j + u < count) x[j + u] = ex2(x[j + u]);
        }
    }
}

// v[c] = v[c] * sl - m for c < N, two columns per packed FFMA2
template <int N, int NV>
__device__ __forceinline__ void scale_shift2(float (&v)[NV], float sl, float m) {
    static_assert(N % 2 == 0 && N <= NV, "pairs");
    const uint64_t s2 = pk(sl, sl), m2 = pk(-m, -m);
#pragma unroll
    for (int c = 0; c < N; c += 2) upk(fma2(pk(v[c], v[c + 1]), s2, m2), v[c], v[c + 1]);
}

// in-place max-pool of width 2*PAD+1: v[o] = max(v[o .. o + 2 PAD]) for o < NOUT
template <int PAD, int NV, int NOUT>
__device__ __forceinline__ void pool_inplace(float (&v)[NV]) {
    static_assert(NOUT + 2 * PAD <= NV, "halo");
    if constexpr (PAD == 1) {
#pragma unroll
        for (int o = 0; o < NOUT; ++o) v[o] = max3(v[o], v[o + 1], v[o + 2]);
    } else if constexpr (PAD >= 2) {
        // b[j] = max(v[j..j+2]); v[j] is dead once b[j] exists
#pragma unroll
        for (int jj = 0; jj < NOUT + 2 * PAD - 2; ++jj) v[jj] = max3(v[jj], v[jj + 1], v[jj + 2]);
        if constexpr (PAD == 2) {
#pragma unroll
            for (int o = 0; o < NOUT; ++o) v[o] = fmaxf(v[o], v[o + 2]);
        } else {
            static_assert(PAD == 3, "pad <= 3");
#pragma unroll
            for (int o = 0; o < NOUT; ++o) v[o] = max3(v[o], v[o + 3], v[o + 4]);
        }
    }
}

// pass-2 epilogue of one 32-output column group cg (outputs [32 cg, min(32 cg + 32, STEP))):
// the column group is a runtime value so all 16 epilogue warps share one code path.  Always
// 32 outputs are formed; the last group's surplus outputs (beyond the tile step) are zeros.
template <int PAD>
__device__ __forceinline__ void pass2_group_rt(int cg, uint32_t taddr, int lane, int r, int key_col0, int n_o,
                                               float sl, float lw2, uint8_t* a2tile, uint64_t* acc_empty_bar,
                                               uint64_t* e_empty_bar, uint32_t e_parity, uint64_t* e_full_bar,
                                               int dbg_flags) {
    constexpr int STEP = kTile - 2 * PAD;
    constexpr int NV = PAD > 0 ? 40 : 32;  // loaded columns incl. the halo
    const int O0 = 32 * cg;
    const int NOUT = (STEP - O0) < 32 ? (STEP - O0) : 32;
    float v[NV];
    tmem_ld_x32<0>(taddr + O0, v);
    if constexpr (NV > 32) {
        if (cg < 3) {
            tmem_ld_x8<32>(taddr + O0 + 32, v);
        } else {
#pragma unroll
            for (int jj = 32; jj < NV; ++jj) v[jj] = -INFINITY;
        }
    }
    tmem_ld_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(acc_empty_bar);
    // keys outside [0, n_o) are excluded from every window (padded cells, policies.hpp:105-106)
    const int k0 = key_col0 + O0;
    if (k0 < 0 || k0 + NV > n_o) {
#pragma unroll
        for (int jj = 0; jj < NV; ++jj)
            if (k0 + jj < 0 || k0 + jj >= n_o) v[jj] = -INFINITY;
    }
    pool_inplace<PAD, NV, 32>(v);
    scale_shift2<32>(v, sl, lw2);
    if (!(dbg_flags & 1024)) exp2_mixed<NV, kPass2Poly>(v, 32);
    mbar_wait(e_empty_bar, e_parity);
    uint8_t* rowbase = a2tile + (r >> 3) * 2048 + (cg >> 1) * 1024 + (r & 7) * 128;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        uint32_t w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int o0 = c * 8 + 2 * u, o1 = o0 + 1;
            const __half2 h2 = __floats2half2_rn(o0 < NOUT ? v[o0] : 0.f, o1 < NOUT ? v[o1] : 0.f);
            w[u] = *reinterpret_cast<const uint32_t*>(&h2);
        }
        const int chunk = 4 * (cg & 1) + c;
        *reinterpret_cast<uint4*>(rowbase + ((chunk ^ (r & 7)) * 16)) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    fence_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(e_full_bar);
}

template <int PAD>
__global__ void __launch_bounds__(kThreads, 1)
score_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                const TcParams prm) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment by offsetting the __shared__ array itself (keeps the shared window:
    // LDS/STS instead of generic LD/ST)
    Smem& S = *reinterpret_cast<Smem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool pass2 = prm.pass == 2;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tm_q);
        prefetch_tmap(&tm_k);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&S.full[s], 1);
            mbar_init(&S.empty[s], 1);
        }
        mbar_init(&S.q_full, 1);
        mbar_init(&S.q_empty, 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&S.acc_full[b], 1);
            mbar_init(&S.acc_empty[b], kEpiWarps);
            mbar_init(&S.e_full[b], kEpiWarps);  // every column group writes its slice of E^T
            mbar_init(&S.e_empty[b], 1);
            mbar_init(&S.d2_full[b], 1);
            mbar_init(&S.d2_empty[b], 4);
        }
        mbar_fence_init();
    }
    if (warp == 1) tmem_alloc<kTmemCols>(&S.tmem_base);
    if (pass2) {
        // head-indicator B operand: Hd[row k][head n] = 1 iff k / m == n < g (K-major, SW128)
        for (int i = threadIdx.x; i < 2 * 16 * 64; i += kThreads) {
            const int hk = i / (16 * 64), n = (i / 64) % 16, kk = i % 64;
            const int krow = hk * 64 + kk;
            const __half val = __float2half((n < prm.gs && krow / prm.m == n) ? 1.f : 0.f);
            *reinterpret_cast<__half*>(&S.b2[hk][n * 128 + (((kk >> 3) ^ (n & 7)) << 4) + (kk & 7) * 2]) = val;
        }
        fence_async_smem();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem_base;
    // Programmatic dependent launch: pass 1 needs nothing from the kernel before it (the
    // previous slice's pass 2), so the next kernel may be scheduled at once; pass 2 lets its
    // TMA / MMA warps start on K immediately and only its epilogue waits for pass 1's
    // statistics (below), after which it releases the next slice's pass 1 (which reuses
    // the pass-1 workspace, so it must not start before this slice's pass 1 is complete).
    if (!pass2) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();  // K streams through once per pass (no L2 reuse)
            const uint64_t pol_q = policy_evict_last();
            uint32_t stage = 0, sphase = 0, qphase = 0;
            long long prod_wait = 0;
            const long long p_start = clock64();
            for (int item = blockIdx.x; item < prm.n_items; item += gridDim.x) {
                const int pg = item / prm.chunks_per_pg, chunk = item % prm.chunks_per_pg;
                const int t0 = chunk * prm.tiles_per_item;
                const int t1 = min(t0 + prm.tiles_per_item, prm.tiles_per_pg);
                mbar_wait(&S.q_empty, qphase ^ 1);
                qphase ^= 1;
                mbar_arrive_expect_tx(&S.q_full, kTileBytes);
                tma_load_3d(S.q[0], &tm_q, 0, 0, pg, &S.q_full, pol_q);
                tma_load_3d(S.q[1], &tm_q, 64, 0, pg, &S.q_full, pol_q);
                for (int t = t0; t < t1; ++t) {
                    const long long w0 = clock64();
                    mbar_wait(&S.empty[stage], sphase ^ 1);
                    prod_wait += clock64() - w0;
                    mbar_arrive_expect_tx(&S.full[stage], kTileBytes);
                    const int row = t * prm.step - prm.pad;
                    tma_load_3d(S.k[stage][0], &tm_k, 0, row, pg / prm.vsplit, &S.full[stage], pol);
                    tma_load_3d(S.k[stage][1], &tm_k, 64, row, pg / prm.vsplit, &S.full[stage], pol);
                    if (++stage == kStages) {
                        stage = 0;
                        sphase ^= 1;
                    }
                }
            }
            if (prm.dbg) {
                long long* ts = prm.dbg + ((prm.pass - 1) * 160 + blockIdx.x) * 16;
                ts[0] = prod_wait;
                ts[1] = clock64() - p_start;
            }
        }
    } else if (warp == 1) {
        // ===================== tcgen05 MMA issuer =====================
        if (lane == 0) {
            constexpr uint32_t idesc1 = idesc_bf16_f32(128, kTile);
            constexpr uint32_t idesc2 = idesc_f16_f32(128, 16, 1);
            uint32_t stage = 0, sphase = 0, qphase = 0;
            uint32_t j = 0;  // tile sequence number of this CTA
            long long mma_wait_acc = 0, mma_wait_full = 0, mma_wait_e = 0, mma_wait_d2 = 0;
            auto mma2 = [&](uint32_t i) {
                const uint32_t b = i & 1, ph = (i >> 1) & 1;
                long long w = clock64();
                mbar_wait(&S.e_full[b], ph);
                mma_wait_e += clock64() - w;
                w = clock64();
                mbar_wait(&S.d2_empty[b], ph ^ 1);
                mma_wait_d2 += clock64() - w;
                tc_fence_after();
#pragma unroll
                for (int s = 0; s < 8; ++s) {
                    const uint64_t ad = desc_mnmajor_sw128(smem_u32(S.a2[b]) + s * 4096, 1024, 2048);
                    const uint64_t bd = desc_kmajor_sw128(smem_u32(S.b2[s >> 2]) + (s & 3) * 32);
                    mma_f16(tmem + kD2Col + 16 * b, ad, bd, idesc2, s > 0 ? 1u : 0u);
                }
                mma_commit(&S.e_empty[b]);
                mma_commit(&S.d2_full[b]);
            };
            for (int item = blockIdx.x; item < prm.n_items; item += gridDim.x) {
                const int chunk = item % prm.chunks_per_pg;
                const int t0 = chunk * prm.tiles_per_item;
                const int t1 = min(t0 + prm.tiles_per_item, prm.tiles_per_pg);
                mbar_wait(&S.q_full, qphase);
                qphase ^= 1;
                for (int t = t0; t < t1; ++t, ++j) {
                    const uint32_t ab = j & 1, aph = (j >> 1) & 1;
                    long long w0 = clock64();
                    mbar_wait(&S.acc_empty[ab], aph ^ 1);
                    mma_wait_acc += clock64() - w0;
                    w0 = clock64();
                    mbar_wait(&S.full[stage], sphase);
                    mma_wait_full += clock64() - w0;
                    tc_fence_after();
                    const uint32_t d = tmem + ab * kTile;
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint32_t off = (kk & 3) * 32;
                        const uint64_t ad = desc_kmajor_sw128(smem_u32(S.q[kk >> 2]) + off);
                        const uint64_t bd = desc_kmajor_sw128(smem_u32(S.k[stage][kk >> 2]) + off);
                        mma_bf16(d, ad, bd, idesc1, kk > 0 ? 1u : 0u);
                    }
                    mma_commit(&S.empty[stage]);
                    mma_commit(&S.acc_full[ab]);
                    if (++stage == kStages) {
                        stage = 0;
                        sphase ^= 1;
                    }
                    // the head-sum MMA of tile j-2 (two tiles of slack: QK of the next tile is
                    // not held back by the slowest epilogue warp of the previous one)
                    if (pass2 && j > 1) mma2(j - 2);
                }
                mma_commit(&S.q_empty);
            }
            if (pass2 && j > 1) mma2(j - 2);
            if (pass2 && j > 0) mma2(j - 1);
            if (prm.dbg) {
                long long* ts = prm.dbg + ((prm.pass - 1) * 160 + blockIdx.x) * 16;
                ts[2] = mma_wait_acc;
                ts[3] = mma_wait_full;
                ts[7] = mma_wait_e;
                ts[8] = mma_wait_d2;
            }
        }
    } else {
        // ===================== epilogue (warps 2..9) =====================
        const int ew = warp - 2;
        const int q = warp & 3;              // TMEM lane quarter == head (m == 32)
        const int cg = ew >> 2;              // 32-column group
        const int r = q * 32 + lane;         // window row == TMEM lane
        const bool active = r < prm.gs * prm.m;
        const int et = ew * 32 + lane;       // 0..511
        const float sl = prm.scale_log2;
        if (pass2) {
            asm volatile("griddepcontrol.wait;" ::: "memory");
            asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        }
        uint32_t j = 0;
        long long epi_wait = 0;
        const long long e_start = clock64();
        int prev_pg = -1, prev_t = 0, prev2_pg = -1, prev2_t = 0;
        auto readout = [&](uint32_t i, int rpg, int rt) {
            // D2 of tile i: lanes = output keys, columns = heads (one warp per lane quarter)
            const uint32_t b = i & 1, ph = (i >> 1) & 1;
            mbar_wait(&S.d2_full[b], ph);
            tc_fence_after();
            float hv[16];
            tmem_ld_x16<0>(tmem + kD2Col + 16 * b + (uint32_t(q * 32) << 16), hv);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.d2_empty[b]);
            const int o = q * 32 + lane;
            const int key = rt * prm.step + o;
            if (o < prm.step && key < prm.n_o) {
                // virtual group gpg = (p G + g) vsplit + half holds heads [gpg gs, gpg gs + gs) of
                // all H = G gs vsplit, and group row p G + g = gpg / vsplit (vsplit = 1, 2, 4): no
                // division by G per readout
                const int gpg = prm.pg_base + rpg;
                constexpr float inv_scale = 1.f / 65536.f;
                float gsum = 0.f;
#pragma unroll
                for (int h = 0; h < 16; ++h) {
                    if (h >= prm.gs) break;
                    const float sh = hv[h] * inv_scale;
                    gsum += sh;
                    if (prm.head_scores) prm.head_scores[(size_t(gpg) * prm.gs + h) * prm.n_o + key] = sh;
                }
                float* gdst = prm.group_scores + size_t(gpg >> (prm.vsplit >> 1)) * prm.n_o + key;
                if (prm.vsplit == 1) *gdst = gsum * prm.inv_g;
                else atomicAdd(gdst, gsum * prm.inv_g);
            }
        };
        for (int item = blockIdx.x; item < prm.n_items; item += gridDim.x) {
            const int pg = item / prm.chunks_per_pg, chunk = item % prm.chunks_per_pg;
            const int t0 = chunk * prm.tiles_per_item;
            const int t1 = min(t0 + prm.tiles_per_item, prm.tiles_per_pg);
            const int gpg = prm.pg_base + pg;
            float run_m = -INFINITY, run_s = 0.f, lw2 = INFINITY;
            if (pass2 && active) lw2 = prm.final_stats[(size_t(gpg) * 128 + r) * 2 + 1] - kEScaleLog2;
            for (int t = t0; t < t1; ++t, ++j) {
                const uint32_t ab = j & 1, aph = (j >> 1) & 1;
                const long long w0 = clock64();
                mbar_wait(&S.acc_full[ab], aph);
                epi_wait += clock64() - w0;
                tc_fence_after();
                const uint32_t taddr = tmem + ab * kTile + (uint32_t(q * 32) << 16);
                if (!pass2) {
                    float v[32];
                    tmem_ld_x32<0>(taddr + 32 * cg, v);
                    tmem_ld_wait();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&S.acc_empty[ab]);
                    const int nvalid = prm.n_o - (t * kTile + 32 * cg);
                    if (nvalid < 32) {
#pragma unroll
                        for (int c = 0; c < 32; ++c)
                            if (c >= nvalid) v[c] = -INFINITY;
                    }
                    float m2[2];
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        float mm = max3(v[16 * c], v[16 * c + 1], v[16 * c + 2]);
#pragma unroll
                        for (int u = 3; u < 15; u += 2) mm = max3(mm, v[16 * c + u], v[16 * c + u + 1]);
                        m2[c] = fmaxf(mm, v[16 * c + 15]);
                    }
                    const float tmx = fmaxf(m2[0], m2[1]);
                    const float nm = fmaxf(run_m, tmx * sl);
                    if (nm != -INFINITY) {
                        scale_shift2<32>(v, sl, nm);
                        // 2 of every 8 exp2 on the FMA pipe (polynomial), 6 on MUFU: measured
                        // fastest split (debug 64: MUFU only)
                        if (prm.debug & 64) exp2_mixed<32, 0>(v, 32);
                        else exp2_mixed<32, kPass1Poly>(v, 32);
                        uint64_t a0 = pk(0.f, 0.f), a1 = pk(0.f, 0.f);
#pragma unroll
                        for (int c = 0; c < 32; c += 4) {
                            a0 = add2(a0, pk(v[c], v[c + 1]));
                            a1 = add2(a1, pk(v[c + 2], v[c + 3]));
                        }
                        float s0, s1, s2, s3;
                        upk(a0, s0, s1);
                        upk(a1, s2, s3);
                        run_s = (run_m == -INFINITY ? 0.f : run_s * ex2(run_m - nm)) + ((s0 + s1) + (s2 + s3));
                        run_m = nm;
                    }
                } else {
                    const uint32_t eb = j & 1, eph = (j >> 1) & 1;
                    const int key_col0 = t * prm.step - prm.pad;
                    const float lw = active ? lw2 : INFINITY;
                    pass2_group_rt<PAD>(cg, taddr, lane, r, key_col0, prm.n_o, sl, lw, S.a2[eb], &S.acc_empty[ab],
                                        &S.e_empty[eb], eph ^ 1, &S.e_full[eb], prm.debug);
                    // one column group (rotating, so the extra work is spread evenly over the
                    // epilogue warps) reads back the scores of tile j-2
                    if (j > 1 && cg == int((j - 2) & 3)) readout(j - 2, prev2_pg, prev2_t);
                    prev2_pg = prev_pg;
                    prev2_t = prev_t;
                    prev_pg = pg;
                    prev_t = t;
                }
            }
            if (!pass2) {
                float* pp = prm.partial + (((size_t(pg) * prm.chunks_per_pg + chunk) * 4 + cg) * 128 + r) * 2;
                pp[0] = active ? run_m : -INFINITY;
                pp[1] = active ? run_s : 0.f;
                if (prm.debug & 4) continue;
                // grid-sync pattern: CTA barrier, then ONE thread fences (cumulative release of
                // every epilogue thread's partial) and takes the ticket (a fence per thread costs
                // ~0.5 ms here); the last arriver fences again (acquire) before the fold.
                named_bar(1, 32 * kEpiWarps);
                if (et == 0) {
                    if (!(prm.debug & 8)) __threadfence();
                    const bool last = atomicAdd(&prm.tickets[pg], 1u) == unsigned(prm.chunks_per_pg - 1);
                    if (last && !(prm.debug & 8)) __threadfence();
                    S.is_last = last;
                }
                named_bar(1, 32 * kEpiWarps);
                if (S.is_last && !(prm.debug & 16)) {
                    // parallel fold: thread (row r, column group cg) folds every 4th partial of
                    // its row (all loads in flight at once), then the 4 groups merge via smem.
                    const float* base = prm.partial + size_t(pg) * prm.chunks_per_pg * 4 * 256;
                    const int nparts = prm.chunks_per_pg * 4;
                    float M = -INFINITY, Ssum = 0.f;
                    for (int c0 = cg; c0 < nparts; c0 += 32) {
                        float2 v8[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int c = c0 + 4 * u;
                            v8[u] = c < nparts ? __ldcg(reinterpret_cast<const float2*>(base + (c * 128 + r) * 2))
                                               : make_float2(-INFINITY, 0.f);
                        }
                        float bm = M;
#pragma unroll
                        for (int u = 0; u < 8; ++u) bm = fmaxf(bm, v8[u].x);
                        if (bm != -INFINITY) {
                            float acc = M == -INFINITY ? 0.f : Ssum * ex2(M - bm);
#pragma unroll
                            for (int u = 0; u < 8; ++u)
                                if (v8[u].x != -INFINITY) acc += v8[u].y * ex2(v8[u].x - bm);
                            Ssum = acc;
                            M = bm;
                        }
                    }
                    // stash in the (now idle) E^T staging buffer: [cg][128 rows][2]
                    float* red = reinterpret_cast<float*>(S.a2[0]);
                    red[(cg * 128 + r) * 2 + 0] = M;
                    red[(cg * 128 + r) * 2 + 1] = Ssum;
                    named_bar(1, 32 * kEpiWarps);
                    if (cg == 0) {
                        float Mf = -INFINITY;
#pragma unroll
                        for (int c = 0; c < 4; ++c) Mf = fmaxf(Mf, red[(c * 128 + r) * 2]);
                        float Sf = 0.f;
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const float mc = red[(c * 128 + r) * 2];
                            if (mc != -INFINITY) Sf += red[(c * 128 + r) * 2 + 1] * ex2(mc - Mf);
                        }
                        float* fs = prm.final_stats + (size_t(gpg) * 128 + r) * 2;
                        // a NaN or +Inf logit anywhere in the row (a non-finite key,
                        // LayerCache::validate, attention.hpp:76-83) leaves a non-finite max or sum
                        if (active && prm.err && !(Mf > -INFINITY && Mf < INFINITY && Sf >= 1.f && Sf < INFINITY))
                            atomicOr(prm.err, ERR_NONFINITE);
                        fs[0] = Mf;
                        fs[1] = active ? Mf + __log2f(Sf) + prm.log2_m : INFINITY;
                        if (et == 0) prm.tickets[pg] = 0u;
                    }
                    named_bar(1, 32 * kEpiWarps);
                }
            }
        }
        if (pass2 && j > 1 && cg == int((j - 2) & 3)) readout(j - 2, prev2_pg, prev2_t);
        if (pass2 && j > 0 && cg == int((j - 1) & 3)) readout(j - 1, prev_pg, prev_t);
        if (prm.dbg && et == 0) {
            long long* ts = prm.dbg + ((prm.pass - 1) * 160 + blockIdx.x) * 16;
            ts[4] = epi_wait;
            ts[5] = clock64() - e_start;
            ts[6] = j;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc<kTmemCols>(tmem);
}

// ------------------------------------------------------------------ host side
long long* g_score_dbg = nullptr;  // (debug) role wait counters, scripts/tc_ts.py
// 3-D bf16 tensor [outer][rows][128] with a {64, 128, 1} box, 128-byte swizzle.
adakv_status make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t outer) {
    ptx::EncodeFn enc = ptx::get_encode();
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

// Tiles per item minimising the makespan: ceil(items / CTAs) items per CTA, each costing its
// tiles plus ~2 tiles of fixed overhead (Q load, pipeline ramp, ticket), plus the serial fold
// of chunks partials per group in the last CTA (~1 tile per 16 chunks).
void balance(int64_t pgs, int64_t tiles, int sms, int* tpi, int* chunks) {
    int64_t best_t = 1, best_cost = INT64_MAX;
    for (int64_t t = 1; t <= tiles; ++t) {
        const int64_t ch = ceil_div(tiles, t);
        const int64_t items = pgs * ch;
        const int64_t cost = 16 * ceil_div(items, sms) * (t + 2) + ch;
        if (cost < best_cost) {
            best_cost = cost;
            best_t = t;
        }
    }
    *tpi = int(best_t);
    *chunks = int(ceil_div(tiles, best_t));
}

struct Plan {
    int64_t slice;
    int tpi1, chunks1, tpi2, chunks2;
};

}  // namespace
int vsplit_of(const adakv_layer_shape& s);
namespace {

Plan make_plan(const adakv_layer_shape& s, int pad) {
    Plan pl{};
    // a slice = a run of KV groups (across problems); default: the whole call (see the header)
    static const int64_t budget = [] {
        const char* e = std::getenv("ADAKV_SCORE_SLICE_MB");
        const int64_t v = e ? std::atoll(e) : 0;
        return v > 0 ? (v << 20) : (int64_t(1) << 62);
    }();
    const int64_t g_bytes = (s.outside + s.window) * s.head_dim * 2;
    pl.slice = std::max<int64_t>(1, std::min<int64_t>(s.problems * s.kv_groups, budget / std::max<int64_t>(g_bytes, 1)));
    const int sms = device_sm_count();
    const int64_t pgs = pl.slice * std::max(1, vsplit_of(s));
    balance(pgs, ceil_div(s.outside, kTile), sms, &pl.tpi1, &pl.chunks1);
    balance(pgs, ceil_div(s.outside, kTile - 2 * pad), sms, &pl.tpi2, &pl.chunks2);
    return pl;
}

}  // namespace

// window-row tiles per KV group: 1 while g*m <= 128; else the smallest split into <= 128-row
// tiles of whole heads (g = 8, m = 32 -> 2)
int vsplit_of(const adakv_layer_shape& s) {
    const int64_t gs = s.kv_groups > 0 ? s.q_heads / s.kv_groups : 0;
    for (int v = 1; v <= 4; v *= 2)
        if (gs % v == 0 && (gs / v) * s.window <= 128) return v;
    return 0;
}

bool score_window_tc_supported(adakv_dtype dt, const adakv_layer_shape& s, int64_t pool_kernel) {
    const int64_t gs = s.kv_groups > 0 ? s.q_heads / s.kv_groups : 0;
    return dt == ADAKV_BF16 && s.head_dim == 128 && s.window == 32 && gs >= 1 && vsplit_of(s) > 0 &&
           (pool_kernel == 1 || pool_kernel == 3 || pool_kernel == 5 || pool_kernel == 7) && s.outside >= 1 &&
           s.outside + s.window < (int64_t(1) << 31) && ptx::get_encode() != nullptr;
}

size_t score_window_tc_workspace(const adakv_layer_shape& s) {
    const Plan pl = make_plan(s, 0);
    const int64_t vs = std::max(1, vsplit_of(s));
    const int64_t pgs_slice = pl.slice * vs;
    return 3 * 256 + size_t(pgs_slice) * pl.chunks1 * 4 * 128 * 2 * 4 +
           size_t(s.problems * s.kv_groups * vs) * 128 * 2 * 4 + size_t(pgs_slice) * 4;
}

adakv_status score_window_tc(const adakv_layer_shape& s, int64_t pool_kernel, int32_t scale, const void* q,
                             const void* k, void* head_scores, void* group_scores, void* ws, uint32_t* err,
                             cudaStream_t stream) {
    const int pad = int((pool_kernel - 1) / 2);
    const Plan pl = make_plan(s, pad);
    const int64_t G = s.kv_groups, H = s.q_heads, gs = H / G, m = s.window, n = s.outside + s.window;
    const int64_t d = s.head_dim;
    const int64_t vs = vsplit_of(s), Gv = G * vs, gst = gs / vs;  // virtual groups of gst heads
    Arena ar(ws);
    float* partial = ar.take<float>(size_t(pl.slice * vs * pl.chunks1 * 4 * 256));
    float* fstats = ar.take<float>(size_t(s.problems * Gv * 256));
    unsigned* tickets = ar.take<unsigned>(size_t(pl.slice * vs));
    ADAKV_CUDA_TRY(cudaMemsetAsync(tickets, 0, size_t(pl.slice * vs) * 4, stream));
    if (vs > 1)  // the virtual groups' halves are added into the group scores
        ADAKV_CUDA_TRY(cudaMemsetAsync(group_scores, 0, size_t(s.problems * G * s.outside) * 4, stream));
    const size_t smem = smem_bytes();
    const int sms = device_sm_count();
    auto k2 = pad == 0 ? score_tc_kernel<0> : pad == 1 ? score_tc_kernel<1> : pad == 2 ? score_tc_kernel<2>
                                                                                       : score_tc_kernel<3>;
    ADAKV_CUDA_TRY(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    ADAKV_CUDA_TRY(cudaFuncSetAttribute(score_tc_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const float sc = scale ? 1.0f / sqrtf(float(d)) : 1.0f;
    for (int64_t g0 = 0; g0 < s.problems * G; g0 += pl.slice) {
        const int64_t ng = std::min(pl.slice, s.problems * G - g0);  // KV groups of this slice
        CUtensorMap tq, tk;
        const auto* qb = static_cast<const __nv_bfloat16*>(q) + g0 * gs * m * d;
        const auto* kb = static_cast<const __nv_bfloat16*>(k) + g0 * n * d;
        ADAKV_TRY(make_map(&tq, qb, uint64_t(gst * m), uint64_t(ng * vs)));
        ADAKV_TRY(make_map(&tk, kb, uint64_t(n), uint64_t(ng)));
        TcParams prm{};
        prm.G = int(G);
        prm.H = int(H);
        prm.gs = int(gst);
        prm.vsplit = int(vs);
        prm.m = int(m);
        prm.n_o = int(s.outside);
        prm.pg_base = int(g0 * vs);
        prm.scale_log2 = sc * 1.4426950408889634f;
        prm.log2_m = log2f(float(m));
        prm.inv_g = 1.0f / float(gs);
        prm.partial = partial;
        prm.final_stats = fstats;
        prm.tickets = tickets;
        prm.head_scores = static_cast<float*>(head_scores);
        prm.group_scores = static_cast<float*>(group_scores);
        static const int dbg = [] {
            const char* e = std::getenv("ADAKV_TC_DEBUG");
            return e ? std::atoi(e) : 0;
        }();
        prm.debug = dbg;
        prm.dbg = g_score_dbg;
        prm.err = err;
        // pass 1: row statistics over 128-key tiles
        prm.pass = 1;
        prm.step = kTile;
        prm.pad = 0;
        prm.tiles_per_pg = int(ceil_div(s.outside, kTile));
        prm.tiles_per_item = pl.tpi1;
        prm.chunks_per_pg = pl.chunks1;
        prm.n_items = int(ng * vs * prm.chunks_per_pg);
        int grid = std::min(prm.n_items, sms);
        cudaLaunchAttribute pdl[1];
        pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        pdl[0].val.programmaticStreamSerializationAllowed = 1;
        cudaLaunchConfig_t lc = {};
        lc.blockDim = dim3(kThreads);
        lc.dynamicSmemBytes = smem;
        lc.stream = stream;
        lc.attrs = pdl;
        lc.gridDim = dim3(unsigned(grid));
        lc.numAttrs = g0 > 0 ? 1 : 0;  // the first pass 1 waits for whatever produced K
        ADAKV_CUDA_TRY(cudaLaunchKernelEx(&lc, score_tc_kernel<0>, tq, tk, prm));
        // pass 2: pooled scores over (128 - 2 pad)-key output tiles
        prm.pass = 2;
        prm.pad = pad;
        prm.step = kTile - 2 * pad;
        prm.tiles_per_pg = int(ceil_div(s.outside, prm.step));
        prm.tiles_per_item = pl.tpi2;
        prm.chunks_per_pg = pl.chunks2;
        prm.n_items = int(ng * vs * prm.chunks_per_pg);
        grid = std::min(prm.n_items, sms);
        if (dbg & 1) continue;  // debug: pass 1 only
        lc.gridDim = dim3(unsigned(grid));
        lc.numAttrs = 1;
        ADAKV_CUDA_TRY(cudaLaunchKernelEx(&lc, k2, tq, tk, prm));
    }
    return ADAKV_OK;
}

}  // namespace adakv_b200

extern "C" void adakv_debug_set_score_counters(void* buf) {
    adakv_b200::g_score_dbg = static_cast<long long*>(buf);
}
