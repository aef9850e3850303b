// decode_tc.cu -- K4 fast path: split-K varlen flash-decoding for bf16, d == 128,
// g = H/G <= 8 query heads per KV group, on warp-level tensor-core MMA (m16n8k16).
//
// Same contract as decode.cu (attention_weights + row_times(a, V) per head over the
// retained cache, attention.hpp:169-196 / report.hpp:133-144, with append_kv fused).
//
// Data movement: every warp owns a contiguous run of 16-row blocks of its group's segment
// and streams them through a private ring of shared-memory slots with TMA
// (cp.async.bulk.tensor, one 4 KB box per block for K and one for V, 128-byte swizzle).
// The copies for the first ring's worth of blocks are issued before griddepcontrol.wait,
// so under programmatic dependent launch a layer's cache streams in while the previous
// layer's decode is still finishing.
//
// Per warp, keys are consumed in blocks of 16, two blocks per step when two are left (their
// S chains overlap; one softmax covers the 32 keys):
//   S  = Q K^T      two m16n8k16 n8 tiles x 8 k-steps; rows = the g heads (padded to 16);
//   P  = exp2(S*c - m)  online softmax (block max over the 4 lanes of a row; the running
//                   max moves only when a step exceeds it by more than 2^8);
//   O^T += V^T P^T  eight m16n8k16 m-tiles over d.
// The per-block cost is the mma.sync issue/latency chain (scripts/micro/dec_block.cu), so
// the first block's wait and K loads are placed before the Q fragments are assembled (the
// Q load's latency overlaps them); the group's query rows arrive by one multicast bulk copy
// from cluster rank 0 into every CTA's shared memory (one L2 read per group instead of one per
// warp: 4.22 -> 4.21 us per step-layer on the bench).  Combine: warp partials merge in shared memory (each
// (warp, head) scale computed once per merging warp and shared by shuffles), then each CTA
// pushes its columns' slice to the owning rank with DSMEM st.async.
// The dot products are invariant to a consistent permutation of d, so Q's and K's
// d-columns are permuted such that each lane's B-fragment words are exactly the 16-byte
// chunks it reads; V's d (the MMA M dimension) is permuted likewise and un-permuted when O
// is written.  Attention is also invariant to a consistent permutation of the keys: MMA key
// slot n of an 8-key tile reads block row kperm(n), chosen with the 128-byte swizzle so that
// both the K reads (2 rows x 64 B per 8-lane phase) and the V reads (4 rows x 32 B) hit 32
// distinct banks.  The S accumulator fragment (row = head, cols = keys 2t, 2t+1) is exactly
// the P^T B-fragment of the PV MMA, so P never leaves registers.
#include <algorithm>
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

constexpr int kBlk = 16;
#ifndef ADAKV_DECODE_W
#define ADAKV_DECODE_W 8
#endif
#ifndef ADAKV_DEC_TRIPLE
#define ADAKV_DEC_TRIPLE 1
#endif
constexpr bool kTriple = ADAKV_DEC_TRIPLE != 0;  // last three blocks of a warp as one step
constexpr int kMaxWarps = ADAKV_DECODE_W;   // warps per CTA (template parameter W <= kMaxWarps)
constexpr int kMaxSlots = 3;               // ring depth per warp (runtime <= kMaxSlots; 227 KB smem)
constexpr int kBoxBytes = kBlk * 256;      // one 16-row box of K (or V): [16 rows][2 halves][128 B]
constexpr int kMaxCS = 16;

// Split-K combine chunk sent by every CTA to each owner rank: (m, l) per head (16 floats),
// then O for the owner's columns as [column][8 heads].
__host__ __device__ constexpr int chunk_floats(int cs) { return 16 + ((128 + cs - 1) / cs) * 8; }

// Shared memory: the split-K combine buffers, then the per-warp TMA rings.
struct DecSmem {
    float s_ml[kMaxWarps][8][2];                    // warp partials: (m, l) per head
    alignas(16) float s_f[kMaxWarps][32];           // CTA merge: each merging warp's 32 scales
    alignas(16) float recv[kMaxCS * 16 + 1024 + kMaxCS * 8];   // one chunk from every rank
    alignas(128) uint8_t qs[8 * 256];               // the group's query rows (Q staging modes 1, 2)
    uint64_t bar[kMaxWarps][kMaxSlots];
    uint64_t rbar;                                  // receive barrier (bulk-copy complete_tx)
    uint64_t qbar;                                  // query rows landed (Q staging modes 1, 2)
};
constexpr size_t kRingOffset = (sizeof(DecSmem) + 1023) / 1024 * 1024;
size_t dec_smem_bytes(int nslots, int warps) { return kRingOffset + size_t(warps) * nslots * 2 * kBoxBytes + 1024; }

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

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// shared::cluster address of the same smem offset in CTA `rank` of this cluster
__device__ __forceinline__ uint32_t mapa(uint32_t addr, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
// 16-byte store into (possibly remote) cluster shared memory, completing tx bytes on its mbarrier
__device__ __forceinline__ void st_async_v4(uint32_t addr, float4 v, uint32_t bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1,%2,%3,%4}, [%5];" ::"r"(addr),
                 "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(bar)
                 : "memory");
}
// bulk copy global -> this CTA's shared memory (mode 1) or the same offset in every CTA of
// the cluster in `mask` (mode 2, multicast), completing tx bytes on the mbarrier at `bar`'s offset
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s_mc(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                            uint16_t mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
        "%4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "h"(mask)
        : "memory");
}
// byte offset of 16-byte chunk c (0..15) of block row r in a swizzled box: line = 2r + half
__device__ __forceinline__ uint32_t box_off(int r, int c) {
    const int line = 2 * r + (c >> 3);
    return uint32_t(line * 128 + (((c & 7) ^ (line & 7)) << 4));
}

// key slot n (0..7) of an 8-key MMA tile -> block row (see header): n = 2t + e -> 4e | (t ^ 2e)
__device__ __forceinline__ int kperm(int n) {
    const int t = n >> 1, e = n & 1;
    return (e << 2) | (t ^ (e << 1));
}

// d column held by (m-tile i, fragment row r) of the PV MMA
__device__ __forceinline__ int v_col(int i, int r) { return (i < 4 ? 0 : 64) + 8 * (r & 7) + 2 * (i & 3) + (r >> 3); }

// One thread-block cluster of CS CTAs per (problem, KV group): CTA rank r takes blocks
// [nblk r / CS, nblk (r+1) / CS) of the group's 16-row blocks, split again over its W warps.
// Warp partials (m, l, O) merge in shared memory; each CTA partial is then split by output
// column and sent with one bulk DSMEM copy per rank to the rank that finishes those columns,
// so the split-K combine needs no global round trips, atomics or remote loads.
template <int CS, int W>
__global__ void __launch_bounds__(32 * W, 1)
decode_tc_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                 const __nv_bfloat16* __restrict__ q, __nv_bfloat16* __restrict__ k_cache,
                 __nv_bfloat16* __restrict__ v_cache, const int32_t* __restrict__ seg_start,
                 const int32_t* __restrict__ seg_cap, int32_t* __restrict__ seqlens,
                 const __nv_bfloat16* __restrict__ k_new, const __nv_bfloat16* __restrict__ v_new,
                 __nv_bfloat16* __restrict__ out, uint32_t* __restrict__ err, int H, int G, float scale_log2,
                 int nslots, int qmode, unsigned long long* __restrict__ dbg) {
    constexpr int d = 128;
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment by offsetting the __shared__ array itself (keeps the shared window,
    // so every access below compiles to LDS/STS rather than generic LD/ST)
    uint8_t* smem_al = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    DecSmem& S = *reinterpret_cast<DecSmem*>(smem_al);
    auto ring_of = [&](int w) { return smem_al + kRingOffset + size_t(w) * nslots * 2 * kBoxBytes; };
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = int(cluster.block_rank());
    const int pg = blockIdx.x / CS;
    const int p = pg / G, g = pg % G;
    const int gs = H / G;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const bool head_ok = gid < gs;
    uint8_t* ring = ring_of(warp);  // this warp's TMA slots
    auto stamp = [&](int k) {       // (debug) per-CTA phase timestamps
        if (dbg && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            dbg[blockIdx.x * 64 + k] = t;
            if (k < 8) dbg[blockIdx.x * 64 + 16 + k] = clock64();
        }
    };
    // this layer's own cache state (written by its previous decode step, long complete)
    const int L_old = __ldcg(seqlens + pg);
    const int base = seg_start[pg];
    ADAKV_DCHECK(L_old >= 0 && base >= 0 && L_old <= seg_cap[pg]);
    // append_kv into a full segment is refused (never written past seg_cap): the step attends
    // the existing rows and ERR_CAPACITY is latched after the dependency wait
    const bool append = k_new != nullptr && L_old < seg_cap[pg];
    stamp(0);
    // rank r finishes output columns [128 r / CS, 128 (r+1) / CS) of every head
    constexpr int chunk = chunk_floats(CS);
    const int col_lo = (d * rank) / CS, ncols = (d * (rank + 1)) / CS - col_lo;
    if (threadIdx.x == 0) {
        // receive barrier: completes when every rank's chunk has landed
        mbar_init(&S.rbar, 1);
        mbar_fence_init();
        const int nq = (gs + 3) >> 2;  // head quads: each (column, quad) arrives as one 16-byte store
        mbar_arrive_expect_tx(&S.rbar, uint32_t(CS * nq * (32 + 16 * ncols)));
        if (qmode >= 1) {
            // query staging barrier: the group's gs rows land by one bulk copy (the cluster
            // barrier below orders this init before any multicast from rank 0)
            mbar_init(&S.qbar, 1);
            mbar_fence_init();
            mbar_arrive_expect_tx(&S.qbar, uint32_t(gs * d * 2));
        }
    }
    // first phase of the cluster barrier: every CTA has started and initialised its receive
    // barrier before any DSMEM copy (waited on before griddepcontrol.wait, off the critical path)
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");

    const int L = L_old + (append ? 1 : 0);
    const int nblk = (L + kBlk - 1) / kBlk;
    const int c_lo = (nblk * rank) / CS, c_hi = (nblk * (rank + 1)) / CS;
    const int w_lo = c_lo + ((c_hi - c_lo) * warp) / W, w_hi = c_lo + ((c_hi - c_lo) * (warp + 1)) / W;
    const int nb = w_hi - w_lo;

    uint64_t* bars = S.bar[warp];
    const uint32_t slot0 = smem_u32(ring);
    auto issue = [&](int j) {  // lane 0: block w_lo + j into slot j % nslots
        const int s = j % nslots;
        const int row = base + (w_lo + j) * kBlk;
        mbar_arrive_expect_tx(&bars[s], 2 * kBoxBytes);
        const uint64_t pol = policy_evict_first();
        tma_load_3d(ring + s * 2 * kBoxBytes, &tm_k, 0, 0, row, &bars[s], pol);
        tma_load_3d(ring + s * 2 * kBoxBytes + kBoxBytes, &tm_v, 0, 0, row, &bars[s], pol);
    };
    if (lane == 0) {
        for (int s = 0; s < nslots; ++s) mbar_init(&bars[s], 1);
        mbar_fence_init();
        for (int j = 0; j < (nb < nslots ? nb : nslots); ++j) issue(j);
    }
    __syncwarp();
    // warm L2 with this lane's Q row while the previous layer finishes: an L2 prefetch is
    // safe before the dependency wait (it fills no L1 line, and L2 is the point of coherence
    // for the producer's writes), and the loads after the wait then hit L2
    {
        const char* qrow = reinterpret_cast<const char*>(q + (int64_t(p) * H + g * gs + (head_ok ? gid : 0)) * d);
        if (warp == 0 && tig < 2) asm volatile("prefetch.global.L2 [%0];" ::"l"(qrow + 128 * tig) : "memory");
    }
    // register set-up that needs nothing produced upstream: done before the dependency wait
    float m_run = -INFINITY, l_run = 0.f;
    float acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;

    const int rk0 = kperm(gid), rk1 = 8 + kperm(gid);                // K rows of this lane (tiles 0, 1)
    const int rv0 = kperm(2 * tig), rv1 = kperm(2 * tig + 1);         // V rows of key slots 2t, 2t+1 (+8)
    // loop-invariant fragment offsets within a slot (the per-block work is then base + offset)
    uint32_t koff[2][4], voff[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        koff[0][i] = box_off(rk0, i * 4 + tig);
        koff[1][i] = box_off(rk1, i * 4 + tig);
    }
#pragma unroll
    for (int jv = 0; jv < 4; ++jv) {
        const int r = (jv >> 1) * 8 + ((jv & 1) ? rv1 : rv0);
        voff[jv][0] = kBoxBytes + box_off(r, gid);
        voff[jv][1] = kBoxBytes + box_off(r, 8 + gid);
    }
    stamp(1);
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (k_new != nullptr && !append && rank == 0 && threadIdx.x == 0) atomicOr(err, ERR_CAPACITY);
    stamp(2);
    // Q staging: mode 0 -- every lane loads its fragments from global memory (72 warps per
    // group hit the same 1 KB); mode 1 -- one bulk copy per CTA into shared memory; mode 2 --
    // rank 0 multicasts the rows to every CTA of the cluster (one L2 read per group)
    const __nv_bfloat16* qgrp = q + (int64_t(p) * H + g * gs) * d;
    if (threadIdx.x == 0) {
        if (qmode == 1)
            bulk_g2s(smem_u32(S.qs), qgrp, uint32_t(gs * d * 2), smem_u32(&S.qbar));
        else if (qmode == 2 && rank == 0)
            bulk_g2s_mc(smem_u32(S.qs), qgrp, uint32_t(gs * d * 2), smem_u32(&S.qbar), uint16_t((1u << CS) - 1u));
    }

    // Q A-fragments for this group's heads; produced upstream.  Padding rows (gid >= g) load
    // head 0's row too -- their probabilities are forced to zero below -- so the loads are
    // unconditional and nothing waits for them before the first block's MMAs (a predicated
    // load would be materialised with predicated moves that stall right here).
    uint4 qv[4];
    if (qmode == 0) {
        const uint4* qrow = reinterpret_cast<const uint4*>(q + (int64_t(p) * H + g * gs + (head_ok ? gid : 0)) * d);
#pragma unroll
        for (int i = 0; i < 4; ++i) qv[i] = qrow[i * 4 + tig];
    }
    // this lane's 16-byte chunk of the appended row (K for lanes 0-15, V for 16-31), loaded
    // once with Q: the end-of-segment block below only stores it
    uint4 new_chunk = make_uint4(0, 0, 0, 0);
    if (append && nb > 0 && (w_hi * kBlk > L_old))
        new_chunk = reinterpret_cast<const uint4*>((lane < 16 ? k_new : v_new) + int64_t(pg) * d)[lane & 15];
    auto wstamp = [&](int j, int k) {  // (debug) warp 1's first two blocks: cycles per phase
        if (dbg && warp == 1 && lane == 0 && j < 2) dbg[blockIdx.x * 64 + 8 + 4 * j + k] = clock64();
    };
    int s = 0;
    uint32_t sphase = 0;  // slot and mbarrier phase of block j (no division in the loop)
    auto slot_addr = [&](int sl) { return slot0 + uint32_t(sl * 2 * kBoxBytes); };
    // block j's K fragments: wait for its slot (sl, ph), patch the segment end, load K
    auto fetch_k = [&](int j, int sl, uint32_t ph, uint4 (&kv)[2][4]) {
        wstamp(j, 0);
        const int blk = (w_lo + j) * kBlk;
        const uint32_t ks = slot_addr(sl), vs = ks + kBoxBytes;
        mbar_wait(&bars[sl], ph);
        wstamp(j, 1);
        if (blk + kBlk > L_old) {
            // the block holding the end of the segment: the appended row (produced upstream)
            // replaces what TMA fetched at L_old; rows past it are zeroed (V must be finite)
            const uint32_t dst = lane < 16 ? ks : vs;
            for (int rr = (L_old > blk ? L_old - blk : 0); rr < kBlk; ++rr) {
                const bool isnew = append && blk + rr == L_old;
                sts128(dst + box_off(rr, lane & 15), isnew ? new_chunk : make_uint4(0, 0, 0, 0));
            }
            // K5 append, by the warp holding the new row's block: no other CTA's boxes cover
            // it, this CTA's own box has landed, and every CTA of the cluster read seqlens
            // before the cluster barrier, so the row and the length are written here, from
            // the registers already holding the row, instead of at the end of the kernel
            if (append && L_old >= blk) {
                reinterpret_cast<uint4*>((lane < 16 ? k_cache : v_cache) + (int64_t(base) + L_old) * d)[lane & 15] =
                    new_chunk;
                if (lane == 0) seqlens[pg] = L;
            }
            __syncwarp();
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            kv[0][i] = lds128(ks + koff[0][i]);
            kv[1][i] = lds128(ks + koff[1][i]);
        }
    };
    auto load_v = [&](int sl, uint4 (&vv)[4][2]) {
        const uint32_t ks = slot_addr(sl);
#pragma unroll
        for (int jv = 0; jv < 4; ++jv) {
            vv[jv][0] = lds128(ks + voff[jv][0]);
            vv[jv][1] = lds128(ks + voff[jv][1]);
        }
    };
    // the first block's wait and K loads go before the Q fragments are assembled (register
    // moves that wait for the Q loads), so they overlap the Q latency
    uint4 kva[2][4], kvb[2][4];
    if (nb > 0) fetch_k(0, 0, 0u, kva);
    // zdep is always 0 but depends on the fetched fragments, which pins the assembly below
    // after fetch_k(0) (otherwise the compiler hoists it, and with it the wait for Q)
    const uint32_t zdep = (kva[0][0].x == 0x7fc00001u && nslots == -12345) ? 1u : 0u;
    if (qmode >= 1) {
        // every warp waits (also those without blocks: no multicast may land in an exited CTA)
        mbar_wait(&S.qbar, 0);
        if (dbg && warp == 1 && lane == 0) dbg[blockIdx.x * 64 + 14] = clock64();  // (debug) Q landed
        if (dbg && lane == 0) dbg[blockIdx.x * 64 + 32 + 4 * warp] = clock64();
        const uint32_t qrow = smem_u32(S.qs) + uint32_t((head_ok ? gid : 0) * d * 2);
#pragma unroll
        for (int i = 0; i < 4; ++i) qv[i] = lds128(qrow + 16u * uint32_t(i * 4 + tig));
    }
    uint32_t qa0[8], qa2[8];
#pragma unroll
    for (int st = 0; st < 8; ++st) {
        const uint4 w = qv[st >> 1];
        qa0[st] = ((st & 1) ? w.z : w.x) ^ zdep;
        qa2[st] = ((st & 1) ? w.w : w.y) ^ zdep;
    }
    // S = Q K^T of block j: two key tiles x two halves of d -> four independent 4-deep MMA
    // chains; keys past the segment end are masked
    auto scores = [&](int j, const uint4 (&kv)[2][4], float (&x)[4]) {
        const int blk = (w_lo + j) * kBlk;
        float s0a[4] = {0.f, 0.f, 0.f, 0.f}, s1a[4] = {0.f, 0.f, 0.f, 0.f};
        float s0b[4] = {0.f, 0.f, 0.f, 0.f}, s1b[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int st = 0; st < 4; ++st) {
            const uint4 w0a = kv[0][st >> 1], w1a = kv[1][st >> 1];
            const uint4 w0b = kv[0][2 + (st >> 1)], w1b = kv[1][2 + (st >> 1)];
            mma16816(s0a, qa0[st], 0u, qa2[st], 0u, (st & 1) ? w0a.z : w0a.x, (st & 1) ? w0a.w : w0a.y);
            mma16816(s1a, qa0[st], 0u, qa2[st], 0u, (st & 1) ? w1a.z : w1a.x, (st & 1) ? w1a.w : w1a.y);
            mma16816(s0b, qa0[4 + st], 0u, qa2[4 + st], 0u, (st & 1) ? w0b.z : w0b.x, (st & 1) ? w0b.w : w0b.y);
            mma16816(s1b, qa0[4 + st], 0u, qa2[4 + st], 0u, (st & 1) ? w1b.z : w1b.x, (st & 1) ? w1b.w : w1b.y);
        }
        x[0] = s0a[0] + s0b[0];
        x[1] = s0a[1] + s0b[1];
        x[2] = s1a[0] + s1b[0];
        x[3] = s1a[1] + s1b[1];
        if (blk + kBlk > L) {
            if (blk + rv0 >= L) x[0] = -INFINITY;
            if (blk + rv1 >= L) x[1] = -INFINITY;
            if (blk + 8 + rv0 >= L) x[2] = -INFINITY;
            if (blk + 8 + rv1 >= L) x[3] = -INFINITY;
        }
    };
    // online softmax over the keys in x[0..NX) (one or two blocks): lazy running max -- it
    // moves only when the keys exceed it by more than 8 (log2 units), so probabilities stay
    // <= 2^8 and the accumulator is rescaled rarely; the first block needs no rescale
    auto softmax = [&](float* x, int nx) {
        float bm = -INFINITY;
        for (int i = 0; i < nx; ++i) bm = fmaxf(bm, x[i]);
        bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 1));
        bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 2));
        const float m_cand = fmaxf(m_run, bm * scale_log2);
        const bool bump = m_cand > m_run + 8.f;
        const float m_new = bump ? m_cand : m_run;
        const float corr = bump ? ex2f(m_run - m_new) : 1.f;
        const bool rescale = bump && m_run != -INFINITY;
        float lsum = 0.f;
        for (int i = 0; i < nx; ++i) {
            x[i] = head_ok ? ex2f(fmaf(x[i], scale_log2, -m_new)) : 0.f;
            lsum += x[i];
        }
        l_run = l_run * corr + lsum;
        m_run = m_new;
        if (__any_sync(0xffffffffu, head_ok && rescale)) {
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
    };
    // O^T += V^T P^T for one block (p = its four probabilities)
    auto pv = [&](const uint4 (&vv)[4][2], const float* pr) {
        const uint32_t b0 = pack_bf16(pr[0], pr[1]), b1 = pack_bf16(pr[2], pr[3]);
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
    };
    auto advance = [&](int& sl, uint32_t& ph) {
        if (++sl == nslots) {
            sl = 0;
            ph ^= 1u;
        }
    };
    // Blocks are taken two at a time when the warp has two left: both blocks' S chains, one
    // softmax over 32 keys, then both PVs -- the two blocks' latency chains overlap.
    int j = 0;
    while (j < nb) {
        if (kTriple && nb - j == 3 && nslots >= 3) {
            // exactly three left (a warp of a CTA whose block count is not a multiple of 2W):
            // one softmax over 48 keys and three S chains in flight instead of a pair + a single
            int s1 = s, s2;
            uint32_t ph1 = sphase, ph2;
            advance(s1, ph1);
            s2 = s1;
            ph2 = ph1;
            advance(s2, ph2);
            uint4 kvc[2][4];
            fetch_k(j + 1, s1, ph1, kvb);
            fetch_k(j + 2, s2, ph2, kvc);
            float x[12];
            scores(j, kva, *reinterpret_cast<float(*)[4]>(&x[0]));
            scores(j + 1, kvb, *reinterpret_cast<float(*)[4]>(&x[4]));
            scores(j + 2, kvc, *reinterpret_cast<float(*)[4]>(&x[8]));
            softmax(x, 12);
            uint4 vv[4][2];
            load_v(s, vv);
            pv(vv, &x[0]);
            load_v(s1, vv);
            pv(vv, &x[4]);
            load_v(s2, vv);
            pv(vv, &x[8]);
            __syncwarp();
            s = s2;
            sphase = ph2;
            advance(s, sphase);
            j += 3;  // the last blocks of this warp: nothing left to issue
            continue;
        }
        if (j + 1 < nb) {
            int s1 = s;
            uint32_t ph1 = sphase;
            advance(s1, ph1);
            fetch_k(j + 1, s1, ph1, kvb);
            float x[8];
            scores(j, kva, *reinterpret_cast<float(*)[4]>(&x[0]));
            scores(j + 1, kvb, *reinterpret_cast<float(*)[4]>(&x[4]));
            wstamp(j, 2);
            if (dbg && lane == 0 && j == 0) dbg[blockIdx.x * 64 + 33 + 4 * warp] = clock64();
            softmax(x, 8);
            uint4 vv[4][2];
            load_v(s, vv);
            pv(vv, &x[0]);
            load_v(s1, vv);
            pv(vv, &x[4]);
            __syncwarp();  // every lane's reads of both slots have been consumed
            if (lane == 0 && j + nslots < nb) issue(j + nslots);
            if (lane == 0 && j + 1 + nslots < nb) issue(j + 1 + nslots);
            wstamp(j, 3);
            if (dbg && lane == 0 && j == 0) dbg[blockIdx.x * 64 + 34 + 4 * warp] = clock64();
            s = s1;
            sphase = ph1;
            advance(s, sphase);
            j += 2;
        } else {
            float x[4];
            scores(j, kva, x);
            softmax(x, 4);
            uint4 vv[4][2];
            load_v(s, vv);
            pv(vv, x);
            __syncwarp();
            if (lane == 0 && j + nslots < nb) issue(j + nslots);
            advance(s, sphase);
            j += 1;
        }
        if (j < nb) fetch_k(j, s, sphase, kva);
    }
    stamp(3);
    if (dbg && lane == 0 && warp < 8) {  // (debug) every warp's loop end + its block count
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        dbg[blockIdx.x * 64 + 24 + warp] = t;
        dbg[blockIdx.x * 64 + 35 + 4 * warp] = clock64();
    }
    // ---- (1) warp partial -> smem: (m, l) per head; O into the warp's idle ring in a skewed
    // [column][8 heads] layout (8 words of padding per 8 columns, so the lanes' float2 (ha, hb)
    // stores cover 32 distinct banks per half-warp)
    auto so_idx = [](int c, int h) { return c * 8 + 8 * (c >> 3) + h; };
    {
        float* s_o = reinterpret_cast<float*>(ring);
        float lsum = l_run + __shfl_xor_sync(0xffffffffu, l_run, 1);
        lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
        if (tig == 0) {
            S.s_ml[warp][gid][0] = m_run;
            S.s_ml[warp][gid][1] = lsum;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int c0 = v_col(i, gid);  // v_col(i, gid + 8) == c0 + 1
            *reinterpret_cast<float2*>(&s_o[so_idx(c0, 2 * tig)]) = make_float2(acc[i][0], acc[i][1]);
            *reinterpret_cast<float2*>(&s_o[so_idx(c0 + 1, 2 * tig)]) = make_float2(acc[i][2], acc[i][3]);
        }
    }
    __syncthreads();
    stamp(4);
    // ---- (2) CTA merge of the W warp partials: thread -> (column c, head quad hq).  The W x 4
    // per-(warp, head) scales are the same for every column, so each lane of a merging warp
    // computes one of them (lane = 4 w + head; W = 8 covers the warp) and the column loop
    // reads them back as broadcast float4s instead of recomputing 32 exponentials per thread.
    static_assert(W <= 8, "one scale per lane: up to 8 warps x 4 heads");
    {
        const int nq = (gs + 3) >> 2;
        for (int t = threadIdx.x; t < 128 * nq; t += 32 * W) {
            const int hq = t >> 7, c = t & 127;  // head quad is uniform over a warp
            const int fw = lane >> 2, fh = 4 * hq + (lane & 3);
            const float mw = fw < W ? S.s_ml[fw][fh][0] : -INFINITY;
            float M = mw;
            M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, 4));
            M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, 8));
            M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, 16));
            const float f = mw == -INFINITY ? 0.f : ex2f(mw - M);
            float lf = fw < W ? S.s_ml[fw][fh][1] * f : 0.f;
            lf += __shfl_xor_sync(0xffffffffu, lf, 4);
            lf += __shfl_xor_sync(0xffffffffu, lf, 8);
            lf += __shfl_xor_sync(0xffffffffu, lf, 16);  // lanes 0..3: the head's scaled sum
            S.s_f[warp][lane] = f;
            __syncwarp();
            float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int w = 0; w < W; ++w) {
                const float4 fw4 = *reinterpret_cast<const float4*>(&S.s_f[warp][4 * w]);  // broadcast
                const float4 o = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(ring_of(w)) + so_idx(c, 4 * hq));
                O.x += o.x * fw4.x;
                O.y += o.y * fw4.y;
                O.z += o.z * fw4.z;
                O.w += o.w * fw4.w;
            }
            __syncwarp();  // s_f[warp] is rewritten by the next column round
            float Mq[4], Lq[4];
#pragma unroll
            for (int jh = 0; jh < 4; ++jh) {
                Mq[jh] = __shfl_sync(0xffffffffu, M, jh);
                Lq[jh] = __shfl_sync(0xffffffffu, lf, jh);
            }
            const int owner = ((c + 1) * CS - 1) / d, cl = c - (d * owner) / CS;
            // straight into the owner's receive chunk for this rank (DSMEM st.async)
            const uint32_t dst = smem_u32(S.recv + rank * chunk), bar = mapa(smem_u32(&S.rbar), owner);
            st_async_v4(mapa(dst + 4u * uint32_t(16 + cl * 8 + 4 * hq), owner), O, bar);
            if (cl == 0) {
                st_async_v4(mapa(dst + 4u * uint32_t(8 * hq), owner), make_float4(Mq[0], Lq[0], Mq[1], Lq[1]), bar);
                st_async_v4(mapa(dst + 4u * uint32_t(8 * hq + 4), owner), make_float4(Mq[2], Lq[2], Mq[3], Lq[3]), bar);
            }
        }
    }
    stamp(5);
    mbar_wait(&S.rbar, 0);
    stamp(6);
    // ---- (4) this rank's columns: merge the CS chunks
    const int gshift = (gs & (gs - 1)) == 0 ? __ffs(gs) - 1 : -1;  // g a power of two: shifts
    for (int t = threadIdx.x; t < ncols * gs; t += 32 * W) {
        const int cl = gshift >= 0 ? t >> gshift : t / gs, h = gshift >= 0 ? t & (gs - 1) : t % gs;
        float M = -INFINITY;
#pragma unroll
        for (int r = 0; r < CS; ++r) M = fmaxf(M, S.recv[r * chunk + 2 * h]);
        float Ls = 0.f, Os = 0.f;
#pragma unroll
        for (int r = 0; r < CS; ++r) {
            const float* ch = S.recv + r * chunk;
            const float mr = ch[2 * h];
            const float f = mr == -INFINITY ? 0.f : ex2f(mr - M);
            Ls += ch[2 * h + 1] * f;
            Os += ch[16 + cl * 8 + h] * f;
        }
        out[(int64_t(p) * H + g * gs + h) * d + col_lo + cl] = __float2bfloat16_rn(__fdividef(Os, Ls));
    }
    stamp(7);
}

// 3-D view of a cache plane [rows][2 halves][64 bf16] with a {64, 2, 16} box (one 16-row
// block, 4 KB) and 128-byte swizzle; rows past the plane read as zeros.
adakv_status make_cache_map(CUtensorMap* m, const void* plane, int64_t rows) {
    EncodeFn enc = get_encode();
    if (!enc) return fail(ADAKV_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[3] = {64, 2, cuuint64_t(rows)};
    const cuuint64_t strides[2] = {128, 256};
    const cuuint32_t box[3] = {64, 2, kBlk};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(plane), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(ADAKV_CUDA_ERROR, "cuTensorMapEncodeTiled failed (decode cache plane)");
    return ADAKV_OK;
}

}  // namespace

// debug: per-CTA phase timestamps, 64 slots per CTA (scripts/dec_ts4.py sets the buffer)
static unsigned long long* g_dbg = nullptr;
unsigned long long* dbg_buf() { return g_dbg; }
extern "C" void adakv_debug_set_decode_timestamps(void* buf) { g_dbg = static_cast<unsigned long long*>(buf); }

bool decode_tc_supported(adakv_dtype dt, int64_t H, int64_t G, int64_t d, int64_t cache_rows) {
    return dt == ADAKV_BF16 && d == 128 && G > 0 && H % G == 0 && H / G <= 8 && cache_rows < (int64_t(1) << 31) &&
           get_encode() != nullptr;
}

constexpr int kWarpsDec = ADAKV_DECODE_W;
static int decode_warps() { return kWarpsDec; }

using DecodeKernel = decltype(&decode_tc_kernel<1, kWarpsDec>);
template <int... CS>
static DecodeKernel kernel_for_impl(int64_t cs, std::integer_sequence<int, CS...>) {
    DecodeKernel k = nullptr;
    ((cs == CS + 1 ? (k = decode_tc_kernel<CS + 1, kWarpsDec>, 0) : 0), ...);
    return k;
}
static DecodeKernel kernel_for(int64_t cs) { return kernel_for_impl(cs, std::make_integer_sequence<int, kMaxCS>{}); }

// TMA ring depth per warp (ADAKV_DECODE_SLOTS overrides; 2..kMaxSlots)
static int decode_slots() {
    static int n = [] {
        const char* e = std::getenv("ADAKV_DECODE_SLOTS");
        // the rings of all warps within 227 KB of shared memory
        int mx = kMaxSlots;
        while (mx > 1 && dec_smem_bytes(mx, kWarpsDec) > 227 * 1024) --mx;
        const int v = e ? std::atoi(e) : mx;
        // >= 2: a warp takes its blocks two at a time, and both must be in flight at once
        return v < 2 ? 2 : v > mx ? mx : v;
    }();
    return n;
}

// Function attributes are per device: set them once for every device this process uses.
static adakv_status prepare_kernel() {
    static std::mutex mu;
    static uint64_t done_mask = 0;
    int dev = 0;
    ADAKV_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    if (dev < 64 && (done_mask >> dev) & 1) return ADAKV_OK;
    for (int64_t cs = 1; cs <= kMaxCS; ++cs) {
        ADAKV_CUDA_TRY(cudaFuncSetAttribute(kernel_for(cs), cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        ADAKV_CUDA_TRY(cudaFuncSetAttribute(kernel_for(cs), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            int(dec_smem_bytes(decode_slots(), decode_warps()))));
    }
    if (dev < 64) done_mask |= uint64_t(1) << dev;
    return ADAKV_OK;
}

// CTAs per cluster (one cluster per (problem, group)), from cudaOccupancyMaxActiveClusters;
// ADAKV_DECODE_CS overrides.
int64_t decode_tc_cluster(int64_t P, int64_t G) {
    static std::mutex mu;
    static int64_t cached_segs = -1, cached_cs = 1;
    static int cached_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    const int64_t segs = std::max<int64_t>(1, P * G);
    if (segs == cached_segs && dev == cached_dev) return cached_cs;
    if (prepare_kernel() != ADAKV_OK) return 1;
    // active clusters the device can hold for each size
    int64_t fit[kMaxCS + 1] = {};
    for (int64_t cs = 2; cs <= kMaxCS; ++cs) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(segs * cs));
        cfg.blockDim = dim3(32 * decode_warps());
        cfg.dynamicSmemBytes = dec_smem_bytes(decode_slots(), decode_warps());
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = unsigned(cs);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, kernel_for(cs), &cfg) == cudaSuccess) fit[cs] = n;
        cudaGetLastError();
    }
    // The largest size for which every cluster of one launch is co-resident -- or one size
    // smaller when that lets two launches' CTAs share the SMs (one CTA each), so every CTA of
    // the next layer's launch starts, and prefetches, while this one runs: config 2 measures
    // 4.11 us per step-layer at 9 against 4.13 at 10.  Smaller still costs more in per-CTA
    // work than the earlier start saves.
    if (std::getenv("ADAKV_DEBUG_FIT"))
        for (int64_t cs = 2; cs <= kMaxCS; ++cs) std::fprintf(stderr, "decode cluster fit cs=%lld: %lld\n", (long long)cs, (long long)fit[cs]);
    int64_t best = 1;
    for (int64_t cs = kMaxCS; cs >= 2 && best == 1; --cs)
        if (fit[cs] >= segs) best = cs;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (best > 2 && 2 * segs * (best - 1) <= sms && 2 * segs * best > sms) best -= 1;
    if (const char* e = std::getenv("ADAKV_DECODE_CS")) {
        const int64_t v = std::atoi(e);
        if (v >= 1 && v <= kMaxCS) best = v;
    }
    cached_segs = segs;
    cached_dev = dev;
    cached_cs = best;
    return best;
}

size_t decode_tc_workspace(int64_t, int64_t, int64_t, int64_t) { return 256; }

extern "C" int adakv_debug_decode_cluster(int64_t P, int64_t G) { return int(decode_tc_cluster(P, G)); }

adakv_status launch_decode_tc(int64_t P, int64_t H, int64_t G, int32_t scale, const void* q, void* kc, void* vc,
                              int64_t cache_rows, const int32_t* ss, const int32_t* cap, int32_t* sl,
                              const void* kn, const void* vn, void* out, uint32_t* err, bool overlap_prev,
                              cudaStream_t stream) {
    ADAKV_TRY(prepare_kernel());
    // tensor maps of the two planes (one pair serves every layer of a model-wide plane)
    static std::mutex mu;
    static const void* c_k = nullptr;
    static const void* c_v = nullptr;
    static int64_t c_rows = -1;
    static CUtensorMap c_tk, c_tv;
    CUtensorMap tk, tv;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (kc != c_k || vc != c_v || cache_rows != c_rows) {
            ADAKV_TRY(make_cache_map(&c_tk, kc, cache_rows));
            ADAKV_TRY(make_cache_map(&c_tv, vc, cache_rows));
            c_k = kc;
            c_v = vc;
            c_rows = cache_rows;
        }
        tk = c_tk;
        tv = c_tv;
    }
    const float sc = (scale ? 1.0f / sqrtf(128.f) : 1.0f) * 1.4426950408889634f;
    const int64_t cs = decode_tc_cluster(P, G);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(P * G * cs));
    cfg.blockDim = dim3(32 * decode_warps());
    const int nslots = decode_slots();
    static const int qmode = [] {
        const char* e = std::getenv("ADAKV_DECODE_QMODE");
        const int v = e ? std::atoi(e) : 2;
        return v < 0 || v > 2 ? 2 : v;
    }();
    cfg.dynamicSmemBytes = dec_smem_bytes(nslots, decode_warps());
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
    ADAKV_CUDA_TRY(cudaLaunchKernelEx(&cfg, kernel_for(cs), tk, tv, static_cast<const __nv_bfloat16*>(q),
                                      static_cast<__nv_bfloat16*>(kc), static_cast<__nv_bfloat16*>(vc), ss, cap, sl,
                                      static_cast<const __nv_bfloat16*>(kn), static_cast<const __nv_bfloat16*>(vn),
                                      static_cast<__nv_bfloat16*>(out), err, int(H), int(G), sc, nslots, cs > 1 ? qmode : (qmode ? 1 : 0), dbg_buf()));
    return ADAKV_OK;
}

}  // namespace adakv_b200
