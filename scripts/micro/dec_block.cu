// Per-block cost of the decode inner loop (decode_tc.cu) with the data already in shared
// memory: W warps each run NB 16-row blocks (S = QK^T, online softmax, O += PV) from a
// swizzled K/V box; prints cycles per block for W = 1, 2, 4, 8.  Variants: full body,
// S only (no softmax/PV), LDS only.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_bf16.h>

constexpr int kBlk = 16, kBoxBytes = kBlk * 256;
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) { uint32_t r; asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo)); return r; }
__device__ __forceinline__ float ex2f(float x) { float r; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
__device__ __forceinline__ uint4 lds128(uint32_t addr) { uint4 v; asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr)); return v; }
__device__ __forceinline__ uint32_t box_off(int r, int c) { const int line = 2 * r + (c >> 3); return uint32_t(line * 128 + (((c & 7) ^ (line & 7)) << 4)); }
__device__ __forceinline__ int kperm(int n) { const int t = n >> 1, e = n & 1; return (e << 2) | (t ^ (e << 1)); }

template <int MODE>
__global__ void k(long long* out, int nblk, int nslots, float scale_log2, int reps) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
    for (int i = threadIdx.x; i < (int)(blockDim.x / 32) * nslots * 2 * kBoxBytes / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
    __syncthreads();
    const uint32_t slot0 = (uint32_t)__cvta_generic_to_shared(sm) + warp * nslots * 2 * kBoxBytes;
    uint32_t qa0[8], qa2[8];
    for (int s = 0; s < 8; ++s) { qa0[s] = 0x3c003c00u + lane; qa2[s] = 0x3c003c00u + s; }
    const int rk0 = kperm(gid), rk1 = 8 + kperm(gid), rv0 = kperm(2 * tig), rv1 = kperm(2 * tig + 1);
    uint32_t koff[2][4], voff[4][2];
    for (int i = 0; i < 4; ++i) { koff[0][i] = box_off(rk0, i * 4 + tig); koff[1][i] = box_off(rk1, i * 4 + tig); }
    for (int jv = 0; jv < 4; ++jv) { const int r = (jv >> 1) * 8 + ((jv & 1) ? rv1 : rv0); voff[jv][0] = kBoxBytes + box_off(r, gid); voff[jv][1] = kBoxBytes + box_off(r, 8 + gid); }
    float m_run = -INFINITY, l_run = 0.f, acc[8][4] = {};
    float sink = 0.f;
    __syncthreads();
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
    if (rep == reps - 1) t0 = clock64();
    if (MODE == 3 || MODE == 6) {
        // K as the A operand (rows = keys): lane reads row gid and gid+8, 4 chunks each
        uint32_t ka[2][4];
        const int rho = (gid & 4) | ((gid & 1) << 1) | ((gid >> 1) & 1);  // quarter-warp rows {r, r+2}
        for (int i = 0; i < 4; ++i) {
            const int rr = MODE == 6 ? rho : gid;
            ka[0][i] = box_off(rr, i * 4 + tig); ka[1][i] = box_off(rr + 8, i * 4 + tig);
        }
        uint32_t qb[8][2];
        for (int st = 0; st < 8; ++st) { qb[st][0] = 0x3c003c00u + lane; qb[st][1] = 0x3c003c00u + st; }
        const int tsrc = ((gid & 3) >> 1) | ((gid & 1) << 1);  // lane (quad) publishing head gid&3
        const int srcA = (2 * tig) * 4 + tsrc, srcB = (2 * tig + 1) * 4 + tsrc;
        float mh[2] = {-INFINITY, -INFINITY}, lh[2] = {0.f, 0.f};
        for (int j = 0; j < nblk; ++j) {
            const int s = j % nslots;
            const uint32_t ks = slot0 + uint32_t(s * 2 * kBoxBytes);
            uint4 kv[2][4], vv[4][2];
#pragma unroll
            for (int i = 0; i < 4; ++i) { kv[0][i] = lds128(ks + ka[0][i]); kv[1][i] = lds128(ks + ka[1][i]); }
#pragma unroll
            for (int jv = 0; jv < 4; ++jv) { vv[jv][0] = lds128(ks + voff[jv][0]); vv[jv][1] = lds128(ks + voff[jv][1]); }
            float sa[4] = {}, sb[4] = {};
#pragma unroll
            for (int st = 0; st < 8; st += 2) {
                const uint4 r0 = kv[0][st >> 1], r8 = kv[1][st >> 1];
                mma16816(sa, r0.x, r8.x, r0.y, r8.y, qb[st][0], qb[st][1]);
                mma16816(sb, r0.z, r8.z, r0.w, r8.w, qb[st + 1][0], qb[st + 1][1]);
            }
            // lane (g, t): S^T[key g][heads 2(t&1), +1], S^T[key g+8][same]
            float x[4] = {sa[0] + sb[0], sa[1] + sb[1], sa[2] + sb[2], sa[3] + sb[3]};
            float bm0 = fmaxf(x[0], x[2]), bm1 = fmaxf(x[1], x[3]);
            const bool over = bm0 * scale_log2 > mh[0] + 8.f || bm1 * scale_log2 > mh[1] + 8.f;
            if (MODE == 3 || __any_sync(0xffffffffu, over)) {
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
                bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, o));
                bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, o));
            }
            } else { bm0 = -INFINITY; bm1 = -INFINITY; }
            float corr[2], mnew[2];
            bool resc = false;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const float mc = fmaxf(mh[e], (e ? bm1 : bm0) * scale_log2);
                const bool bump = mc > mh[e] + 8.f;
                mnew[e] = bump ? mc : mh[e];
                corr[e] = bump ? ex2f(mh[e] - mnew[e]) : 1.f;
                resc |= bump && mh[e] != -INFINITY;
            }
            const float p0 = ex2f(fmaf(x[0], scale_log2, -mnew[0])), p1 = ex2f(fmaf(x[1], scale_log2, -mnew[1]));
            const float p2 = ex2f(fmaf(x[2], scale_log2, -mnew[0])), p3 = ex2f(fmaf(x[3], scale_log2, -mnew[1]));
            lh[0] = lh[0] * corr[0] + (p0 + p2);
            lh[1] = lh[1] * corr[1] + (p1 + p3);
            mh[0] = mnew[0];
            mh[1] = mnew[1];
            if (__any_sync(0xffffffffu, resc)) {
#pragma unroll
                for (int i = 0; i < 8; ++i) { acc[i][0] *= corr[0]; acc[i][1] *= corr[1]; acc[i][2] *= corr[0]; acc[i][3] *= corr[1]; }
            }
            // publish head (t>>1) of this lane's pair as (key g, key g+8); pull keys 2t', 2t'+1 (+8)
            const uint32_t wpub = (tig >> 1) ? pack_bf16(p1, p3) : pack_bf16(p0, p2);
            const uint32_t wa = __shfl_sync(0xffffffffu, wpub, srcA), wb = __shfl_sync(0xffffffffu, wpub, srcB);
            const uint32_t b0 = __byte_perm(wa, wb, 0x5410), b1 = __byte_perm(wa, wb, 0x7632);
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
            __syncwarp();
        }
        l_run = lh[0] + lh[1];
    } else
    if (MODE == 8) {
        for (int j = 0; j < nblk; j += 2) {
            uint4 kv[2][2][4], vv[2][4][2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const uint32_t ks = slot0 + uint32_t(((j + u) % nslots) * 2 * kBoxBytes);
#pragma unroll
                for (int i = 0; i < 4; ++i) { kv[u][0][i] = lds128(ks + koff[0][i]); kv[u][1][i] = lds128(ks + koff[1][i]); }
#pragma unroll
                for (int jv = 0; jv < 4; ++jv) { vv[u][jv][0] = lds128(ks + voff[jv][0]); vv[u][jv][1] = lds128(ks + voff[jv][1]); }
            }
            float x[2][4];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                float s0a[4] = {}, s1a[4] = {}, s0b[4] = {}, s1b[4] = {};
#pragma unroll
                for (int st = 0; st < 4; ++st) {
                    const uint4 w0a = kv[u][0][st >> 1], w1a = kv[u][1][st >> 1], w0b = kv[u][0][2 + (st >> 1)], w1b = kv[u][1][2 + (st >> 1)];
                    mma16816(s0a, qa0[st], 0u, qa2[st], 0u, (st & 1) ? w0a.z : w0a.x, (st & 1) ? w0a.w : w0a.y);
                    mma16816(s1a, qa0[st], 0u, qa2[st], 0u, (st & 1) ? w1a.z : w1a.x, (st & 1) ? w1a.w : w1a.y);
                    mma16816(s0b, qa0[4 + st], 0u, qa2[4 + st], 0u, (st & 1) ? w0b.z : w0b.x, (st & 1) ? w0b.w : w0b.y);
                    mma16816(s1b, qa0[4 + st], 0u, qa2[4 + st], 0u, (st & 1) ? w1b.z : w1b.x, (st & 1) ? w1b.w : w1b.y);
                }
                x[u][0] = s0a[0] + s0b[0]; x[u][1] = s0a[1] + s0b[1]; x[u][2] = s1a[0] + s1b[0]; x[u][3] = s1a[1] + s1b[1];
            }
            float bm = fmaxf(fmaxf(fmaxf(x[0][0], x[0][1]), fmaxf(x[0][2], x[0][3])), fmaxf(fmaxf(x[1][0], x[1][1]), fmaxf(x[1][2], x[1][3])));
            bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 1));
            bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 2));
            const float m_cand = fmaxf(m_run, bm * scale_log2);
            const bool bump = m_cand > m_run + 8.f;
            const float m_new = bump ? m_cand : m_run;
            const float corr = bump ? ex2f(m_run - m_new) : 1.f;
            const bool rescale = bump && m_run != -INFINITY;
            float pp[2][4];
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int e = 0; e < 4; ++e) pp[u][e] = ex2f(fmaf(x[u][e], scale_log2, -m_new));
            l_run = l_run * corr + ((pp[0][0] + pp[0][1]) + (pp[0][2] + pp[0][3])) + ((pp[1][0] + pp[1][1]) + (pp[1][2] + pp[1][3]));
            m_run = m_new;
            if (__any_sync(0xffffffffu, rescale)) {
                const float ca = __shfl_sync(0xffffffffu, corr, 8 * tig), cb = __shfl_sync(0xffffffffu, corr, 8 * tig + 4);
#pragma unroll
                for (int i = 0; i < 8; ++i) { acc[i][0] *= ca; acc[i][1] *= cb; acc[i][2] *= ca; acc[i][3] *= cb; }
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const uint32_t b0 = pack_bf16(pp[u][0], pp[u][1]), b1 = pack_bf16(pp[u][2], pp[u][3]);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int h = i >> 2, wd = i & 3;
                    const uint32_t* r0w = reinterpret_cast<const uint32_t*>(&vv[u][0][h]);
                    const uint32_t* r1w = reinterpret_cast<const uint32_t*>(&vv[u][1][h]);
                    const uint32_t* r8w = reinterpret_cast<const uint32_t*>(&vv[u][2][h]);
                    const uint32_t* r9w = reinterpret_cast<const uint32_t*>(&vv[u][3][h]);
                    mma16816(acc[i], __byte_perm(r0w[wd], r1w[wd], 0x5410), __byte_perm(r0w[wd], r1w[wd], 0x7632),
                             __byte_perm(r8w[wd], r9w[wd], 0x5410), __byte_perm(r8w[wd], r9w[wd], 0x7632), b0, b1);
                }
            }
            __syncwarp();
        }
    } else
    for (int j = 0; j < nblk; ++j) {
        const int s = j % nslots;
        const uint32_t ks = slot0 + uint32_t(s * 2 * kBoxBytes);
        uint4 kv[2][4], vv[4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (MODE == 5) { kv[0][i] = make_uint4(ks + i, j, lane, 7); kv[1][i] = make_uint4(ks, i, j, lane); }
            else { kv[0][i] = lds128(ks + koff[0][i]); kv[1][i] = lds128(ks + koff[1][i]); }
        }
#pragma unroll
        for (int jv = 0; jv < 4; ++jv) {
            if (MODE == 5) { vv[jv][0] = make_uint4(ks + jv, j, lane, 9); vv[jv][1] = make_uint4(ks, jv, j, lane); }
            else { vv[jv][0] = lds128(ks + voff[jv][0]); vv[jv][1] = lds128(ks + voff[jv][1]); }
        }
        if (MODE == 2) { sink += __uint_as_float(kv[0][0].x ^ kv[1][3].w ^ vv[0][0].x ^ vv[3][1].y); continue; }
        float x0, x1, x2, x3;
        if (MODE == 4) {  // 8 chains of depth 2
            float c[8][4] = {};
#pragma unroll
            for (int st = 0; st < 8; ++st) {
                const int ch = st >> 1;  // chain per (k half) x tile
                const uint4 w0 = kv[0][st >> 1], w1 = kv[1][st >> 1];
                mma16816(c[ch], qa0[st], 0u, qa2[st], 0u, (st & 1) ? w0.z : w0.x, (st & 1) ? w0.w : w0.y);
                mma16816(c[4 + ch], qa0[st], 0u, qa2[st], 0u, (st & 1) ? w1.z : w1.x, (st & 1) ? w1.w : w1.y);
            }
            x0 = (c[0][0] + c[1][0]) + (c[2][0] + c[3][0]);
            x1 = (c[0][1] + c[1][1]) + (c[2][1] + c[3][1]);
            x2 = (c[4][0] + c[5][0]) + (c[6][0] + c[7][0]);
            x3 = (c[4][1] + c[5][1]) + (c[6][1] + c[7][1]);
        } else {
        float s0a[4] = {}, s1a[4] = {}, s0b[4] = {}, s1b[4] = {};
#pragma unroll
        for (int st = 0; st < 4; ++st) {
            const uint4 w0a = kv[0][st >> 1], w1a = kv[1][st >> 1], w0b = kv[0][2 + (st >> 1)], w1b = kv[1][2 + (st >> 1)];
            mma16816(s0a, qa0[st], 0u, qa2[st], 0u, (st & 1) ? w0a.z : w0a.x, (st & 1) ? w0a.w : w0a.y);
            mma16816(s1a, qa0[st], 0u, qa2[st], 0u, (st & 1) ? w1a.z : w1a.x, (st & 1) ? w1a.w : w1a.y);
            mma16816(s0b, qa0[4 + st], 0u, qa2[4 + st], 0u, (st & 1) ? w0b.z : w0b.x, (st & 1) ? w0b.w : w0b.y);
            mma16816(s1b, qa0[4 + st], 0u, qa2[4 + st], 0u, (st & 1) ? w1b.z : w1b.x, (st & 1) ? w1b.w : w1b.y);
        }
        x0 = s0a[0] + s0b[0]; x1 = s0a[1] + s0b[1]; x2 = s1a[0] + s1b[0]; x3 = s1a[1] + s1b[1];
        }
        if (MODE == 1) { sink += x0 + x1 + x2 + x3 + __uint_as_float(vv[0][0].x ^ vv[3][1].y); continue; }
        float bm = fmaxf(fmaxf(x0, x1), fmaxf(x2, x3));
        if (MODE != 7 || __any_sync(0xffffffffu, bm * scale_log2 > m_run + 8.f)) {
            bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 1));
            bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 2));
        } else bm = -INFINITY;
        const float m_cand = fmaxf(m_run, bm * scale_log2);
        const bool bump = m_cand > m_run + 8.f;
        const float m_new = bump ? m_cand : m_run;
        const float corr = bump ? ex2f(m_run - m_new) : 1.f;
        const bool rescale = bump && m_run != -INFINITY;
        float p0 = ex2f(fmaf(x0, scale_log2, -m_new)), p1 = ex2f(fmaf(x1, scale_log2, -m_new));
        float p2 = ex2f(fmaf(x2, scale_log2, -m_new)), p3 = ex2f(fmaf(x3, scale_log2, -m_new));
        l_run = l_run * corr + ((p0 + p1) + (p2 + p3));
        m_run = m_new;
        if (__any_sync(0xffffffffu, rescale)) {
            const float ca = __shfl_sync(0xffffffffu, corr, 8 * tig), cb = __shfl_sync(0xffffffffu, corr, 8 * tig + 4);
#pragma unroll
            for (int i = 0; i < 8; ++i) { acc[i][0] *= ca; acc[i][1] *= cb; acc[i][2] *= ca; acc[i][3] *= cb; }
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
        __syncwarp();
    }
    for (int i = 0; i < 8; ++i) sink += acc[i][0] + acc[i][3];
    }  // reps
    const long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * 64 + warp] = t1 - t0;
    if (sink == 1234.5f + l_run) out[0] = 0;
}

int main() {
    long long* d; cudaMalloc(&d, 64 * 64 * sizeof(long long));
    const int nslots = 3;
    const int nblk = getenv("NBLK") ? atoi(getenv("NBLK")) : 64;
    const int reps = getenv("REPS") ? atoi(getenv("REPS")) : 1;
    for (int mode : {0, 1, 2, 7, 8}) {
        for (int W : {1, 2, 4, 8, 12, 16}) {
            const int ns = W <= 8 ? nslots : (W <= 12 ? 2 : 1);  // the rings within 227 KB
            const size_t smem = size_t(W) * ns * 2 * kBoxBytes + 1024;
            auto kern = mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : mode == 7 ? k<7> : k<8>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (smem > 227 * 1024) continue;
            kern<<<1, 32 * W, smem>>>(d, nblk, ns, 0.127f, reps);
            kern<<<1, 32 * W, smem>>>(d, nblk, ns, 0.127f, reps);
            if (cudaGetLastError() != cudaSuccess) { printf("W=%d launch failed\n", W); continue; }
            long long h[64]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            long long mx = 0; for (int w = 0; w < W; ++w) mx = h[w] > mx ? h[w] : mx;
            printf("mode %d (%s) W=%2d: %6.1f cycles/block/warp  (smem %.0f B/clk)\n", mode, mode == 0 ? "full" : mode == 1 ? "S+LDS" : mode == 2 ? "LDS" : mode == 3 ? "S^T full" : mode == 7 ? "vote-max" : "pairs", W,
                   double(mx) / nblk, double(W) * nblk * 8192 / double(mx));
        }
    }
    cudaError_t e = cudaDeviceSynchronize(); printf("%s\n", cudaGetErrorString(e));
}
