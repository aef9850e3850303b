// decode.cu -- K4 split-K varlen flash-decoding over the compressed cache, with
// the K5 append fused in.
//
// Replaces, for one new token per problem, attention_weights (attention.hpp:169-179:
// softmax of q.K^T/sqrt(d) over the head's retained keys) followed by
// row_times(a, V) (matrix.hpp:79-89), the context half of attention_output
// (attention.hpp:182-196) as applied to the retained cache in report.hpp:133-144;
// and append_kv (attention.hpp:126-134, the new row goes at the END of the head's
// rows, i.e. after the window rows).
//
// Grid (split, group, problem).  Each CTA streams one chunk of one KV group's
// variable-length segment ONCE for all g = H/G query heads of the group (GQA
// sharing), keeping a per-head online softmax (running max, sum, context) in
// registers; partials go to the workspace and the last CTA of each (p, g) to
// finish (atomic ticket) merges them, writes out[p, h, :], bumps seqlens and
// re-arms the ticket -- one launch per decode step, graph-capturable (the grid is
// sized from max_rows, so lengths can grow on the device between replays).
#include <algorithm>

#include "common.cuh"

namespace adakv_b200 {

namespace {

constexpr int kDecThreads = 128;
constexpr int kDecWarps = kDecThreads / 32;
constexpr int kMaxGroupHeads = 16;

template <class T, class A, int J, int GH>
__global__ void __launch_bounds__(kDecThreads)
decode_kernel(const T* __restrict__ q, T* __restrict__ k_cache, T* __restrict__ v_cache,
              const int32_t* __restrict__ seg_start, const int32_t* __restrict__ seg_cap,
              int32_t* __restrict__ seqlens, const T* __restrict__ k_new, const T* __restrict__ v_new,
              T* __restrict__ out, int64_t H, int64_t G, int64_t d, A inv_scale, int64_t chunk,
              A* __restrict__ part_ml, A* __restrict__ part_o, uint32_t* __restrict__ tickets,
              uint32_t* __restrict__ err) {
    const int64_t split = blockIdx.x, g = blockIdx.y, p = blockIdx.z;
    const int64_t nsplit = gridDim.x;
    const int64_t gs = H / G;
    const int64_t pg = p * G + g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t L_old = seqlens[pg];
    // append_kv into a full segment is refused (no write past its capacity); the step then
    // attends the existing rows and the error is latched for adakv_workspace_status
    const bool append = k_new != nullptr && L_old < seg_cap[pg];
    if (k_new != nullptr && !append && split == 0 && threadIdx.x == 0) atomicOr(err, ERR_CAPACITY);
    const int64_t L = L_old + (append ? 1 : 0);
    const int64_t base = seg_start[pg];
    const T* kn = append ? k_new + pg * d : nullptr;
    const T* vn = append ? v_new + pg * d : nullptr;

    extern __shared__ __align__(16) unsigned char dsm[];
    A (*s_q)[32 * J] = reinterpret_cast<A (*)[32 * J]>(dsm);                       // [GH][32J]
    A (*s_o)[GH][32 * J] = reinterpret_cast<A (*)[GH][32 * J]>(dsm + sizeof(A) * GH * 32 * J);  // [W][GH][32J]
    __shared__ A s_m[kDecWarps][GH], s_l[kDecWarps][GH];
    __shared__ bool s_last;

    for (int64_t i = tid; i < GH * 32 * J; i += kDecThreads) s_q[i / (32 * J)][i % (32 * J)] = A(0);
    __syncthreads();
    for (int64_t i = tid; i < gs * d; i += kDecThreads)
        s_q[i / d][i % d] = A(to_acc(q[(p * H + g * gs) * d + i]));
    if (append && split == 0) {  // K5: the new token lands after the window rows
        for (int64_t i = tid; i < d; i += kDecThreads) {
            k_cache[(base + L_old) * d + i] = kn[i];
            v_cache[(base + L_old) * d + i] = vn[i];
        }
    }
    __syncthreads();

    A m_run[GH], l_run[GH], o_run[GH][J];
#pragma unroll
    for (int h = 0; h < GH; ++h) {
        m_run[h] = -INFINITY;
        l_run[h] = A(0);
#pragma unroll
        for (int j = 0; j < J; ++j) o_run[h][j] = A(0);
    }
    const int64_t r0 = split * chunk, r1 = min(r0 + chunk, L);
    for (int64_t r = r0 + warp; r < r1; r += kDecWarps) {
        const T* krow = (append && r == L_old) ? kn : k_cache + (base + r) * d;
        const T* vrow = (append && r == L_old) ? vn : v_cache + (base + r) * d;
        A kx[J], vx[J];
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int64_t c = int64_t(lane) * J + j;
            kx[j] = c < d ? A(to_acc(krow[c])) : A(0);
            vx[j] = c < d ? A(to_acc(vrow[c])) : A(0);
        }
#pragma unroll
        for (int h = 0; h < GH; ++h) {
            if (h >= gs) break;
            A s = A(0);
#pragma unroll
            for (int j = 0; j < J; ++j) s += s_q[h][lane * J + j] * kx[j];
#pragma unroll
            for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            s *= inv_scale;
            const A nm = s > m_run[h] ? s : m_run[h];
            const A corr = acc_exp(m_run[h] - nm);
            const A pr = acc_exp(s - nm);
            l_run[h] = l_run[h] * corr + pr;
#pragma unroll
            for (int j = 0; j < J; ++j) o_run[h][j] = o_run[h][j] * corr + pr * vx[j];
            m_run[h] = nm;
        }
    }
    // merge the warps
#pragma unroll
    for (int h = 0; h < GH; ++h) {
        if (h >= gs) break;
        if (lane == 0) {
            s_m[warp][h] = m_run[h];
            s_l[warp][h] = l_run[h];
        }
#pragma unroll
        for (int j = 0; j < J; ++j) s_o[warp][h][lane * J + j] = o_run[h][j];
    }
    __syncthreads();
    for (int64_t i = tid; i < gs * d; i += kDecThreads) {
        const int64_t h = i / d, c = i % d;
        A M = -INFINITY;
        for (int w = 0; w < kDecWarps; ++w) M = s_m[w][h] > M ? s_m[w][h] : M;
        A Ls = A(0), Os = A(0);
        for (int w = 0; w < kDecWarps; ++w) {
            if (s_m[w][h] == A(-INFINITY)) continue;
            const A f = acc_exp(s_m[w][h] - M);
            Ls += s_l[w][h] * f;
            Os += s_o[w][h][c] * f;
        }
        const int64_t slot = (pg * nsplit + split) * gs + h;
        part_o[slot * d + c] = Os;
        if (c == 0) {
            part_ml[slot * 2 + 0] = M;
            part_ml[slot * 2 + 1] = Ls;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // one fence + ticket per CTA (grid-sync pattern)
        __threadfence();
        s_last = atomicAdd(&tickets[pg], 1u) == uint32_t(nsplit - 1);
        if (s_last) __threadfence();
    }
    __syncthreads();
    if (!s_last) return;
    for (int64_t i = tid; i < gs * d; i += kDecThreads) {
        const int64_t h = i / d, c = i % d;
        A M = -INFINITY;
        for (int64_t sp = 0; sp < nsplit; ++sp) {
            const A mm = part_ml[((pg * nsplit + sp) * gs + h) * 2];
            M = mm > M ? mm : M;
        }
        A Ls = A(0), Os = A(0);
        for (int64_t sp = 0; sp < nsplit; ++sp) {
            const int64_t slot = (pg * nsplit + sp) * gs + h;
            const A mm = part_ml[slot * 2];
            if (mm == A(-INFINITY)) continue;
            const A f = acc_exp(mm - M);
            Ls += part_ml[slot * 2 + 1] * f;
            Os += part_o[slot * d + c] * f;
        }
        out[(p * H + g * gs + h) * d + c] = from_acc<T>(Os / Ls);
    }
    if (tid == 0) {
        tickets[pg] = 0u;
        if (append) seqlens[pg] = int32_t(L);
    }
}

// append_kv (attention.hpp:126-134), `rows` rows per segment: block s appends
// new[s, 0..rows) after the segment's current end and advances seqlens[s] by rows.
__global__ void append_kernel(int64_t segments, int64_t rows, int64_t d, const int32_t* __restrict__ seg_start,
                              const int32_t* __restrict__ seg_cap, int32_t* __restrict__ seqlens,
                              const uint16_t* __restrict__ kn, const uint16_t* __restrict__ vn,
                              uint16_t* __restrict__ kc, uint16_t* __restrict__ vc, int64_t esz_units,
                              uint32_t* __restrict__ err) {
    const int64_t s = blockIdx.x;
    if (int64_t(seqlens[s]) + rows > int64_t(seg_cap[s])) {  // capacity exhausted: refuse, latch
        if (threadIdx.x == 0) atomicOr(err, ERR_CAPACITY);
        return;
    }
    const int64_t row0 = int64_t(seg_start[s]) + seqlens[s];
    ADAKV_DCHECK(seqlens[s] >= 0 && row0 + rows <= int64_t(seg_start[s]) + seg_cap[s]);
    const int64_t w = d * esz_units;  // row width in 16-bit units
    for (int64_t i = threadIdx.x; i < rows * w; i += blockDim.x) {
        kc[row0 * w + i] = kn[s * rows * w + i];
        vc[row0 * w + i] = vn[s * rows * w + i];
    }
    __syncthreads();
    if (threadIdx.x == 0) seqlens[s] += int32_t(rows);
}

template <class T, int J, int GH>
adakv_status launch_t(int64_t P, int64_t H, int64_t G, int64_t d, int32_t scale, const void* q,
                      void* kc, void* vc, const int32_t* ss, const int32_t* cap, int32_t* sl, int64_t max_rows,
                      const void* kn, const void* vn, void* out, void* ws, uint32_t* err, int64_t chunk,
                      int64_t nsplit, cudaStream_t stream) {
    using A = typename Acc<T>::type;
    Arena ar(ws);
    uint32_t* tickets = ar.take<uint32_t>(size_t(P * G));
    A* part_ml = ar.take<A>(size_t(P * G * nsplit * (H / G) * 2));
    A* part_o = ar.take<A>(size_t(P * G * nsplit * (H / G) * d));
    const A inv = scale ? A(1) / sqrt(A(d)) : A(1);
    const dim3 grid{unsigned(nsplit), unsigned(G), unsigned(P)};
    const size_t smem = sizeof(A) * (GH * 32 * J + kDecWarps * GH * 32 * J);
    auto kfn = decode_kernel<T, A, J, GH>;
    ADAKV_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kfn<<<grid, kDecThreads, smem, stream>>>(
        static_cast<const T*>(q), static_cast<T*>(kc), static_cast<T*>(vc), ss, cap, sl,
        static_cast<const T*>(kn), static_cast<const T*>(vn), static_cast<T*>(out), H, G, d, inv,
        chunk, part_ml, part_o, tickets, err);
    ADAKV_CUDA_TRY(cudaGetLastError());
    (void)max_rows;
    return ADAKV_OK;
}

}  // namespace

void decode_plan(int64_t P, int64_t G, int64_t max_rows, int64_t* chunk, int64_t* nsplit) {
    // ~1.5 CTAs per SM over the P*G segments; chunks of >= 128 rows (multiples of 64,
    // 16-row blocks x 4 warps); at most 64 splits per segment (the combine's fan-in).
    const int64_t sms = device_sm_count();
    const int64_t segs = P * G > 0 ? P * G : 1;
    const int64_t rows = max_rows > 0 ? max_rows : 1;
    const int64_t want_splits = std::max<int64_t>(1, (3 * sms / 2 + segs - 1) / segs);
    int64_t c = ceil_div(rows, want_splits);
    c = std::max<int64_t>(128, ((c + 63) / 64) * 64);
    c = std::max<int64_t>(c, ((ceil_div(rows, 64) + 63) / 64) * 64);
    *chunk = c;
    *nsplit = ceil_div(rows, c);
}

size_t decode_tc_workspace(int64_t P, int64_t H, int64_t G, int64_t d);

size_t decode_workspace_bytes(int64_t P, int64_t H, int64_t G, int64_t d, int64_t max_rows, size_t acc) {
    int64_t chunk, nsplit;
    decode_plan(P, G, max_rows, &chunk, &nsplit);
    return std::max<size_t>(3 * 256 + size_t(P * G) * 4 + size_t(P * G * nsplit * (H / G)) * (2 + d) * acc,
                            decode_tc_workspace(P, H, G, d));
}

bool decode_tc_supported(adakv_dtype dt, int64_t H, int64_t G, int64_t d, int64_t cache_rows);
adakv_status launch_decode_tc(int64_t P, int64_t H, int64_t G, int32_t scale, const void* q, void* kc, void* vc,
                              int64_t cache_rows, const int32_t* ss, const int32_t* cap, int32_t* sl,
                              const void* kn, const void* vn, void* out, uint32_t* err, bool overlap_prev,
                              cudaStream_t stream);

adakv_status launch_decode(adakv_dtype dt, int64_t P, int64_t H, int64_t G, int64_t d, int32_t scale,
                           const void* q, void* kc, void* vc, int64_t cache_rows, const int32_t* ss,
                           const int32_t* cap, int32_t* sl, int64_t max_rows, const void* kn, const void* vn,
                           void* out, void* ws, uint32_t* err, bool overlap_prev, cudaStream_t stream) {
    if (decode_tc_supported(dt, H, G, d, cache_rows))
        return launch_decode_tc(P, H, G, scale, q, kc, vc, cache_rows, ss, cap, sl, kn, vn, out, err, overlap_prev,
                                stream);
    int64_t chunk, nsplit;
    decode_plan(P, G, max_rows, &chunk, &nsplit);
    if (H / G > kMaxGroupHeads) return fail(ADAKV_UNSUPPORTED, "decode: more than 16 query heads per KV group");
    if (d > 256) return fail(ADAKV_UNSUPPORTED, "decode: head_dim > 256");
    const int J = int(ceil_div(d, 32));
    const int64_t gs = H / G;
    const int GHs = gs <= 1 ? 1 : gs <= 2 ? 2 : gs <= 4 ? 4 : gs <= 8 ? 8 : 16;
    const int Js = J <= 1 ? 1 : J <= 2 ? 2 : J <= 4 ? 4 : 8;
#define ADAKV_DEC_GH(T, JJ)                                                                     \
    switch (GHs) {                                                                              \
        case 1: return launch_t<T, JJ, 1>(P, H, G, d, scale, q, kc, vc, ss, cap, sl, max_rows, kn, vn, out, ws, err, chunk, nsplit, stream); \
        case 2: return launch_t<T, JJ, 2>(P, H, G, d, scale, q, kc, vc, ss, cap, sl, max_rows, kn, vn, out, ws, err, chunk, nsplit, stream); \
        case 4: return launch_t<T, JJ, 4>(P, H, G, d, scale, q, kc, vc, ss, cap, sl, max_rows, kn, vn, out, ws, err, chunk, nsplit, stream); \
        case 8: return launch_t<T, JJ, 8>(P, H, G, d, scale, q, kc, vc, ss, cap, sl, max_rows, kn, vn, out, ws, err, chunk, nsplit, stream); \
        default: return launch_t<T, JJ, 16>(P, H, G, d, scale, q, kc, vc, ss, cap, sl, max_rows, kn, vn, out, ws, err, chunk, nsplit, stream); \
    }
#define ADAKV_DEC_SWITCH(T)                 \
    switch (Js) {                           \
        case 1: ADAKV_DEC_GH(T, 1)          \
        case 2: ADAKV_DEC_GH(T, 2)          \
        case 4: ADAKV_DEC_GH(T, 4)          \
        default: ADAKV_DEC_GH(T, 8)         \
    }
    switch (dt) {
        case ADAKV_BF16: ADAKV_DEC_SWITCH(__nv_bfloat16)
        case ADAKV_F32: ADAKV_DEC_SWITCH(float)
        case ADAKV_F64: ADAKV_DEC_SWITCH(double)
    }
#undef ADAKV_DEC_SWITCH
#undef ADAKV_DEC_GH
    return fail(ADAKV_INVALID_ARGUMENT, "decode: unknown dtype");
}

adakv_status launch_append(adakv_dtype dt, int64_t segments, int64_t rows, int64_t d, void* kc, void* vc,
                           const int32_t* ss, const int32_t* cap, int32_t* sl, const void* kn, const void* vn,
                           uint32_t* err, cudaStream_t stream) {
    if (segments == 0 || rows == 0) return ADAKV_OK;
    const int64_t units = int64_t(dtype_size(dt)) / 2;
    append_kernel<<<unsigned(segments), 128, 0, stream>>>(
        segments, rows, d, ss, cap, sl, static_cast<const uint16_t*>(kn), static_cast<const uint16_t*>(vn),
        static_cast<uint16_t*>(kc), static_cast<uint16_t*>(vc), units, err);
    ADAKV_CUDA_TRY(cudaGetLastError());
    return ADAKV_OK;
}

}  // namespace adakv_b200
