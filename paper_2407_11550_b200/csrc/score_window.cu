// score_window.cu -- K1 generic: observation-window scoring for any dtype / shape.
//
// Replaces, per KV group (p, g) and its g member heads:
//   attention_weights (attention.hpp:169-179) with scores_row (159-163) and the
//   max-subtracted softmax (141-157) over the OUTSIDE keys only (no causal mask,
//   policies.hpp:244); maxpool_same (policies.hpp:99-112, stride 1, pad (k-1)/2,
//   padded cells excluded); the row mean (125-131: sum rows in order, then /m);
//   and group_mean_scores (136-156: sum heads in order, then /g).
//
// Two launches over a grid of (key chunk, problem*group):
//   stats_kernel   per chunk, per window row: partial (max, sum exp(l - max)).
//   scores_kernel  combines the partials into (M_r, S_r), recomputes the logits
//                  of its chunk plus a (k-1)/2 halo, pools the LOGITS (exp is
//                  monotone so max(exp(l)) == exp(max(l)); division by S_r is
//                  monotone too), and reduces rows then heads in the reference's
//                  order.
// fp64 instantiation: logits use the reference's dot order without FMA, so every
// logit is bit-identical; scores then differ only by exp() ulps and the order of
// the S_r sum (~1e-15 relative).  bf16/f32 use fp32 math.  The bf16, d == 128,
// g*m <= 128 perf path is score_window_tc.cu (tcgen05).
#include <cfloat>

#include "common.cuh"

namespace adakv_b200 {

namespace {

constexpr int kThreads = 256;
constexpr int kRowBlock = 32;   // window rows per smem tile
constexpr int kKeyTile = 32;    // keys per smem tile
constexpr int kChunk = 256;     // keys per CTA

template <class A>
__device__ __forceinline__ A dot_seq(const A* __restrict__ q, const A* __restrict__ k, int d) {
    A s = A(0);
    for (int c = 0; c < d; ++c) {
        if constexpr (sizeof(A) == 8) s = dadd(s, dmul(q[c], k[c]));
        else s = __fadd_rn(s, __fmul_rn(q[c], k[c]));
    }
    return s;
}

template <class A>
__device__ __forceinline__ A neg_inf() { return -INFINITY; }

template <class T, class A>
__global__ void __launch_bounds__(kThreads)
stats_kernel(const T* __restrict__ q, const T* __restrict__ k, int64_t H, int64_t G, int64_t m,
             int64_t n_o, int64_t n_rows, int64_t d, A inv_scale, A* __restrict__ stats,
             int64_t nchunks) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    A* sq = reinterpret_cast<A*>(smem_raw);            // [kRowBlock][d]
    A* sk = sq + kRowBlock * d;                        // [kKeyTile][d + 1]
    const int64_t pg = blockIdx.y;
    const int64_t p = pg / G, g = pg % G;
    const int64_t gs = H / G;
    const int64_t R = gs * m;
    const T* qg = q + (p * H + g * gs) * m * d;
    const T* kg = k + pg * n_rows * d;
    const int64_t c0 = int64_t(blockIdx.x) * kChunk;
    const int64_t c1 = min(c0 + int64_t(kChunk), n_o);
    const int tid = threadIdx.x;
    const int r_local = tid / 8, kq = tid % 8;

    for (int64_t rb = 0; rb < R; rb += kRowBlock) {
        __syncthreads();
        for (int64_t i = tid; i < kRowBlock * d; i += kThreads) {
            const int64_t r = rb + i / d;
            sq[i] = r < R ? A(to_acc(qg[r * d + i % d])) : A(0);
        }
        A run_m = neg_inf<A>(), run_s = A(0);
        for (int64_t kt = c0; kt < c1; kt += kKeyTile) {
            __syncthreads();
            for (int64_t i = tid; i < kKeyTile * d; i += kThreads) {
                const int64_t j = kt + i / d;
                sk[(i / d) * (d + 1) + i % d] = j < c1 ? A(to_acc(kg[j * d + i % d])) : A(0);
            }
            __syncthreads();
            if (rb + r_local < R) {
                for (int jj = kq; jj < kKeyTile; jj += 8) {
                    if (kt + jj >= c1) break;
                    A l = dot_seq(sq + r_local * d, sk + jj * (d + 1), int(d));
                    if constexpr (sizeof(A) == 8) l = dmul(l, inv_scale);
                    else l = __fmul_rn(l, inv_scale);
                    if (l > run_m) {
                        run_s = run_s * acc_exp(run_m - l) + A(1);
                        run_m = l;
                    } else {
                        run_s += acc_exp(l - run_m);
                    }
                }
            }
        }
        // combine the 8 lanes that share a row (consecutive lanes)
        for (int o = 4; o >= 1; o >>= 1) {
            const A om = __shfl_xor_sync(0xffffffffu, run_m, o);
            const A os = __shfl_xor_sync(0xffffffffu, run_s, o);
            const A nm = om > run_m ? om : run_m;
            A ns = A(0);
            if (run_m != neg_inf<A>()) ns += run_s * acc_exp(run_m - nm);
            if (om != neg_inf<A>()) ns += os * acc_exp(om - nm);
            run_m = nm;
            run_s = ns;
        }
        if (kq == 0 && rb + r_local < R) {
            A* st = stats + ((pg * R + rb + r_local) * nchunks + blockIdx.x) * 2;
            st[0] = run_m;
            st[1] = run_s;
        }
    }
}

template <class T, class A>
__global__ void __launch_bounds__(kThreads)
scores_kernel(const T* __restrict__ q, const T* __restrict__ k, int64_t H, int64_t G, int64_t m,
              int64_t n_o, int64_t n_rows, int64_t d, A inv_scale, int pad,
              const A* __restrict__ stats, int64_t nchunks, A* __restrict__ head_scores,
              A* __restrict__ group_scores, uint32_t* __restrict__ err) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int64_t pg = blockIdx.y;
    const int64_t p = pg / G, g = pg % G;
    const int64_t gs = H / G;
    const int64_t R = gs * m;
    const int TKH = kKeyTile + 2 * pad;                      // tile keys incl. halo
    A* rowM = reinterpret_cast<A*>(smem_raw);                // [R]
    A* rowS = rowM + R;                                      // [R]
    A* acc = rowS + R;                                       // [gs][kChunk]
    A* sq = acc + gs * kChunk;                               // [kRowBlock][d]
    A* sk = sq + kRowBlock * d;                              // [TKH][d+1]
    A* sl = sk + TKH * (d + 1);                              // [kRowBlock][TKH]
    A* sp = sl + kRowBlock * TKH;                            // [kRowBlock][kKeyTile]
    const T* qg = q + (p * H + g * gs) * m * d;
    const T* kg = k + pg * n_rows * d;
    const int64_t c0 = int64_t(blockIdx.x) * kChunk;
    const int64_t c1 = min(c0 + int64_t(kChunk), n_o);
    const int tid = threadIdx.x;

    // final row statistics from the per-chunk partials
    for (int64_t r = tid; r < R; r += kThreads) {
        const A* st = stats + (pg * R + r) * nchunks * 2;
        A M = neg_inf<A>();
        for (int64_t c = 0; c < nchunks; ++c) M = st[2 * c] > M ? st[2 * c] : M;
        A S = A(0);
        for (int64_t c = 0; c < nchunks; ++c)
            if (st[2 * c] != neg_inf<A>()) S += st[2 * c + 1] * acc_exp(st[2 * c] - M);
        rowM[r] = M;
        rowS[r] = S;
        // a NaN or +Inf logit anywhere in the row (a non-finite key, LayerCache::validate,
        // attention.hpp:76-83) leaves a non-finite maximum or sum
        if (blockIdx.x == 0 && err && !(M > neg_inf<A>() && M < A(INFINITY) && S >= A(1) && S < A(INFINITY)))
            atomicOr(err, ERR_NONFINITE);
    }
    for (int64_t i = tid; i < gs * kChunk; i += kThreads) acc[i] = A(0);

    for (int64_t rb = 0; rb < R; rb += kRowBlock) {
        __syncthreads();
        for (int64_t i = tid; i < kRowBlock * d; i += kThreads) {
            const int64_t r = rb + i / d;
            sq[i] = r < R ? A(to_acc(qg[r * d + i % d])) : A(0);
        }
        for (int64_t kt = c0; kt < c1; kt += kKeyTile) {
            const int64_t lo = kt - pad;  // first key of the haloed tile (may be < 0)
            __syncthreads();
            for (int64_t i = tid; i < TKH * d; i += kThreads) {
                const int64_t j = lo + i / d;
                sk[(i / d) * (d + 1) + i % d] = (j >= 0 && j < n_o) ? A(to_acc(kg[j * d + i % d])) : A(0);
            }
            __syncthreads();
            for (int64_t i = tid; i < kRowBlock * TKH; i += kThreads) {
                const int64_t r = i / TKH, jj = i % TKH;
                const int64_t j = lo + jj;
                A l = neg_inf<A>();
                if (rb + r < R && j >= 0 && j < n_o) {
                    l = dot_seq(sq + r * d, sk + jj * (d + 1), int(d));
                    if constexpr (sizeof(A) == 8) l = dmul(l, inv_scale);
                    else l = __fmul_rn(l, inv_scale);
                }
                sl[i] = l;
            }
            __syncthreads();
            // pooled probability: exp(max over window of l - M) / S
            for (int64_t i = tid; i < kRowBlock * kKeyTile; i += kThreads) {
                const int64_t r = i / kKeyTile, jj = i % kKeyTile;
                A v = A(0);
                if (rb + r < R && kt + jj < c1) {
                    const A* row = sl + r * TKH + jj;  // window [jj, jj + 2pad]
                    A mx = row[pad];
                    for (int t = 0; t <= 2 * pad; ++t) mx = (mx < row[t]) ? row[t] : mx;
                    const A e = acc_exp(mx - rowM[rb + r]);
                    if constexpr (sizeof(A) == 8) v = ddiv(e, rowS[rb + r]);
                    else v = __fdiv_rn(e, rowS[rb + r]);
                }
                sp[i] = v;
            }
            __syncthreads();
            // accumulate rows in ascending order into their head (policies.hpp:126-129)
            for (int64_t jj = tid; jj < kKeyTile; jj += kThreads) {
                if (kt + jj >= c1) continue;
                const int64_t col = kt + jj - c0;
                for (int64_t r = 0; r < kRowBlock && rb + r < R; ++r) {
                    const int64_t h = (rb + r) / m;
                    if constexpr (sizeof(A) == 8) acc[h * kChunk + col] = dadd(acc[h * kChunk + col], sp[r * kKeyTile + jj]);
                    else acc[h * kChunk + col] = __fadd_rn(acc[h * kChunk + col], sp[r * kKeyTile + jj]);
                }
            }
        }
    }
    __syncthreads();
    for (int64_t col = tid; col < c1 - c0; col += kThreads) {
        A gsum = A(0);
        for (int64_t h = 0; h < gs; ++h) {
            A mean;
            if constexpr (sizeof(A) == 8) mean = ddiv(acc[h * kChunk + col], double(m));
            else mean = __fdiv_rn(acc[h * kChunk + col], float(m));
            if (head_scores) head_scores[((p * H + g * gs + h) * n_o) + c0 + col] = mean;
            if constexpr (sizeof(A) == 8) gsum = dadd(gsum, mean);
            else gsum = __fadd_rn(gsum, mean);
        }
        if constexpr (sizeof(A) == 8) group_scores[pg * n_o + c0 + col] = ddiv(gsum, double(gs));
        else group_scores[pg * n_o + c0 + col] = __fdiv_rn(gsum, float(gs));
    }
}

template <class T>
adakv_status launch_generic(const adakv_layer_shape& s, int64_t pool_kernel, int32_t scale,
                            const void* q, const void* k, void* head_scores, void* group_scores,
                            void* ws, uint32_t* err, cudaStream_t stream) {
    using A = typename Acc<T>::type;
    const int64_t P = s.problems, H = s.q_heads, G = s.kv_groups, m = s.window, n_o = s.outside,
                  d = s.head_dim;
    const int64_t gs = H / G, R = gs * m;
    const int64_t nchunks = ceil_div(n_o, kChunk);
    const int pad = int((pool_kernel - 1) / 2);
    const A inv = scale ? A(1) / sqrt(A(d)) : A(1);
    Arena ar(ws);
    A* stats = ar.take<A>(size_t(P * G * R * nchunks * 2));
    const dim3 grid(unsigned(nchunks), unsigned(P * G));
    const size_t smem1 = sizeof(A) * (kRowBlock * d + kKeyTile * (d + 1));
    const int TKH = kKeyTile + 2 * pad;
    const size_t smem2 = sizeof(A) * (2 * R + gs * kChunk + kRowBlock * d + TKH * (d + 1) +
                                      kRowBlock * TKH + kRowBlock * kKeyTile);
    auto k1 = stats_kernel<T, A>;
    auto k2 = scores_kernel<T, A>;
    ADAKV_CUDA_TRY(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem1)));
    ADAKV_CUDA_TRY(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem2)));
    k1<<<grid, kThreads, smem1, stream>>>(static_cast<const T*>(q), static_cast<const T*>(k), H, G, m,
                                         n_o, n_o + m, d, inv, stats, nchunks);
    ADAKV_CUDA_TRY(cudaGetLastError());
    k2<<<grid, kThreads, smem2, stream>>>(static_cast<const T*>(q), static_cast<const T*>(k), H, G, m,
                                         n_o, n_o + m, d, inv, pad, stats, nchunks,
                                         static_cast<A*>(head_scores), static_cast<A*>(group_scores), err);
    ADAKV_CUDA_TRY(cudaGetLastError());
    return ADAKV_OK;
}

}  // namespace

size_t score_window_generic_workspace(adakv_dtype dt, const adakv_layer_shape& s) {
    const size_t a = dt == ADAKV_F64 ? 8 : 4;
    const int64_t R = (s.q_heads / s.kv_groups) * s.window;
    const int64_t nchunks = ceil_div(s.outside, kChunk);
    return 256 + size_t(s.problems * s.kv_groups * R * nchunks * 2) * a;
}

size_t score_window_generic_smem(adakv_dtype dt, const adakv_layer_shape& s, int64_t pool_kernel) {
    const size_t a = dt == ADAKV_F64 ? 8 : 4;
    const int64_t gs = s.q_heads / s.kv_groups, R = gs * s.window, d = s.head_dim;
    const int64_t TKH = kKeyTile + (pool_kernel - 1);
    return a * size_t(2 * R + gs * kChunk + kRowBlock * d + TKH * (d + 1) + kRowBlock * TKH +
                      kRowBlock * kKeyTile);
}

adakv_status score_window_generic(adakv_dtype dt, const adakv_layer_shape& s, int64_t pool_kernel,
                                  int32_t scale, const void* q, const void* k, void* head_scores,
                                  void* group_scores, void* ws, uint32_t* err, cudaStream_t stream) {
    switch (dt) {
        case ADAKV_F64: return launch_generic<double>(s, pool_kernel, scale, q, k, head_scores, group_scores, ws, err, stream);
        case ADAKV_F32: return launch_generic<float>(s, pool_kernel, scale, q, k, head_scores, group_scores, ws, err, stream);
        case ADAKV_BF16: return launch_generic<__nv_bfloat16>(s, pool_kernel, scale, q, k, head_scores, group_scores, ws, err, stream);
    }
    return fail(ADAKV_INVALID_ARGUMENT, "window_scores: unknown dtype");
}

}  // namespace adakv_b200
