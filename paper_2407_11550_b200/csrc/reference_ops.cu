// reference_ops.cu -- fp64 device kernels behind the reference-typed C++ API
// (include/adakv_b200/adakv.hpp) for the entry points that are not part of the
// bf16 fast path: each one reproduces the reference's loop order without FMA
// contraction (__dmul_rn/__dadd_rn), so results match the host reference bit for
// bit except where exp() is involved.
#include "common.cuh"

namespace adakv_b200 {
namespace {

// matmul (matrix.hpp:91-102): out(i,j) = sum_k a(i,k) * b(k,j), k ascending, a(i,k)==0 skipped.
// Q_h = X * W_h for every head h (policies.hpp:243).  x [m, D], w [H, D, d] -> q [H, m, d].
__global__ void project_kernel(const double* __restrict__ x, const double* __restrict__ w, int64_t H,
                               int64_t m, int64_t D, int64_t d, double* __restrict__ q) {
    const int64_t total = H * m * d;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t h = t / (m * d), i = (t / d) % m, j = t % d;
        double acc = 0.0;
        for (int64_t k = 0; k < D; ++k) {
            const double aik = x[i * D + k];
            if (aik == 0.0) continue;
            acc = dadd(acc, dmul(aik, w[(h * D + k) * d + j]));
        }
        q[t] = acc;
    }
}

// group_mean_scores (policies.hpp:136-156): members summed in order, then / g.
__global__ void group_mean_kernel(const double* __restrict__ s, int64_t h, int64_t n, int64_t g,
                                  double* __restrict__ out) {
    const int64_t groups = h / g;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < groups * n; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t gi = t / n, j = t % n;
        double acc = 0.0;
        for (int64_t k = 0; k < g; ++k) acc = dadd(acc, s[(gi * g + k) * n + j]);
        out[t] = ddiv(acc, double(g));
    }
}

// attention_weights (attention.hpp:169-179): one CTA per query row; logits in the
// reference's dot order, max, exp(l - max), sum (block tree), divide.
__global__ void attention_weights_kernel(const double* __restrict__ q, const double* __restrict__ k, int64_t n,
                                         int64_t d, double inv, double* __restrict__ out) {
    const int64_t r = blockIdx.x;
    double* row = out + r * n;
    __shared__ double red[256];
    double mx = -INFINITY;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
        double s = 0.0;
        for (int64_t c = 0; c < d; ++c) s = dadd(s, dmul(q[r * d + c], k[j * d + c]));
        s = dmul(s, inv);
        row[j] = s;
        mx = s > mx ? s : mx;
    }
    red[threadIdx.x] = mx;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] = red[threadIdx.x + o] > red[threadIdx.x] ? red[threadIdx.x + o] : red[threadIdx.x];
        __syncthreads();
    }
    mx = red[0];
    __syncthreads();
    double sum = 0.0;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
        const double e = exp(dsub(row[j], mx));
        row[j] = e;
        sum = dadd(sum, e);
    }
    red[threadIdx.x] = sum;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] = dadd(red[threadIdx.x], red[threadIdx.x + o]);
        __syncthreads();
    }
    const double denom = red[0];
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) row[j] = ddiv(row[j], denom);
}

// attention_output (attention.hpp:182-196): per head ctx = row_times(w_i, V_i) then
// contrib = row_times(ctx, Wo_i) (matrix.hpp:79-89, zero multipliers skipped); one thread
// per (head, output column) writes contrib[h][c]; heads are summed in order afterwards.
__global__ void ctx_kernel(const double* __restrict__ w, const int64_t* __restrict__ woff,
                           const double* __restrict__ v, const int64_t* __restrict__ voff, int64_t H, int64_t dh,
                           double* __restrict__ ctx) {
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < H * dh; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t h = t / dh, c = t % dh;
        const int64_t n = woff[h + 1] - woff[h];
        double acc = 0.0;
        for (int64_t r = 0; r < n; ++r) {
            const double xr = w[woff[h] + r];
            if (xr == 0.0) continue;
            acc = dadd(acc, dmul(xr, v[(voff[h] + r) * dh + c]));
        }
        ctx[t] = acc;
    }
}
__global__ void out_kernel(const double* __restrict__ ctx, const double* __restrict__ wo, int64_t H, int64_t dh,
                           int64_t D, double* __restrict__ y) {
    for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < D; c += int64_t(gridDim.x) * blockDim.x) {
        double yc = 0.0;
        for (int64_t h = 0; h < H; ++h) {
            double contrib = 0.0;
            for (int64_t r = 0; r < dh; ++r) {
                const double xr = ctx[h * dh + r];
                if (xr == 0.0) continue;
                contrib = dadd(contrib, dmul(xr, wo[(h * dh + r) * D + c]));
            }
            yc = dadd(yc, contrib);
        }
        y[c] = yc;
    }
}

// select_and_compact (flat_cache.hpp:92-120): per segment, rows with mask != 0 are copied in
// order.  One CTA per segment; block-wide ballot scan over the mask in 1024-row chunks.
__global__ void compact_rows_kernel(const uint8_t* __restrict__ mask, const int64_t* __restrict__ off,
                                    const double* __restrict__ src_k, const double* __restrict__ src_v, int64_t d,
                                    const int64_t* __restrict__ out_off, double* __restrict__ dst_k,
                                    double* __restrict__ dst_v) {
    const int64_t s = blockIdx.x;
    __shared__ int warp_sum[32];
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t base = off[s]; base < off[s + 1]; base += blockDim.x) {
        const int64_t r = base + threadIdx.x;
        const bool keep = r < off[s + 1] && mask[r] != 0;
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) warp_sum[warp] = __popc(bal);
        __syncthreads();
        int before = 0;
        for (int w = 0; w < warp; ++w) before += warp_sum[w];
        const int64_t rank = carry + before + __popc(bal & ((1u << lane) - 1u));
        if (keep) {
            for (int64_t c = 0; c < d; ++c) {
                dst_k[(out_off[s] + rank) * d + c] = src_k[r * d + c];
                dst_v[(out_off[s] + rank) * d + c] = src_v[r * d + c];
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int tot = 0;
            for (int w = 0; w < int(blockDim.x / 32); ++w) tot += warp_sum[w];
            carry += tot;
        }
        __syncthreads();
    }
}

int grid_for(int64_t n) { return int(std::min<int64_t>(ceil_div(std::max<int64_t>(n, 1), 256), 4096)); }

}  // namespace
}  // namespace adakv_b200

using namespace adakv_b200;

extern "C" {

adakv_status adakv_project_queries_f64(const double* x, const double* w, int64_t H, int64_t m, int64_t D,
                                       int64_t d, double* q, adakv_stream_t stream) {
    if (H <= 0 || m <= 0 || D <= 0 || d <= 0) return fail(ADAKV_INVALID_ARGUMENT, "matmul: inner dimension mismatch");
    project_kernel<<<grid_for(H * m * d), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(x, w, H, m, D, d, q);
    ADAKV_CUDA_TRY(cudaGetLastError());
    return ADAKV_OK;
}

adakv_status adakv_group_mean_scores_f64(const double* scores, int64_t h, int64_t n, int64_t g, double* out,
                                         adakv_stream_t stream) {
    if (g <= 0) return fail(ADAKV_INVALID_ARGUMENT, "group_mean_scores: zero group size");
    if (h % g != 0) return fail(ADAKV_INVALID_ARGUMENT, "group_mean_scores: head count not divisible by group size");
    if (h == 0 || n == 0) return ADAKV_OK;
    group_mean_kernel<<<grid_for(h / g * n), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(scores, h, n, g, out);
    ADAKV_CUDA_TRY(cudaGetLastError());
    return ADAKV_OK;
}

adakv_status adakv_attention_weights_f64(const double* q, int64_t m, const double* k, int64_t n, int64_t d,
                                         int32_t scale, double* out, adakv_stream_t stream) {
    if (n == 0) return fail(ADAKV_INVALID_ARGUMENT, "attention_weights: empty key set");
    if (m == 0) return ADAKV_OK;
    const double inv = scale ? 1.0 / sqrt(double(d)) : 1.0;
    attention_weights_kernel<<<unsigned(m), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(q, k, n, d, inv, out);
    ADAKV_CUDA_TRY(cudaGetLastError());
    return ADAKV_OK;
}

adakv_status adakv_attention_output_f64(const double* w, const int64_t* woff, const double* v,
                                        const int64_t* voff, int64_t H, int64_t dh, const double* wo, int64_t D,
                                        double* ctx_ws, double* y, adakv_stream_t stream) {
    const cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    ctx_kernel<<<grid_for(H * dh), 256, 0, st>>>(w, woff, v, voff, H, dh, ctx_ws);
    ADAKV_CUDA_TRY(cudaGetLastError());
    out_kernel<<<grid_for(D), 256, 0, st>>>(ctx_ws, wo, H, dh, D, y);
    ADAKV_CUDA_TRY(cudaGetLastError());
    return ADAKV_OK;
}

adakv_status adakv_compact_rows_f64(int64_t segments, const uint8_t* mask, const int64_t* off, const double* src_k,
                                    const double* src_v, int64_t d, const int64_t* out_off, double* dst_k,
                                    double* dst_v, adakv_stream_t stream) {
    if (segments == 0) return ADAKV_OK;
    compact_rows_kernel<<<unsigned(segments), 1024, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        mask, off, src_k, src_v, d, out_off, dst_k, dst_v);
    ADAKV_CUDA_TRY(cudaGetLastError());
    return ADAKV_OK;
}

}  // extern "C"
