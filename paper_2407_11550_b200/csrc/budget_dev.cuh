// budget_dev.cuh -- bit-exact fp64 budget integerisation on the device.
//
// Restates budget.hpp:45-93 (detail::apportion), 103-113 (uniform_allocation),
// 145-158 (safeguard_blend), 169-191 (pyramid_layer_budgets) and
// policies.hpp:178-196 (repair_zero_budgets).  Every fp64 operation is an
// explicit round-to-nearest intrinsic (__dmul_rn, __dadd_rn, ...), so nvcc can
// never contract a*b+c into an FMA: the results are bit-identical to the
// reference's x86-64 Release build.  Runs on one thread (O(h) work, h <= 64).
#pragma once

#include "common.cuh"

namespace adakv_b200 {

constexpr int kMaxSeg = 64;
constexpr uint64_t kAmpleCap = ~uint64_t(0) / 2;  // budget.hpp:95-97

__device__ inline uint32_t apportion_dev(const double* quotas, int h, uint64_t total,
                                         const uint64_t* caps, uint64_t* out) {
    uint64_t cap_sum = 0;
    for (int i = 0; i < h; ++i)
        cap_sum = (cap_sum > ~uint64_t(0) - caps[i]) ? ~uint64_t(0) : cap_sum + caps[i];
    if (total > cap_sum) return ERR_BUDGET;
    uint64_t assigned = 0;
    for (int i = 0; i < h; ++i) {
        if (!(quotas[i] >= 0.0)) return ERR_BUDGET;
        const uint64_t base = __double2ull_rz(floor(quotas[i]));
        out[i] = base < caps[i] ? base : caps[i];
        assigned += out[i];
    }
    while (assigned < total) {
        int pick = h;
        double best = -INFINITY;
        for (int i = 0; i < h; ++i) {
            if (out[i] >= caps[i]) continue;
            const double deficit = dsub(quotas[i], __ull2double_rn(out[i]));
            if (deficit > best) {
                best = deficit;
                pick = i;
            }
        }
        if (pick == h) return ERR_BUDGET;
        ++out[pick];
        ++assigned;
    }
    while (assigned > total) {
        int pick = h;
        double best = -INFINITY;
        for (int i = 0; i < h; ++i) {
            if (out[i] == 0) continue;
            const double surplus = dsub(__ull2double_rn(out[i]), quotas[i]);
            if (surplus > best) {
                best = surplus;
                pick = i;
            }
        }
        if (pick == h) return ERR_BUDGET;
        --out[pick];
        --assigned;
    }
    return 0;
}

// ---- warp-parallel forms used by the selection kernel (one warp, lane i holds segments
// i, i + 32): the same fp64 operations per element, so the same results bit for bit.
//
// apportion's increment loop (budget.hpp:73-82) picks, each round, the eligible element
// (out < cap) with the largest deficit q - out, lowest index on ties.  An eligible element has
// out = floor(q) <= q, so its deficit lies in [0, 1); once picked it drops below 0 and every
// other eligible deficit is >= 0, so it is not picked again while unpicked eligible elements
// remain.  Hence, when the remainder R does not exceed the eligible count, the R rounds pick
// exactly the top R eligible deficits ordered (deficit desc, index asc): one rank computation
// instead of R scans.  Otherwise (R larger, or a surplus to remove) lane 0 runs the sequential
// loop itself.
__device__ inline uint64_t sat_add_u64(uint64_t a, uint64_t b) { return a > ~uint64_t(0) - b ? ~uint64_t(0) : a + b; }

__device__ inline uint32_t apportion_warp(const double* quotas, int h, uint64_t total, const uint64_t* caps,
                                          uint64_t* out, int lane) {
    uint64_t cap_sum = 0, assigned = 0;
    bool bad = false;
    for (int i = lane; i < h; i += 32) {
        cap_sum = sat_add_u64(cap_sum, caps[i]);
        const double q = quotas[i];
        if (!(q >= 0.0)) {
            bad = true;
            continue;
        }
        const uint64_t base = __double2ull_rz(floor(q));
        out[i] = base < caps[i] ? base : caps[i];
        assigned += out[i];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        cap_sum = sat_add_u64(cap_sum, __shfl_xor_sync(0xffffffffu, cap_sum, o));
        assigned += __shfl_xor_sync(0xffffffffu, assigned, o);
    }
    if (total > cap_sum) return ERR_BUDGET;
    if (__any_sync(0xffffffffu, bad)) return ERR_BUDGET;
    if (assigned == total) return 0;
    // eligible elements (and their deficits) of this lane: slots i = lane, lane + 32
    double d[2];
    bool el[2];
    int n_el = 0;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int i = lane + 32 * u;
        el[u] = i < h && out[i] < caps[i];
        d[u] = el[u] ? dsub(quotas[i], __ull2double_rn(out[i])) : 0.0;
        n_el += __popc(__ballot_sync(0xffffffffu, el[u]));
    }
    if (assigned < total && total - assigned <= uint64_t(n_el)) {
        const uint64_t R = total - assigned;
        uint32_t rank[2] = {0u, 0u};
        for (int j = 0; j < h; ++j) {
            const int u = j >> 5;
            const double dj = __shfl_sync(0xffffffffu, d[u], j & 31);
            const bool ej = __shfl_sync(0xffffffffu, el[u], j & 31);
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int i = lane + 32 * v;
                if (ej && (dj > d[v] || (dj == d[v] && j < i))) ++rank[v];
            }
        }
#pragma unroll
        for (int v = 0; v < 2; ++v)
            if (el[v] && rank[v] < R) ++out[lane + 32 * v];
        __syncwarp();
        return 0;
    }
    // rare: several increments per element, or a surplus -- the sequential loops on lane 0
    __syncwarp();
    uint32_t e = 0;
    if (lane == 0) {
        while (assigned < total) {
            int pick = h;
            double best = -INFINITY;
            for (int i = 0; i < h; ++i) {
                if (out[i] >= caps[i]) continue;
                const double deficit = dsub(quotas[i], __ull2double_rn(out[i]));
                if (deficit > best) {
                    best = deficit;
                    pick = i;
                }
            }
            if (pick == h) {
                e = ERR_BUDGET;
                break;
            }
            ++out[pick];
            ++assigned;
        }
        while (!e && assigned > total) {
            int pick = h;
            double best = -INFINITY;
            for (int i = 0; i < h; ++i) {
                if (out[i] == 0) continue;
                const double surplus = dsub(__ull2double_rn(out[i]), quotas[i]);
                if (surplus > best) {
                    best = surplus;
                    pick = i;
                }
            }
            if (pick == h) {
                e = ERR_BUDGET;
                break;
            }
            --out[pick];
            --assigned;
        }
    }
    __syncwarp();
    return __shfl_sync(0xffffffffu, e, 0);
}

__device__ inline uint32_t uniform_warp(uint64_t total, int h, const uint64_t* caps, double* quotas, uint64_t* out,
                                        int lane) {
    const double q = ddiv(__ull2double_rn(total), __ull2double_rn(uint64_t(h)));
    for (int i = lane; i < h; i += 32) quotas[i] = q;
    __syncwarp();
    return apportion_warp(quotas, h, total, caps, out, lane);
}

__device__ inline uint32_t safeguard_warp(const uint64_t* adaptive, uint64_t total, int h, double alpha,
                                          const uint64_t* caps, double* quotas, uint64_t* out, int lane) {
    if (!(alpha >= 0.0 && alpha <= 1.0)) return ERR_BUDGET;
    const double share = ddiv(__ull2double_rn(total), __ull2double_rn(uint64_t(h)));
    const double beta = dsub(1.0, alpha);
    for (int i = lane; i < h; i += 32) quotas[i] = dadd(dmul(alpha, __ull2double_rn(adaptive[i])), dmul(beta, share));
    __syncwarp();
    return apportion_warp(quotas, h, total, caps, out, lane);
}

__device__ inline uint32_t uniform_dev(uint64_t total, int h, const uint64_t* caps, double* quotas,
                                       uint64_t* out) {
    const double q = ddiv(__ull2double_rn(total), __ull2double_rn(uint64_t(h)));
    for (int i = 0; i < h; ++i) quotas[i] = q;
    return apportion_dev(quotas, h, total, caps, out);
}

__device__ inline uint32_t safeguard_dev(const uint64_t* adaptive, uint64_t total, int h,
                                         double alpha, const uint64_t* caps, double* quotas,
                                         uint64_t* out) {
    if (!(alpha >= 0.0 && alpha <= 1.0)) return ERR_BUDGET;
    const double share = ddiv(__ull2double_rn(total), __ull2double_rn(uint64_t(h)));
    const double beta = dsub(1.0, alpha);
    for (int i = 0; i < h; ++i)
        quotas[i] = dadd(dmul(alpha, __ull2double_rn(adaptive[i])), dmul(beta, share));
    return apportion_dev(quotas, h, total, caps, out);
}

__device__ inline uint32_t repair_dev(uint64_t* counts, const uint64_t* caps, int h) {
    for (int gi = 0; gi < h; ++gi) {
        while (counts[gi] == 0) {
            int donor = h;
            uint64_t best = 1;
            for (int k = 0; k < h; ++k)
                if (counts[k] > best) {
                    best = counts[k];
                    donor = k;
                }
            if (donor == h || caps[gi] == 0) return ERR_REPAIR;
            --counts[donor];
            ++counts[gi];
        }
    }
    return 0;
}

__device__ inline uint32_t pyramid_dev(uint64_t avg, int layers, double bmax, double bmin,
                                       double* quotas, uint64_t* caps, uint64_t* out) {
    if (layers == 1) {
        out[0] = avg;
        return 0;
    }
    const double a = __ull2double_rn(avg);
    double qsum = 0.0;
    for (int l = 0; l < layers; ++l) {
        const double t = ddiv(__ull2double_rn(uint64_t(l)), __ull2double_rn(uint64_t(layers - 1)));
        quotas[l] = dmul(a, dsub(bmax, dmul(dsub(bmax, bmin), t)));
        qsum = dadd(qsum, quotas[l]);
    }
    const uint64_t total = avg * uint64_t(layers);
    if (qsum > 0.0) {
        const double sc = ddiv(__ull2double_rn(total), qsum);
        for (int l = 0; l < layers; ++l) quotas[l] = dmul(quotas[l], sc);
    }
    for (int l = 0; l < layers; ++l) caps[l] = kAmpleCap;
    return apportion_dev(quotas, layers, total, caps, out);
}

}  // namespace adakv_b200
