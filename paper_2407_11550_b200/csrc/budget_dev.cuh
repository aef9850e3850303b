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
