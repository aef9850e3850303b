// tc_ptx.cuh -- thin inline-PTX wrappers for sm_100a: mbarrier, TMA, tcgen05 (MMA, TMEM).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

namespace adakv_b200 {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE_%=;\n"
        "bra WAIT_%=;\n"
        "DONE_%=:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* m) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* m, int c0, int c1, int c2,
                                            uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// ---------------------------------------------------------------- tcgen05
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {  // whole warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {  // whole warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}

// K-major operand in shared memory, 128-byte swizzle: 8-row atoms of 8 x 16 B, atoms
// 1024 B apart (SBO); LBO unused for swizzled K-major; descriptor version 1 (sm_100).
__device__ __forceinline__ uint64_t desc_kmajor_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFFu);
    d |= uint64_t(1) << 16;            // LBO (16 B units, ignored)
    d |= uint64_t(1024 >> 4) << 32;    // SBO
    d |= uint64_t(1) << 46;            // version
    d |= uint64_t(2) << 61;            // SWIZZLE_128B
    return d;
}

// Instruction descriptor: kind::f16, A/B = BF16, D = F32, both K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(uint32_t M, uint32_t N) {
    return (1u << 4)            // c_format F32
           | (1u << 7)          // a_format BF16
           | (1u << 10)         // b_format BF16
           | ((N >> 3) << 17)   // n_dim
           | ((M >> 4) << 24);  // m_dim
}

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns: thread t receives lane (base + t).
template <int OFF, int N>
__device__ __forceinline__ void tmem_ld_x32(uint32_t taddr, float (&v)[N]) {
    static_assert(OFF + 32 <= N, "range");
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=f"(v[OFF + 0]), "=f"(v[OFF + 1]), "=f"(v[OFF + 2]), "=f"(v[OFF + 3]), "=f"(v[OFF + 4]), "=f"(v[OFF + 5]), "=f"(v[OFF + 6]), "=f"(v[OFF + 7]), "=f"(v[OFF + 8]), "=f"(v[OFF + 9]), "=f"(v[OFF + 10]), "=f"(v[OFF + 11]), "=f"(v[OFF + 12]), "=f"(v[OFF + 13]), "=f"(v[OFF + 14]), "=f"(v[OFF + 15]), "=f"(v[OFF + 16]), "=f"(v[OFF + 17]), "=f"(v[OFF + 18]), "=f"(v[OFF + 19]), "=f"(v[OFF + 20]), "=f"(v[OFF + 21]), "=f"(v[OFF + 22]), "=f"(v[OFF + 23]), "=f"(v[OFF + 24]), "=f"(v[OFF + 25]), "=f"(v[OFF + 26]), "=f"(v[OFF + 27]), "=f"(v[OFF + 28]), "=f"(v[OFF + 29]), "=f"(v[OFF + 30]), "=f"(v[OFF + 31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float max3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ float ex2(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ void named_bar(uint32_t id, uint32_t count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <int OFF, int N>
__device__ __forceinline__ void tmem_ld_x16(uint32_t taddr, float (&v)[N]) {
    static_assert(OFF + 16 <= N, "range");
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=f"(v[OFF + 0]), "=f"(v[OFF + 1]), "=f"(v[OFF + 2]), "=f"(v[OFF + 3]), "=f"(v[OFF + 4]),
          "=f"(v[OFF + 5]), "=f"(v[OFF + 6]), "=f"(v[OFF + 7]), "=f"(v[OFF + 8]), "=f"(v[OFF + 9]),
          "=f"(v[OFF + 10]), "=f"(v[OFF + 11]), "=f"(v[OFF + 12]), "=f"(v[OFF + 13]), "=f"(v[OFF + 14]),
          "=f"(v[OFF + 15])
        : "r"(taddr));
}
template <int OFF, int N>
__device__ __forceinline__ void tmem_ld_x8(uint32_t taddr, float (&v)[N]) {
    static_assert(OFF + 8 <= N, "range");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(v[OFF + 0]), "=f"(v[OFF + 1]), "=f"(v[OFF + 2]), "=f"(v[OFF + 3]), "=f"(v[OFF + 4]),
                   "=f"(v[OFF + 5]), "=f"(v[OFF + 6]), "=f"(v[OFF + 7])
                 : "r"(taddr));
}

// MN-major operand, 128-byte swizzle: atoms of 64 MN-elements (128 B) x 8 K-rows;
// lbo = byte stride between MN-atoms, sbo = byte stride between K-atoms.
__device__ __forceinline__ uint64_t desc_mnmajor_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFFu);
    d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(2) << 61;
    return d;
}

// kind::f16 with F16 A/B, F32 D; A major selectable (1 = MN-major), B K-major.
__host__ __device__ constexpr uint32_t idesc_f16_f32(uint32_t M, uint32_t N, uint32_t a_mn_major) {
    return (1u << 4) | (0u << 7) | (0u << 10) | (a_mn_major << 15) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// make generic-proxy shared-memory writes visible to the async proxy (tensor core / TMA)
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- packed fp32x2
__device__ __forceinline__ uint64_t pk(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void upk(uint64_t v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

// 2^x for two lanes on the FMA pipe (FA4-style MUFU offload): x = n + f, n = rint(x) by the
// 1.5*2^23 trick, f in [-0.5, 0.5], degree-6 Taylor of 2^f (|rel err| < 2e-7), exponent
// added as integer bits.  Inputs are clamped to >= -125 so the result stays normal (2^-125 ~ 2e-38
// where MUFU would flush to 0 -- harmless for sums and exactly 0 once rounded to fp16).
__device__ __forceinline__ void exp2_poly2(float& a, float& b) {
    a = fmaxf(a, -125.f);
    b = fmaxf(b, -125.f);
    const uint64_t magic = pk(12582912.f, 12582912.f);
    const uint64_t x = pk(a, b);
    const uint64_t t = add2(x, magic);                        // rint(x) + 1.5*2^23
    const uint64_t r = add2(t, pk(-12582912.f, -12582912.f)); // rint(x)
    float r0, r1;
    upk(r, r0, r1);
    const uint64_t f = add2(x, pk(-r0, -r1));                 // f = x - rint(x)
    uint64_t p = pk(1.5403530e-4f, 1.5403530e-4f);
    p = fma2(p, f, pk(1.3333558e-3f, 1.3333558e-3f));
    p = fma2(p, f, pk(9.6181291e-3f, 9.6181291e-3f));
    p = fma2(p, f, pk(5.5504109e-2f, 5.5504109e-2f));
    p = fma2(p, f, pk(2.4022651e-1f, 2.4022651e-1f));
    p = fma2(p, f, pk(6.9314718e-1f, 6.9314718e-1f));
    p = fma2(p, f, pk(1.f, 1.f));
    float p0, p1, t0, t1;
    upk(p, p0, p1);
    upk(t, t0, t1);
    a = __int_as_float(__float_as_int(p0) + ((__float_as_int(t0) - 0x4B400000) << 23));
    b = __int_as_float(__float_as_int(p1) + ((__float_as_int(t1) - 0x4B400000) << 23));
}

// ---------------------------------------------------------------- host: tensor-map encoder
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
            qr == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

}  // namespace ptx
}  // namespace adakv_b200
