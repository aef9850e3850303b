// common.cuh -- shared device/host helpers for the Ada-KV B200 kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <string>

#include "adakv_b200.h"

namespace adakv_b200 {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
adakv_status fail(adakv_status st, const std::string& msg);
adakv_status cuda_fail(cudaError_t e, const char* what);

#define ADAKV_CUDA_TRY(expr)                                                \
    do {                                                                    \
        cudaError_t _e = (expr);                                            \
        if (_e != cudaSuccess) return ::adakv_b200::cuda_fail(_e, #expr);   \
    } while (0)

#define ADAKV_TRY(expr)                                 \
    do {                                                \
        adakv_status _s = (expr);                       \
        if (_s != ADAKV_OK) return _s;                  \
    } while (0)

// Device error word bits latched in the workspace header.
enum : uint32_t {
    ERR_NONFINITE = 1u << 0,   // LayerCache::validate (attention.hpp:76-83)
    ERR_BUDGET = 1u << 1,      // topk_decision k > n (policies.hpp:83), apportion capacity
    ERR_REPAIR = 1u << 2,      // repair_zero_budgets (policies.hpp:190-191)
    ERR_CAPACITY = 1u << 3,    // decode append beyond reserved capacity
    ERR_MAXROWS = 1u << 4,     // a decode segment longer than the call's max_rows bound
};

// Device-side bounds assertions (a checked build: make EXTRA=-DADAKV_DEVICE_CHECKS; used in
// place of compute-sanitizer, which this GPU pool does not allow).  Compiled out otherwise.
#ifdef ADAKV_DEVICE_CHECKS
#define ADAKV_DCHECK(cond)                                                                      \
    do {                                                                                        \
        if (!(cond)) {                                                                          \
            printf("ADAKV_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
                   int(blockIdx.x), int(threadIdx.x));                                          \
            __trap();                                                                           \
        }                                                                                       \
    } while (0)
#else
#define ADAKV_DCHECK(cond) \
    do {                   \
    } while (0)
#endif

// ---------------------------------------------------------------- workspace
// Bump allocator: the same code computes sizes (base == nullptr) and carves.
struct Arena {
    char* base;
    size_t off = 0;
    explicit Arena(void* b) : base(static_cast<char*>(b)) {}
    template <class T>
    T* take(size_t count) {
        off = (off + 255) & ~size_t(255);
        T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
        off += count * sizeof(T);
        return p;
    }
};
// Every workspace begins with a 256-byte header holding the error word.
constexpr size_t kWsHeader = 256;

// ---------------------------------------------------------------- dtypes
template <class T> struct Acc { using type = float; };
template <> struct Acc<double> { using type = double; };

__device__ __forceinline__ float to_acc(float x) { return x; }
__device__ __forceinline__ double to_acc(double x) { return x; }
__device__ __forceinline__ float to_acc(__nv_bfloat16 x) { return __bfloat162float(x); }

template <class T> __device__ __forceinline__ T from_acc(float x);
template <> __device__ __forceinline__ float from_acc<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16>(float x) {
    return __float2bfloat16_rn(x);
}
template <class T> __device__ __forceinline__ T from_acc(double x);
template <> __device__ __forceinline__ double from_acc<double>(double x) { return x; }

__device__ __forceinline__ float acc_exp(float x) { return expf(x); }
__device__ __forceinline__ double acc_exp(double x) { return exp(x); }

// Exact (no-FMA) fp64 arithmetic for bit-exact parity with the host reference.
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

inline size_t dtype_size(adakv_dtype t) {
    return t == ADAKV_F64 ? 8 : (t == ADAKV_F32 ? 4 : 2);
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

int device_sm_count();

}  // namespace adakv_b200
