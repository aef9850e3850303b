// mma.sync m16n8k16 bf16 latency / throughput and LDS.128 latency on this GPU (one warp).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void mma(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__global__ void k(long long* out, uint32_t x) {
    float c[8][4] = {};
    __shared__ uint4 sm[1024];
    for (int i = threadIdx.x; i < 1024; i += 32) sm[i] = make_uint4(x, x, x, x);
    __syncwarp();
    long long t0 = clock64();
    for (int i = 0; i < 64; ++i) mma(c[0], x, x, x, x, x, x);           // dependent chain
    long long t1 = clock64();
    for (int i = 0; i < 64; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) mma(c[j], x, x, x, x, x, x);          // 8 independent chains
    long long t2 = clock64();
    uint32_t a = threadIdx.x * 16;
    uint4 v = make_uint4(0, 0, 0, 0);
    for (int i = 0; i < 64; ++i) {                                          // dependent LDS.128
        asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a + (uint32_t)__cvta_generic_to_shared(sm)));
        a = (v.x & 0xf) * 16 + threadIdx.x * 16;
    }
    long long t3 = clock64();
    float s = 0;
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
    if (threadIdx.x == 0) {
        out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = (long long)s + v.x;
    }
}
int main() {
    long long* d; cudaMalloc(&d, 64);
    long long h[4];
    for (int r = 0; r < 3; ++r) {
        k<<<1, 32>>>(d, 0x3f803f80u);
        cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    }
    printf("mma dep latency %.1f cyc, 8-chain per-mma %.1f cyc, lds128 dep latency %.1f cyc\n", h[0] / 64.0, h[1] / 512.0, h[2] / 64.0);
    return 0;
}
