// Throughput of f32 -> bf16 rounding variants on sm_100a (per SM per clock).
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t f2bf_f2f(float x) { return __bfloat16_as_ushort(__float2bfloat16_rn(x)); }
__device__ __forceinline__ uint32_t cvt2(float lo, float hi) {
    uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo)); return r; }
__device__ __forceinline__ uint32_t rne_int(float x) {
    uint32_t b = __float_as_uint(x); return (b + 0x7FFFu + ((b >> 16) & 1u)) >> 16; }
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
template <int MODE>
__global__ void k(float* out, int iters, long long* cyc) {
    float a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001f + i;
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
            if (MODE == 0) acc += f2bf_f2f(a[i]) + f2bf_f2f(a[i + 1]);
            if (MODE == 1) acc += cvt2(a[i], a[i + 1]);
            if (MODE == 2) acc += rne_int(a[i]) + rne_int(a[i + 1]);
            if (MODE == 3) { a[i] = ex2(a[i]); a[i+1] = ex2(a[i+1]); }
            a[i] += 1.0f; a[i + 1] += 1.0f;
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + a[0] + a[2] + a[4] + a[6];
}
int main() {
    float* o; long long* c; cudaMalloc(&o, 148 * 1024 * 4 * 4); cudaMalloc(&c, 8);
    const char* names[4] = {"F2F.BF16 (1 value/instr)", "cvt.rn.bf16x2 (2 values/instr)", "integer RNE", "ex2.approx"};
    for (int mode = 0; mode < 4; ++mode) {
        int iters = 4096;
        for (int rep = 0; rep < 2; ++rep) {
            if (mode == 0) k<0><<<148 * 2, 1024>>>(o, iters, c);
            if (mode == 1) k<1><<<148 * 2, 1024>>>(o, iters, c);
            if (mode == 2) k<2><<<148 * 2, 1024>>>(o, iters, c);
            if (mode == 3) k<3><<<148 * 2, 1024>>>(o, iters, c);
        }
        cudaDeviceSynchronize();
        long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
        // values per SM per clock: 2 CTAs x 1024 threads x iters x 8 values / cycles
        printf("%-34s %.1f values/clk/SM\n", names[mode], 2.0 * 1024 * iters * 8 / (double)cy);
    }
    return 0;
}
