// Cycles per element of the sequential f32 sum-of-squares chain (RMSNorm) for one
// thread per row: (A) row in shared memory, (B) row streamed from global memory.
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void unpack8(const uint4 u, float (&f)[8]) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) { f[2 * j] = __uint_as_float(w[j] << 16); f[2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u); }
}
template <int D>
__global__ void chain_smem(float* out, long long* cyc) {
    extern __shared__ __align__(16) uint8_t sm[];
    const int r = threadIdx.x, stride = 2 * D + 16;
    for (int i = r; i < 16 * D / 8; i += 16) {
        const int row = i / (D / 8), c = i % (D / 8);
        *reinterpret_cast<uint4*>(sm + row * stride + c * 16) = make_uint4(0x3f803f80u + i, 0x3f803f81u, 0x3f803f82u, 0x3f803f83u);
    }
    __syncthreads();
    const uint4* p = reinterpret_cast<const uint4*>(sm + r * stride);
    long long t0 = clock64();
    float s = 0.0f;
    for (int c = 0; c < D / 8; c += 4) {
        uint4 u[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) u[k] = p[c + k];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            float a[8]; unpack8(u[k], a);
            float q[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) q[j] = __fmul_rn(a[j], a[j]);
#pragma unroll
            for (int j = 0; j < 8; ++j) s = __fadd_rn(s, q[j]);
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * 32 + r] = s;
    if (r == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int D, int PF>
__global__ void chain_global(const uint4* __restrict__ x, float* out, long long* cyc) {
    const int r = blockIdx.x * 32 + threadIdx.x;
    const uint4* p = x + (size_t)r * (D / 8);
    long long t0 = clock64();
    float s = 0.0f;
    uint4 nx[PF];
#pragma unroll
    for (int k = 0; k < PF; ++k) nx[k] = __ldg(p + k);
    for (int c = 0; c < D / 8; c += PF) {
        uint4 u[PF];
#pragma unroll
        for (int k = 0; k < PF; ++k) u[k] = nx[k];
        if (c + PF < D / 8) {
#pragma unroll
            for (int k = 0; k < PF; ++k) nx[k] = __ldg(p + c + PF + k);
        }
#pragma unroll
        for (int k = 0; k < PF; ++k) {
            float a[8]; unpack8(u[k], a);
            float q[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) q[j] = __fmul_rn(a[j], a[j]);
#pragma unroll
            for (int j = 0; j < 8; ++j) s = __fadd_rn(s, q[j]);
        }
    }
    long long t1 = clock64();
    out[r] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    constexpr int D = 4096;
    float* o; long long* c; uint4* x;
    cudaMalloc(&o, 8192 * 4); cudaMalloc(&c, 8); cudaMalloc(&x, (size_t)8192 * D * 2);
    cudaMemset(x, 0x3f, (size_t)8192 * D * 2);
    const int smem = 16 * (2 * D + 16);
    cudaFuncSetAttribute(chain_smem<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    long long cy;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a); chain_smem<D><<<256, 16, smem>>>(o, c); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
        printf("smem  : %.2f cycles/element, kernel %.1f us (%s)\n", (double)cy / D, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
#define RUNG(PF) \
        cudaEventRecord(a); chain_global<D, PF><<<256, 32>>>(x, o, c); cudaEventRecord(b); cudaEventSynchronize(b); \
        cudaEventElapsedTime(&ms, a, b); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); \
        printf("global PF=%d: %.2f cycles/element, kernel %.1f us\n", PF, (double)cy / D, ms * 1e3);
        cudaMemset(x, 0x3f, (size_t)8192 * D * 2);  // evict L2 (memset of 67 MB) -- rows cold-ish
        RUNG(8) RUNG(16) RUNG(32)
    }
    return 0;
}
