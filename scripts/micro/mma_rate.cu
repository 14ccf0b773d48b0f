// tcgen05.mma kind::f16 issue/execution rate for the shapes the attention
// backward uses: cycles per MMA for back-to-back issue, SS vs TS (A in TMEM).
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"
using namespace qtb::sm100;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                 "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

__device__ __forceinline__ void mma_ss_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred P, p;\n\telect.sync _|P, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "@P tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__global__ void rate(int mode, int N, int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 1) tmem_alloc(&slot, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (mode == 7 && warp == 0) {  // whole warp, elect inside the asm
        const uint32_t base = smem_u32(sm);
        const uint32_t idesc = make_idesc(1, 1, false, false, 128, N);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint64_t bd = make_sdesc_sw128(base + 32768 + (i & 3) * 32, 16, 1024);
            const uint64_t ad = make_sdesc_sw128(base + (i & 3) * 32, 16, 1024);
            mma_ss_elect(tmem + 256, ad, bd, idesc, 1);
        }
        long long t1 = clock64();
        if (lane == 0) {
            tc_commit(&bar);
            mbar_wait(&bar, 0);
            long long t2 = clock64();
            out[0] = t1 - t0;
            out[1] = t2 - t0;
        }
        __syncwarp();
    } else if (mode >= 3 && mode < 7 && warp == 0) {  // whole warp, elect.sync picks the issuing lane
        const uint32_t base = smem_u32(sm);
        const uint32_t idesc = make_idesc(1, 1, false, false, 128, N);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint64_t bd = make_sdesc_sw128(base + 32768 + (i & 3) * 32, 16, 1024);
            const uint64_t ad = make_sdesc_sw128(base + (i & 3) * 32, 16, 1024);
            uint32_t e;
            asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(e));
            if (e) {
                if (mode == 3) mma_bf16(tmem + 256, ad, bd, idesc, 1);
                else mma_ts(tmem + 256, tmem + (i & 7) * 8, bd, idesc, 1);
            }
            __syncwarp();
        }
        long long t1 = clock64();
        if (lane == 0) {
            tc_commit(&bar);
            mbar_wait(&bar, 0);
            long long t2 = clock64();
            out[0] = t1 - t0;
            out[1] = t2 - t0;
        }
        __syncwarp();
    } else if ((mode < 3 || mode == 5 || mode == 6) && threadIdx.x == 0) {
        const uint32_t base = smem_u32(sm);
        const uint32_t idesc = make_idesc(1, 1, false, mode == 2, 128, N);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint64_t bd = make_sdesc_sw128(base + 32768 + (i & 3) * 32, mode == 2 ? 16384 : 16, 1024);
            if (mode == 5) mma_bf16(tmem + (i & 3) * 64, make_sdesc_sw128(base + (i & 3) * 32, 16, 1024), bd, idesc, 1);
            else if (mode == 6) {  // 8 independent MMAs per iteration, constant descriptors
                const uint64_t ad = make_sdesc_sw128(base, 16, 1024);
#pragma unroll
                for (int u = 0; u < 8; ++u) mma_bf16(tmem + (u & 3) * 64, ad + 2 * u, bd, idesc, 1);
            } else if (mode == 0) mma_bf16(tmem + 256, make_sdesc_sw128(base + (i & 3) * 32, 16, 1024), bd, idesc, 1);
            else mma_ts(tmem + 256, tmem + (i & 7) * 8, bd, idesc, 1);
        }
        long long t1 = clock64();
        tc_commit(&bar);
        mbar_wait(&bar, 0);
        long long t2 = clock64();
        out[0] = t1 - t0;
        out[1] = t2 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
    long long* d; cudaMalloc(&d, 16);
    cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    const char* names[] = {"SS K-major B", "TS K-major B", "TS MN-major B", "warp SS", "warp TS", "SS rot D",
                           "SS 8/iter", "warp elect-in-asm"};
    for (int mode = 0; mode < 8; ++mode)
        for (int N : {64, 128, 256}) {
            if (mode == 2 && N == 256) continue;
            if ((mode == 5 || mode == 6) && N > 64) continue;
            long long h[2];
            for (int rep = 0; rep < 2; ++rep) {
                rate<<<1, 128, 65536>>>(mode, N, 2000, d);
                cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            }
            const double per = mode == 6 ? 16000.0 : 2000.0;
            printf("%-14s M128 N%-3d K16: issue %.1f cyc/mma, complete %.1f cyc/mma (ideal %d) %s\n", names[mode], N,
                   h[0] / per, h[1] / per, 128 * N / 256, cudaGetErrorString(cudaGetLastError()));
        }
}
