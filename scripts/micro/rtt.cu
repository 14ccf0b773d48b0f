// Round-trip latency of the MMA-issuer <-> elementwise-warp handoff used by the
// attention backward: mode 0 tcgen05.commit, 1 plain mbarrier.arrive,
// 2 = 0 + TMEM ld x32 x2 / st x16 x4 in the elementwise warps.
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"
using namespace qtb::sm100;

__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}

__global__ void rtt(int mode, int iters, long long* out) {
    __shared__ uint64_t bar[2];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x / 32 - 4;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], nw);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    long long t0 = clock64();
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < iters; ++i) {
            if (mode != 1) tc_commit(&bar[0]); else mbar_arrive(&bar[0]);
            mbar_wait(&bar[1], i & 1);
        }
        out[0] = clock64() - t0;
    } else if (warp >= 4) {
        const uint32_t lb = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 32;
        uint32_t acc = 0;
        for (int i = 0; i < iters; ++i) {
            mbar_wait(&bar[0], i & 1);
            tc_fence_after();
            if (mode == 2) {
                uint32_t r[32], q[32];
                tmem_ld32(lb, r);
                tmem_ld32(lb + 64, q);
                tmem_ld_wait();
                uint32_t h[16];
                for (int j = 0; j < 16; ++j) h[j] = r[j] ^ q[j + 16] ^ acc;
                st16(lb, h); st16(lb + 16, h); st16(lb + 64, h); st16(lb + 80, h);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                acc += h[3];
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar[1]);
        }
        if (acc == 12345) out[1] = acc;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
    long long* d; cudaMalloc(&d, 16);
    const char* names[] = {"tc_commit", "mbar_arrive", "tc_commit+tmem ld/st"};
    for (int nw : {1, 8})
        for (int mode = 0; mode < 3; ++mode) {
            rtt<<<1, 128 + 32 * nw>>>(mode, 1000, d);
            rtt<<<1, 128 + 32 * nw>>>(mode, 1000, d);
            long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            printf("%d warps, %-22s: %.1f cycles per round trip (%s)\n", nw, names[mode], h / 1000.0,
                   cudaGetErrorString(cudaGetLastError()));
        }
}
