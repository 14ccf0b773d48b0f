// Per-boundary cost of back-to-back kernels in a CUDA graph, with and without
// programmatic dependent launch (griddepcontrol).  Each kernel streams a
// buffer (HBM-bound, ~148*8 CTAs) so the tail of one overlaps the prologue of
// the next only under PDL.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 pdl_gap.cu -o pdl_gap
#include <cstdio>
#include <cuda_runtime.h>

template <bool PDL>
__global__ void __launch_bounds__(256) stream_kernel(const float4* __restrict__ in, float4* __restrict__ out, long n) {
    if (PDL) {
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    for (long i = blockIdx.x * 256L + threadIdx.x; i < n; i += (long)gridDim.x * 256) {
        float4 v = in[i];
        v.x += 1.0f;
        out[i] = v;
    }
}

int main() {
    const int K = 400;
    for (long n4 : {1L << 16, 1L << 18, 1L << 20, 1L << 22}) {
        float4 *a, *b;
        cudaMalloc(&a, n4 * 16);
        cudaMalloc(&b, n4 * 16);
        cudaMemset(a, 0, n4 * 16);
        cudaMemset(b, 0, n4 * 16);
        for (int pdl = 0; pdl < 2; ++pdl) {
            cudaStream_t s;
            cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
            cudaGraph_t g;
            cudaGraphExec_t ge;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
            for (int k = 0; k < K; ++k) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(148 * 8);
                cfg.blockDim = dim3(256);
                cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = pdl ? 1 : 0;
                const float4* in = (k & 1) ? b : a;
                float4* out = (k & 1) ? a : b;
                if (pdl)
                    cudaLaunchKernelEx(&cfg, stream_kernel<true>, in, out, n4);
                else
                    cudaLaunchKernelEx(&cfg, stream_kernel<false>, in, out, n4);
            }
            cudaStreamEndCapture(s, &g);
            cudaGraphInstantiate(&ge, g, 0);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            float best = 1e30f;
            for (int r = 0; r < 6; ++r) {
                cudaEventRecord(e0, s);
                cudaGraphLaunch(ge, s);
                cudaEventRecord(e1, s);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (r > 0 && ms < best) best = ms;
            }
            printf("bytes/kernel %8.1f MB  pdl=%d  %.3f us per kernel  (%s)\n", n4 * 32 / 1e6, pdl, best * 1e3 / K,
                   cudaGetErrorString(cudaGetLastError()));
            cudaGraphExecDestroy(ge);
            cudaGraphDestroy(g);
            cudaStreamDestroy(s);
        }
        cudaFree(a);
        cudaFree(b);
    }
    return 0;
}
