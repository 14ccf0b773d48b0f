// Stable sort of token positions by id for the ordered embedding backward
// (src/tensorops.cpp:326-332: std::stable_sort + per-token ascending
// positions).  LSD radix sort is stable, so equal ids keep ascending
// position order exactly like the reference.  Uses CUB from the CUDA toolkit
// (a library sort on 16K keys, off the critical path).
#include "common.cuh"
#include "kernels.h"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>

namespace qtb {
__global__ void iota_kernel(int32_t* p, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = i;
}
__global__ void finish_offsets_kernel(int32_t* off, const int* nseg, int n) { off[*nseg] = n; }
}  // namespace qtb

using namespace qtb;

extern "C" {

static int bits_for(int64_t V) {
    int b = 1;
    while ((int64_t(1) << b) < V) ++b;
    return b;
}

// scratch layout (ints unless noted): keys_out[n], pos_in[n], counts[n], then CUB temp
size_t qtk_embed_sort_scratch_bytes(int n, int64_t V) {
    size_t a = 0, b = 0, c = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (int32_t*)nullptr, (int32_t*)nullptr, (int32_t*)nullptr,
                                    (int32_t*)nullptr, n, 0, bits_for(V));
    cub::DeviceRunLengthEncode::Encode(nullptr, b, (int32_t*)nullptr, (int32_t*)nullptr, (int32_t*)nullptr,
                                       (int*)nullptr, n);
    cub::DeviceScan::ExclusiveSum(nullptr, c, (int32_t*)nullptr, (int32_t*)nullptr, n);
    size_t t = a > b ? a : b;
    t = t > c ? t : c;
    return 3 * (size_t)n * sizeof(int32_t) + t + 256;
}

// ids[n] -> sorted_pos[n], seg_tok[n], seg_off[n+1], *nseg (device)
int qtk_embed_sort(const int32_t* ids, int n, int64_t V, void* scratch, size_t scratch_bytes, int32_t* sorted_pos,
                   int32_t* seg_tok, int32_t* seg_off, int* nseg, cudaStream_t s) {
    int32_t* keys_out = (int32_t*)scratch;
    int32_t* pos_in = keys_out + n;
    int32_t* counts = pos_in + n;
    uint8_t* temp = (uint8_t*)(counts + n);
    temp = (uint8_t*)(((uintptr_t)temp + 255) & ~uintptr_t(255));
    size_t tb = scratch_bytes - (size_t)(temp - (uint8_t*)scratch);
    iota_kernel<<<(n + 255) / 256, 256, 0, s>>>(pos_in, n);
    cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, tb, ids, keys_out, pos_in, sorted_pos, n, 0, bits_for(V), s);
    if (e != cudaSuccess) return (int)e;
    cudaMemsetAsync(counts, 0, (size_t)n * sizeof(int32_t), s);
    tb = scratch_bytes - (size_t)(temp - (uint8_t*)scratch);
    e = cub::DeviceRunLengthEncode::Encode(temp, tb, keys_out, seg_tok, counts, nseg, n, s);
    if (e != cudaSuccess) return (int)e;
    tb = scratch_bytes - (size_t)(temp - (uint8_t*)scratch);
    e = cub::DeviceScan::ExclusiveSum(temp, tb, counts, seg_off, n, s);
    if (e != cudaSuccess) return (int)e;
    finish_offsets_kernel<<<1, 1, 0, s>>>(seg_off, nseg, n);
    return (int)cudaGetLastError();
}

}  // extern "C"
