// Per-tensor absmax and FP8 cast kernels (north-star item 1).
//
// Reference semantics: absmax / absmax_or_nan (src/numerics.cpp:141-148,
// src/model.cpp:133-140), absmax_scale (src/numerics.cpp:150-158),
// quantize_with_absmax (src/numerics.cpp:160-176) and
// transpose_quantize_with_absmax (src/tensorops.cpp:164-182).  All outputs are
// bit-exact: max is order-free, the scale is computed in f64 exactly as the
// reference does, and cvt.rn.satfinite equals the reference encoder.
//
// HBM roofline: absmax reads 2 B/elem; cast reads 2 B and writes 1 B per
// elem; the dual-layout cast (row-major + transposed codes) writes 2 B.
#include "common.cuh"
#include "kernels.h"

namespace qtb {

// ---------------------------------------------------------------------------
// absmax: 16-B vector loads, grid-stride, one atomicMax per CTA
// ---------------------------------------------------------------------------
template <int NT>
__global__ void __launch_bounds__(NT) absmax_bf16_kernel(const uint4* __restrict__ x, int64_t nvec,
                                                         const uint16_t* __restrict__ tail, int ntail,
                                                         uint32_t* __restrict__ out) {
    uint32_t m = 0;
    const int64_t stride = (int64_t)gridDim.x * NT;
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    // 4 independent 16-B loads in flight per thread
    for (; i + 3 * stride < nvec; i += 4 * stride) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldcs(x + i + u * stride);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                m = max(m, (w[j] & 0x7FFFu) << 16);
                m = max(m, (w[j] & 0x7FFF0000u));
            }
        }
    }
    for (; i < nvec; i += stride) {
        const uint4 v = __ldcs(x + i);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            m = max(m, (w[j] & 0x7FFFu) << 16);
            m = max(m, (w[j] & 0x7FFF0000u));
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < ntail) m = max(m, ((uint32_t)tail[threadIdx.x] & 0x7FFFu) << 16);
    block_absmax_commit<NT>(m, out);
}

template <int NT>
__global__ void __launch_bounds__(NT) absmax_f32_kernel(const float* __restrict__ x, int64_t n,
                                                        uint32_t* __restrict__ out) {
    uint32_t m = 0;
    for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT)
        m = max(m, abs_bits(x[i]));
    block_absmax_commit<NT>(m, out);
}

// ---------------------------------------------------------------------------
// cast: 16 bf16 in (2 x 16 B) -> 16 codes out (16 B)
// ---------------------------------------------------------------------------
__device__ __forceinline__ float load_amax(const uint32_t* p) { return __uint_as_float(*p); }

// cast: lane i of the grid converts 8 consecutive bf16 (one 16-B load) to 8
// codes (one 8-B store) -- a warp moves 512 contiguous bytes in and 256 out;
// 4 vectors per thread in flight.
template <int NT>
__global__ void __launch_bounds__(NT) quantize_bf16_kernel(const uint16_t* __restrict__ x, int64_t n, int kind,
                                                           const uint32_t* __restrict__ amax_bits,
                                                           uint8_t* __restrict__ codes,
                                                           float* __restrict__ scale_out) {
    const float scale = absmax_scale(load_amax(amax_bits), kind);
    if (blockIdx.x == 0 && threadIdx.x == 0 && scale_out) *scale_out = scale;
    const int64_t n8 = n / 8;
    const uint4* xv = reinterpret_cast<const uint4*>(x);
    uint2* cv = reinterpret_cast<uint2*>(codes);
    constexpr int U = 4;
    const int64_t stride = (int64_t)gridDim.x * NT;
    for (int64_t i0 = (int64_t)blockIdx.x * NT + threadIdx.x; i0 < n8; i0 += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int k = 0; k < U; ++k)
            if (i0 + k * stride < n8) v[k] = __ldcs(xv + i0 + k * stride);
#pragma unroll
        for (int k = 0; k < U; ++k) {
            if (i0 + k * stride < n8) {
                const uint32_t w[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
                uint32_t o[2];
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const uint32_t p0 = quant2(__uint_as_float(w[2 * j] << 16), __uint_as_float(w[2 * j] & 0xFFFF0000u),
                                               scale, kind);
                    const uint32_t p1 = quant2(__uint_as_float(w[2 * j + 1] << 16),
                                               __uint_as_float(w[2 * j + 1] & 0xFFFF0000u), scale, kind);
                    o[j] = p0 | (p1 << 16);
                }
                cv[i0 + k * stride] = make_uint2(o[0], o[1]);
            }
        }
    }
    // tail
    for (int64_t i = n8 * 8 + (int64_t)blockIdx.x * NT + threadIdx.x; i < n; i += stride)
        codes[i] = (uint8_t)(quant2(bfbits2f(x[i]), 0.0f, scale, kind) & 0xFF);
}

// transpose cast: x (rows, cols) bf16 -> codes_t (cols, rows); optionally also
// the row-major codes.  64x64 tile through smem; each thread writes 16 B.
constexpr int TT = 64;
__global__ void __launch_bounds__(256) quantize_transpose_bf16_kernel(
    const uint16_t* __restrict__ x, int64_t rows, int64_t cols, int kind, const uint32_t* __restrict__ amax_bits,
    uint8_t* __restrict__ codes_t, uint8_t* __restrict__ codes_rm, float* __restrict__ scale_out) {
    __shared__ uint8_t tile[TT][TT + 16];
    const float scale = absmax_scale(load_amax(amax_bits), kind);
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && scale_out) *scale_out = scale;
    const int64_t r0 = (int64_t)blockIdx.y * TT, c0 = (int64_t)blockIdx.x * TT;
    // load: 64 rows x 64 cols bf16 = 64 x 128 B; 256 threads x 16 cols each
    const int tr = threadIdx.x / 4, tc = (threadIdx.x % 4) * 16;
    const int64_t r = r0 + tr;
    uint8_t q[16];
    const bool full = (r < rows) && (c0 + tc + 16 <= cols) && ((cols & 7) == 0);
    if (full) {
        const uint4* p = reinterpret_cast<const uint4*>(x + r * cols + c0 + tc);
        const uint4 a = p[0], b = p[1];
        const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint16_t pr = quant2(__uint_as_float(w[j] << 16), __uint_as_float(w[j] & 0xFFFF0000u), scale, kind);
            q[2 * j] = pr & 0xFF;
            q[2 * j + 1] = pr >> 8;
        }
    } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int64_t c = c0 + tc + j;
            q[j] = (r < rows && c < cols) ? (uint8_t)(quant2(bfbits2f(x[r * cols + c]), 0.0f, scale, kind) & 0xFF) : 0;
        }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) tile[tr][tc + j] = q[j];
    if (codes_rm) {
        if (full && (cols % 16) == 0) {
            *reinterpret_cast<uint4*>(codes_rm + r * cols + c0 + tc) = *reinterpret_cast<const uint4*>(q);
        } else {
            for (int j = 0; j < 16; ++j) {
                const int64_t c = c0 + tc + j;
                if (r < rows && c < cols) codes_rm[r * cols + c] = q[j];
            }
        }
    }
    __syncthreads();
    // store transposed: out row = c (64 of them), 64 codes each = 4 x 16 B
    const int oc = threadIdx.x / 4, orr = (threadIdx.x % 4) * 16;
    const int64_t c = c0 + oc;
    uint8_t o[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) o[j] = tile[orr + j][oc];
    if (c < cols) {
        if (r0 + orr + 16 <= rows && (rows % 16) == 0) {
            *reinterpret_cast<uint4*>(codes_t + c * rows + r0 + orr) = *reinterpret_cast<const uint4*>(o);
        } else {
            for (int j = 0; j < 16; ++j)
                if (r0 + orr + j < rows) codes_t[c * rows + r0 + orr + j] = o[j];
        }
    }
}

}  // namespace qtb

using namespace qtb;

extern "C" {

int qtk_absmax_bf16(const void* x, int64_t n, uint32_t* amax_bits, cudaStream_t s) {
    if (n <= 0) return 0;
    const int64_t nvec = n / 8;
    const int ntail = (int)(n - nvec * 8);
    const int64_t want = ceil_div(nvec, 256 * 4);
    const int grid = (int)(want < 4 * kNumSMs ? (want < 1 ? 1 : want) : 4 * kNumSMs);
    absmax_bf16_kernel<256><<<grid, 256, 0, s>>>(reinterpret_cast<const uint4*>(x), nvec,
                                                 reinterpret_cast<const uint16_t*>(x) + nvec * 8, ntail, amax_bits);
    return (int)cudaGetLastError();
}

int qtk_absmax_f32(const float* x, int64_t n, uint32_t* amax_bits, cudaStream_t s) {
    if (n <= 0) return 0;
    const int64_t want = ceil_div(n, 256 * 8);
    const int grid = (int)(want < 4 * kNumSMs ? (want < 1 ? 1 : want) : 4 * kNumSMs);
    absmax_f32_kernel<256><<<grid, 256, 0, s>>>(x, n, amax_bits);
    return (int)cudaGetLastError();
}

int qtk_quantize_bf16(const void* x, int64_t n, int kind, const uint32_t* amax_bits, uint8_t* codes,
                      float* scale_out, cudaStream_t s) {
    if (n <= 0) return 0;
    const int64_t want = ceil_div(n / 32 + 1, 256);  // >= 4 vectors of 8 per thread
    const int grid = (int)(want < 8 * kNumSMs ? want : 8 * kNumSMs);
    quantize_bf16_kernel<256><<<grid, 256, 0, s>>>(reinterpret_cast<const uint16_t*>(x), n, kind, amax_bits, codes,
                                                   scale_out);
    return (int)cudaGetLastError();
}

int qtk_quantize_transpose_bf16(const void* x, int64_t rows, int64_t cols, int kind, const uint32_t* amax_bits,
                                uint8_t* codes_t, uint8_t* codes_rm, float* scale_out, cudaStream_t s) {
    if (rows <= 0 || cols <= 0) return 0;
    dim3 grid((unsigned)ceil_div(cols, TT), (unsigned)ceil_div(rows, TT));
    quantize_transpose_bf16_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const uint16_t*>(x), rows, cols, kind,
                                                        amax_bits, codes_t, codes_rm, scale_out);
    return (int)cudaGetLastError();
}

}  // extern "C"
