// Shared device helpers for the qtrain-b200 kernels (sm_100a only).
//
// Bit-exactness contract (SURVEY.md §8a'): every value the reference rounds
// is rounded here at the same point with the same mode; every f32 expression
// on a bit-exact path uses __f*_rn intrinsics so nvcc cannot contract it into
// an FMA (the reference's x86-64 build has none).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace qtb {

constexpr int kNumSMs = 148;

// ---------------------------------------------------------------------------
// FP8 formats (reference include/qtrain/numerics.hpp:20-23): 0 = E4M3 (OCP FN,
// fmax 448), 1 = E5M2 (IEEE-like, fmax 57344).
// ---------------------------------------------------------------------------
enum F8 : int { kE4M3 = 0, kE5M2 = 1 };

__host__ __device__ inline float f8_fmax(int kind) { return kind == kE4M3 ? 448.0f : 57344.0f; }

// absmax_scale (reference src/numerics.cpp:150-158): fmax/absmax computed in
// f64, converted to f32 and bumped one ulp up when the conversion rounded
// down, so fmax/scale <= absmax holds exactly.  0 -> 1.
__host__ __device__ inline float absmax_scale(float amax, int kind) {
    if (amax == 0.0f) return 1.0f;
    const double exact = (double)f8_fmax(kind) / (double)amax;
    float s = (float)exact;
    if ((double)s < exact) {
#ifdef __CUDA_ARCH__
        s = __uint_as_float(__float_as_uint(s) + 1u);  // s > 0 finite: nextafter(+inf)
#else
        union { float f; uint32_t u; } v{s};
        v.u += 1u;
        s = v.f;
#endif
    }
    return s;
}

// Saturating RNE encode of two f32 into two fp8 codes: cvt.rn.satfinite, proven
// equal to the reference's table encoder (src/numerics.cpp:87-112) on every
// finite input.  Low byte = lo.
__device__ __forceinline__ uint16_t cvt_f8x2(float lo, float hi, int kind) {
    uint16_t r;
    if (kind == kE4M3)
        asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
    else
        asm("cvt.rn.satfinite.e5m2x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
    return r;
}

// quantize_with_absmax element rule (src/numerics.cpp:170-173):
// encode(clamp(x*scale, +-fmax)).  satfinite performs the clamp.
__device__ __forceinline__ uint16_t quant2(float a, float b, float scale, int kind) {
    return cvt_f8x2(__fmul_rn(a, scale), __fmul_rn(b, scale), kind);
}

// fp8 code -> f32 (exact).
__device__ __forceinline__ float f8_decode(uint8_t c, int kind) {
    if (kind == kE4M3) {
        __nv_fp8_e4m3 v;
        v.__x = c;
        return float(v);
    }
    __nv_fp8_e5m2 v;
    v.__x = c;
    return float(v);
}

// ---------------------------------------------------------------------------
// BF16 helpers.  bf16_round (src/numerics.cpp:237-243) is RNE == cvt.rn.bf16.
// ---------------------------------------------------------------------------
// f32 -> bf16 round-to-nearest-even through the packed converter
// (cvt.rn.bf16x2.f32 = F2FP.BF16.F32.PACK_AB): same rounding as
// __float2bfloat16_rn, ~4x the throughput of the scalar F2F.BF16.F32 on sm_100
// (scripts/micro/cvt_rate.cu: 129 vs 32 values/clk/SM).
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ float bf16r(float x) { return __uint_as_float(pack_bf16x2(0.0f, x) & 0xFFFF0000u); }
__device__ __forceinline__ float bf2f(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ float bfbits2f(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }
__device__ __forceinline__ uint16_t f2bfbits(float x) { return (uint16_t)(pack_bf16x2(0.0f, x) >> 16); }

// ---------------------------------------------------------------------------
// Counter RNG (src/numerics.cpp:192-210) and stochastic rounding
// (src/numerics.cpp:249-258).  Streams (fnv1a64 of names) are hashed on the host.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}
// The first two mixing rounds depend only on (seed, stream): rng_key() is
// hoisted out of element loops, rng_uniform_k() finishes per counter.
__host__ __device__ __forceinline__ uint64_t rng_key(uint64_t seed, uint64_t stream) {
    return mix64(mix64(0x9E3779B97F4A7C15ull ^ seed) ^ stream);
}
__host__ __device__ __forceinline__ uint32_t rng_uniform_k(uint64_t key, uint64_t counter) {
    const uint64_t z = mix64(mix64(key ^ counter));
    return (uint32_t)(z >> 32) ^ (uint32_t)z;
}
__host__ __device__ __forceinline__ uint32_t rng_uniform(uint64_t seed, uint64_t stream, uint64_t counter) {
    return rng_uniform_k(rng_key(seed, stream), counter);
}
// Returns the f32 bit pattern of SR_bf16(x); representable inputs (and NaN)
// pass through unchanged.
__device__ __forceinline__ float sr_bf16k(float x, uint64_t key, uint64_t counter) {
    uint32_t bits = __float_as_uint(x);
    if ((bits & 0xFFFFu) == 0u || x != x) return x;
    bits += rng_uniform_k(key, counter) & 0xFFFFu;
    bits &= 0xFFFF0000u;
    return __uint_as_float(bits);
}
__device__ __forceinline__ float sr_bf16(float x, uint64_t seed, uint64_t stream, uint64_t counter) {
    return sr_bf16k(x, rng_key(seed, stream), counter);
}

// n / d and n % d for 0 <= n < 2^31 by multiply-high (d fixed per launch)
struct FastDiv {
    uint32_t d, m, l;
    __host__ FastDiv() : d(1), m(0), l(0) {}
    __host__ explicit FastDiv(uint32_t dv) : d(dv) {
        l = 0;
        while ((1ull << l) < dv) ++l;
        m = (uint32_t)((((1ull << l) - dv) << 32) / dv + 1);
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        if (l == 0) return n;
        const uint32_t t = __umulhi(n, m);
        return (t + ((n - t) >> 1)) >> (l - 1);
    }
};

// ---------------------------------------------------------------------------
// absmax as an order-free u32 max of |x| bit patterns: NaN (0x7FC..) > inf >
// every finite, so a NaN anywhere is sticky exactly like absmax_or_nan
// (src/model.cpp:133-140).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t abs_bits(float x) { return __float_as_uint(x) & 0x7FFFFFFFu; }
__device__ __forceinline__ uint32_t warp_max_u32(uint32_t v) {
    return __reduce_max_sync(0xffffffffu, v);
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// block-wide u32 max, then one atomicMax per CTA
template <int NT>
__device__ __forceinline__ void block_absmax_commit(uint32_t v, uint32_t* dst) {
    __shared__ uint32_t red[NT / 32];
    v = warp_max_u32(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        uint32_t w = threadIdx.x < NT / 32 ? red[threadIdx.x] : 0u;
        w = warp_max_u32(w);
        if (threadIdx.x == 0 && w != 0u) atomicMax(dst, w);
    }
}

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace qtb
