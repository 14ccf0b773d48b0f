// Cross-entropy softmax stage (fused_cross_entropy_chunked,
// src/tensorops.cpp:344-410), the deterministic gradient norm
// (src/optim.cpp:87-110) and the AdamW update (src/optim.cpp:37-85).
//
// The LM-head logits and both CE backward matmuls run on the tcgen05 GEMM
// (gemm.cu); this file holds the per-row softmax/loss/dlogits pass and the
// HBM-bound optimizer kernels.
#include "common.cuh"
#include "kernels.h"

#include <algorithm>

namespace qtb {

// ---------------------------------------------------------------------------
// CE: one CTA per token row of f32 logits.
//   mx = max_v l ; denom = sum_v exp(l - mx) ; lse = mx + log(denom)
//   loss_row = lse - l[target]
//   dlogits[v] = (exp(l - mx) * (1/denom) - [v == target]) * inv_n   (bf16)
// The row is read twice; the second read is served by L2 (rows in flight
// across all SMs are far below the 126 MB L2).
// ---------------------------------------------------------------------------
constexpr int CE_T = 512;

__device__ __forceinline__ float block_reduce_max(float v, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    float r = -INFINITY;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r = fmaxf(r, red[i]);
    __syncthreads();
    return r;
}
__device__ __forceinline__ float block_reduce_sum(float v, float* red) {
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    float r = 0.0f;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r += red[i];  // fixed order
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(CE_T) ce_softmax_kernel(const float* __restrict__ logits, int64_t ldl, int V,
                                                          const int32_t* __restrict__ targets, float inv_n,
                                                          uint16_t* __restrict__ dlogits,
                                                          uint16_t* __restrict__ dlogits_lo, int64_t ldd,
                                                          float* __restrict__ loss_rows) {
    __shared__ float red[CE_T / 32];
    const int64_t row = blockIdx.x;
    const float* l = logits + row * ldl;
    const int V4 = V / 4;
    const float4* l4 = reinterpret_cast<const float4*>(l);
    // one pass for (max, sum exp): each thread keeps a running max and rescales
    // its partial sum when the max grows; partials meet at the block max
    float mx = -INFINITY, s = 0.0f;
    for (int i = threadIdx.x; i < V4; i += CE_T) {
        const float4 v = l4[i];
        const float m4 = fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w));
        if (m4 > mx) {
            s *= expf(mx - m4);
            mx = m4;
        }
        s += expf(v.x - mx) + expf(v.y - mx) + expf(v.z - mx) + expf(v.w - mx);
    }
    for (int i = V4 * 4 + threadIdx.x; i < V; i += CE_T) {
        const float x = l[i];
        if (x > mx) {
            s *= expf(mx - x);
            mx = x;
        }
        s += expf(x - mx);
    }
    const float bmx = block_reduce_max(mx, red);
    if (mx != -INFINITY) s *= expf(mx - bmx);
    mx = bmx;
    const float denom = block_reduce_sum(s, red);
    const int tgt = targets[row];
    if (threadIdx.x == 0) loss_rows[row] = (mx + logf(denom)) - l[tgt];
    if (!dlogits) return;
    const float inv_denom = 1.0f / denom;
    // dlogits stays f32 in the reference (tensorops.cpp:389-393): it is carried
    // here as a bf16 hi part plus a bf16 lo part (the residual), which the
    // split-A GEMMs consume as one f32-faithful operand
    uint16_t* dl = dlogits + row * ldd;
    uint16_t* dlo = dlogits_lo ? dlogits_lo + row * ldd : nullptr;
    for (int i = threadIdx.x; i < V4; i += CE_T) {
        const float4 v = l4[i];
        float p[4] = {expf(v.x - mx) * inv_denom, expf(v.y - mx) * inv_denom, expf(v.z - mx) * inv_denom,
                      expf(v.w - mx) * inv_denom};
        float hi[4], lo[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (4 * i + j == tgt) p[j] -= 1.0f;
            p[j] *= inv_n;
            hi[j] = bf16r(p[j]);
            lo[j] = p[j] - hi[j];
        }
        *reinterpret_cast<uint2*>(dl + 4 * i) = make_uint2(pack_bf16x2(hi[0], hi[1]), pack_bf16x2(hi[2], hi[3]));
        if (dlo)
            *reinterpret_cast<uint2*>(dlo + 4 * i) = make_uint2(pack_bf16x2(lo[0], lo[1]), pack_bf16x2(lo[2], lo[3]));
    }
    for (int i = V4 * 4 + threadIdx.x; i < V; i += CE_T) {
        float p = expf(l[i] - mx) * inv_denom;
        if (i == tgt) p -= 1.0f;
        p *= inv_n;
        const float hi = bf16r(p);
        dl[i] = f2bfbits(hi);
        if (dlo) dlo[i] = f2bfbits(p - hi);
    }
}


// deterministic sum of per-row losses, then * inv_n (fixed tree order)
__global__ void loss_reduce_kernel(const float* __restrict__ rows, int64_t n, float inv_n, float* __restrict__ out,
                                   float* __restrict__ accum) {
    __shared__ float red[32];
    float s = 0.0f;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += rows[i];
    s = block_reduce_sum(s, red);
    if (threadIdx.x == 0) {
        const float loss = s * inv_n;
        if (out) *out = loss;
        if (accum) *accum += loss;
    }
}

// ---------------------------------------------------------------------------
// gradient norm: f64 sum of squares over fixed 256-element blocks of each
// tensor (src/optim.cpp:87-105); block partials exactly as the reference,
// combined by a fixed-order tree (deterministic; ~1e-16 relative).
// ---------------------------------------------------------------------------
struct Seg {
    int64_t off;     // element offset in the flat buffer
    int64_t n;       // elements in this buffer
    int64_t gstart;  // global element index of off within the full tensor
    int64_t gnumel;  // full tensor numel (RNG counter base)
    uint64_t sm, sv, sw;  // fnv1a64("adamw/<name>/{m,v,w}")
    int64_t blk0;    // first norm block index of this segment
    int64_t poff;    // element offset of (gstart) in the full parameter buffer
};

template <typename G>
__device__ __forceinline__ float gval(const G* g, int64_t i);
template <>
__device__ __forceinline__ float gval<uint16_t>(const uint16_t* g, int64_t i) {
    return bfbits2f(g[i]);
}
template <>
__device__ __forceinline__ float gval<float>(const float* g, int64_t i) {
    return g[i];
}

// one warp per 256-element block: lane l holds elements [8l, 8l+8) of the
// block (16-B loads), squares in f64 (exact), lane-sequential then a fixed
// shuffle tree -- deterministic, ~1e-16 relative to the sequential sum
// 8 gradient values starting at i (zero past n) as raw bits, unpacked later: the
// loads of a warp's U blocks are all issued before the first is consumed
template <typename G>
struct Raw8;
template <>
struct Raw8<uint16_t> {
    uint4 u;
    __device__ __forceinline__ void load(const uint16_t* g, int64_t i, int64_t n) {
        if (i + 8 <= n && ((i & 7) == 0)) {
            u = *reinterpret_cast<const uint4*>(g + i);
        } else {
            uint32_t w[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t lo = (i + 2 * j < n) ? g[i + 2 * j] : 0u;
                const uint32_t hi = (i + 2 * j + 1 < n) ? g[i + 2 * j + 1] : 0u;
                w[j] = lo | (hi << 16);
            }
            u = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
    __device__ __forceinline__ void unpack(float (&x)[8]) const {
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            x[2 * j] = __uint_as_float(w[j] << 16);
            x[2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
        }
    }
};
template <>
struct Raw8<float> {
    float4 a, b;
    __device__ __forceinline__ void load(const float* g, int64_t i, int64_t n) {
        if (i + 8 <= n && ((i & 3) == 0)) {
            a = *reinterpret_cast<const float4*>(g + i);
            b = *reinterpret_cast<const float4*>(g + i + 4);
        } else {
            float x[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = (i + j < n) ? g[i + j] : 0.0f;
            a = make_float4(x[0], x[1], x[2], x[3]);
            b = make_float4(x[4], x[5], x[6], x[7]);
        }
    }
    __device__ __forceinline__ void unpack(float (&x)[8]) const {
        x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
    }
};

template <typename G>
__global__ void norm_partials_kernel(const G* __restrict__ g, const Seg* __restrict__ segs, int nseg, int64_t nblk,
                                     double* __restrict__ part) {
    // each warp owns a contiguous run of 256-element blocks, so the segment changes
    // rarely along it (tracked incrementally; one binary search per warp); U blocks'
    // loads in flight.  Per block: lane-sequential f64 squares then a fixed xor tree.
    extern __shared__ int64_t s_blk0[];
    for (int i = threadIdx.x; i < nseg; i += blockDim.x) s_blk0[i] = segs[i].blk0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t per = (nblk + nw - 1) / nw;
    const int64_t b_begin = w * per, b_end = min(nblk, b_begin + per);
    if (b_begin >= b_end) return;
    int sg = 0;
    {
        int lo = 0, hi = nseg - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_blk0[mid] <= b_begin) lo = mid;
            else hi = mid - 1;
        }
        sg = lo;
    }
    constexpr int U = 4;
    for (int64_t b0 = b_begin; b0 < b_end; b0 += U) {
        Raw8<G> raw[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t b = b0 + u;
            if (b < b_end) {
                while (sg + 1 < nseg && s_blk0[sg + 1] <= b) ++sg;
                raw[u].load(g + segs[sg].off, (b - s_blk0[sg]) * 256 + lane * 8, segs[sg].n);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t b = b0 + u;
            if (b >= b_end) break;
            float x[8];
            raw[u].unpack(x);
            double p = 0.0;
#pragma unroll
            for (int j = 0; j < 8; ++j) p = __dadd_rn(p, __dmul_rn((double)x[j], (double)x[j]));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) p = __dadd_rn(p, __shfl_xor_sync(0xffffffffu, p, o));
            if (lane == 0) part[b] = p;
        }
    }
}

__global__ void sum_f64_kernel(const double* __restrict__ in, int64_t n, double* __restrict__ out) {
    __shared__ double red[32];
    double s = 0.0;
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t b0 = blockIdx.x * per, b1 = min(n, b0 + per);
    for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) s += in[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
        out[blockIdx.x] = t;
    }
}

// ---------------------------------------------------------------------------
// AdamW (src/optim.cpp:37-59), exact f32 expression order, no FMA:
//   g  = grad*scale ; m' = b1*m + (1-b1)*g ; v' = b2*v + ((1-b2)*g)*g
//   upd = (m'/bc1)/(sqrt(v'/bc2)+eps) + wd*p ; p' = p - lr*upd
//   bf16 fields written with SR, key {seed, fnv("adamw/<name>/<field>"), (step-1)*numel + i}
// Optional per-segment absmax of the new weights (next step's FP8 weight
// quantization, fused so the weights are not re-read).
// ---------------------------------------------------------------------------
// device-resident per-step values (CUDA-graph replay): the host writes them before
// each launch; bc1 / bc2 still come from the host's powf (src/optim.cpp:63-64)
struct AdamStepDev {
    int64_t step;  // 1-based step being applied
    float bc1, bc2;
};
struct AdamHyper {
    float lr, b1, b2, eps, wd, bc1, bc2;
    const float* grad_scale;  // device scalar (trainer clip * mean scale)
    uint64_t seed;
    int64_t step;  // 1-based step being applied
    int bf16_moments;
    const AdamStepDev* sd;  // when set, step / bc1 / bc2 are read here
};

constexpr int ADAM_T = 256;
constexpr int ADAM_CHUNK = ADAM_T * 8 * 4;  // elements per CTA

// chunk table entry: (segment, first element of the chunk within the segment)
struct AdamChunk {
    int32_t seg;
    int32_t pad;
    int64_t start;
};

__device__ __forceinline__ void store8_bf16(uint16_t* p, const float (&x)[8]) {
    *reinterpret_cast<uint4*>(p) = make_uint4(pack_bf16x2(x[0], x[1]), pack_bf16x2(x[2], x[3]),
                                              pack_bf16x2(x[4], x[5]), pack_bf16x2(x[6], x[7]));
}

// x / c for a per-launch constant c from rc = RN(1/c): q = RN(x*rc) is within
// 1 ulp, the FMA residual is exact and one correction gives the correctly
// rounded quotient (Markstein) -- bitwise __fdiv_rn(x, c) in 3 instructions.
// Tiny |x| (residual could leave the normal range) takes the IEEE division.
__device__ __forceinline__ float div_const(float x, float c, float rc) {
    if (fabsf(x) < 1.0e-30f) return __fdiv_rn(x, c);
    const float q = __fmul_rn(x, rc);
    return __fmaf_rn(__fmaf_rn(-q, c, x), rc, q);
}

struct AdamConst {
    float b1, b2, omb1, omb2, bc1, bc2, rbc1, rbc2, eps, wd, lr, gscale;
    uint64_t km, kv, kw;
    int bf16_moments;
};

// one element of src/optim.cpp:37-59; returns false for a non-finite gradient
template <bool BF16M>
__device__ __forceinline__ bool adam_elem(const AdamConst& c, float g, float& p, float& m, float& v, uint64_t ctr) {
    const float gi = __fmul_rn(g, c.gscale);
    const float m_new = __fadd_rn(__fmul_rn(c.b1, m), __fmul_rn(c.omb1, gi));
    const float v_new = __fadd_rn(__fmul_rn(c.b2, v), __fmul_rn(__fmul_rn(c.omb2, gi), gi));
    const float mhat = div_const(m_new, c.bc1, c.rbc1);
    const float vhat = div_const(v_new, c.bc2, c.rbc2);
    const float upd = __fadd_rn(__fdiv_rn(mhat, __fadd_rn(__fsqrt_rn(vhat), c.eps)), __fmul_rn(c.wd, p));
    const float p_new = __fsub_rn(p, __fmul_rn(c.lr, upd));
    if (BF16M) {
        m = sr_bf16k(m_new, c.km, ctr);
        v = sr_bf16k(v_new, c.kv, ctr);
    } else {
        m = m_new;
        v = v_new;
    }
    p = sr_bf16k(p_new, c.kw, ctr);
    return isfinite(gi);
}

template <typename G>
__device__ __forceinline__ float4 ld4g(const G* g, int64_t i);
template <>
__device__ __forceinline__ float4 ld4g<uint16_t>(const uint16_t* g, int64_t i) {
    const uint2 u = *reinterpret_cast<const uint2*>(g + i);
    return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u), __uint_as_float(u.y << 16),
                       __uint_as_float(u.y & 0xFFFF0000u));
}
template <>
__device__ __forceinline__ float4 ld4g<float>(const float* g, int64_t i) {
    return *reinterpret_cast<const float4*>(g + i);
}
__device__ __forceinline__ void st4bf(uint16_t* p, int64_t i, float4 x) {
    *reinterpret_cast<uint2*>(p + i) = make_uint2(pack_bf16x2(x.x, x.y), pack_bf16x2(x.z, x.w));
}

// Lane t of the CTA owns 4 consecutive elements per iteration, so a warp
// touches 128 consecutive elements of every stream (coalesced 8/16-B accesses).
template <typename G, bool BF16M>
__global__ void __launch_bounds__(ADAM_T) adamw_kernel(uint16_t* __restrict__ p, float* __restrict__ m,
                                                       float* __restrict__ v, uint16_t* __restrict__ m16,
                                                       uint16_t* __restrict__ v16, const G* __restrict__ grad,
                                                       const Seg* __restrict__ segs,
                                                       const AdamChunk* __restrict__ chunks, AdamHyper h,
                                                       int* __restrict__ err, uint32_t* __restrict__ seg_amax) {
    if (err && *err != 0) return;  // gated step: earlier non-finite / out-of-range error (nothing updated)
    const AdamChunk ch = chunks[blockIdx.x];
    const Seg sg = segs[ch.seg];
    AdamConst c;
    c.b1 = h.b1;
    c.b2 = h.b2;
    c.omb1 = __fsub_rn(1.0f, h.b1);
    c.omb2 = __fsub_rn(1.0f, h.b2);
    int64_t step = h.step;
    float bc1 = h.bc1, bc2 = h.bc2;
    if (h.sd) {
        step = h.sd->step;
        bc1 = h.sd->bc1;
        bc2 = h.sd->bc2;
    }
    c.bc1 = bc1;
    c.bc2 = bc2;
    c.rbc1 = __frcp_rn(bc1);
    c.rbc2 = __frcp_rn(bc2);
    c.eps = h.eps;
    c.wd = h.wd;
    c.lr = h.lr;
    c.gscale = *h.grad_scale;
    c.kw = rng_key(h.seed, sg.sw);
    c.km = BF16M ? rng_key(h.seed, sg.sm) : 0;
    c.kv = BF16M ? rng_key(h.seed, sg.sv) : 0;
    c.bf16_moments = BF16M;
    const int64_t end = min(sg.n, ch.start + (int64_t)ADAM_CHUNK);
    const uint64_t ctr_base = (uint64_t)(step - 1) * (uint64_t)sg.gnumel + (uint64_t)sg.gstart;
    const bool vec_ok = ((sg.off | sg.poff) & 3) == 0;
    G const* gs = grad + sg.off;
    uint16_t* ps = p + sg.poff;
    uint32_t amax = 0;
    bool ok = true;
    if (vec_ok && end - ch.start == ADAM_CHUNK) {
        // full aligned chunk: 32-bit offsets from chunk-local base pointers, no bounds checks
        const G* gc = gs + ch.start;
        uint16_t* pc = ps + ch.start;
        float* mc = m + sg.off + ch.start;
        float* vc = v + sg.off + ch.start;
        uint16_t* m16c = m16 + sg.off + ch.start;
        uint16_t* v16c = v16 + sg.off + ch.start;
        const uint64_t cb = ctr_base + (uint64_t)ch.start;
#pragma unroll 2
        for (int j = threadIdx.x * 4; j < ADAM_CHUNK; j += ADAM_T * 4) {
            const float4 g4 = ld4g<G>(gc, j);
            float4 p4 = ld4g<uint16_t>(pc, j);
            float4 m4, v4;
            if (BF16M) {
                m4 = ld4g<uint16_t>(m16c, j);
                v4 = ld4g<uint16_t>(v16c, j);
            } else {
                m4 = *reinterpret_cast<const float4*>(mc + j);
                v4 = *reinterpret_cast<const float4*>(vc + j);
            }
            const uint64_t ctr = cb + (uint32_t)j;
            ok &= adam_elem<BF16M>(c, g4.x, p4.x, m4.x, v4.x, ctr);
            ok &= adam_elem<BF16M>(c, g4.y, p4.y, m4.y, v4.y, ctr + 1);
            ok &= adam_elem<BF16M>(c, g4.z, p4.z, m4.z, v4.z, ctr + 2);
            ok &= adam_elem<BF16M>(c, g4.w, p4.w, m4.w, v4.w, ctr + 3);
            amax = max(max(max(amax, abs_bits(p4.x)), abs_bits(p4.y)), max(abs_bits(p4.z), abs_bits(p4.w)));
            st4bf(pc, j, p4);
            if (BF16M) {
                st4bf(m16c, j, m4);
                st4bf(v16c, j, v4);
            } else {
                *reinterpret_cast<float4*>(mc + j) = m4;
                *reinterpret_cast<float4*>(vc + j) = v4;
            }
        }
    } else
    for (int64_t j = ch.start + threadIdx.x * 4; j < end; j += ADAM_T * 4) {
        const uint64_t ctr = ctr_base + (uint64_t)j;
        if (vec_ok && j + 4 <= end) {
            const float4 g4 = ld4g<G>(gs, j);
            float4 p4 = ld4g<uint16_t>(ps, j);
            float4 m4, v4;
            if (BF16M) {
                m4 = ld4g<uint16_t>(m16 + sg.off, j);
                v4 = ld4g<uint16_t>(v16 + sg.off, j);
            } else {
                m4 = *reinterpret_cast<const float4*>(m + sg.off + j);
                v4 = *reinterpret_cast<const float4*>(v + sg.off + j);
            }
            ok &= adam_elem<BF16M>(c, g4.x, p4.x, m4.x, v4.x, ctr);
            ok &= adam_elem<BF16M>(c, g4.y, p4.y, m4.y, v4.y, ctr + 1);
            ok &= adam_elem<BF16M>(c, g4.z, p4.z, m4.z, v4.z, ctr + 2);
            ok &= adam_elem<BF16M>(c, g4.w, p4.w, m4.w, v4.w, ctr + 3);
            amax = max(max(max(amax, abs_bits(p4.x)), abs_bits(p4.y)), max(abs_bits(p4.z), abs_bits(p4.w)));
            st4bf(ps, j, p4);
            if (BF16M) {
                st4bf(m16 + sg.off, j, m4);
                st4bf(v16 + sg.off, j, v4);
            } else {
                *reinterpret_cast<float4*>(m + sg.off + j) = m4;
                *reinterpret_cast<float4*>(v + sg.off + j) = v4;
            }
        } else {
            for (int64_t e = j; e < min(j + 4, end); ++e) {
                const int64_t i = sg.off + e;
                float pe = bfbits2f(ps[e]);
                float me = BF16M ? bfbits2f(m16[i]) : m[i];
                float ve = BF16M ? bfbits2f(v16[i]) : v[i];
                ok &= adam_elem<BF16M>(c, gval<G>(gs, e), pe, me, ve, ctr_base + (uint64_t)e);
                amax = max(amax, abs_bits(pe));
                ps[e] = f2bfbits(pe);
                if (BF16M) {
                    m16[i] = f2bfbits(me);
                    v16[i] = f2bfbits(ve);
                } else {
                    m[i] = me;
                    v[i] = ve;
                }
            }
        }
    }
    if (!ok) atomicExch(err, 3);  // adamw_step: non-finite gradient (src/optim.cpp:47)
    if (seg_amax && amax) atomicMax(&seg_amax[ch.seg], amax);
}


// Single-pass CE softmax from the logits GEMM's per-row statistics: the row's
// (max, sum exp) is combined from its 128-column blocks, then one pass writes
// dlogits = (exp(l - mx) / denom - [target]) / N as bf16 hi + lo
// (tensorops.cpp:372-393); loss = mx + log(denom) - l[target].
__global__ void __launch_bounds__(CE_T) ce_softmax_stats_kernel(const float* __restrict__ logits, int64_t ldl, int V,
                                                                const int32_t* __restrict__ targets,
                                                                const float2* __restrict__ stats, int nstat,
                                                                const float* __restrict__ tgt_logit, float inv_n,
                                                                uint16_t* __restrict__ dlogits,
                                                                uint16_t* __restrict__ dlogits_lo, int64_t ldd,
                                                                float* __restrict__ loss_rows,
                                                                float* __restrict__ dl_tgt) {
    __shared__ float red[CE_T / 32];
    const int64_t row = blockIdx.x;
    const float2* st = stats + row * nstat;
    float mx = -INFINITY;
    for (int i = threadIdx.x; i < nstat; i += CE_T) mx = fmaxf(mx, st[i].x);
    mx = block_reduce_max(mx, red);
    float s = 0.0f;
    for (int i = threadIdx.x; i < nstat; i += CE_T) {
        const float2 v = st[i];
        if (v.x != -INFINITY) s += v.y * expf(v.x - mx);
    }
    const float denom = block_reduce_sum(s, red);
    const int tgt = targets[row];
    if (threadIdx.x == 0) loss_rows[row] = (mx + logf(denom)) - tgt_logit[row];
    if (!dlogits) return;
    const float inv_denom = 1.0f / denom;
    const float* l = logits + row * ldl;
    const float4* l4 = reinterpret_cast<const float4*>(l);
    const int V4 = V / 4;
    uint16_t* dl = dlogits + row * ldd;
    uint16_t* dlo = dlogits_lo ? dlogits_lo + row * ldd : nullptr;
    for (int i = threadIdx.x; i < V4; i += CE_T) {
        const float4 v = __ldcs(l4 + i);
        float p[4] = {expf(v.x - mx) * inv_denom, expf(v.y - mx) * inv_denom, expf(v.z - mx) * inv_denom,
                      expf(v.w - mx) * inv_denom};
        float hi[4], lo[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (4 * i + j == tgt) {
                p[j] -= 1.0f;
                if (dl_tgt) {  // the target entry leaves the bf16 operand, kept exact in f32
                    dl_tgt[row] = p[j] * inv_n;
                    p[j] = 0.0f;
                }
            }
            p[j] *= inv_n;
            hi[j] = bf16r(p[j]);
            lo[j] = p[j] - hi[j];
        }
        *reinterpret_cast<uint2*>(dl + 4 * i) = make_uint2(pack_bf16x2(hi[0], hi[1]), pack_bf16x2(hi[2], hi[3]));
        if (dlo)
            *reinterpret_cast<uint2*>(dlo + 4 * i) = make_uint2(pack_bf16x2(lo[0], lo[1]), pack_bf16x2(lo[2], lo[3]));
    }
    for (int i = V4 * 4 + threadIdx.x; i < V; i += CE_T) {
        float p = expf(l[i] - mx) * inv_denom;
        if (i == tgt) {
            p -= 1.0f;
            if (dl_tgt) {
                dl_tgt[row] = p * inv_n;
                p = 0.0f;
            }
        }
        p *= inv_n;
        const float hi = bf16r(p);
        dl[i] = f2bfbits(hi);
        if (dlo) dlo[i] = f2bfbits(p - hi);
    }
}

// LM-head backward with the target term kept exact (the "target-exact" CE
// backward, DESIGN.md §2 A15).  dlogits = (p - 1[target]) / N
// (tensorops.cpp:372-393) is split into the bf16 operand of the two GEMMs with
// the target entry zeroed, and the f32 target term dl_t[m] = (p_t - 1) / N:
//   d_hidden[m]  = bf16( sum_v bf16(dl[m,v]) W[v]  +  dl_t[m] * W[t_m] )
//   d_lm_w[v]   += sum_{m : t_m = v} dl_t[m] * h[m]     (ascending m)
// The non-target entries p_v / N are small (sum_v p_v <= 1), so their bf16
// rounding moves the sum by less than the tensor core's own f32 accumulation;
// the one O(1/N) entry per row is never rounded.
__global__ void lm_dgrad_finish_kernel(const float* __restrict__ acc, int64_t M, int d, const float* __restrict__ dl_t,
                                       const int32_t* __restrict__ targets, const uint16_t* __restrict__ W,
                                       uint16_t* __restrict__ out) {
    const int d4 = d / 4;
    const int64_t total = M * d4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = i / d4;
        const int c = (int)(i - m * d4) * 4;
        const float4 a = reinterpret_cast<const float4*>(acc + m * d)[c / 4];
        const float t = dl_t[m];
        const uint2 wb = *reinterpret_cast<const uint2*>(W + (int64_t)targets[m] * d + c);
        const float w0 = bfbits2f((uint16_t)(wb.x & 0xFFFF)), w1 = bfbits2f((uint16_t)(wb.x >> 16));
        const float w2 = bfbits2f((uint16_t)(wb.y & 0xFFFF)), w3 = bfbits2f((uint16_t)(wb.y >> 16));
        const float r0 = bf16r(__fadd_rn(a.x, __fmul_rn(t, w0)));
        const float r1 = bf16r(__fadd_rn(a.y, __fmul_rn(t, w1)));
        const float r2 = bf16r(__fadd_rn(a.z, __fmul_rn(t, w2)));
        const float r3 = bf16r(__fadd_rn(a.w, __fmul_rn(t, w3)));
        *reinterpret_cast<uint2*>(out + m * d + c) = make_uint2(pack_bf16x2(r0, r1), pack_bf16x2(r2, r3));
    }
}

// one CTA per distinct target id (segments of the stable sort of the targets):
// acc[v] += dl_t[m] * h[m] over the segment's positions in ascending order
__global__ void lm_wgrad_targets_kernel(float* __restrict__ acc, int d, const int32_t* __restrict__ sorted_pos,
                                        const int32_t* __restrict__ seg_tok, const int32_t* __restrict__ seg_off,
                                        const int* __restrict__ nseg, const float* __restrict__ dl_t,
                                        const uint16_t* __restrict__ h) {
    const int ns = *nseg;
    for (int sgi = blockIdx.x; sgi < ns; sgi += gridDim.x) {
        const int v = seg_tok[sgi], b = seg_off[sgi], e = seg_off[sgi + 1];
        float* row = acc + (int64_t)v * d;
        for (int c = threadIdx.x; c < d; c += blockDim.x) {
            float x = row[c];
            for (int k = b; k < e; ++k) {
                const int m = sorted_pos[k];
                x = __fadd_rn(x, __fmul_rn(dl_t[m], bfbits2f(h[(int64_t)m * d + c])));
            }
            row[c] = x;
        }
    }
}

}  // namespace qtb

using namespace qtb;

extern "C" {

int qtk_ce_softmax(const float* logits, int64_t ldl, int64_t rows, int V, const int32_t* targets, float inv_n,
                   void* dlogits, void* dlogits_lo, int64_t ldd, float* loss_rows, cudaStream_t s) {
    if (rows <= 0) return 0;
    if ((ldl & 3) || (dlogits && (ldd & 3))) return 1;
    ce_softmax_kernel<<<(unsigned)rows, CE_T, 0, s>>>(logits, ldl, V, targets, inv_n, (uint16_t*)dlogits,
                                                      (uint16_t*)dlogits_lo, ldd, loss_rows);
    return (int)cudaGetLastError();
}

int qtk_ce_softmax_stats(const float* logits, int64_t ldl, int64_t rows, int V, const int32_t* targets,
                         const float* stats, const float* tgt_logit, float inv_n, void* dlogits, void* dlogits_lo,
                         int64_t ldd, float* loss_rows, cudaStream_t s) {
    if (rows <= 0) return 0;
    if ((ldl & 3) || (dlogits && (ldd & 3)) || !stats || !tgt_logit) return 1;
    ce_softmax_stats_kernel<<<(unsigned)rows, CE_T, 0, s>>>(logits, ldl, V, targets, (const float2*)stats,
                                                            (int)ceil_div(V, 128), tgt_logit, inv_n,
                                                            (uint16_t*)dlogits, (uint16_t*)dlogits_lo, ldd, loss_rows,
                                                            nullptr);
    return (int)cudaGetLastError();
}

int qtk_ce_softmax_stats_tx(const float* logits, int64_t ldl, int64_t rows, int V, const int32_t* targets,
                            const float* stats, const float* tgt_logit, float inv_n, void* dlogits, int64_t ldd,
                            float* loss_rows, float* dl_tgt, cudaStream_t s) {
    if (rows <= 0) return 0;
    if ((ldl & 3) || !dlogits || (ldd & 3) || !stats || !tgt_logit || !dl_tgt) return 1;
    ce_softmax_stats_kernel<<<(unsigned)rows, CE_T, 0, s>>>(logits, ldl, V, targets, (const float2*)stats,
                                                            (int)ceil_div(V, 128), tgt_logit, inv_n,
                                                            (uint16_t*)dlogits, nullptr, ldd, loss_rows, dl_tgt);
    return (int)cudaGetLastError();
}

int qtk_lm_dgrad_finish(const float* acc, int64_t M, int d, const float* dl_tgt, const int32_t* targets,
                        const void* lm_w, void* d_hidden, cudaStream_t s) {
    if (M <= 0) return 0;
    if (d % 4) return 1;
    const int64_t n4 = M * (d / 4);
    const unsigned g = (unsigned)std::min<int64_t>(ceil_div(n4, 256), 16 * kNumSMs);
    lm_dgrad_finish_kernel<<<g, 256, 0, s>>>(acc, M, d, dl_tgt, targets, (const uint16_t*)lm_w, (uint16_t*)d_hidden);
    return (int)cudaGetLastError();
}

int qtk_lm_wgrad_targets(float* acc, int d, const int32_t* sorted_pos, const int32_t* seg_tok, const int32_t* seg_off,
                         const int* nseg, int64_t max_segs, const float* dl_tgt, const void* hidden, cudaStream_t s) {
    if (max_segs <= 0) return 0;
    const unsigned g = (unsigned)std::min<int64_t>(max_segs, 16 * kNumSMs);
    lm_wgrad_targets_kernel<<<g, 128, 0, s>>>(acc, d, sorted_pos, seg_tok, seg_off, nseg, dl_tgt,
                                              (const uint16_t*)hidden);
    return (int)cudaGetLastError();
}

int qtk_loss_reduce(const float* loss_rows, int64_t n, float inv_n, float* out, float* accum, cudaStream_t s) {
    loss_reduce_kernel<<<1, 1024, 0, s>>>(loss_rows, n, inv_n, out, accum);
    return (int)cudaGetLastError();
}

int qtk_seg_size(void) { return (int)sizeof(Seg); }

// segs: device array of QtkSeg (layout == qtb::Seg); partials: nblk doubles;
// scratch: >= 1024 doubles; out: one double (sum of squares)
int qtk_grad_sumsq(const void* grad, int grad_f32, const void* segs, int nseg, int64_t nblk, double* partials,
                   double* scratch, double* out, cudaStream_t s) {
    if (nblk <= 0) return cudaMemsetAsync(out, 0, sizeof(double), s);
    const unsigned g = (unsigned)std::min<int64_t>(ceil_div(nblk * 32, 256), 32 * kNumSMs);
    if (grad_f32)
        norm_partials_kernel<float><<<g, 256, nseg * sizeof(int64_t), s>>>((const float*)grad, (const Seg*)segs, nseg, nblk, partials);
    else
        norm_partials_kernel<uint16_t><<<g, 256, nseg * sizeof(int64_t), s>>>((const uint16_t*)grad, (const Seg*)segs, nseg, nblk, partials);
    const int nb = (int)std::min<int64_t>(1024, ceil_div(nblk, 256));
    sum_f64_kernel<<<nb, 256, 0, s>>>(partials, nblk, scratch);
    sum_f64_kernel<<<1, 256, 0, s>>>(scratch, nb, out);
    return (int)cudaGetLastError();
}

int qtk_adamw_chunk_size(void) { return ADAM_CHUNK; }
int qtk_adamw_chunk_entry_size(void) { return (int)sizeof(AdamChunk); }

// chunks: device table of qtk_adamw_nchunks entries {int32 seg, int32 pad, int64 start},
// one per ADAM_CHUNK elements of every segment (built on the host)
int qtk_adamw_dev_sd(void* p, float* m, float* v, void* m16, void* v16, const void* grad, int grad_f32, const void* segs,
                  const void* chunks, int nchunks, float lr, float b1, float b2, float eps, float wd, float bc1,
                  float bc2, const float* grad_scale_dev, uint64_t seed, int64_t step, int bf16_moments, int* err,
                  uint32_t* seg_amax, const void* step_dev, cudaStream_t s) {
    if (nchunks <= 0) return 0;
    AdamHyper h{lr, b1, b2, eps, wd, bc1, bc2, grad_scale_dev, seed, step, bf16_moments,
                static_cast<const AdamStepDev*>(step_dev)};
    if (grad_f32)
        (bf16_moments ? adamw_kernel<float, true> : adamw_kernel<float, false>)<<<nchunks, ADAM_T, 0, s>>>(
            (uint16_t*)p, m, v, (uint16_t*)m16, (uint16_t*)v16, (const float*)grad, (const Seg*)segs,
            (const AdamChunk*)chunks, h, err, seg_amax);
    else
        (bf16_moments ? adamw_kernel<uint16_t, true> : adamw_kernel<uint16_t, false>)<<<nchunks, ADAM_T, 0, s>>>(
            (uint16_t*)p, m, v, (uint16_t*)m16, (uint16_t*)v16, (const uint16_t*)grad, (const Seg*)segs,
            (const AdamChunk*)chunks, h, err, seg_amax);
    return (int)cudaGetLastError();
}

int qtk_adamw_dev(void* p, float* m, float* v, void* m16, void* v16, const void* grad, int grad_f32, const void* segs,
                  const void* chunks, int nchunks, float lr, float b1, float b2, float eps, float wd, float bc1,
                  float bc2, const float* grad_scale_dev, uint64_t seed, int64_t step, int bf16_moments, int* err,
                  uint32_t* seg_amax, cudaStream_t s) {
    return qtk_adamw_dev_sd(p, m, v, m16, v16, grad, grad_f32, segs, chunks, nchunks, lr, b1, b2, eps, wd, bc1, bc2,
                            grad_scale_dev, seed, step, bf16_moments, err, seg_amax, nullptr, s);
}

}  // extern "C"
