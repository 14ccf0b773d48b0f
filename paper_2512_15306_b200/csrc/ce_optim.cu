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
    float mx = -INFINITY;
    for (int i = threadIdx.x; i < V4; i += CE_T) {
        const float4 v = l4[i];
        mx = fmaxf(mx, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
    }
    for (int i = V4 * 4 + threadIdx.x; i < V; i += CE_T) mx = fmaxf(mx, l[i]);
    mx = block_reduce_max(mx, red);
    float s = 0.0f;
    for (int i = threadIdx.x; i < V4; i += CE_T) {
        const float4 v = l4[i];
        s += expf(v.x - mx) + expf(v.y - mx) + expf(v.z - mx) + expf(v.w - mx);
    }
    for (int i = V4 * 4 + threadIdx.x; i < V; i += CE_T) s += expf(l[i] - mx);
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

template <typename G>
__global__ void norm_partials_kernel(const G* __restrict__ g, const Seg* __restrict__ segs, int nseg, int64_t nblk,
                                     double* __restrict__ part) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nblk) return;
    // find segment: last s with blk0 <= b
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (segs[mid].blk0 <= b) lo = mid;
        else hi = mid - 1;
    }
    const Seg sg = segs[lo];
    const int64_t i0 = (b - sg.blk0) * 256;
    const int64_t i1 = min(i0 + 256, sg.n);
    double p = 0.0;
    for (int64_t i = i0; i < i1; ++i) {
        const double x = (double)gval<G>(g, sg.off + i);
        p = __dadd_rn(p, __dmul_rn(x, x));
    }
    part[b] = p;
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
struct AdamHyper {
    float lr, b1, b2, eps, wd, bc1, bc2;
    const float* grad_scale;  // device scalar (trainer clip * mean scale)
    uint64_t seed;
    int64_t step;  // 1-based step being applied
    int bf16_moments;
};

template <typename G>
__global__ void adamw_kernel(uint16_t* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                             uint16_t* __restrict__ m16, uint16_t* __restrict__ v16, const G* __restrict__ grad,
                             const Seg* __restrict__ segs, int nseg, int64_t total, AdamHyper h, int* __restrict__ err,
                             uint32_t* __restrict__ seg_amax) {
    __shared__ int64_t s_off[1024];
    const int ns = min(nseg, 1024);
    for (int i = threadIdx.x; i < ns; i += blockDim.x) s_off[i] = segs[i].off;
    __syncthreads();
    const float one_m_b1 = __fsub_rn(1.0f, h.b1), one_m_b2 = __fsub_rn(1.0f, h.b2);
    const float gscale = *h.grad_scale;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = ns - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_off[mid] <= i) lo = mid;
            else hi = mid - 1;
        }
        const Seg& sg = segs[lo];
        const int64_t j = i - sg.off;
        if (j >= sg.n) continue;  // padding between segments
        const float gi = __fmul_rn(gval<G>(grad, i), gscale);
        if (!isfinite(gi)) {
            atomicExch(err, 3);
            continue;
        }
        const float mo = h.bf16_moments ? bfbits2f(m16[i]) : m[i];
        const float vo = h.bf16_moments ? bfbits2f(v16[i]) : v[i];
        const int64_t pidx = sg.poff + j;
        const float pi = bfbits2f(p[pidx]);
        const float m_new = __fadd_rn(__fmul_rn(h.b1, mo), __fmul_rn(one_m_b1, gi));
        const float v_new = __fadd_rn(__fmul_rn(h.b2, vo), __fmul_rn(__fmul_rn(one_m_b2, gi), gi));
        const float mhat = __fdiv_rn(m_new, h.bc1);
        const float vhat = __fdiv_rn(v_new, h.bc2);
        const float upd = __fadd_rn(__fdiv_rn(mhat, __fadd_rn(__fsqrt_rn(vhat), h.eps)), __fmul_rn(h.wd, pi));
        const float p_new = __fsub_rn(pi, __fmul_rn(h.lr, upd));
        const uint64_t ctr = (uint64_t)(h.step - 1) * (uint64_t)sg.gnumel + (uint64_t)(sg.gstart + j);
        if (h.bf16_moments) {
            m16[i] = f2bfbits(sr_bf16(m_new, h.seed, sg.sm, ctr));
            v16[i] = f2bfbits(sr_bf16(v_new, h.seed, sg.sv, ctr));
        } else {
            m[i] = m_new;
            v[i] = v_new;
        }
        const float pw = sr_bf16(p_new, h.seed, sg.sw, ctr);
        p[pidx] = f2bfbits(pw);
        if (seg_amax) {
            const uint32_t a = abs_bits(pw);
            if (a) atomicMax(&seg_amax[lo], a);
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
    const unsigned g = (unsigned)ceil_div(nblk, 256);
    if (grad_f32)
        norm_partials_kernel<float><<<g, 256, 0, s>>>((const float*)grad, (const Seg*)segs, nseg, nblk, partials);
    else
        norm_partials_kernel<uint16_t><<<g, 256, 0, s>>>((const uint16_t*)grad, (const Seg*)segs, nseg, nblk, partials);
    const int nb = (int)std::min<int64_t>(1024, ceil_div(nblk, 256));
    sum_f64_kernel<<<nb, 256, 0, s>>>(partials, nblk, scratch);
    sum_f64_kernel<<<1, 256, 0, s>>>(scratch, nb, out);
    return (int)cudaGetLastError();
}

int qtk_adamw_dev(void* p, float* m, float* v, void* m16, void* v16, const void* grad, int grad_f32, const void* segs,
                  int nseg, int64_t total, float lr, float b1, float b2, float eps, float wd, float bc1, float bc2,
                  const float* grad_scale_dev, uint64_t seed, int64_t step, int bf16_moments, int* err,
                  uint32_t* seg_amax, cudaStream_t s) {
    if (nseg > 1024) return 1;
    AdamHyper h{lr, b1, b2, eps, wd, bc1, bc2, grad_scale_dev, seed, step, bf16_moments};
    const int grid = (int)std::min<int64_t>(ceil_div(total, 256), 16 * kNumSMs);
    if (grad_f32)
        adamw_kernel<float><<<grid, 256, 0, s>>>((uint16_t*)p, m, v, (uint16_t*)m16, (uint16_t*)v16,
                                                 (const float*)grad, (const Seg*)segs, nseg, total, h, err, seg_amax);
    else
        adamw_kernel<uint16_t><<<grid, 256, 0, s>>>((uint16_t*)p, m, v, (uint16_t*)m16, (uint16_t*)v16,
                                                    (const uint16_t*)grad, (const Seg*)segs, nseg, total, h, err,
                                                    seg_amax);
    return (int)cudaGetLastError();
}

}  // extern "C"
