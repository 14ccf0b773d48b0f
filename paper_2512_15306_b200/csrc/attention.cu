// Causal GQA attention, forward + deterministic backward (north-star item 3,
// "attention softmax").  Reference: sdpa_chunked / sdpa_chunked_backward /
// attn_row_forward (src/tensorops.cpp:191-303) with split/merge_heads
// (src/model.cpp:195-219).
//
// The kernels read q/k/v straight out of the (rows, qkv_dim) RoPE'd tensor
// and write att (rows, d) / d_qkv (rows, qkv_dim) in place of split/merge.
// Softmax statistics are f32; QK^T and PV run on BF16 tensor cores with f32
// accumulation.  Backward is FA2-style and atomic-free: dK/dV are owned by a
// KV-block CTA that loops over every query block of every head in its GQA
// group, dQ by a Q-block CTA; each gradient is accumulated in f32 registers
// and rounded to bf16 once, as the reference does (src/tensorops.cpp:298-301).
#include "common.cuh"
#include "kernels.h"

#include <algorithm>
#include <cstdlib>

namespace qtb { namespace attn { __device__ __forceinline__ uint32_t sm100_smem(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); } } }

namespace qtb {
namespace attn {

constexpr float LOG2E = 1.4426950408889634f;

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool pred) {
    const int n = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

// two f32 C fragments (n-tiles 2kk, 2kk+1) -> A fragments of the bf16 hi and lo parts
__device__ __forceinline__ void split_frag(const float (&c0)[4], const float (&c1)[4], uint32_t (&hi)[4],
                                           uint32_t (&lo)[4]) {
    const float* cs[2] = {c0, c1};
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        float h[4], l[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            h[e] = bf16r(cs[half][e]);
            l[e] = cs[half][e] - h[e];
        }
        hi[half * 2 + 0] = pack_bf16(h[0], h[1]);
        hi[half * 2 + 1] = pack_bf16(h[2], h[3]);
        lo[half * 2 + 0] = pack_bf16(l[0], l[1]);
        lo[half * 2 + 1] = pack_bf16(l[2], l[3]);
    }
}

// smem tile of ROWS x HD bf16, 16-B chunks XOR-swizzled by (row % 8)
template <int HD>
struct Tile {
    static constexpr int CH = HD / 8;  // 16-B chunks per row
    __device__ static __forceinline__ uint32_t off(int row, int chunk) {
        // 8+ chunks per row: XOR with row%8; 4 chunks (hd 32): XOR with (row/2)%4
        const int sw = CH >= 8 ? (row & 7) : ((row >> 1) & 3);
        return (uint32_t)(row * HD * 2 + ((chunk ^ sw) * 16));
    }
};

// async load of a ROWS x HD tile from a strided bf16 matrix; rows >= valid -> 0
template <int HD, int ROWS, int NT>
__device__ __forceinline__ void load_tile(uint32_t s_base, const uint16_t* g, int64_t ld, int valid) {
    constexpr int CH = HD / 8;
    for (int i = threadIdx.x; i < ROWS * CH; i += NT) {
        const int r = i / CH, c = i % CH;
        const bool ok = r < valid;
        cp_async16(s_base + Tile<HD>::off(r, c), g + (ok ? (int64_t)r * ld + c * 8 : 0), ok);
    }
}

// A fragment (16 rows x 16 k) at (row0, k0) of a swizzled tile
template <int HD>
__device__ __forceinline__ void ld_a(uint32_t (&a)[4], uint32_t s, int row0, int k0) {
    const int lane = threadIdx.x & 31;
    const int r = row0 + (lane & 15), c = (k0 >> 3) + (lane >> 4);
    ldsm_x4(a, s + Tile<HD>::off(r, c));
}
// B fragments for two n8 tiles (n0..n0+15) x k16 from a tile stored [n][k] (k contiguous)
template <int HD>
__device__ __forceinline__ void ld_b_nk(uint32_t (&b)[4], uint32_t s, int n0, int k0) {
    const int lane = threadIdx.x & 31;
    const int r = n0 + (lane & 7) + ((lane >> 4) << 3), c = (k0 >> 3) + ((lane >> 3) & 1);
    ldsm_x4(b, s + Tile<HD>::off(r, c));  // b[0],b[1] -> n-tile 0 ; b[2],b[3] -> n-tile 1
}
// B fragments for two n8 tiles x k16 from a tile stored [k][n] (n contiguous)
template <int HD>
__device__ __forceinline__ void ld_b_kn(uint32_t (&b)[4], uint32_t s, int k0, int n0) {
    const int lane = threadIdx.x & 31;
    const int r = k0 + (lane & 7) + (((lane >> 3) & 1) << 3), c = (n0 >> 3) + (lane >> 4);
    ldsm_x4_t(b, s + Tile<HD>::off(r, c));
}

// ===========================================================================
// forward: grid (ceil(T/64), H, B), 4 warps x 16 query rows
// ===========================================================================
template <bool FAST>
__device__ __forceinline__ float att_exp(float x) {
    if constexpr (FAST) return __expf(x);
    else return expf(x);
}

template <int HD, bool FAST = false>
__global__ void __launch_bounds__(128) fwd_kernel(const uint16_t* __restrict__ qkv, int T, int H, int Hkv, int qkv_dim,
                                                  float inv_sqrt_d, uint16_t* __restrict__ out, int64_t ldo,
                                                  float* __restrict__ out32, float* __restrict__ lse,
                                                  uint32_t* __restrict__ amax) {
    constexpr int BQ = 64, BK = 64;
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t sQ = sm100_smem(smem);
    const uint32_t sK = sQ + BQ * HD * 2;
    const uint32_t sV = sK + 2 * BK * HD * 2;
    const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int kvh = h / (H / Hkv);
    const int d = H * HD;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t rowbase = (int64_t)b * T;
    const uint16_t* gq = qkv + (rowbase + qb * BQ) * qkv_dim + h * HD;
    const uint16_t* gk = qkv + rowbase * qkv_dim + d + kvh * HD;
    const uint16_t* gv = qkv + rowbase * qkv_dim + d + Hkv * HD + kvh * HD;
    const int qvalid = min(BQ, T - qb * BQ);

    load_tile<HD, BQ, 128>(sQ, gq, qkv_dim, qvalid);
    load_tile<HD, BK, 128>(sK, gk, qkv_dim, min(BK, T));
    load_tile<HD, BK, 128>(sV, gv, qkv_dim, min(BK, T));
    cp_commit();

    float o[HD / 8][4];
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.0f;
    float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.0f, 0.0f};
    uint32_t qf[HD / 16][4];
    const float sl2 = inv_sqrt_d * LOG2E;
    const int g = lane >> 2, c4 = lane & 3;
    const int qrow0 = qb * BQ + warp * 16 + g;  // query positions of this thread's rows: qrow0, qrow0+8

    const int nkb = qb + 1;  // causal: key blocks 0..qb (BQ == BK)
    for (int j = 0; j < nkb; ++j) {
        if (j + 1 < nkb) {
            const int buf = (j + 1) & 1;
            load_tile<HD, BK, 128>(sK + buf * BK * HD * 2, gk + (int64_t)(j + 1) * BK * qkv_dim, qkv_dim,
                                   min(BK, T - (j + 1) * BK));
            load_tile<HD, BK, 128>(sV + buf * BK * HD * 2, gv + (int64_t)(j + 1) * BK * qkv_dim, qkv_dim,
                                   min(BK, T - (j + 1) * BK));
            cp_commit();
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        if (j == 0) {
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) ld_a<HD>(qf[kk], sQ, warp * 16, kk * 16);
        }
        const uint32_t k_s = sK + (j & 1) * BK * HD * 2, v_s = sV + (j & 1) * BK * HD * 2;
        float s[BK / 8][4];
#pragma unroll
        for (int i = 0; i < BK / 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.0f;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
            for (int nn = 0; nn < BK / 16; ++nn) {
                uint32_t bf[4];
                ld_b_nk<HD>(bf, k_s, nn * 16, kk * 16);
                mma16816(s[2 * nn], qf[kk], bf[0], bf[1]);
                mma16816(s[2 * nn + 1], qf[kk], bf[2], bf[3]);
            }
        }
        // scale, mask, online softmax
        float mx[2] = {m_r[0], m_r[1]};
#pragma unroll
        for (int i = 0; i < BK / 8; ++i) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int key = j * BK + i * 8 + 2 * c4 + (e & 1);
                const int q = qrow0 + (e >> 1) * 8;
                float x = s[i][e] * inv_sqrt_d;
                if (key > q || key >= T) x = -INFINITY;
                s[i][e] = x;
                mx[e >> 1] = fmaxf(mx[e >> 1], x);
            }
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
            mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
        }
        float corr[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            corr[r] = (m_r[r] == -INFINITY) ? 0.0f : att_exp<FAST>(m_r[r] - mx[r]);
            m_r[r] = mx[r];
            l_r[r] *= corr[r];
        }
#pragma unroll
        for (int i = 0; i < HD / 8; ++i) {
            o[i][0] *= corr[0];
            o[i][1] *= corr[0];
            o[i][2] *= corr[1];
            o[i][3] *= corr[1];
        }
        // p = exp(x - m) in f32 (std::exp semantics, src/tensorops.cpp:207)
#pragma unroll
        for (int i = 0; i < BK / 8; ++i) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float p = (s[i][e] == -INFINITY) ? 0.0f : att_exp<FAST>(s[i][e] - m_r[e >> 1]);
                s[i][e] = p;
                l_r[e >> 1] += p;
            }
        }
        // O += P V with P split into bf16 hi + lo parts (16 significant bits):
        // the reference multiplies f32 probabilities by bf16 values in f32
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk) {
            uint32_t ph[4], pl[4];
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const float* pv = s[2 * kk + half];
                float hi[4], lo[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    hi[e] = bf16r(pv[e]);
                    lo[e] = pv[e] - hi[e];
                }
                ph[half * 2 + 0] = pack_bf16(hi[0], hi[1]);
                ph[half * 2 + 1] = pack_bf16(hi[2], hi[3]);
                pl[half * 2 + 0] = pack_bf16(lo[0], lo[1]);
                pl[half * 2 + 1] = pack_bf16(lo[2], lo[3]);
            }
#pragma unroll
            for (int nn = 0; nn < HD / 16; ++nn) {
                uint32_t bf[4];
                ld_b_kn<HD>(bf, v_s, kk * 16, nn * 16);
                mma16816(o[2 * nn], ph, bf[0], bf[1]);
                mma16816(o[2 * nn + 1], ph, bf[2], bf[3]);
                mma16816(o[2 * nn], pl, bf[0], bf[1]);
                mma16816(o[2 * nn + 1], pl, bf[2], bf[3]);
            }
        }
        __syncthreads();
    }
    (void)sl2;
    // finalize
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 1);
        l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 2);
    }
    uint32_t m = 0;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int q = qrow0 + r * 8;
        if (q >= T) continue;
        const float inv_l = 1.0f / l_r[r];
        uint16_t* op = out + (rowbase + q) * ldo + h * HD;
#pragma unroll
        for (int i = 0; i < HD / 8; ++i) {
            const float f0 = o[i][2 * r] * inv_l, f1 = o[i][2 * r + 1] * inv_l;
            const float v0 = bf16r(f0), v1 = bf16r(f1);
            m = max(m, max(abs_bits(v0), abs_bits(v1)));
            *reinterpret_cast<uint32_t*>(op + i * 8 + 2 * c4) = pack_bf16(v0, v1);
            if (out32) *reinterpret_cast<float2*>(out32 + (rowbase + q) * ldo + h * HD + i * 8 + 2 * c4) = make_float2(f0, f1);
        }
        if (c4 == 0) lse[((int64_t)b * H + h) * T + q] = m_r[r] + logf(l_r[r]);
    }
    if (amax) block_absmax_commit<128>(m, amax);
}

// ===========================================================================
// backward preprocess: Dv[b,h,t] = sum_i dO[i] * O[i]   (src/tensorops.cpp:280-281)
// ===========================================================================
__global__ void bwd_dot_kernel(const uint16_t* __restrict__ dout, const float* __restrict__ o, int64_t ld, int T,
                               int H, int hd, int64_t rows, float* __restrict__ D) {
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= rows * H) return;
    const int64_t row = wid / H;
    const int h = (int)(wid % H);
    const uint16_t* a = dout + row * ld + h * hd;
    const float* bq = o + row * ld + h * hd;
    float s = 0.0f;
    for (int i = lane; i < hd; i += 32) s += bfbits2f(a[i]) * bq[i];
    s = warp_sum(s);
    if (lane == 0) {
        const int64_t bb = row / T, t = row % T;
        D[(bb * H + h) * T + t] = s;
    }
}

// Vectorised D: G = hd/8 threads per (row, head), 8 columns each (one 16 B
// dO load, two 16 B O loads).  The sum reproduces bwd_dot_kernel's order bit
// for bit -- lane l of a warp sums columns l, l+32, ... from 0, then the
// xor-16/8/4/2/1 tree -- because the first query row's dQ is exactly zero
// only when D matches dP's rounding there (P = 1, O = V).  Column l = 8j + k
// lives in thread j; the per-lane partials p_l (l < 32) end in threads 0..3,
// the tree's levels 16 and 8 cross threads (shfl_down 2, 1), 4/2/1 are in-thread.
template <int G>
__global__ void __launch_bounds__(256) bwd_dot_vec_kernel(const uint16_t* __restrict__ dout,
                                                          const float* __restrict__ o, int64_t ld, int T, int H,
                                                          int64_t rows, float* __restrict__ D) {
    constexpr int R = G / 4;  // columns per warp lane in bwd_dot_kernel (hd / 32)
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const int j = threadIdx.x % G;
    const bool live = gid < rows * H;
    const int64_t row = live ? gid / H : 0;
    const int h = live ? (int)(gid % H) : 0;
    float x[8];
    if (live) {
        const int64_t off = row * ld + (int64_t)h * (G * 8) + j * 8;
        const uint4 a = *reinterpret_cast<const uint4*>(dout + off);
        const float4 b0 = *reinterpret_cast<const float4*>(o + off), b1 = *reinterpret_cast<const float4*>(o + off + 4);
        const uint32_t w[4] = {a.x, a.y, a.z, a.w};
        const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            x[2 * k] = __fmul_rn(__uint_as_float(w[k] << 16), bv[2 * k]);
            x[2 * k + 1] = __fmul_rn(__uint_as_float(w[k] & 0xFFFF0000u), bv[2 * k + 1]);
        }
    } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = 0.0f;
    }
    // p_l = ((0 + x_l) + x_{l+32}) + ... : column l + 32r sits in thread j + 4r
    float p[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) p[k] = __fadd_rn(0.0f, x[k]);
#pragma unroll
    for (int r = 1; r < R; ++r)
#pragma unroll
        for (int k = 0; k < 8; ++k) p[k] = __fadd_rn(p[k], __shfl_down_sync(0xffffffffu, x[k], 4 * r, G));
    // tree level 16 (p_l + p_{l+16}: thread j + 2) and 8 (thread j + 1)
#pragma unroll
    for (int k = 0; k < 8; ++k) p[k] = __fadd_rn(p[k], __shfl_down_sync(0xffffffffu, p[k], 2, G));
#pragma unroll
    for (int k = 0; k < 8; ++k) p[k] = __fadd_rn(p[k], __shfl_down_sync(0xffffffffu, p[k], 1, G));
    // levels 4, 2, 1 inside thread 0
#pragma unroll
    for (int k = 0; k < 4; ++k) p[k] = __fadd_rn(p[k], p[k + 4]);
    p[0] = __fadd_rn(p[0], p[2]);
    p[1] = __fadd_rn(p[1], p[3]);
    if (live && j == 0) {
        const int64_t bb = row / T, t = row % T;
        D[(bb * H + h) * T + t] = __fadd_rn(p[0], p[1]);
    }
}

// D[b, h, t] = sum_c dO[row, h, c] * O[row, h, c] (row = b*T + t), f32
void launch_bwd_dot(const uint16_t* dout, const float* o, int64_t ld, int T, int H, int hd, int64_t rows, float* D,
                    cudaStream_t s) {
    const bool vec = (ld % 8 == 0) && ((uintptr_t)dout % 16 == 0) && ((uintptr_t)o % 16 == 0);
    const int64_t units = rows * H;
    if (vec && hd == 64) {
        bwd_dot_vec_kernel<8><<<(unsigned)ceil_div(units * 8, 256), 256, 0, s>>>(dout, o, ld, T, H, rows, D);
    } else if (vec && hd == 128) {
        bwd_dot_vec_kernel<16><<<(unsigned)ceil_div(units * 16, 256), 256, 0, s>>>(dout, o, ld, T, H, rows, D);
    } else if (vec && hd == 32) {
        bwd_dot_vec_kernel<4><<<(unsigned)ceil_div(units * 4, 256), 256, 0, s>>>(dout, o, ld, T, H, rows, D);
    } else {
        bwd_dot_kernel<<<(unsigned)ceil_div(units * 32, 256), 256, 0, s>>>(dout, o, ld, T, H, hd, rows, D);
    }
}

// ===========================================================================
// dK/dV: grid (ceil(T/64), Hkv, B); each warp owns 16 kv rows; loops over the
// GQA group's heads and every query block at or after the kv block
// ===========================================================================
template <int HD, int BQ, bool SPLIT = true, bool FAST = false>
__global__ void __launch_bounds__(128) bwd_dkdv_kernel(const uint16_t* __restrict__ qkv, const uint16_t* __restrict__ dout,
                                                       int64_t ldd, const float* __restrict__ lse,
                                                       const float* __restrict__ Dv, int T, int H, int Hkv,
                                                       int qkv_dim, float inv_sqrt_d, uint16_t* __restrict__ dqkv,
                                                       float* __restrict__ ws) {
    // grid (kv blocks, query heads, batch): one CTA per (kv block, query head);
    // with GQA (group > 1) the per-head f32 dK/dV go to ws and a second kernel
    // adds the group's heads in ascending order (deterministic)
    constexpr int BKV = 64;
    constexpr int TILE = BQ * HD * 2;
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t sK = sm100_smem(smem);
    const uint32_t sV = sK + BKV * HD * 2;
    const uint32_t sQ0 = sV + BKV * HD * 2;        // [2][Q, dO] double buffer
    const uint32_t sLD0 = sQ0 + 4 * TILE;          // [2][L(BQ), D(BQ)] floats
    float* sLDf = reinterpret_cast<float*>(smem + (sLD0 - sK));
    const int kb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int d = H * HD;
    const int group = H / Hkv;
    const int kvh = h / group;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, c4 = lane & 3;
    const int64_t rowbase = (int64_t)b * T;
    const int kvvalid = min(BKV, T - kb * BKV);
    const uint16_t* gk = qkv + (rowbase + kb * BKV) * qkv_dim + d + kvh * HD;
    const uint16_t* gv = qkv + (rowbase + kb * BKV) * qkv_dim + d + Hkv * HD + kvh * HD;
    const float* gL = lse + ((int64_t)b * H + h) * T;
    const float* gD = Dv + ((int64_t)b * H + h) * T;
    load_tile<HD, BKV, 128>(sK, gk, qkv_dim, kvvalid);
    load_tile<HD, BKV, 128>(sV, gv, qkv_dim, kvvalid);

    const int q_first = (kb * BKV) / BQ;
    const int nqb = (T + BQ - 1) / BQ;
    auto issue = [&](int qi, int buf) {
        const int qvalid = min(BQ, T - qi * BQ);
        const uint32_t sq = sQ0 + buf * 2 * TILE;
        load_tile<HD, BQ, 128>(sq, qkv + (rowbase + qi * BQ) * qkv_dim + h * HD, qkv_dim, qvalid);
        load_tile<HD, BQ, 128>(sq + TILE, dout + (rowbase + qi * BQ) * ldd + h * HD, ldd, qvalid);
        const uint32_t sld = sLD0 + buf * 2 * BQ * 4;
        for (int i = threadIdx.x; i < 2 * (BQ / 4); i += 128) {
            const int which = i / (BQ / 4), c = i % (BQ / 4);
            const int q = qi * BQ + c * 4;
            const float* src = (which ? gD : gL) + q;
            cp_async16(sld + which * BQ * 4 + c * 16, q < T ? src : gL, q < T);
        }
        cp_commit();
    };
    issue(q_first, 0);

    float dk[HD / 8][4], dv[HD / 8][4];
#pragma unroll
    for (int i = 0; i < HD / 8; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.0f;
    const int kv0 = kb * BKV + warp * 16 + g;  // kv positions of this thread's rows: kv0, kv0+8

    for (int qi = q_first, it = 0; qi < nqb; ++qi, ++it) {
        const int buf = it & 1;
        if (qi + 1 < nqb) {
            issue(qi + 1, buf ^ 1);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        const uint32_t sQ = sQ0 + buf * 2 * TILE, sO = sQ + TILE;
        const float* sL = sLDf + buf * 2 * BQ;
        const float* sD = sL + BQ;
        // S^T = K Q^T and dP^T = V dO^T  (16 kv x BQ q per warp)
        float st[BQ / 8][4], dpt[BQ / 8][4];
#pragma unroll
        for (int i = 0; i < BQ / 8; ++i)
#pragma unroll
            for (int e = 0; e < 4; ++e) st[i][e] = dpt[i][e] = 0.0f;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
            uint32_t ka[4], va[4];
            ld_a<HD>(ka, sK, warp * 16, kk * 16);
            ld_a<HD>(va, sV, warp * 16, kk * 16);
#pragma unroll
            for (int nn = 0; nn < BQ / 16; ++nn) {
                uint32_t bq[4], bo[4];
                ld_b_nk<HD>(bq, sQ, nn * 16, kk * 16);
                ld_b_nk<HD>(bo, sO, nn * 16, kk * 16);
                mma16816(st[2 * nn], ka, bq[0], bq[1]);
                mma16816(st[2 * nn + 1], ka, bq[2], bq[3]);
                mma16816(dpt[2 * nn], va, bo[0], bo[1]);
                mma16816(dpt[2 * nn + 1], va, bo[2], bo[3]);
            }
        }
        // P^T and dS^T (f32), then dV += P^T dO and dK += dS^T Q with both
        // left operands split into bf16 hi + lo parts (f32-faithful products)
#pragma unroll
        for (int i = 0; i < BQ / 8; ++i) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int kv = kv0 + (e >> 1) * 8;
                const int qc = i * 8 + 2 * c4 + (e & 1);
                const int q = qi * BQ + qc;
                const bool ok = (q >= kv) && (q < T) && (kv < T);
                const float x = st[i][e] * inv_sqrt_d;
                const float p = ok ? att_exp<FAST>(x - sL[qc]) : 0.0f;
                st[i][e] = p;
                dpt[i][e] = p * (dpt[i][e] - sD[qc]) * inv_sqrt_d;
            }
        }
#pragma unroll
        for (int kk = 0; kk < BQ / 16; ++kk) {
            uint32_t ph[4], pl[4], dh[4], dl[4];
            split_frag(st[2 * kk], st[2 * kk + 1], ph, pl);
            split_frag(dpt[2 * kk], dpt[2 * kk + 1], dh, dl);
#pragma unroll
            for (int nn = 0; nn < HD / 16; ++nn) {
                uint32_t bo[4], bq[4];
                ld_b_kn<HD>(bo, sO, kk * 16, nn * 16);
                ld_b_kn<HD>(bq, sQ, kk * 16, nn * 16);
                mma16816(dv[2 * nn], ph, bo[0], bo[1]);
                mma16816(dv[2 * nn + 1], ph, bo[2], bo[3]);
                mma16816(dk[2 * nn], dh, bq[0], bq[1]);
                mma16816(dk[2 * nn + 1], dh, bq[2], bq[3]);
                if constexpr (SPLIT) {
                    mma16816(dv[2 * nn], pl, bo[0], bo[1]);
                    mma16816(dv[2 * nn + 1], pl, bo[2], bo[3]);
                    mma16816(dk[2 * nn], dl, bq[0], bq[1]);
                    mma16816(dk[2 * nn + 1], dl, bq[2], bq[3]);
                }
            }
        }
        __syncthreads();  // this buffer is refilled by the prefetch two iterations on
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int kv = kv0 + r * 8;
        if (kv >= T) continue;
        if (group == 1) {
            uint16_t* pk = dqkv + (rowbase + kv) * qkv_dim + d + kvh * HD;
            uint16_t* pv = dqkv + (rowbase + kv) * qkv_dim + d + Hkv * HD + kvh * HD;
#pragma unroll
            for (int i = 0; i < HD / 8; ++i) {
                *reinterpret_cast<uint32_t*>(pk + i * 8 + 2 * c4) = pack_bf16(dk[i][2 * r], dk[i][2 * r + 1]);
                *reinterpret_cast<uint32_t*>(pv + i * 8 + 2 * c4) = pack_bf16(dv[i][2 * r], dv[i][2 * r + 1]);
            }
        } else {
            // ws layout: [2][B][H][T][HD] f32 (dk then dv)
            const int64_t base = (((int64_t)b * H + h) * T + kv) * HD;
            const int64_t half = (int64_t)gridDim.z * H * T * HD;
#pragma unroll
            for (int i = 0; i < HD / 8; ++i) {
                *reinterpret_cast<float2*>(ws + base + i * 8 + 2 * c4) = make_float2(dk[i][2 * r], dk[i][2 * r + 1]);
                *reinterpret_cast<float2*>(ws + half + base + i * 8 + 2 * c4) =
                    make_float2(dv[i][2 * r], dv[i][2 * r + 1]);
            }
        }
    }
}

// dK/dV of a kv head = sum over its GQA group's query heads in ascending
// order (the reference accumulates h-outer, src/tensorops.cpp:268-296), rounded once
__global__ void dkdv_reduce_kernel(const float* __restrict__ ws, int B, int T, int H, int Hkv, int hd, int qkv_dim,
                                   uint16_t* __restrict__ dqkv) {
    const int group = H / Hkv;
    const int d = H * hd;
    const int64_t half = (int64_t)B * H * T * hd;
    const int64_t n = (int64_t)B * Hkv * T * hd;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % hd);
        const int64_t r = i / hd;
        const int t = (int)(r % T);
        const int kvh = (int)((r / T) % Hkv);
        const int b = (int)(r / ((int64_t)T * Hkv));
        float sk = 0.0f, sv = 0.0f;
        for (int hh = 0; hh < group; ++hh) {
            const int64_t o = (((int64_t)b * H + kvh * group + hh) * T + t) * hd + c;
            sk = __fadd_rn(sk, ws[o]);
            sv = __fadd_rn(sv, ws[half + o]);
        }
        const int64_t row = (int64_t)b * T + t;
        dqkv[row * qkv_dim + d + kvh * hd + c] = f2bfbits(sk);
        dqkv[row * qkv_dim + d + Hkv * hd + kvh * hd + c] = f2bfbits(sv);
    }
}

// ===========================================================================
// dQ: grid (ceil(T/64), H, B); each warp owns 16 query rows
// ===========================================================================
template <int HD, bool SPLIT = true, bool FAST = false>
__global__ void __launch_bounds__(128) bwd_dq_kernel(const uint16_t* __restrict__ qkv, const uint16_t* __restrict__ dout,
                                                     int64_t ldd, const float* __restrict__ lse,
                                                     const float* __restrict__ Dv, int T, int H, int Hkv, int qkv_dim,
                                                     float inv_sqrt_d, uint16_t* __restrict__ dqkv) {
    constexpr int BQ = 64, BKV = 64;
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t sQ = sm100_smem(smem);
    const uint32_t sO = sQ + BQ * HD * 2;
    const uint32_t sKV0 = sO + BQ * HD * 2;  // [2][K, V] double buffer
    const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int kvh = h / (H / Hkv);
    const int d = H * HD;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, c4 = lane & 3;
    const int64_t rowbase = (int64_t)b * T;
    const int qvalid = min(BQ, T - qb * BQ);
    const uint16_t* gk = qkv + rowbase * qkv_dim + d + kvh * HD;
    const uint16_t* gv = qkv + rowbase * qkv_dim + d + Hkv * HD + kvh * HD;
    load_tile<HD, BQ, 128>(sQ, qkv + (rowbase + qb * BQ) * qkv_dim + h * HD, qkv_dim, qvalid);
    load_tile<HD, BQ, 128>(sO, dout + (rowbase + qb * BQ) * ldd + h * HD, ldd, qvalid);
    auto issue = [&](int j, int buf) {
        const uint32_t k_s = sKV0 + buf * 2 * BKV * HD * 2;
        load_tile<HD, BKV, 128>(k_s, gk + (int64_t)j * BKV * qkv_dim, qkv_dim, min(BKV, T - j * BKV));
        load_tile<HD, BKV, 128>(k_s + BKV * HD * 2, gv + (int64_t)j * BKV * qkv_dim, qkv_dim, min(BKV, T - j * BKV));
        cp_commit();
    };
    issue(0, 0);  // commits Q, dO and K/V block 0 together
    const int q0 = qb * BQ + warp * 16 + g;
    float L[2], Dd[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int q = q0 + r * 8;
        L[r] = q < T ? lse[((int64_t)b * H + h) * T + q] : 0.0f;
        Dd[r] = q < T ? Dv[((int64_t)b * H + h) * T + q] : 0.0f;
    }
    float dq[HD / 8][4];
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.0f;
    uint32_t qf[HD / 16][4], of[HD / 16][4];
    for (int j = 0; j <= qb; ++j) {
        const int buf = j & 1;
        if (j + 1 <= qb) {
            issue(j + 1, buf ^ 1);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        const uint32_t sK = sKV0 + buf * 2 * BKV * HD * 2, sV = sK + BKV * HD * 2;
        if (j == 0) {
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) {
                ld_a<HD>(qf[kk], sQ, warp * 16, kk * 16);
                ld_a<HD>(of[kk], sO, warp * 16, kk * 16);
            }
        }
        float s[BKV / 8][4], dp[BKV / 8][4];
#pragma unroll
        for (int i = 0; i < BKV / 8; ++i)
#pragma unroll
            for (int e = 0; e < 4; ++e) s[i][e] = dp[i][e] = 0.0f;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
            for (int nn = 0; nn < BKV / 16; ++nn) {
                uint32_t bk[4], bv[4];
                ld_b_nk<HD>(bk, sK, nn * 16, kk * 16);
                ld_b_nk<HD>(bv, sV, nn * 16, kk * 16);
                mma16816(s[2 * nn], qf[kk], bk[0], bk[1]);
                mma16816(s[2 * nn + 1], qf[kk], bk[2], bk[3]);
                mma16816(dp[2 * nn], of[kk], bv[0], bv[1]);
                mma16816(dp[2 * nn + 1], of[kk], bv[2], bv[3]);
            }
        }
#pragma unroll
        for (int i = 0; i < BKV / 8; ++i) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int r = e >> 1;
                const int q = q0 + r * 8;
                const int key = j * BKV + i * 8 + 2 * c4 + (e & 1);
                const bool ok = key <= q && key < T && q < T;
                const float x = s[i][e] * inv_sqrt_d;
                const float p = ok ? att_exp<FAST>(x - L[r]) : 0.0f;
                s[i][e] = p * (dp[i][e] - Dd[r]) * inv_sqrt_d;
            }
        }
        // dQ += dS K   (k = kv index; K tile stored [kv][hd]); dS split hi + lo
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk) {
            uint32_t dh[4], dl[4];
            split_frag(s[2 * kk], s[2 * kk + 1], dh, dl);
#pragma unroll
            for (int nn = 0; nn < HD / 16; ++nn) {
                uint32_t bk[4];
                ld_b_kn<HD>(bk, sK, kk * 16, nn * 16);
                mma16816(dq[2 * nn], dh, bk[0], bk[1]);
                mma16816(dq[2 * nn + 1], dh, bk[2], bk[3]);
                if constexpr (SPLIT) {
                    mma16816(dq[2 * nn], dl, bk[0], bk[1]);
                    mma16816(dq[2 * nn + 1], dl, bk[2], bk[3]);
                }
            }
        }
        __syncthreads();  // buffer reused by the prefetch of block j+2
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int q = q0 + r * 8;
        if (q >= T) continue;
        uint16_t* pq = dqkv + (rowbase + q) * qkv_dim + h * HD;
#pragma unroll
        for (int i = 0; i < HD / 8; ++i)
            *reinterpret_cast<uint32_t*>(pq + i * 8 + 2 * c4) = pack_bf16(dq[i][2 * r], dq[i][2 * r + 1]);
    }
}

}  // namespace attn
}  // namespace qtb

using namespace qtb;
using namespace qtb::attn;

static int g_fast_exp = 1, g_bwd_split = 1;  // ex2.approx: same parity as expf (scripts/attn_modes.py)

extern "C" {

// precision mode of the attention kernels: fast_exp = __expf (ex2.approx) in
// place of expf; bwd_split = carry P and dS as bf16 hi+lo in the backward
void qtk_attn_set_mode(int fast_exp, int bwd_split) {
    g_fast_exp = fast_exp;
    g_bwd_split = bwd_split;
}

int qtk_attn_fwd_tc(const void* qkv, int B, int T, int H, int Hkv, int hd, int qkv_dim, void* out, int64_t ldo,
                    float* out32, float* lse, uint32_t* amax, cudaStream_t s);

int qtk_attn_fwd(const void* qkv, int B, int T, int H, int Hkv, int hd, int qkv_dim, void* out, int64_t ldo,
                 float* out32, float* lse, uint32_t* amax, cudaStream_t s) {
    if (H % Hkv) return 1;
    static int use_tc = -1;
    if (use_tc < 0) {
        const char* e = getenv("QTB_ATTN_TC");
        use_tc = e ? atoi(e) : 1;  // tcgen05 forward for hd 64 (QTB_ATTN_TC=0: the mma.sync kernel)
    }
    // tcgen05 path for head_dim 64/128; the mma.sync kernel covers the rest
    if (use_tc && (hd == 64 || hd == 128))
        return qtk_attn_fwd_tc(qkv, B, T, H, Hkv, hd, qkv_dim, out, ldo, out32, lse, amax, s);
    const float inv_sqrt_d = 1.0f / sqrtf((float)hd);
    dim3 grid((unsigned)ceil_div(T, 64), H, B);
    if (hd == 64) {
        const int smem = (64 + 2 * 64 * 2) * 64 * 2;
        if (g_fast_exp)
            fwd_kernel<64, true><<<grid, 128, smem, s>>>((const uint16_t*)qkv, T, H, Hkv, qkv_dim, inv_sqrt_d,
                                                         (uint16_t*)out, ldo, out32, lse, amax);
        else
            fwd_kernel<64><<<grid, 128, smem, s>>>((const uint16_t*)qkv, T, H, Hkv, qkv_dim, inv_sqrt_d, (uint16_t*)out,
                                                   ldo, out32, lse, amax);
    } else if (hd == 128) {
        const int smem = (64 + 2 * 64 * 2) * 128 * 2;
        cudaFuncSetAttribute(fwd_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        fwd_kernel<128><<<grid, 128, smem, s>>>((const uint16_t*)qkv, T, H, Hkv, qkv_dim, inv_sqrt_d, (uint16_t*)out,
                                                ldo, out32, lse, amax);
    } else if (hd == 32) {
        const int smem = (64 + 2 * 64 * 2) * 32 * 2;
        fwd_kernel<32><<<grid, 128, smem, s>>>((const uint16_t*)qkv, T, H, Hkv, qkv_dim, inv_sqrt_d, (uint16_t*)out,
                                               ldo, out32, lse, amax);
    } else {
        return 1;
    }
    return (int)cudaGetLastError();
}

// Dv scratch: B*H*T floats; ws: 2*B*H*T*hd floats when H > Hkv (GQA partials), else unused
size_t qtk_attn_bwd_ws_bytes(int B, int T, int H, int Hkv, int hd) {
    return H > Hkv ? (size_t)2 * B * H * T * hd * sizeof(float) : 0;
}

int qtk_attn_bwd_tc(const void* qkv, const float* out32, const void* dout, int64_t ldo, const float* lse,
                    float* Dv, int B, int T, int H, int Hkv, int hd, int qkv_dim, void* dqkv, float* ws, cudaStream_t s);

int qtk_attn_bwd_tc2(const void* qkv, const float* out32, const void* dout, int64_t ldo, const float* lse,
                     float* Dv, int B, int T, int H, int Hkv, int hd, int qkv_dim, void* dqkv, float* ws, cudaStream_t s,
                     cudaStream_t s2);
// two-stream form: the tcgen05 path runs its dQ kernel on s2 next to dK/dV on s
int qtk_attn_bwd2(const void* qkv, const float* out32, const void* dout, int64_t ldo, const float* lse, float* Dv,
                  int B, int T, int H, int Hkv, int hd, int qkv_dim, void* dqkv, float* ws, cudaStream_t s,
                  cudaStream_t s2) {
    static int use_tc = -1;
    if (use_tc < 0) {
        const char* e = getenv("QTB_ATTN_BWD_TC");
        use_tc = e ? atoi(e) : 1;
    }
    if (use_tc && (hd == 64 || hd == 128) && !(H % Hkv) && !(T % 4))
        return qtk_attn_bwd_tc2(qkv, out32, dout, ldo, lse, Dv, B, T, H, Hkv, hd, qkv_dim, dqkv, ws, s, s2);
    return qtk_attn_bwd(qkv, out32, dout, ldo, lse, Dv, B, T, H, Hkv, hd, qkv_dim, dqkv, ws, s);
}

int qtk_attn_bwd(const void* qkv, const float* out32, const void* dout, int64_t ldo, const float* lse, float* Dv, int B,
                 int T, int H, int Hkv, int hd, int qkv_dim, void* dqkv, float* ws, cudaStream_t s) {
    if (H % Hkv || T % 4) return 1;
    if (H > Hkv && !ws) return 1;
    static int use_tc = -1;
    if (use_tc < 0) {
        const char* e = getenv("QTB_ATTN_BWD_TC");
        use_tc = e ? atoi(e) : 1;
    }
    if (use_tc && (hd == 64 || hd == 128))
        return qtk_attn_bwd_tc(qkv, out32, dout, ldo, lse, Dv, B, T, H, Hkv, hd, qkv_dim, dqkv, ws, s);
    const float inv_sqrt_d = 1.0f / sqrtf((float)hd);
    const int64_t rows = (int64_t)B * T;
    launch_bwd_dot((const uint16_t*)dout, out32, ldo, T, H, hd, rows, Dv, s);
    dim3 gkv((unsigned)ceil_div(T, 64), H, B), gq((unsigned)ceil_div(T, 64), H, B);
#define QTB_ATTN_BWD_V(HD, BQ, SP, FA)                                                                           \
    {                                                                                                             \
        const int smem_kv = (2 * 64 + 4 * BQ) * HD * 2 + 4 * BQ * 4;                                              \
        cudaFuncSetAttribute(bwd_dkdv_kernel<HD, BQ, SP, FA>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kv); \
        bwd_dkdv_kernel<HD, BQ, SP, FA><<<gkv, 128, smem_kv, s>>>((const uint16_t*)qkv, (const uint16_t*)dout, ldo,  \
                                                                  lse, Dv, T, H, Hkv, qkv_dim, inv_sqrt_d,         \
                                                                  (uint16_t*)dqkv, ws);                            \
        const int smem_q = 6 * 64 * HD * 2;                                                                       \
        cudaFuncSetAttribute(bwd_dq_kernel<HD, SP, FA>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_q);     \
        bwd_dq_kernel<HD, SP, FA><<<gq, 128, smem_q, s>>>((const uint16_t*)qkv, (const uint16_t*)dout, ldo, lse, Dv, \
                                                          T, H, Hkv, qkv_dim, inv_sqrt_d, (uint16_t*)dqkv);         \
    }
#define QTB_ATTN_BWD(HD, BQ)                                     \
    {                                                            \
        if (g_bwd_split && g_fast_exp) QTB_ATTN_BWD_V(HD, BQ, true, true)       \
        else if (g_bwd_split) QTB_ATTN_BWD_V(HD, BQ, true, false)               \
        else if (g_fast_exp) QTB_ATTN_BWD_V(HD, BQ, false, true)                \
        else QTB_ATTN_BWD_V(HD, BQ, false, false)                               \
    }
    if (hd == 64)
        QTB_ATTN_BWD(64, 64)
    else if (hd == 128)
        QTB_ATTN_BWD(128, 32)
    else if (hd == 32)
        QTB_ATTN_BWD(32, 64)
    else
        return 1;
#undef QTB_ATTN_BWD
    if (H > Hkv) {
        const int64_t n = (int64_t)B * Hkv * T * hd;
        dkdv_reduce_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 16 * kNumSMs), 256, 0, s>>>(
            ws, B, T, H, Hkv, hd, qkv_dim, (uint16_t*)dqkv);
    }
    return (int)cudaGetLastError();
}

}  // extern "C"
