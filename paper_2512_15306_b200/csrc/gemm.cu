// Warp-specialised persistent tcgen05 GEMM for sm_100a (north-star item 2).
//
//   D[m, n] = sum_k A[m, k] * B[n, k]          (f32 accumulation in TMEM)
//
// Operands come from HBM through TMA (128-B swizzle) into a STAGES-deep smem
// ring; one elected thread issues tcgen05.mma (kind::f8f6f4 for E4M3/E5M2,
// kind::f16 for BF16) into a double-buffered TMEM accumulator; four epilogue
// warps drain TMEM with tcgen05.ld and apply the reference's rounding:
//
//   EPI_BF16      out = bf16( acc / (sa*sb) )              src/tensorops.cpp:47,55
//   EPI_F32       out = acc (f32)                          src/tensorops.cpp:372-376 (CE logits)
//   EPI_BF16_RES  out = bf16( bf16(acc/(sa*sb)) + res )    src/model.cpp:281-283 (r_out)
//   EPI_BF16_ACC  buf = SR_bf16( buf + bf16(acc/(sa*sb)) ) src/model.cpp:455-462 (GradAccumulator)
//   EPI_F32_ACC   buf = SR_bf16( buf + acc )               (f32 grads, e.g. d_lm_w)
//
// Either operand may be K-major (row-major [rows][K]) or MN-major (stored
// [K][rows]); MN-major FP8/BF16 is legal on sm_100 (UMMA a_major/b_major), so
// dgrad and wgrad read the forward-layout tensors directly with no transposed
// copies.  Warp roles: 0 = TMA producer, 1 = MMA issuer, 2 = TMEM allocator,
// 4..7 = epilogue (warp%4 selects the TMEM lane quarter).
#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"

#include <cudaTypedefs.h>
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <mutex>

namespace qtb {
namespace gemm {

using namespace sm100;

constexpr int BM = 128;

struct alignas(64) Params {
    CUtensorMap ta;
    CUtensorMap tb;
    CUtensorMap ta2;  // split-A: D = A.B + A2.B (the K loop runs twice, B repeats)
    CUtensorMap to;   // output (and EPI_*_ACC accumulator) map, 128-B x 32-row boxes
    CUtensorMap tr;   // EPI_BF16_RES residual map
    int tma_out;      // epilogue stages tiles through smem and stores them with TMA
    uint32_t* amax;   // EPI_SWIGLU_BWD: absmax of the output
    const int32_t* ce_targets;  // EPI_F32 logits: per-row softmax statistics (see QtkGemm)
    float2* ce_stats;
    float* ce_tgt_logit;
    int ce_nstat;
    int n_fast;       // tile order: N-tiles of one M panel adjacent (they share the A panel in L2)
    int M, N, K;
    int num_m, num_n, num_k;
    int split_a;
    int splits, kb_per_split;  // split-K: partial f32 tiles to out + s*M*ldo
    uint32_t idesc;
    const float* a_scale;
    const float* b_scale;
    void* out;
    int64_t ldo;
    const uint16_t* res;
    int64_t ldr;
    uint64_t sr_seed, sr_stream, sr_base;
    const uint64_t* sr_ms;  // device micro-step: base = *sr_ms * sr_mn + sr_off (graph replay), else sr_base
    uint64_t sr_mn, sr_off;  // full GEMM's M*N and this launch's first-row counter offset (tail split)
};

// CG = CTAs per MMA (tcgen05 cta_group): 2 pairs two SMs on a 256-row tile
// and splits the B tile between them (half the per-SM operand traffic)
__host__ __device__ constexpr bool epi_loads(int epi) {
    return epi == EPI_BF16_RES || epi == EPI_BF16_ACC || epi == EPI_F32_ACC || epi == EPI_SWIGLU_BWD;
}

template <int KIND, int BN, int CG = 1, int EPI = EPI_BF16>
struct Cfg {
    static constexpr int ELEM = KIND == 0 ? 1 : 2;
    static constexpr int BK = 128 / ELEM;  // K elements per pipeline stage (one 128-B swizzle row)
    static constexpr int UK = 32 / ELEM;   // K per tcgen05.mma
    static constexpr int BN_CTA = BN / CG; // B rows held by each CTA
    static constexpr int A_BYTES = BM * 128;
    static constexpr int B_BYTES = BN_CTA * 128;
    static constexpr int STAGE = A_BYTES + B_BYTES;
    // per epilogue warp: one 32-row x 128-B staging box, or -- for the
    // epilogues that read the output tile first -- the warp's whole 32-row
    // slice of its columns, prefetched while the tile's MMAs run
    // 8 epilogue warps (two per TMEM lane quarter, each owning half of the
    // tile's columns); a LOADS warp keeps its whole 32 x BN/2 slice
    static constexpr int EPI_WARPS = 8;
    static constexpr int EPI_GROUPS = EPI == EPI_SWIGLU_BWD ? 2 : (epi_loads(EPI) ? BN / 128 : 1);
    static constexpr int EPI_BYTES = EPI_WARPS * EPI_GROUPS * 4096;
    static constexpr int STAGE_BUDGET = 232448 - 1536 - EPI_BYTES;  // 227 KB opt-in max, less align + barriers
    static constexpr int STAGES = STAGE_BUDGET / STAGE > 8 ? 8 : STAGE_BUDGET / STAGE;
    static constexpr int TMEM_COLS = 2 * BN;
    static constexpr int SMEM = STAGES * STAGE + EPI_BYTES + 1024 + 256;
};

__device__ __forceinline__ void store_bf16x32(uint16_t* dst, const float (&v)[32]) {
    uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int q = 0; q < 4; ++q)
        d[q] = make_uint4(pack_bf16x2(v[8 * q + 0], v[8 * q + 1]), pack_bf16x2(v[8 * q + 2], v[8 * q + 3]),
                          pack_bf16x2(v[8 * q + 4], v[8 * q + 5]), pack_bf16x2(v[8 * q + 6], v[8 * q + 7]));
}
__device__ __forceinline__ void load_bf16x32(const uint16_t* src, float (&v)[32]) {
    const uint4* s = reinterpret_cast<const uint4*>(src);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint4 u = s[q];
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            v[8 * q + 2 * j] = __uint_as_float(w[j] << 16);
            v[8 * q + 2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
        }
    }
}

// x / d correctly rounded from rcp = RN(1/d): q = RN(x*rcp) is within 1 ulp, the
// FMA residual x - q*d is exact, and one correction q + res*rcp rounds to the
// correctly rounded quotient (Markstein's theorem) -- the same bits as the
// reference's f32 division acc / denom (src/tensorops.cpp:55) in 3 instructions.
__device__ __forceinline__ float exp2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float div_exact(float x, float d, float rcp) {
    const float q = __fmul_rn(x, rcp);
    const float e = __fmaf_rn(-q, d, x);
    return __fmaf_rn(e, rcp, q);
}

template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const Params& p, int row, int col0, float denom, float rcp,
                                               const uint32_t (&r)[32]) {
    if (col0 >= p.N) return;
    const bool vec = (col0 + 32 <= p.N) && ((p.ldo & 7) == 0);
    float v[32];
    if constexpr (EPI == EPI_F32 || EPI == EPI_F32_ACC) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
    } else if constexpr (EPI == EPI_BF16) {
        // rounding happens once, in the bf16x2 pack of the store
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = div_exact(__uint_as_float(r[j]), denom, rcp);
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = bf16r(div_exact(__uint_as_float(r[j]), denom, rcp));
    }
    if constexpr (EPI == EPI_BF16 || EPI == EPI_BF16_RES) {
        uint16_t* out = reinterpret_cast<uint16_t*>(p.out) + (int64_t)row * p.ldo + col0;
        if constexpr (EPI == EPI_BF16_RES) {
            const uint16_t* rs = p.res + (int64_t)row * p.ldr + col0;
            if (vec && (p.ldr & 7) == 0) {
                float rv[32];
                load_bf16x32(rs, rv);
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __fadd_rn(v[j], rv[j]);
            } else {
                for (int j = 0; j < 32 && col0 + j < p.N; ++j) v[j] = __fadd_rn(v[j], bfbits2f(rs[j]));
            }
        }
        if (vec) {
            store_bf16x32(out, v);
        } else {
            for (int j = 0; j < 32 && col0 + j < p.N; ++j) out[j] = f2bfbits(v[j]);
        }
    } else if constexpr (EPI == EPI_F32) {
        float* out = reinterpret_cast<float*>(p.out) + (int64_t)row * p.ldo + col0;
        if (vec) {
            float4* o4 = reinterpret_cast<float4*>(out);
#pragma unroll
            for (int q = 0; q < 8; ++q) o4[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else {
            for (int j = 0; j < 32 && col0 + j < p.N; ++j) out[j] = v[j];
        }
    } else {  // *_ACC: GradAccumulator::accumulate fused (src/model.cpp:455-462)
        uint16_t* buf = reinterpret_cast<uint16_t*>(p.out) + (int64_t)row * p.ldo + col0;
        const uint64_t sb = p.sr_ms ? *p.sr_ms * p.sr_mn + p.sr_off : p.sr_base;
        const uint64_t ctr0 = sb + (uint64_t)row * (uint64_t)p.N + (uint64_t)col0;
        const uint64_t key = rng_key(p.sr_seed, p.sr_stream);
        if (vec) {
            float b[32];
            load_bf16x32(buf, b);
#pragma unroll
            for (int j = 0; j < 32; ++j) b[j] = sr_bf16k(__fadd_rn(b[j], v[j]), key, ctr0 + j);
            store_bf16x32(buf, b);
        } else {
            for (int j = 0; j < 32 && col0 + j < p.N; ++j)
                buf[j] = f2bfbits(sr_bf16k(__fadd_rn(bfbits2f(buf[j]), v[j]), key, ctr0 + j));
        }
    }
}

// ---------------------------------------------------------------------------
// Staged epilogue: one 128-B column group (64 bf16 or 32 f32 output columns) of
// this warp's 32 rows at a time: TMEM -> registers -> rounding -> 128-B-swizzled
// smem box (lane = row, 16-B chunk c at c ^ (row & 7): conflict-free) -> TMA
// store.  Two boxes per warp alternate so the store of one overlaps the next
// group's math.  EPI_BF16_RES / *_ACC first TMA-load the residual / the grad
// accumulator box into the same smem (zero-filled out of bounds; the store clips).
// ---------------------------------------------------------------------------
// Prefetch (lane 0) of the residual / accumulator slice a LOADS epilogue reads:
// the warp's 32 rows x BNt columns, one 4-KB box per 64 columns, on ebar.
template <int EPI>
__device__ __forceinline__ void epilogue_prefetch(const Params& p, int m_row0, int n0, int BNt, uint8_t* stg,
                                                  uint64_t* ebar) {
    bulk_wait_read<0>();  // the previous tile's stores have left these boxes
    if constexpr (EPI == EPI_SWIGLU_BWD) {  // group 0's gate and up boxes (later groups load in turn)
        mbar_arrive_expect_tx(ebar, 2 * 4096);
        tma_load_2d(&p.tr, ebar, stg, n0, m_row0);
        tma_load_2d(&p.tr, ebar, stg + 4096, n0 + p.N, m_row0);
        return;
    }
    const int ng = max(0, min(BNt, p.N - n0 + 63)) / 64;  // 0 when this half lies past N
    mbar_arrive_expect_tx(ebar, ng * 4096);
    for (int g = 0; g < ng; ++g) tma_load_2d(EPI == EPI_BF16_RES ? &p.tr : &p.to, ebar, stg + g * 4096, n0 + g * 64, m_row0);
}

template <int EPI>
__device__ __forceinline__ void epilogue_tile_tma(const Params& p, uint32_t tmem_cols, int m_row0, int n0, int BNt,
                                                  float denom, float rcp, uint8_t* stg, uint64_t* ebar,
                                                  uint32_t& ephase, int& buf) {
    constexpr bool F32OUT = EPI == EPI_F32;
    constexpr int GC = F32OUT ? 32 : 64;  // output columns per 128-B group
    constexpr bool LOADS = epi_loads(EPI);
    const int lane = threadIdx.x & 31;
    const int row = m_row0 + lane;
    const uint64_t key = (EPI == EPI_BF16_ACC || EPI == EPI_F32_ACC) ? rng_key(p.sr_seed, p.sr_stream) : 0;
    const uint64_t sr_base = (EPI == EPI_BF16_ACC || EPI == EPI_F32_ACC) && p.sr_ms
                                 ? *p.sr_ms * p.sr_mn + p.sr_off
                                 : p.sr_base;
    constexpr bool SWI = EPI == EPI_SWIGLU_BWD;
    if constexpr (LOADS && !SWI) {
        mbar_wait(ebar, ephase);
        ephase ^= 1;
    }
    uint32_t smax = 0;
    // EPI_F32 logits: online (max, sum exp) of this thread's row over its BNt columns
    const bool stats = EPI == EPI_F32 && p.ce_stats != nullptr;
    float cm = -INFINITY, cs = 0.0f;
    int ctgt = -1;
    if (EPI == EPI_F32 && stats && row < p.M) ctgt = p.ce_targets[row];
    for (int g = 0; g < BNt / GC; ++g) {
        const int col0 = n0 + g * GC;
        if (col0 >= p.N) break;
        if constexpr (SWI) {
            if (g > 0 && lane == 0) {  // this group's gate / up boxes, once the previous stores have read them
                bulk_wait_read<0>();
                mbar_arrive_expect_tx(ebar, 2 * 4096);
                tma_load_2d(&p.tr, ebar, stg, col0, m_row0);
                tma_load_2d(&p.tr, ebar, stg + 4096, col0 + p.N, m_row0);
            }
        }
        uint32_t r[GC];
        tmem_ld32(tmem_cols + g * GC, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
        if constexpr (GC == 64) tmem_ld32(tmem_cols + g * GC + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
        uint8_t* box;
        if constexpr (SWI) {
            box = stg;
        } else if constexpr (LOADS) {
            box = stg + g * 4096;
        } else {
            box = stg;
            // the store issued from this box by the previous group must have finished reading it
            if (lane == 0) bulk_wait_read<0>();
            __syncwarp();
        }
        tmem_ld_wait();
        float v[GC];
        if constexpr (EPI == EPI_F32 || EPI == EPI_F32_ACC) {
#pragma unroll
            for (int j = 0; j < GC; ++j) v[j] = __uint_as_float(r[j]);
            if (EPI == EPI_F32 && stats) {
                constexpr float L2E = 1.4426950408889634f;
                const int nv = min(GC, p.N - col0);
                float gm = -INFINITY;
#pragma unroll
                for (int j = 0; j < GC; ++j)
                    if (j < nv) gm = fmaxf(gm, v[j]);
                if (gm > cm) {
                    cs = cm == -INFINITY ? 0.0f : cs * exp2_approx((cm - gm) * L2E);
                    cm = gm;
                }
                const float mb = cm * L2E;
                float s4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
                for (int j = 0; j < GC; ++j)
                    if (j < nv) s4[j & 3] += exp2_approx(__fmaf_rn(v[j], L2E, -mb));
                cs += (s4[0] + s4[1]) + (s4[2] + s4[3]);
                if (ctgt >= col0 && ctgt < col0 + GC) {
                    float tv = 0.0f;
#pragma unroll
                    for (int j = 0; j < GC; ++j)
                        if (col0 + j == ctgt) tv = v[j];
                    p.ce_tgt_logit[row] = tv;
                }
            }
        } else if constexpr (EPI == EPI_BF16) {
#pragma unroll
            for (int j = 0; j < GC; ++j) v[j] = div_exact(__uint_as_float(r[j]), denom, rcp);  // rounded by the pack
        } else {
#pragma unroll
            for (int j = 0; j < GC; ++j) v[j] = bf16r(div_exact(__uint_as_float(r[j]), denom, rcp));
        }
        uint4* rowp = reinterpret_cast<uint4*>(box + lane * 128);
        if constexpr (SWI) {
            // dh = bf16(acc / (sa*sb)) (the reference's dgrad output), then swiglu_backward
            // (tensorops.cpp:133-153) with gate / up from the staged boxes, in place
            mbar_wait(ebar, ephase);
            ephase ^= 1;
            uint4* rowu = reinterpret_cast<uint4*>(box + 4096 + lane * 128);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const int sl = c ^ (lane & 7);
                const uint4 ug = rowp[sl], uu = rowu[sl];
                const uint32_t wg[4] = {ug.x, ug.y, ug.z, ug.w}, wu[4] = {uu.x, uu.y, uu.z, uu.w};
                float dg[8], du[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const float gv = e & 1 ? __uint_as_float(wg[e >> 1] & 0xFFFF0000u) : __uint_as_float(wg[e >> 1] << 16);
                    const float uv = e & 1 ? __uint_as_float(wu[e >> 1] & 0xFFFF0000u) : __uint_as_float(wu[e >> 1] << 16);
                    const float go = v[c * 8 + e];
                    const float sig = __frcp_rn(__fadd_rn(1.0f, expf(-gv)));
                    const float dsilu = __fmul_rn(sig, __fadd_rn(1.0f, __fmul_rn(gv, __fsub_rn(1.0f, sig))));
                    dg[e] = bf16r(__fmul_rn(__fmul_rn(go, uv), dsilu));
                    du[e] = bf16r(__fmul_rn(go, __fmul_rn(gv, sig)));
                    smax = max(smax, max(abs_bits(dg[e]), abs_bits(du[e])));
                }
                rowp[sl] = make_uint4(pack_bf16x2(dg[0], dg[1]), pack_bf16x2(dg[2], dg[3]), pack_bf16x2(dg[4], dg[5]),
                                      pack_bf16x2(dg[6], dg[7]));
                rowu[sl] = make_uint4(pack_bf16x2(du[0], du[1]), pack_bf16x2(du[2], du[3]), pack_bf16x2(du[4], du[5]),
                                      pack_bf16x2(du[6], du[7]));
            }
            fence_async_shared();
            __syncwarp();
            if (lane == 0) {
                tma_store_2d(&p.to, box, col0, m_row0);
                tma_store_2d(&p.to, box + 4096, col0 + p.N, m_row0);
                bulk_commit();
            }
            continue;
        }
        if constexpr (LOADS) {
            const uint64_t ctr0 = sr_base + (uint64_t)row * (uint64_t)p.N + (uint64_t)col0;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const uint4 u = rowp[c ^ (lane & 7)];
                const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int j = c * 8 + 2 * e;
                    const float in0 = __uint_as_float(w[e] << 16), in1 = __uint_as_float(w[e] & 0xFFFF0000u);
                    if constexpr (EPI == EPI_BF16_RES) {
                        v[j] = __fadd_rn(v[j], in0);
                        v[j + 1] = __fadd_rn(v[j + 1], in1);
                    } else {
                        v[j] = sr_bf16k(__fadd_rn(in0, v[j]), key, ctr0 + j);
                        v[j + 1] = sr_bf16k(__fadd_rn(in1, v[j + 1]), key, ctr0 + j + 1);
                    }
                }
            }
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            uint4 u;
            if constexpr (F32OUT) {
                u = make_uint4(__float_as_uint(v[4 * c]), __float_as_uint(v[4 * c + 1]), __float_as_uint(v[4 * c + 2]),
                               __float_as_uint(v[4 * c + 3]));
            } else {
                u = make_uint4(pack_bf16x2(v[8 * c], v[8 * c + 1]), pack_bf16x2(v[8 * c + 2], v[8 * c + 3]),
                               pack_bf16x2(v[8 * c + 4], v[8 * c + 5]), pack_bf16x2(v[8 * c + 6], v[8 * c + 7]));
            }
            rowp[c ^ (lane & 7)] = u;
        }
        fence_async_shared();
        __syncwarp();
        if (lane == 0) {
            tma_store_2d(&p.to, box, col0, m_row0);
            bulk_commit();
        }
        buf ^= 1;
    }
    if constexpr (SWI) {
        smax = warp_max_u32(smax);
        if (lane == 0 && smax) atomicMax(p.amax, smax);
    }
    if (EPI == EPI_F32 && stats && row < p.M && n0 < p.N) p.ce_stats[(int64_t)row * p.ce_nstat + n0 / 128] = make_float2(cm, cs);
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_rank0(uint32_t local) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(local));
    return r;
}

constexpr int GEMM_THREADS = 384;  // warps: 0 TMA, 1 MMA, 2 TMEM alloc, 3 idle, 4..11 epilogue

template <int KIND, bool A_MN, bool B_MN, int BN, int EPI, int CG>
__global__ void __launch_bounds__(GEMM_THREADS, 1) gemm_kernel(const __grid_constant__ Params p) {
    using C = Cfg<KIND, BN, CG, EPI>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stg_base = base + C::STAGES * C::STAGE;  // epilogue staging boxes
    uint64_t* full = reinterpret_cast<uint64_t*>(stg_base + C::EPI_BYTES);
    uint64_t* empty = full + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* ebar = tempty + 2;  // [4] epilogue TMA-load barriers
    uint32_t* tslot = reinterpret_cast<uint32_t*>(ebar + C::EPI_WARPS);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = CG == 2 ? cluster_rank() : 0;
    const bool leader = crank == 0;
    if (warp == 0 && lane == 0) {
        tma_prefetch(&p.ta);
        tma_prefetch(&p.tb);
        if (p.split_a) tma_prefetch(&p.ta2);
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], C::EPI_WARPS * CG);
        }
        for (int w = 0; w < C::EPI_WARPS; ++w) mbar_init(&ebar[w], 1);
        fence_barrier_init();
        fence_async_shared();
    }
    if (warp == 2) {
        if constexpr (CG == 1) {
            tmem_alloc(tslot, C::TMEM_COLS);
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                         "r"(C::TMEM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const int tiles = p.num_m * p.num_n;
    const int all_tiles = tiles * p.splits;
    const int cid = blockIdx.x / CG, ncl = gridDim.x / CG;

    if (warp == 0 && lane == 0) {
        // ===== TMA producer (both CTAs of a pair load their halves) =====
        int stage = 0;
        uint32_t phase = 0;
        for (int tt = cid; tt < all_tiles; tt += ncl) {
            const int t = tt % tiles, sp = tt / tiles;
            const int tm = p.n_fast ? t / p.num_n : t % p.num_m, tn = p.n_fast ? t % p.num_n : t / p.num_m;
            const int m0 = tm * BM * CG + (int)crank * BM;
            const int n0 = tn * BN + (int)crank * C::BN_CTA;
            const int kb0 = sp * p.kb_per_split, kb1 = min(p.num_k, kb0 + p.kb_per_split);
            const int kn = kb1 - kb0;
            const int kiters = p.split_a ? 2 * kn : kn;
            for (int kq = 0; kq < kiters; ++kq) {
                mbar_wait(&empty[stage], phase ^ 1);
                uint8_t* sa = base + stage * C::STAGE;
                uint8_t* sb = sa + C::A_BYTES;
                uint32_t bar = smem_u32(&full[stage]);
                if constexpr (CG == 2) {
                    bar = mapa_rank0(bar);
                    if (leader)
                        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[stage])),
                                     "r"(C::STAGE * CG)
                                     : "memory");
                } else {
                    mbar_arrive_expect_tx(&full[stage], C::STAGE);
                }
                const bool second = kq >= kn;
                const CUtensorMap* tA = second ? &p.ta2 : &p.ta;
                const int k0 = (kb0 + (second ? kq - kn : kq)) * C::BK;
                auto load = [&](const CUtensorMap* m, void* dst, int c0, int c1) {
                    if constexpr (CG == 2)
                        asm volatile(
                            "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
                            "[%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
                            "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1)
                            : "memory");
                    else
                        tma_load_2d(m, &full[stage], dst, c0, c1);
                };
                if constexpr (!A_MN) {
                    load(tA, sa, k0, m0);
                } else {
#pragma unroll
                    for (int i = 0; i < BM * C::ELEM / 128; ++i)
                        load(tA, sa + i * C::BK * 128, m0 + i * (128 / C::ELEM), k0);
                }
                if constexpr (!B_MN) {
                    load(&p.tb, sb, k0, n0);
                } else {
#pragma unroll
                    for (int i = 0; i < C::BN_CTA * C::ELEM / 128; ++i)
                        load(&p.tb, sb + i * C::BK * 128, n0 + i * (128 / C::ELEM), k0);
                }
                if (++stage == C::STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1 && leader) {
        // ===== MMA issuer (warp-collective, one elected lane issues; leader CTA) =====
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        for (int tt = cid; tt < all_tiles; tt += ncl, ++it) {
            const int sp = tt / tiles;
            const int kb0 = sp * p.kb_per_split, kb1 = min(p.num_k, kb0 + p.kb_per_split);
            const int kiters = p.split_a ? 2 * (kb1 - kb0) : (kb1 - kb0);
            const int acc = it & 1;
            const uint32_t aphase = (it >> 1) & 1;
            mbar_wait(&tempty[acc], aphase ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem + acc * BN;
            for (int kb = 0; kb < kiters; ++kb) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                const uint32_t sa = smem_u32(base + stage * C::STAGE);
                const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
                for (int kk = 0; kk < C::BK / C::UK; ++kk) {
                    const uint64_t ad = A_MN ? make_sdesc_sw128(sa + kk * C::UK * 128, C::BK * 128, 1024)
                                             : make_sdesc_sw128(sa + kk * 32, 16, 1024);
                    const uint64_t bd = B_MN ? make_sdesc_sw128(sb + kk * C::UK * 128, C::BK * 128, 1024)
                                             : make_sdesc_sw128(sb + kk * 32, 16, 1024);
                    const uint32_t accum = (kb | kk) != 0;
                    if constexpr (CG == 1) {
                        if constexpr (KIND == 0) mma_f8(d_tmem, ad, bd, p.idesc, accum);
                        else mma_bf16(d_tmem, ad, bd, p.idesc, accum);
                    } else {
                        if constexpr (KIND == 0) mma_f8_pair(d_tmem, ad, bd, p.idesc, accum);
                        else mma_bf16_pair(d_tmem, ad, bd, p.idesc, accum);
                    }
                }
                if constexpr (CG == 1)
                    tc_commit(&empty[stage]);
                else
                    tc_commit_pair(&empty[stage]);
                if (++stage == C::STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if constexpr (CG == 1)
                tc_commit(&tfull[acc]);
            else
                tc_commit_pair(&tfull[acc]);
        }
    } else if (warp >= 4) {
        // ===== epilogue: TMEM -> registers -> rounding -> HBM =====
        const int ew = warp - 4, wq = warp & 3, half = ew >> 2;  // TMEM lane quarter = warp % 4
        constexpr int BNH = BN / 2;                               // this warp's columns of the tile
        uint8_t* stg = stg_base + ew * C::EPI_GROUPS * 4096;
        float denom = 1.0f;
        if (p.a_scale && p.b_scale) denom = __fmul_rn(*p.a_scale, *p.b_scale);
        const float rcp = __frcp_rn(denom);
        uint32_t ephase = 0;
        int ebuf = 0;
        int it = 0;
        for (int tt = cid; tt < all_tiles; tt += ncl, ++it) {
            const int t = tt % tiles, sp = tt / tiles;
            const int acc = it & 1;
            const uint32_t aphase = (it >> 1) & 1;
            const int tm = p.n_fast ? t / p.num_n : t % p.num_m, tn = p.n_fast ? t % p.num_n : t / p.num_m;
            const int m0 = tm * BM * CG + (int)crank * BM, n0 = tn * BN + half * BNH;
            if constexpr (epi_loads(EPI)) {
                if (p.tma_out && lane == 0) epilogue_prefetch<EPI>(p, m0 + wq * 32, n0, BNH, stg, &ebar[ew]);
            }
            mbar_wait(&tfull[acc], aphase);
            tc_fence_after();
            const uint32_t tcols = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(acc * BN + half * BNH);
            if (p.tma_out) {
                epilogue_tile_tma<EPI>(p, tcols, m0 + wq * 32, n0, BNH, denom, rcp, stg, &ebar[ew], ephase, ebuf);
            } else {
                const int row = m0 + wq * 32 + lane + sp * p.M;  // split partials stack along rows
#pragma unroll 1
                for (int c = 0; c < BNH / 32; ++c) {
                    uint32_t r[32];
                    tmem_ld32(tcols + c * 32, r);
                    tmem_ld_wait();
                    if (row - sp * p.M < p.M) epilogue_chunk<EPI>(p, row, n0 + c * 32, denom, rcp, r);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (CG == 1) {
                    mbar_arrive(&tempty[acc]);
                } else {
                    const uint32_t rb = mapa_rank0(smem_u32(&tempty[acc]));
                    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(rb) : "memory");
                }
            }
        }
        if (p.tma_out && lane == 0) bulk_wait<0>();  // staged stores done before the CTA's smem goes away
    }
    __syncthreads();
    if constexpr (CG == 2) cluster_sync_all();
    if (warp == 2) {
        tc_fence_after();
        if constexpr (CG == 1)
            tmem_dealloc(tmem, C::TMEM_COLS);
        else
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS)
                         : "memory");
    }
}

// ---------------------------------------------------------------------------
// split-K reduction: sum the S f32 partial tiles in split order (fixed, so the
// result is deterministic) and apply the requested epilogue
// ---------------------------------------------------------------------------
// Sums the split-K partials in split order and applies the epilogue; 4 columns
// per thread (N % 4 == 0, checked by the launcher), rows/cols by FastDiv.
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int S, int M, int N, FastDiv n4div, int epi,
                                     const float* __restrict__ a_scale, const float* __restrict__ b_scale,
                                     void* __restrict__ out, int64_t ldo, const uint16_t* __restrict__ res,
                                     int64_t ldr, uint64_t seed, uint64_t stream, uint64_t base,
                                     const uint64_t* ms, uint64_t ms_mn, uint64_t ms_off) {
    if (ms) base = *ms * ms_mn + ms_off;
    float denom = 1.0f;
    if (a_scale && b_scale) denom = __fmul_rn(*a_scale, *b_scale);
    const float rcp = __frcp_rn(denom);
    const int64_t total = (int64_t)M * N;
    const uint32_t n4 = (uint32_t)(N / 4), tot4 = (uint32_t)(total / 4);
    const uint64_t key = rng_key(seed, stream);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < tot4; i += gridDim.x * blockDim.x) {
        float4 acc = reinterpret_cast<const float4*>(ws)[i];
        for (int sp = 1; sp < S; ++sp) {
            const float4 w = reinterpret_cast<const float4*>(ws + (int64_t)sp * total)[i];
            acc.x = __fadd_rn(acc.x, w.x);
            acc.y = __fadd_rn(acc.y, w.y);
            acc.z = __fadd_rn(acc.z, w.z);
            acc.w = __fadd_rn(acc.w, w.w);
        }
        const uint32_t r = n4div.div(i), c = (i - r * n4) * 4;
        const float a[4] = {acc.x, acc.y, acc.z, acc.w};
        if (epi == EPI_F32) {
            *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + r * ldo + c) = acc;
            continue;
        }
        uint16_t* o = reinterpret_cast<uint16_t*>(out) + r * ldo + c;
        const uint64_t ctr = base + (uint64_t)r * (uint64_t)N + c;
        float v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (epi == EPI_F32_ACC) {
                v[j] = sr_bf16k(__fadd_rn(bfbits2f(o[j]), a[j]), key, ctr + j);
                continue;
            }
            v[j] = bf16r(div_exact(a[j], denom, rcp));
            if (epi == EPI_BF16_RES)
                v[j] = __fadd_rn(v[j], bfbits2f(res[r * ldr + c + j]));
            else if (epi == EPI_BF16_ACC)
                v[j] = sr_bf16k(__fadd_rn(bfbits2f(o[j]), v[j]), key, ctr + j);
        }
        *reinterpret_cast<uint2*>(o) = make_uint2(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]));
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

// 2-D map over a row-major matrix [outer][inner] with the given row stride.
int make_tmap(CUtensorMap* m, const void* ptr, int elem, uint64_t inner, uint64_t outer, uint64_t row_stride_elems,
              uint32_t box_inner, uint32_t box_outer) {
    auto fn = encode_fn();
    if (!fn) return 900;
    const CUtensorMapDataType dt = elem == 1   ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                  : elem == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                              : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_stride_elems * (uint64_t)elem};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(m, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : 901;
}

using KernelFn = void (*)(Params);

template <int KIND, bool A_MN, bool B_MN, int BN, int EPI, int CG>
int launch_cg(const Params& p, int grid, cudaStream_t s) {
    using C = Cfg<KIND, BN, CG, EPI>;
    // an MN-major operand tile must span whole 128-B swizzle atoms per CTA
    if constexpr (B_MN && (C::BN_CTA * C::ELEM) % 128 != 0) {
        return 903;
    } else {
    auto k = gemm_kernel<KIND, A_MN, B_MN, BN, EPI, CG>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return (int)e;
        attr_set = true;
    }
    if constexpr (CG == 1) {
        k<<<grid, GEMM_THREADS, C::SMEM, s>>>(p);
    } else {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(GEMM_THREADS);
        cfg.dynamicSmemBytes = C::SMEM;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CG;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, k, p);
        if (e != cudaSuccess) return (int)e;
    }
    return (int)cudaGetLastError();
    }
}

template <int KIND, bool A_MN, bool B_MN, int BN, int EPI>
int launch(const Params& p, int grid, int cg, cudaStream_t s) {
    return cg == 2 ? launch_cg<KIND, A_MN, B_MN, BN, EPI, 2>(p, grid, s)
                   : launch_cg<KIND, A_MN, B_MN, BN, EPI, 1>(p, grid, s);
}

int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = kNumSMs;
    }
    return n;
}

#define QTB_GEMM_CASE(KIND, AMN, BMN, EPI)                                                            \
    if (kind == KIND && a_mn == AMN && b_mn == BMN && epi == EPI)                                     \
        return bn == 256 ? launch<KIND, AMN, BMN, 256, EPI>(p, grid, cg, s)                           \
                         : launch<KIND, AMN, BMN, 128, EPI>(p, grid, cg, s);

int dispatch(int kind, bool a_mn, bool b_mn, int bn, int epi, const Params& p, int grid, int cg, cudaStream_t s) {
    // FP8 block linears: fwd (K,K), dgrad (K,MN), wgrad (MN,MN); plus (K,K) for transposed-operand callers
    QTB_GEMM_CASE(0, false, false, EPI_BF16)
    QTB_GEMM_CASE(0, false, false, EPI_BF16_RES)
    QTB_GEMM_CASE(0, false, true, EPI_BF16)
    QTB_GEMM_CASE(0, false, true, EPI_F32)  // split-K partials of a small-M dgrad
    QTB_GEMM_CASE(0, false, false, EPI_F32)  // split-K partials of a small-M forward
    QTB_GEMM_CASE(0, false, true, EPI_SWIGLU_BWD)
    QTB_GEMM_CASE(0, true, true, EPI_BF16)
    QTB_GEMM_CASE(0, true, true, EPI_BF16_ACC)
    QTB_GEMM_CASE(0, true, true, EPI_F32)
    QTB_GEMM_CASE(0, false, false, EPI_BF16_ACC)
    // BF16: LM-head logits (K,K)->f32, CE dgrad (K,MN)->bf16, CE wgrad (MN,MN)->f32 SR-accumulate
    QTB_GEMM_CASE(1, false, false, EPI_F32)
    QTB_GEMM_CASE(1, false, false, EPI_BF16)
    QTB_GEMM_CASE(1, false, true, EPI_BF16)
    QTB_GEMM_CASE(1, false, true, EPI_F32)
    QTB_GEMM_CASE(1, true, true, EPI_F32)
    QTB_GEMM_CASE(1, true, true, EPI_F32_ACC)
    QTB_GEMM_CASE(1, true, true, EPI_BF16)
    return 902;  // unsupported combination
}

// Tile configuration from a small cost model: for each (cta_group, BN) the
// time is  waves x (per-SM tile work) / (per-SM rate), where the rate is the
// tensor peak capped by this SM's share of L2 bandwidth times the tile's
// arithmetic intensity (2*128*BN flops per (128 + BN/cg) operand rows).
// QTB_GEMM_CG=1 forces single-CTA tiles.
struct TileCfg {
    int cg, bn;
};
TileCfg choose_cfg(int64_t M, int64_t N, int kind, bool b_mn, int64_t K = 1 << 20) {
    static int forced = -1;
    if (forced < 0) {
        const char* e = getenv("QTB_GEMM_CG");
        forced = e ? atoi(e) : 0;
    }
    const int sms = num_sms();
    const double elem = kind == 0 ? 1.0 : 2.0;
    const double peak = kind == 0 ? 21.6e12 : 10.9e12;  // per SM, dense
    const double l2 = 11.0e12 / sms;                   // bytes/s per SM (measured LTS cap, B300_MICROARCH.md)
    TileCfg best{1, 256};
    // short-K FP8 GEMMs (the K = d_model linears): the pair's cluster handshakes are not
    // amortised over a few k-blocks; single-CTA 128x256 tiles measured 15-20 % faster
    // at K = 896 (scripts/gemm_small.py), equal at K = 1152, slower at K >= 4864
    if (kind == 0 && K <= 1024 && N >= 256 && N <= 2048 && forced != 2) return best;  // wide N (gate_up): pairs win
    double best_t = 1e30;
    for (int cg = 1; cg <= 2; ++cg) {
        if (forced == 1 && cg == 2) continue;
        if (forced == 2 && cg == 1 && M >= 256) continue;  // QTB_GEMM_CG=2: pairs whenever legal
        if (cg == 2 && M < 256) continue;
        for (int bn = 128; bn <= 256; bn += 128) {
            if (cg == 2 && kind == 0 && b_mn && bn == 128) continue;  // half-atom MN-major B
            const int64_t tiles = ceil_div(M, (int64_t)BM * cg) * ceil_div(N, bn);
            const int64_t waves = ceil_div(tiles, sms / cg);
            const double inten = 2.0 * BM * bn / ((BM + (double)bn / cg) * elem);
            const double rate = std::min(peak, l2 * inten);
            const double t = (double)waves * BM * bn / rate;
            if (t < best_t * 0.999) {
                best_t = t;
                best = {cg, bn};
            }
        }
    }
    return best;
}
int pick_cg(int64_t M) { return choose_cfg(M, 1 << 20, 0, false).cg; }
int pick_bn(int64_t N) { return choose_cfg(1 << 20, N, 0, false).bn; }

// split-K factor for a GEMM (0 = no split): only when the tile grid leaves
// most SMs idle and K is long enough to amortise the reduction
int choose_splits(int64_t M, int64_t N, int64_t K, int kind, int bn, int cg) {
    const int bk = kind == 0 ? 128 : 64;
    const int64_t tiles = ceil_div(M, BM * cg) * ceil_div(N, bn);
    const int64_t nk = ceil_div(K, bk);
    if (tiles * cg * 2 > num_sms() || nk < 16) return 1;
    int64_t s = num_sms() / (tiles * cg);
    s = std::min<int64_t>(s, nk / 8);
    s = std::min<int64_t>(s, 8);
    return (int)std::max<int64_t>(s, 1);
}

// Tail split: when the persistent tile loop's last round is at most half full and K is
// long, the GEMM runs as a head of whole M panels filling the earlier rounds exactly plus
// a split-K tail over the remaining panels (the idle CTAs of the last round share its K
// loop).  0.5B gate_up wgrad (M 9728, N 896, K 16384): 152 pair tiles on 74 pairs = 2.05
// rounds -> 148 tiles + 4 tiles split 16 ways.  ws_bytes < 0: no workspace bound (sizing).
bool tail_plan(int64_t M, int64_t N, int64_t K, int kind, int cg, int bn, int64_t ws_bytes, int64_t* m_head,
               int* s_tail) {
    const int slots = num_sms() / cg;
    const int64_t bmc = (int64_t)BM * cg;
    const int64_t num_m = ceil_div(M, bmc), num_n = ceil_div(N, (int64_t)bn), tiles = num_m * num_n;
    const int64_t rounds = ceil_div(tiles, (int64_t)slots);
    if (rounds < 2 || N % 4) return false;
    if ((tiles - (rounds - 1) * slots) * 2 > slots) return false;
    // the head + split tail + reduce cost two extra launch ramps (~15 us): only worth it for
    // long K split many ways (measured: gate_up wgrad 130 -> 120 us at K = 16384, S = 16; the
    // down forward / gate_up dgrad at K = 4864 / 9728, S = 2 got slower, scripts/gemm_tail.py)
    const int64_t nk = ceil_div(K, (int64_t)(kind == 0 ? 128 : 64));
    if (nk < 64) return false;
    const int64_t hp = (rounds - 1) * slots / num_n;  // head M panels
    if (hp < 1 || hp >= num_m) return false;
    const int64_t mt = M - hp * bmc, tt = (num_m - hp) * num_n;
    int64_t sp = std::min<int64_t>(std::min<int64_t>(slots / tt, nk / 4), 16);
    while (ws_bytes >= 0 && sp >= 4 && sp * mt * N * 4 > ws_bytes) --sp;
    if (sp < 4) return false;
    *m_head = hp * bmc;
    *s_tail = (int)sp;
    return true;
}
bool tail_split_enabled() {
    static int f = -1;
    if (f < 0) {
        const char* e = getenv("QTB_GEMM_TAIL");
        f = e ? atoi(e) : 1;
    }
    return f != 0;
}

}  // namespace gemm
}  // namespace qtb

using namespace qtb;

extern "C" int qtk_gemm_splitk_ws_bytes(int64_t M, int64_t N, int64_t K, int kind) {
    int best = 0;
    for (int bmn = 0; bmn < 2; ++bmn) {  // the bound over both operand layouts
        const auto tc = qtb::gemm::choose_cfg(M, N, kind, bmn != 0, K);
        const int bn = (tc.cg == 2 && kind == 0 && bmn && tc.bn == 128) ? 256 : tc.bn;
        const int s = qtb::gemm::choose_splits(M, N, K, kind, bn, tc.cg);
        if (s > 1) best = std::max(best, (int)std::min<int64_t>((int64_t)s * M * N * 4, INT32_MAX));
        int64_t mh = 0;
        int st = 0;
        if (s <= 1 && qtb::gemm::tail_split_enabled() && qtb::gemm::tail_plan(M, N, K, kind, tc.cg, bn, -1, &mh, &st))
            best = std::max(best, (int)std::min<int64_t>((int64_t)st * (M - mh) * N * 4, INT32_MAX));
    }
    return best;
}

namespace qtb {
namespace gemm {
// The launch decision of qtk_gemm (cta_group, BN, split-K factor), shared with
// qtk_gemm_plan so tests can assert which instantiation a shape runs.
struct Decision {
    int cg, bn, splits;
};
Decision decide(const QtkGemm* g, int force_cg = 0) {
    TileCfg tc = choose_cfg(g->M, g->N, g->kind, g->b_mn != 0, g->K);
    if (force_cg) tc.cg = force_cg;  // tail-split head: the full GEMM's tile shape
    Decision d{tc.cg, (g->bn == 128 || g->bn == 256) ? g->bn : tc.bn, 1};
    const bool ce = g->ce_stats != nullptr;
    if (ce) d.bn = 256;  // one 128-column statistics block per epilogue warp half
    // FP8 MN-major B split over a CTA pair needs >= 128 N-columns per CTA
    if (d.cg == 2 && g->kind == 0 && g->b_mn && d.bn == 128) d.bn = 256;
    // the reduce pass works on 4-column vectors with 32-bit indices
    const bool reducible = g->N % 4 == 0 && g->ldo % 4 == 0 && g->M * g->N / 4 < (int64_t(1) << 31);
    if (g->ws && g->split_k != 1 && reducible && g->epi != EPI_SWIGLU_BWD && !ce) {
        d.splits = g->split_k > 1 ? g->split_k : choose_splits(g->M, g->N, g->K, g->kind, d.bn, d.cg);
        if ((int64_t)d.splits * g->M * g->N * 4 > g->ws_bytes) d.splits = 1;
    }
    if (d.splits > 1) {
        const int bk = g->kind == 0 ? 128 : 64;
        const int nk = (int)ceil_div(g->K, bk);
        d.splits = (int)ceil_div(nk, (int)ceil_div(nk, d.splits));  // no empty splits
    }
    return d;
}
}  // namespace gemm
}  // namespace qtb

// Which kernel instantiation qtk_gemm would launch for *g (no launch):
// cta_group (1 or 2), BN (128 or 256), split-K factor, grid size (CTAs) and
// output tiles per CTA (the persistent loop's trip count, rounded up).
extern "C" int qtk_gemm_plan(const QtkGemm* g, int* cg, int* bn, int* splits, int* grid, int* tiles_per_cta) {
    using namespace qtb::gemm;
    if (g->M <= 0 || g->N <= 0 || g->K <= 0) return 1;
    const Decision d = decide(g);
    const int64_t tiles = ceil_div(g->M, (int64_t)BM * d.cg) * ceil_div(g->N, (int64_t)d.bn) * d.splits;
    const int64_t ctas = std::min<int64_t>(tiles, num_sms() / d.cg) * d.cg;
    *cg = d.cg;
    *bn = d.bn;
    *splits = d.splits;
    *grid = (int)ctas;
    *tiles_per_cta = (int)ceil_div(tiles, ctas / d.cg);
    return 0;
}

// One launch (or split-K launch + reduce) of *g.  sr_row0 = global row of g's first row
// and M_full = the full GEMM's M when g is a tail-split part (the SR counters stay those of
// the unsplit GEMM); force_cg = the full GEMM's cta_group for the head part.
static int gemm_run(const QtkGemm* g, cudaStream_t s, int64_t sr_row0, int64_t M_full, int force_cg) {
    using namespace qtb::gemm;
    if (g->M <= 0 || g->N <= 0 || g->K <= 0) return 0;
    const int elem = g->kind == 0 ? 1 : 2;
    const int bk = 128 / elem;
    // TMA: 16-B aligned base and row strides, leading dims cover the extents
    if ((reinterpret_cast<uintptr_t>(g->a) & 15) || (reinterpret_cast<uintptr_t>(g->b) & 15) ||
        ((g->lda * elem) & 15) || ((g->ldb * elem) & 15))
        return 1;
    if (g->lda < (g->a_mn ? g->M : g->K) || g->ldb < (g->b_mn ? g->N : g->K)) return 1;
    const Decision dec = decide(g, force_cg);
    const int cg = dec.cg;
    const int bn = dec.bn;
    const bool ce = g->ce_stats != nullptr;
    if (ce && (g->epi != EPI_F32 || !g->ce_targets || !g->ce_tgt_logit)) return 1;
    Params p;
    memset(&p, 0, sizeof(p));
    int rc;
    // A: K-major stored [M][lda]; MN-major stored [K][lda]
    if (!g->a_mn)
        rc = make_tmap(&p.ta, g->a, elem, g->K, g->M, g->lda, bk, BM);
    else
        rc = make_tmap(&p.ta, g->a, elem, g->M, g->K, g->lda, 128 / elem, bk);
    if (rc) return rc;
    if (!g->b_mn)
        rc = make_tmap(&p.tb, g->b, elem, g->K, g->N, g->ldb, bk, bn / cg);
    else
        rc = make_tmap(&p.tb, g->b, elem, g->N, g->K, g->ldb, 128 / elem, bk);
    if (rc) return rc;
    if (g->a2) {
        if (reinterpret_cast<uintptr_t>(g->a2) & 15) return 1;
        if (!g->a_mn)
            rc = make_tmap(&p.ta2, g->a2, elem, g->K, g->M, g->lda, bk, BM);
        else
            rc = make_tmap(&p.ta2, g->a2, elem, g->M, g->K, g->lda, 128 / elem, bk);
        if (rc) return rc;
        p.split_a = 1;
    }
    p.M = (int)g->M;
    p.N = (int)g->N;
    p.K = (int)g->K;
    p.num_m = (int)ceil_div(g->M, BM * cg);
    p.num_n = (int)ceil_div(g->N, bn);
    p.num_k = (int)ceil_div(g->K, bk);
    const uint32_t afmt = g->kind == 0 ? (uint32_t)g->a_fmt : 1u;  // bf16 = 1 in the F16 format table
    const uint32_t bfmt = g->kind == 0 ? (uint32_t)g->b_fmt : 1u;
    p.idesc = sm100::make_idesc(afmt, bfmt, g->a_mn != 0, g->b_mn != 0, BM * cg, bn);
    p.a_scale = g->a_scale;
    p.b_scale = g->b_scale;
    p.out = g->out;
    p.ldo = g->ldo;
    p.res = reinterpret_cast<const uint16_t*>(g->res);
    p.ldr = g->ldr;
    p.sr_seed = g->sr_seed;
    p.sr_stream = g->sr_stream;
    const uint64_t sr_off = (uint64_t)sr_row0 * (uint64_t)g->N;
    p.sr_base = g->sr_base + sr_off;
    p.sr_ms = g->sr_micro_step;
    p.sr_mn = (uint64_t)M_full * (uint64_t)g->N;
    p.sr_off = sr_off;
    const int tiles = p.num_m * p.num_n;
    const int splits = dec.splits;
    p.splits = splits;
    // L2-aware order: when an M panel is shared by few N tiles, run those N tiles side by side
    // (split-K too: the LM-head dgrad's 4 N tiles then share each dlogits panel in L2 instead
    // of re-streaming it once per N tile, 20.3 -> 15.6 GB per launch; with hundreds of M
    // panels -- the LM-head wgrad, M = vocab -- the M-fast order measured better, 13.1 vs 15.9 GB)
    p.n_fast = p.num_n <= p.num_m && (splits == 1 || p.num_m <= 256);
    p.kb_per_split = (int)ceil_div(p.num_k, splits);
    if (splits > 1) {
        p.splits = (int)ceil_div(p.num_k, p.kb_per_split);  // no empty splits (== splits, see decide)
        p.out = g->ws;
        p.ldo = g->N;
        const int all = tiles * p.splits;
        const int grid = std::min(all, num_sms() / cg) * cg;
        int rc2 = dispatch(g->kind, g->a_mn != 0, g->b_mn != 0, bn, EPI_F32, p, grid, cg, s);
        if (rc2) return rc2;
        const int64_t total = g->M * g->N;
        const int rg = (int)std::min<int64_t>(ceil_div(total / 4, 256), 8 * num_sms());
        splitk_reduce_kernel<<<rg, 256, 0, s>>>((const float*)g->ws, p.splits, (int)g->M, (int)g->N,
                                                FastDiv((uint32_t)(g->N / 4)), g->epi,
                                                g->a_scale, g->b_scale, g->out, g->ldo,
                                                reinterpret_cast<const uint16_t*>(g->res), g->ldr, g->sr_seed,
                                                g->sr_stream, g->sr_base + sr_off, g->sr_micro_step, p.sr_mn, sr_off);
        return (int)cudaGetLastError();
    }
    // staged TMA-store epilogue: 16-B aligned output (and residual) rows
    {
        const int oel = g->epi == EPI_F32 ? 4 : 2;
        static int no_tma = -1;
        if (no_tma < 0) {
            const char* e = getenv("QTB_GEMM_NO_TMA_EPI");
            no_tma = e ? atoi(e) : 0;
        }
        const int64_t ncols = g->epi == EPI_SWIGLU_BWD ? 2 * g->N : g->N;  // gate | up halves
        // pinned host buffers (offloaded gradient accumulators, zero-copy) take the direct path
        auto on_device = [](const void* ptr) {
            cudaPointerAttributes a{};
            if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
                cudaGetLastError();
                return true;
            }
            return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
        };
        bool ok = !no_tma && !(reinterpret_cast<uintptr_t>(g->out) & 15) && ((g->ldo * oel) & 15) == 0 &&
                  g->ldo >= ncols && on_device(g->out) && (!g->res || on_device(g->res));
        if (ok && g->epi == EPI_BF16_RES)
            ok = g->res && !(reinterpret_cast<uintptr_t>(g->res) & 15) && ((g->ldr * 2) & 15) == 0 && g->ldr >= g->N;
        if (ok && g->epi == EPI_SWIGLU_BWD)
            ok = g->res && g->amax && !(reinterpret_cast<uintptr_t>(g->res) & 15) && ((g->ldr * 2) & 15) == 0 &&
                 g->ldr >= ncols && g->N % 64 == 0;
        if (ok) ok = make_tmap(&p.to, g->out, oel, ncols, g->M, g->ldo, 128 / oel, 32) == 0;
        if (ok && (g->epi == EPI_BF16_RES || g->epi == EPI_SWIGLU_BWD))
            ok = make_tmap(&p.tr, g->res, 2, ncols, g->M, g->ldr, 64, 32) == 0;
        p.tma_out = ok ? 1 : 0;
        p.amax = g->amax;
    p.ce_targets = g->ce_targets;
    p.ce_stats = reinterpret_cast<float2*>(g->ce_stats);
    p.ce_tgt_logit = g->ce_tgt_logit;
    p.ce_nstat = (int)ceil_div(g->N, 128);
        if ((g->epi == EPI_SWIGLU_BWD || ce) && !ok) return 1;  // no direct-store variant of these epilogues
    }
    const int grid = std::min(tiles, num_sms() / cg) * cg;
    return dispatch(g->kind, g->a_mn != 0, g->b_mn != 0, bn, g->epi, p, grid, cg, s);
}

static bool use_tail(const QtkGemm* g, const qtb::gemm::Decision& d, int64_t* m_head, int* s_tail) {
    using namespace qtb::gemm;
    return tail_split_enabled() && d.splits == 1 && g->ws && g->split_k == 0 && !g->ce_stats && !g->a2 &&
           g->epi != EPI_SWIGLU_BWD && g->ldo % 4 == 0 &&
           tail_plan(g->M, g->N, g->K, g->kind, d.cg, d.bn, g->ws_bytes, m_head, s_tail);
}

extern "C" int qtk_gemm_tail_plan(const QtkGemm* g, int64_t* m_head, int* s_tail) {
    *m_head = g->M;
    *s_tail = 1;
    if (g->M <= 0 || g->N <= 0 || g->K <= 0) return 0;
    return use_tail(g, qtb::gemm::decide(g), m_head, s_tail) ? 1 : 0;
}

extern "C" int qtk_gemm(const QtkGemm* g, cudaStream_t s) {
    using namespace qtb::gemm;
    if (g->M <= 0 || g->N <= 0 || g->K <= 0) return 0;
    const Decision d = decide(g);
    int64_t m_head = 0;
    int s_tail = 0;
    if (use_tail(g, d, &m_head, &s_tail)) {
        const int elem = g->kind == 0 ? 1 : 2;
        const int oel = g->epi == EPI_F32 ? 4 : 2;
        QtkGemm h = *g;
        h.M = m_head;
        h.split_k = 1;
        h.bn = d.bn;
        int rc = gemm_run(&h, s, 0, g->M, d.cg);
        if (rc) return rc;
        QtkGemm t = *g;
        t.M = g->M - m_head;
        t.split_k = s_tail;
        t.a = static_cast<const uint8_t*>(g->a) + (g->a_mn ? m_head : m_head * g->lda) * elem;
        t.out = static_cast<uint8_t*>(g->out) + m_head * g->ldo * oel;
        if (g->res) t.res = static_cast<const uint8_t*>(g->res) + m_head * g->ldr * 2;
        return gemm_run(&t, s, m_head, g->M, 0);
    }
    return gemm_run(g, s, 0, g->M, 0);
}
