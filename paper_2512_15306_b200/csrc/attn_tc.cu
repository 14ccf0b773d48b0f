// Causal GQA attention forward on tcgen05 (sm_100a): reference sdpa_chunked /
// attn_row_forward (src/tensorops.cpp:191-255).
//
// CTA = 128 query rows of one head; 8 warps: 0 TMA producer, 1 MMA issuer
// (one thread), 2 TMEM allocator, 4..7 softmax (thread = query row = TMEM
// lane).  Two passes over the causal KV tiles (128 keys each):
//   pass 1  S = Q K^T (tcgen05 kind::f16, f32 in TMEM, double buffered);
//           softmax warps keep the running row max m and sum l in f32
//   pass 2  S again; P = exp(x - m) / l -- normalised before P.V exactly as
//           the reference does (probs *= inv_denom, then out = sum p v) --
//           written to SMEM as bf16 hi + lo (16 significant bits) in the
//           UMMA 128-B-swizzled K-major layout; O += P_hi V + P_lo V in TMEM
// then O (f32) -> bf16 att, the unrounded f32 copy for the backward's
// D = rowsum(dO o O), LSE = m + log(l), and the fused absmax.
#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

namespace qtb {
namespace attn_tc {

using namespace sm100;

constexpr int BQ = 128, BKV = 128;
constexpr int NT = 384;  // 12 warps: 0 TMA, 1 MMA, 2 TMEM alloc, 3 idle, 4..11 softmax
constexpr int NSW = 8;   // softmax warps: (lane quarter w%4) x (key half (w-4)/4)

template <int HD>
struct Smem {
    static constexpr int Q = BQ * HD * 2;    // Q tile: HD/64 atom columns of 16 KB
    static constexpr int K = BKV * HD * 2;   // one K stage
    static constexpr int V = BKV * HD * 2;   // one V stage
    static constexpr int P = BQ * BKV * 2;   // one P part (hi or lo): 2 atom columns
    static constexpr int NPB = HD == 64 ? 2 : 1;  // P (hi+lo) buffers: double-buffered when they fit
    static constexpr int NVS = HD == 64 ? 2 : 1;  // V stages (hd 128: one, to stay within 227 KB)
    static constexpr int OFF_Q = 0;
    static constexpr int OFF_K = OFF_Q + Q;
    static constexpr int OFF_V = OFF_K + 2 * K;
    static constexpr int OFF_PH = OFF_V + NVS * V;  // buffer b: hi at OFF_PH + 2*b*P, lo at + P
    static constexpr int OFF_BAR = OFF_PH + 2 * NPB * P;
    static constexpr int BYTES = OFF_BAR + 256 + 4 * BQ * 4 + 1024;  // barriers, (m, l) exchange, align
};

__device__ __forceinline__ void mma_bf16_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    mma_bf16(d, a, b, idesc, acc);
}

// K-major SW128 descriptor for a tile whose 64-element atom columns are
// `atom_stride` bytes apart; k-step kk of UK=16 bf16
__device__ __forceinline__ uint64_t kdesc(uint32_t base, int kk, int atom_stride) {
    return make_sdesc_sw128(base + (kk >> 2) * atom_stride + (kk & 3) * 32, 16, 1024);
}
// MN-major SW128 descriptor (N contiguous in 64-element atoms LBO apart), k-step kk of 16 rows
__device__ __forceinline__ uint64_t mndesc(uint32_t base, int kk, int lbo) {
    return make_sdesc_sw128(base + kk * 16 * 128, lbo, 1024);
}

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
constexpr float LOG2E = 1.4426950408889634f;

// fork/join events of the two-stream backward: one pair per host thread (sessions of a peer
// group run on different threads)
inline cudaEvent_t fork_ev() {
    thread_local cudaEvent_t e = [] {
        cudaEvent_t x;
        cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
        return x;
    }();
    return e;
}
inline cudaEvent_t join_ev() {
    thread_local cudaEvent_t e = [] {
        cudaEvent_t x;
        cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
        return x;
    }();
    return e;
}

// forward kernel: 1 = two Q tiles per CTA (fwd2q_tc_kernel), 0 = one (fwd1p_tc_kernel);
// QTB_ATTN_FWD2Q, qtk_attn_set_fwd2q
static int g_fwd2q = -1;
inline int fwd2q_mode() {
    if (g_fwd2q < 0) {
        const char* e = getenv("QTB_ATTN_FWD2Q");
        g_fwd2q = e ? atoi(e) : 1;
    }
    return g_fwd2q;
}

// P (forward) and P / dS (backward) as MMA operands: bf16 hi + lo (16 significant bits,
// f32-faithful products) or bf16 alone (one MMA per k-step instead of two).
// QTB_ATTN_PLO=1|0; qtk_attn_set_plo overrides (tests/A-B).
static int g_plo = -1;
inline int p_lo_mode() {
    if (g_plo < 0) {
        const char* e = getenv("QTB_ATTN_PLO");
        g_plo = e ? atoi(e) : 1;
    }
    return g_plo;
}

template <int HD>
__global__ void __launch_bounds__(NT, 1) fwd_tc_kernel(const __grid_constant__ CUtensorMap tm, int T, int H, int Hkv,
                                                       float inv_sqrt_d, uint16_t* __restrict__ out, int64_t ldo,
                                                       float* __restrict__ out32, float* __restrict__ lse,
                                                       uint32_t* __restrict__ amax) {
    using S = Smem<HD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + S::OFF_BAR);
    uint64_t* q_full = bar + 0;
    uint64_t* k_full = bar + 1;   // [2]
    uint64_t* k_empty = bar + 3;  // [2]
    uint64_t* v_full = bar + 5;   // [2]
    uint64_t* v_empty = bar + 7;  // [2]
    uint64_t* s_full = bar + 9;   // [2]
    uint64_t* s_empty = bar + 11; // [2]
    uint64_t* p_full = bar + 13;   // [2]
    uint64_t* p_empty = bar + 15;  // [2]
    uint64_t* o_full = bar + 17;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 18);

    const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int kvh = h / (H / Hkv);
    const int d = H * HD;
    const int nj = qt + 1;  // causal KV tiles (BQ == BKV)
    const int row0 = b * T + qt * BQ;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) tma_prefetch(&tm);
    if (warp == 1 && lane == 0) {
        mbar_init(q_full, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&k_empty[i], 1);
            mbar_init(&v_full[i], 1);
            mbar_init(&v_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&s_empty[i], NSW);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&p_full[i], NSW);
            mbar_init(&p_empty[i], 1);
        }
        mbar_init(o_full, 1);
        fence_barrier_init();
        fence_async_shared();
    }
    if (warp == 2) tmem_alloc(tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t s_base = smem_u32(sm);

    if (warp == 0 && lane == 0) {
        // ===== TMA producer: Q once; pass 1 K tiles; pass 2 (K, V) tiles =====
        mbar_arrive_expect_tx(q_full, S::Q);
        for (int c = 0; c < HD / 64; ++c) tma_load_2d(&tm, q_full, sm + S::OFF_Q + c * BQ * 128, h * HD + c * 64, row0);
        int ks = 0, vs = 0;
        uint32_t kph = 0, vph = 0;
        for (int pass = 0; pass < 2; ++pass) {
            for (int j = 0; j < nj; ++j) {
                const int krow = b * T + j * BKV;
                mbar_wait(&k_empty[ks], kph ^ 1);
                mbar_arrive_expect_tx(&k_full[ks], S::K);
                for (int c = 0; c < HD / 64; ++c)
                    tma_load_2d(&tm, &k_full[ks], sm + S::OFF_K + ks * S::K + c * BKV * 128, d + kvh * HD + c * 64, krow);
                if (++ks == 2) { ks = 0; kph ^= 1; }
                if (pass == 1) {
                    mbar_wait(&v_empty[vs], vph ^ 1);
                    mbar_arrive_expect_tx(&v_full[vs], S::V);
                    for (int c = 0; c < HD / 64; ++c)
                        tma_load_2d(&tm, &v_full[vs], sm + S::OFF_V + vs * S::V + c * BKV * 128,
                                    d + Hkv * HD + kvh * HD + c * 64, krow);
                    if (++vs == S::NVS) { vs = 0; vph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {  // MMA issuer: whole warp, elected lane issues
        // ===== MMA issuer =====
        const uint32_t idesc_s = make_idesc(1, 1, false, false, BQ, BKV);  // S: M128 N128, both K-major
        const uint32_t idesc_o = make_idesc(1, 1, false, true, BQ, HD);    // O: A = P K-major, B = V MN-major
        mbar_wait(q_full, 0);
        int ks = 0, vs = 0, sc = 0;
        uint32_t kph = 0, vph = 0;
        auto issue_s = [&]() {
            mbar_wait(&k_full[ks], kph);
            const int sb = sc & 1;
            mbar_wait(&s_empty[sb], ((sc >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t qa = s_base + S::OFF_Q, ka = s_base + S::OFF_K + ks * S::K;
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk)
                mma_bf16_ss(tmem + sb * BKV, kdesc(qa, kk, BQ * 128), kdesc(ka, kk, BKV * 128), idesc_s, kk > 0);
            tc_commit(&k_empty[ks]);
            tc_commit(&s_full[sb]);
            if (++ks == 2) { ks = 0; kph ^= 1; }
            ++sc;
        };
        for (int j = 0; j < nj; ++j) issue_s();  // pass 1
        issue_s();                                // pass 2, tile 0
        for (int j = 0; j < nj; ++j) {
            if (j + 1 < nj) issue_s();
            const int pb = S::NPB == 2 ? (j & 1) : 0;
            const uint32_t pph = S::NPB == 2 ? ((j >> 1) & 1) : (j & 1);
            mbar_wait(&p_full[pb], pph);
            mbar_wait(&v_full[vs], vph);
            tc_fence_after();
            const uint32_t va = s_base + S::OFF_V + vs * S::V;
            const uint32_t ph = s_base + S::OFF_PH + pb * 2 * S::P, pl = ph + S::P;
#pragma unroll
            for (int kk = 0; kk < BKV / 16; ++kk) {
                const uint64_t bd = mndesc(va, kk, BKV * 128);
                mma_bf16_ss(tmem + 256, kdesc(ph, kk, BQ * 128), bd, idesc_o, (j | kk) != 0);
                mma_bf16_ss(tmem + 256, kdesc(pl, kk, BQ * 128), bd, idesc_o, 1);
            }
            tc_commit(&v_empty[vs]);
            tc_commit(&p_empty[pb]);
            if (++vs == S::NVS) { vs = 0; vph ^= 1; }
        }
        tc_commit(o_full);
    } else if (warp >= 4) {
        // ===== softmax: thread = (query row, key half) =====
        // Scores stay in raw QK^T units; x = s/sqrt(hd) enters only through
        // a = log2(e)/sqrt(hd): exp(x - m) = ex2(s*a - m_raw*a) (one FMA).
        const int wq = warp & 3, half = (warp - 4) >> 2;
        const int r = wq * 32 + lane;
        const int q = qt * BQ + r;  // position in the sequence
        const uint32_t lane_base = tmem + ((uint32_t)(wq * 32) << 16);
        const int c0 = half * (BKV / 2);  // this thread's 64 keys of each tile
        const float a = inv_sqrt_d * LOG2E;
        float* xch = reinterpret_cast<float*>(sm + S::OFF_BAR + 256);  // [4][BQ] (m, l) exchange
        float m = -INFINITY, l = 0.0f;  // m: running max of the raw scores
        int sc = 0;
        // S tile -> 64 registers, and the TMEM buffer handed back at once
        auto load_s = [&](uint32_t (&rr)[64]) {
            const int sb = sc & 1;
            mbar_wait(&s_full[sb], (sc >> 1) & 1);
            tc_fence_after();
            tmem_ld32(lane_base + sb * BKV + c0, *reinterpret_cast<uint32_t(*)[32]>(&rr[0]));
            tmem_ld32(lane_base + sb * BKV + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&rr[32]));
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[sb]);
            ++sc;
        };
        // keys past the query position exist only in the diagonal tile (BQ == BKV)
        auto masked = [&](int j, int i) { return j == qt && (j * BKV + c0 + i > q); };
        // pass 1: running max / sum over this half's keys
        for (int j = 0; j < nj; ++j) {
            uint32_t rr[64];
            load_s(rr);
            float mt = -INFINITY;
            if (j == qt) {
#pragma unroll
                for (int i = 0; i < 64; ++i)
                    if (!masked(j, i)) mt = fmaxf(mt, __uint_as_float(rr[i]));
            } else {
#pragma unroll
                for (int i = 0; i < 64; ++i) mt = fmaxf(mt, __uint_as_float(rr[i]));
            }
            const float mn = fmaxf(m, mt);
            if (mn != -INFINITY) {
                const float mb = mn * a;
                float ssum = 0.0f;
                if (j == qt) {
#pragma unroll
                    for (int i = 0; i < 64; ++i)
                        if (!masked(j, i)) ssum += ex2(__fmaf_rn(__uint_as_float(rr[i]), a, -mb));
                } else {
                    float s2[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
                    for (int i = 0; i < 64; ++i) s2[i & 3] += ex2(__fmaf_rn(__uint_as_float(rr[i]), a, -mb));
                    ssum = (s2[0] + s2[1]) + (s2[2] + s2[3]);
                }
                l = (m == -INFINITY ? 0.0f : l * ex2((m - mn) * a)) + ssum;
                m = mn;
            }
        }
        // combine the two halves' (m, l) once
        if (half == 1) {
            xch[r] = m;
            xch[BQ + r] = l;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(NSW * 32) : "memory");
        if (half == 0) {
            const float m1 = xch[r], l1 = xch[BQ + r];
            const float mg = fmaxf(m, m1);
            float lg = 0.0f;
            if (mg != -INFINITY) {
                lg = (m == -INFINITY ? 0.0f : l * ex2((m - mg) * a)) + (m1 == -INFINITY ? 0.0f : l1 * ex2((m1 - mg) * a));
            }
            xch[2 * BQ + r] = mg;
            xch[3 * BQ + r] = lg;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(NSW * 32) : "memory");
        m = xch[2 * BQ + r];
        l = xch[3 * BQ + r];
        const float inv_l = l > 0.0f ? 1.0f / l : 0.0f;
        const float mb = m * a;
        // pass 2: normalised probabilities -> P hi/lo in SMEM (this half = one atom column)
        for (int j = 0; j < nj; ++j) {
            uint32_t rr[64];
            load_s(rr);
            const int pb = S::NPB == 2 ? (j & 1) : 0;
            const uint32_t pph = S::NPB == 2 ? ((j >> 1) & 1) : (j & 1);
            uint8_t* ph = sm + S::OFF_PH + pb * 2 * S::P + half * BQ * 128;
            uint8_t* pl = ph + S::P;
            uint32_t hi[32], lo[32];
#pragma unroll
            for (int i = 0; i < 64; i += 2) {
                float pp[2];
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    pp[e] = masked(j, i + e) ? 0.0f : ex2(__fmaf_rn(__uint_as_float(rr[i + e]), a, -mb)) * inv_l;
                const float h0 = bf16r(pp[0]), h1 = bf16r(pp[1]);
                hi[i / 2] = pack_bf16x2(h0, h1);
                lo[i / 2] = pack_bf16x2(pp[0] - h0, pp[1] - h1);
            }
            mbar_wait(&p_empty[pb], pph ^ 1);
            // K-major SW128: key chunk cc (8 keys) at r*128 + ((cc ^ (r&7)) * 16)
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {
                const int off = r * 128 + ((cc ^ (r & 7)) << 4);
                *reinterpret_cast<uint4*>(ph + off) = make_uint4(hi[cc * 4 + 0], hi[cc * 4 + 1], hi[cc * 4 + 2], hi[cc * 4 + 3]);
                *reinterpret_cast<uint4*>(pl + off) = make_uint4(lo[cc * 4 + 0], lo[cc * 4 + 1], lo[cc * 4 + 2], lo[cc * 4 + 3]);
            }
            fence_async_shared();  // generic-proxy stores -> visible to the tensor core
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[pb]);
        }
        // epilogue: this half's HD/2 columns of the O row -> bf16 att + f32 copy; LSE; absmax
        mbar_wait(o_full, 0);
        tc_fence_after();
        uint32_t mx = 0;
        const bool valid = q < T;
        const int64_t grow = (int64_t)b * T + q;
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
            const int col = half * (HD / 2) + c * 32;
            uint32_t rr[32];
            tmem_ld32(lane_base + 256 + col, rr);
            tmem_ld_wait();
            if (valid) {
                uint4* o16 = reinterpret_cast<uint4*>(out + grow * ldo + h * HD + col);
                float4* o32 = reinterpret_cast<float4*>(out32 + grow * ldo + h * HD + col);
#pragma unroll
                for (int v4 = 0; v4 < 4; ++v4) {
                    float f[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        f[e] = __uint_as_float(rr[v4 * 8 + e]);
                        mx = max(mx, abs_bits(bf16r(f[e])));
                    }
                    o16[v4] = make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                                         pack_bf16x2(f[6], f[7]));
                    if (out32) {
                        o32[2 * v4] = make_float4(f[0], f[1], f[2], f[3]);
                        o32[2 * v4 + 1] = make_float4(f[4], f[5], f[6], f[7]);
                    }
                }
            }
        }
        if (valid && half == 0) lse[((int64_t)b * H + h) * T + q] = m * inv_sqrt_d + logf(l);  // m: raw-score max
        mx = warp_max_u32(mx);
        if (lane == 0 && amax && mx) atomicMax(amax, mx);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}



// ===========================================================================
// One-pass forward (online softmax).  Same roles and buffers as fwd_tc_kernel,
// but every KV tile is visited once: S(j) = QK^T in TMEM (double-buffered);
// the two softmax threads of a row (key halves) agree on the tile max through
// shared memory; p~ = exp(x - m_used) with a lazily updated m_used (moved only
// when the row max grows by more than 2^8, so p~ <= 256 and O is rescaled in
// TMEM rarely -- after PV(j-1) has landed); P~ as bf16 hi + lo in double-
// buffered smem; O += P~_hi V + P~_lo V.  At the end O / l (l = sum of p~)
// is the reference's sum_k (p_k) v_k up to f32 rounding order.
// ===========================================================================
__device__ __forceinline__ void tmem_ld32_raw(uint32_t taddr, uint32_t (&r)[32]) { tmem_ld32(taddr, r); }
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}

template <int HD>
__global__ void __launch_bounds__(NT, 1) fwd1_tc_kernel(const __grid_constant__ CUtensorMap tm, int T, int H, int Hkv,
                                                        float inv_sqrt_d, uint16_t* __restrict__ out, int64_t ldo,
                                                        float* __restrict__ out32, float* __restrict__ lse,
                                                        uint32_t* __restrict__ amax) {
    using S = Smem<HD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + S::OFF_BAR);
    uint64_t* q_full = bar + 0;
    uint64_t* k_full = bar + 1;    // [2]
    uint64_t* k_empty = bar + 3;   // [2]
    uint64_t* v_full = bar + 5;    // [2]
    uint64_t* v_empty = bar + 7;   // [2]
    uint64_t* s_full = bar + 9;    // [2]
    uint64_t* s_empty = bar + 11;  // [2]
    uint64_t* p_full = bar + 13;   // [2]
    uint64_t* p_empty = bar + 15;  // [2]
    uint64_t* o_full = bar + 17;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 18);

    const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int kvh = h / (H / Hkv);
    const int d = H * HD;
    const int nj = qt + 1;  // causal KV tiles (BQ == BKV)
    const int row0 = b * T + qt * BQ;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) tma_prefetch(&tm);
    if (warp == 1 && lane == 0) {
        mbar_init(q_full, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&k_empty[i], 1);
            mbar_init(&v_full[i], 1);
            mbar_init(&v_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&s_empty[i], NSW);
            mbar_init(&p_full[i], NSW);
            mbar_init(&p_empty[i], 1);
        }
        mbar_init(o_full, 1);
        fence_barrier_init();
        fence_async_shared();
    }
    if (warp == 2) tmem_alloc(tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t s_base = smem_u32(sm);

    if (warp == 0 && lane == 0) {
        // ===== TMA producer: Q once, then (K, V) per tile =====
        mbar_arrive_expect_tx(q_full, S::Q);
        for (int c = 0; c < HD / 64; ++c) tma_load_2d(&tm, q_full, sm + S::OFF_Q + c * BQ * 128, h * HD + c * 64, row0);
        int ks = 0, vs = 0;
        uint32_t kph = 0, vph = 0;
        for (int j = 0; j < nj; ++j) {
            const int krow = b * T + j * BKV;
            mbar_wait(&k_empty[ks], kph ^ 1);
            mbar_arrive_expect_tx(&k_full[ks], S::K);
            for (int c = 0; c < HD / 64; ++c)
                tma_load_2d(&tm, &k_full[ks], sm + S::OFF_K + ks * S::K + c * BKV * 128, d + kvh * HD + c * 64, krow);
            if (++ks == 2) { ks = 0; kph ^= 1; }
            mbar_wait(&v_empty[vs], vph ^ 1);
            mbar_arrive_expect_tx(&v_full[vs], S::V);
            for (int c = 0; c < HD / 64; ++c)
                tma_load_2d(&tm, &v_full[vs], sm + S::OFF_V + vs * S::V + c * BKV * 128, d + Hkv * HD + kvh * HD + c * 64,
                            krow);
            if (++vs == S::NVS) { vs = 0; vph ^= 1; }
        }
    } else if (warp == 1) {
        // ===== MMA issuer: S(0), then S(j+1) ahead of PV(j) =====
        const uint32_t idesc_s = make_idesc(1, 1, false, false, BQ, BKV);
        const uint32_t idesc_o = make_idesc(1, 1, false, true, BQ, HD);
        mbar_wait(q_full, 0);
        int ks = 0, vs = 0;
        uint32_t kph = 0, vph = 0;
        auto issue_s = [&](int j) {
            mbar_wait(&k_full[ks], kph);
            const int sb = j & 1;
            mbar_wait(&s_empty[sb], ((j >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t qa = s_base + S::OFF_Q, ka = s_base + S::OFF_K + ks * S::K;
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk)
                mma_bf16_ss(tmem + sb * BKV, kdesc(qa, kk, BQ * 128), kdesc(ka, kk, BKV * 128), idesc_s, kk > 0);
            tc_commit(&k_empty[ks]);
            tc_commit(&s_full[sb]);
            if (++ks == 2) { ks = 0; kph ^= 1; }
        };
        issue_s(0);
        for (int j = 0; j < nj; ++j) {
            if (j + 1 < nj) issue_s(j + 1);
            const int pb = S::NPB == 2 ? (j & 1) : 0;
            const uint32_t pph = S::NPB == 2 ? ((j >> 1) & 1) : (j & 1);
            mbar_wait(&p_full[pb], pph);
            mbar_wait(&v_full[vs], vph);
            tc_fence_after();
            const uint32_t va = s_base + S::OFF_V + vs * S::V;
            const uint32_t ph = s_base + S::OFF_PH + pb * 2 * S::P, pl = ph + S::P;
#pragma unroll
            for (int kk = 0; kk < BKV / 16; ++kk) {
                const uint64_t bd = mndesc(va, kk, BKV * 128);
                mma_bf16_ss(tmem + 256, kdesc(ph, kk, BQ * 128), bd, idesc_o, (j | kk) != 0);
                mma_bf16_ss(tmem + 256, kdesc(pl, kk, BQ * 128), bd, idesc_o, 1);
            }
            tc_commit(&v_empty[vs]);
            tc_commit(&p_empty[pb]);
            if (++vs == S::NVS) { vs = 0; vph ^= 1; }
        }
        tc_commit(o_full);
    } else if (warp >= 4) {
        // ===== softmax: thread = (query row, key half) =====
        const int wq = warp & 3, half = (warp - 4) >> 2;
        const int r = wq * 32 + lane;
        const int q = qt * BQ + r;
        const uint32_t lane_base = tmem + ((uint32_t)(wq * 32) << 16);
        const uint32_t o_cols = lane_base + 256 + half * (HD / 2);  // this thread's half of the O row
        const int c0 = half * (BKV / 2);
        const float a = inv_sqrt_d * LOG2E;
        constexpr float RESCALE = 8.0f;  // log2 headroom of p~ before O is rescaled
        float* xch = reinterpret_cast<float*>(sm + S::OFF_BAR + 256);  // [2][BQ] tile maxima, later l
        const int pair_bar = 2 + wq;  // named barrier of the two warps sharing these rows
        float m = -INFINITY, l = 0.0f;  // m: m_used in raw-score units; l: this half's sum of p~
        for (int j = 0; j < nj; ++j) {
            const int sb = j & 1;
            mbar_wait(&s_full[sb], (j >> 1) & 1);
            tc_fence_after();
            uint32_t rr[64];
            tmem_ld32(lane_base + sb * BKV + c0, *reinterpret_cast<uint32_t(*)[32]>(&rr[0]));
            tmem_ld32(lane_base + sb * BKV + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&rr[32]));
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[sb]);
            const bool diag = j == qt;
            const int kbase = j * BKV + c0;
            float mt = -INFINITY;
            if (diag) {
#pragma unroll
                for (int i = 0; i < 64; ++i)
                    if (kbase + i <= q) mt = fmaxf(mt, __uint_as_float(rr[i]));
            } else {
#pragma unroll
                for (int i = 0; i < 64; ++i) mt = fmaxf(mt, __uint_as_float(rr[i]));
            }
            xch[half * BQ + r] = mt;
            asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");
            mt = fmaxf(mt, xch[(half ^ 1) * BQ + r]);
            asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");  // xch reusable next tile
            const int pb = S::NPB == 2 ? (j & 1) : 0;
            const uint32_t pph = S::NPB == 2 ? ((j >> 1) & 1) : (j & 1);
            // P buffer pb free (PV(j - NPB) done)
            mbar_wait(&p_empty[pb], pph ^ 1);
            const bool grow = mt > m && (m == -INFINITY || (mt - m) * a > RESCALE);
            if (__any_sync(0xffffffffu, grow && m != -INFINITY)) {
                // O holds PV(0..j-1): wait for PV(j-1), then scale this thread's O columns
                if (j >= 1) {
                    const int pb1 = S::NPB == 2 ? ((j - 1) & 1) : 0;
                    const uint32_t ph1 = S::NPB == 2 ? (((j - 1) >> 1) & 1) : ((j - 1) & 1);
                    mbar_wait(&p_empty[pb1], ph1);
                }
                tc_fence_after();
                const float alpha = (grow && m != -INFINITY) ? ex2((m - mt) * a) : 1.0f;
#pragma unroll
                for (int c = 0; c < HD / 64; ++c) {
                    uint32_t ov[32];
                    tmem_ld32(o_cols + c * 32, ov);
                    tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
                    tmem_st32(o_cols + c * 32, ov);
                }
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                l *= alpha;
            }
            if (grow) m = mt;
            const float mb = m * a;
            uint8_t* ph = sm + S::OFF_PH + pb * 2 * S::P + half * BQ * 128;
            uint8_t* pl = ph + S::P;
            uint32_t hi[32], lo[32];
            float s4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
            for (int i = 0; i < 64; i += 2) {
                float pp[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const bool live = !diag || (kbase + i + e <= q);
                    pp[e] = live ? ex2(__fmaf_rn(__uint_as_float(rr[i + e]), a, -mb)) : 0.0f;
                }
                s4[(i >> 1) & 3] += pp[0] + pp[1];
                const float h0 = bf16r(pp[0]), h1 = bf16r(pp[1]);
                hi[i / 2] = pack_bf16x2(h0, h1);
                lo[i / 2] = pack_bf16x2(pp[0] - h0, pp[1] - h1);
            }
            l += (s4[0] + s4[1]) + (s4[2] + s4[3]);
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {
                const int off = r * 128 + ((cc ^ (r & 7)) << 4);
                *reinterpret_cast<uint4*>(ph + off) = make_uint4(hi[cc * 4 + 0], hi[cc * 4 + 1], hi[cc * 4 + 2], hi[cc * 4 + 3]);
                *reinterpret_cast<uint4*>(pl + off) = make_uint4(lo[cc * 4 + 0], lo[cc * 4 + 1], lo[cc * 4 + 2], lo[cc * 4 + 3]);
            }
            fence_async_shared();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[pb]);
        }
        // l of the whole row
        xch[half * BQ + r] = l;
        asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");
        const float lt = l + xch[(half ^ 1) * BQ + r];
        const float inv_l = lt > 0.0f ? 1.0f / lt : 0.0f;
        mbar_wait(o_full, 0);
        tc_fence_after();
        uint32_t mx = 0;
        const bool valid = q < T;
        const int64_t grow_ = (int64_t)b * T + q;
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
            const int col = half * (HD / 2) + c * 32;
            uint32_t rr[32];
            tmem_ld32(lane_base + 256 + col, rr);
            tmem_ld_wait();
            if (valid) {
                uint4* o16 = reinterpret_cast<uint4*>(out + grow_ * ldo + h * HD + col);
                float4* o32 = reinterpret_cast<float4*>(out32 + grow_ * ldo + h * HD + col);
#pragma unroll
                for (int v4 = 0; v4 < 4; ++v4) {
                    float f[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        f[e] = __uint_as_float(rr[v4 * 8 + e]) * inv_l;
                        mx = max(mx, abs_bits(bf16r(f[e])));
                    }
                    o16[v4] = make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                                         pack_bf16x2(f[6], f[7]));
                    if (out32) {
                        o32[2 * v4] = make_float4(f[0], f[1], f[2], f[3]);
                        o32[2 * v4 + 1] = make_float4(f[4], f[5], f[6], f[7]);
                    }
                }
            }
        }
        if (valid && half == 0) lse[((int64_t)b * H + h) * T + q] = m * inv_sqrt_d + logf(lt);
        mx = warp_max_u32(mx);
        if (lane == 0 && amax && mx) atomicMax(amax, mx);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}


// ===========================================================================
// Persistent one-pass forward: one CTA per SM walks the (q tile, head, batch)
// items longest-first (item i -> q tile nq-1-i/(H*B)), keeping TMEM, barriers
// and the K/V/S/P rings alive across items, so an item's prologue (Q load) and
// epilogue (O drain) overlap its neighbours' MMAs and softmax instead of being
// exposed once per CTA wave.  Extra barriers: q_empty (last S MMA of an item has
// read Q) and o_empty (the softmax warps have drained O).
// ===========================================================================
template <int HD>
__global__ void __launch_bounds__(NT, 1) fwd1p_tc_kernel(const __grid_constant__ CUtensorMap tm, int T, int H,
                                                         int Hkv, int B, float inv_sqrt_d, uint16_t* __restrict__ out,
                                                         int64_t ldo, float* __restrict__ out32, float* __restrict__ lse,
                                                         uint32_t* __restrict__ amax, int plo) {
    using S = Smem<HD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + S::OFF_BAR);
    uint64_t* q_full = bar + 0;
    uint64_t* k_full = bar + 1;    // [2]
    uint64_t* k_empty = bar + 3;   // [2]
    uint64_t* v_full = bar + 5;    // [2]
    uint64_t* v_empty = bar + 7;   // [2]
    uint64_t* s_full = bar + 9;    // [2]
    uint64_t* s_empty = bar + 11;  // [2]
    uint64_t* p_full = bar + 13;   // [2]
    uint64_t* p_empty = bar + 15;  // [2]
    uint64_t* o_full = bar + 17;
    uint64_t* q_empty = bar + 18;
    uint64_t* o_empty = bar + 19;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 20);

    const int nq = (T + BQ - 1) / BQ;
    const int items = nq * H * B;
    const int d = H * HD;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto decode = [&](int it, int& qt, int& h, int& b) {
        qt = nq - 1 - it / (H * B);
        const int r = it % (H * B);
        h = r % H;
        b = r / H;
    };

    if (warp == 0 && lane == 0) tma_prefetch(&tm);
    if (warp == 1 && lane == 0) {
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        mbar_init(o_full, 1);
        mbar_init(o_empty, NSW);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&k_empty[i], 1);
            mbar_init(&v_full[i], 1);
            mbar_init(&v_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&s_empty[i], NSW);
            mbar_init(&p_full[i], NSW);
            mbar_init(&p_empty[i], 1);
        }
        fence_barrier_init();
        fence_async_shared();
    }
    if (warp == 2) tmem_alloc(tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t s_base = smem_u32(sm);

    if (warp == 0 && lane == 0) {
        // ===== TMA producer =====
        int ks = 0, vs = 0;
        uint32_t kph = 0, vph = 0;
        int n_it = 0;
        for (int it = blockIdx.x; it < items; it += gridDim.x, ++n_it) {
            int qt, h, b;
            decode(it, qt, h, b);
            const int kvh = h / (H / Hkv);
            if (n_it > 0) mbar_wait(q_empty, (n_it - 1) & 1);  // previous item's S MMAs have read Q
            mbar_arrive_expect_tx(q_full, S::Q);
            for (int c = 0; c < HD / 64; ++c)
                tma_load_2d(&tm, q_full, sm + S::OFF_Q + c * BQ * 128, h * HD + c * 64, b * T + qt * BQ);
            for (int j = 0; j <= qt; ++j) {
                const int krow = b * T + j * BKV;
                mbar_wait(&k_empty[ks], kph ^ 1);
                mbar_arrive_expect_tx(&k_full[ks], S::K);
                for (int c = 0; c < HD / 64; ++c)
                    tma_load_2d(&tm, &k_full[ks], sm + S::OFF_K + ks * S::K + c * BKV * 128, d + kvh * HD + c * 64, krow);
                if (++ks == 2) { ks = 0; kph ^= 1; }
                mbar_wait(&v_empty[vs], vph ^ 1);
                mbar_arrive_expect_tx(&v_full[vs], S::V);
                for (int c = 0; c < HD / 64; ++c)
                    tma_load_2d(&tm, &v_full[vs], sm + S::OFF_V + vs * S::V + c * BKV * 128,
                                d + Hkv * HD + kvh * HD + c * 64, krow);
                if (++vs == S::NVS) { vs = 0; vph ^= 1; }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer =====
        const uint32_t idesc_s = make_idesc(1, 1, false, false, BQ, BKV);
        const uint32_t idesc_o = make_idesc(1, 1, false, true, BQ, HD);
        int ks = 0, vs = 0;
        uint32_t kph = 0, vph = 0;
        int sc = 0, pc = 0;  // S tiles / P tiles issued so far (all items)
        int n_it = 0;
        for (int it = blockIdx.x; it < items; it += gridDim.x, ++n_it) {
            int qt, h, b;
            decode(it, qt, h, b);
            const int nj = qt + 1;
            mbar_wait(q_full, n_it & 1);
            int s_issued = 0;
            auto issue_s = [&]() {
                mbar_wait(&k_full[ks], kph);
                const int sb = sc & 1;
                mbar_wait(&s_empty[sb], ((sc >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t qa = s_base + S::OFF_Q, ka = s_base + S::OFF_K + ks * S::K;
#pragma unroll
                for (int kk = 0; kk < HD / 16; ++kk)
                    mma_bf16_ss(tmem + sb * BKV, kdesc(qa, kk, BQ * 128), kdesc(ka, kk, BKV * 128), idesc_s, kk > 0);
                tc_commit(&k_empty[ks]);
                tc_commit(&s_full[sb]);
                if (++ks == 2) { ks = 0; kph ^= 1; }
                ++sc;
                if (++s_issued == nj) tc_commit(q_empty);  // Q no longer read by this item
            };
            issue_s();
            if (n_it > 0) mbar_wait(o_empty, (n_it - 1) & 1);  // previous item's O drained
            for (int j = 0; j < nj; ++j) {
                if (j + 1 < nj) issue_s();
                const int pb = S::NPB == 2 ? (pc & 1) : 0;
                const uint32_t pph = S::NPB == 2 ? ((pc >> 1) & 1) : (pc & 1);
                mbar_wait(&p_full[pb], pph);
                mbar_wait(&v_full[vs], vph);
                tc_fence_after();
                const uint32_t va = s_base + S::OFF_V + vs * S::V;
                const uint32_t ph = s_base + S::OFF_PH + pb * 2 * S::P, pl = ph + S::P;
#pragma unroll
                for (int kk = 0; kk < BKV / 16; ++kk) {
                    const uint64_t bd = mndesc(va, kk, BKV * 128);
                    mma_bf16_ss(tmem + 256, kdesc(ph, kk, BQ * 128), bd, idesc_o, (j | kk) != 0);
                    if (plo) mma_bf16_ss(tmem + 256, kdesc(pl, kk, BQ * 128), bd, idesc_o, 1);
                }
                tc_commit(&v_empty[vs]);
                tc_commit(&p_empty[pb]);
                if (++vs == S::NVS) { vs = 0; vph ^= 1; }
                ++pc;
            }
            tc_commit(o_full);
        }
    } else if (warp >= 4) {
        // ===== softmax (see fwd1_tc_kernel) =====
        const int wq = warp & 3, half = (warp - 4) >> 2;
        const int r = wq * 32 + lane;
        const uint32_t lane_base = tmem + ((uint32_t)(wq * 32) << 16);
        const uint32_t o_cols = lane_base + 256 + half * (HD / 2);
        const int c0 = half * (BKV / 2);
        const float a = inv_sqrt_d * LOG2E;
        constexpr float RESCALE = 8.0f;
        float* xch = reinterpret_cast<float*>(sm + S::OFF_BAR + 256);
        const int pair_bar = 2 + wq;
        int sc = 0, pc = 0;
        int n_it = 0;
        uint32_t mx = 0;
        for (int it = blockIdx.x; it < items; it += gridDim.x, ++n_it) {
            int qt, h, b;
            decode(it, qt, h, b);
            const int nj = qt + 1;
            const int q = qt * BQ + r;
            float m = -INFINITY, l = 0.0f;
            for (int j = 0; j < nj; ++j, ++sc, ++pc) {
                const int sb = sc & 1;
                mbar_wait(&s_full[sb], (sc >> 1) & 1);
                tc_fence_after();
                uint32_t rr[64];
                tmem_ld32(lane_base + sb * BKV + c0, *reinterpret_cast<uint32_t(*)[32]>(&rr[0]));
                tmem_ld32(lane_base + sb * BKV + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&rr[32]));
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s_empty[sb]);
                const bool diag = j == qt;
                const int kbase = j * BKV + c0;
                float mt = -INFINITY;
                if (diag) {
#pragma unroll
                    for (int i = 0; i < 64; ++i)
                        if (kbase + i <= q) mt = fmaxf(mt, __uint_as_float(rr[i]));
                } else {
#pragma unroll
                    for (int i = 0; i < 64; ++i) mt = fmaxf(mt, __uint_as_float(rr[i]));
                }
                xch[half * BQ + r] = mt;
                asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");
                mt = fmaxf(mt, xch[(half ^ 1) * BQ + r]);
                asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");
                const int pb = S::NPB == 2 ? (pc & 1) : 0;
                const uint32_t pph = S::NPB == 2 ? ((pc >> 1) & 1) : (pc & 1);
                mbar_wait(&p_empty[pb], pph ^ 1);
                const bool grow = mt > m && (m == -INFINITY || (mt - m) * a > RESCALE);
                if (__any_sync(0xffffffffu, grow && m != -INFINITY)) {
                    if (j >= 1) {  // O holds PV(..j-1) of this item: wait for PV(j-1)
                        const int pb1 = S::NPB == 2 ? ((pc - 1) & 1) : 0;
                        const uint32_t ph1 = S::NPB == 2 ? (((pc - 1) >> 1) & 1) : ((pc - 1) & 1);
                        mbar_wait(&p_empty[pb1], ph1);
                    }
                    tc_fence_after();
                    const float alpha = (grow && m != -INFINITY) ? ex2((m - mt) * a) : 1.0f;
#pragma unroll
                    for (int c = 0; c < HD / 64; ++c) {
                        uint32_t ov[32];
                        tmem_ld32(o_cols + c * 32, ov);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
                        tmem_st32(o_cols + c * 32, ov);
                    }
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                    l *= alpha;
                }
                if (grow) m = mt;
                const float mb = m * a;
                uint8_t* ph = sm + S::OFF_PH + pb * 2 * S::P + half * BQ * 128;
                uint8_t* pl = ph + S::P;
                uint32_t hi[32], lo[32];
                float s4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
                for (int i = 0; i < 64; i += 2) {
                    float pp[2];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const bool live = !diag || (kbase + i + e <= q);
                        pp[e] = live ? ex2(__fmaf_rn(__uint_as_float(rr[i + e]), a, -mb)) : 0.0f;
                    }
                    s4[(i >> 1) & 3] += pp[0] + pp[1];
                    const float h0 = bf16r(pp[0]), h1 = bf16r(pp[1]);
                    hi[i / 2] = pack_bf16x2(h0, h1);
                    if (plo) lo[i / 2] = pack_bf16x2(pp[0] - h0, pp[1] - h1);
                }
                l += (s4[0] + s4[1]) + (s4[2] + s4[3]);
#pragma unroll
                for (int cc = 0; cc < 8; ++cc) {
                    const int off = r * 128 + ((cc ^ (r & 7)) << 4);
                    *reinterpret_cast<uint4*>(ph + off) = make_uint4(hi[cc * 4 + 0], hi[cc * 4 + 1], hi[cc * 4 + 2], hi[cc * 4 + 3]);
                    if (plo)
                        *reinterpret_cast<uint4*>(pl + off) =
                            make_uint4(lo[cc * 4 + 0], lo[cc * 4 + 1], lo[cc * 4 + 2], lo[cc * 4 + 3]);
                }
                fence_async_shared();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&p_full[pb]);
            }
            xch[half * BQ + r] = l;
            asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");
            const float lt = l + xch[(half ^ 1) * BQ + r];
            asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");  // xch reusable by the next item
            const float inv_l = lt > 0.0f ? 1.0f / lt : 0.0f;
            mbar_wait(o_full, n_it & 1);
            tc_fence_after();
            const bool valid = q < T;
            const int64_t grow_ = (int64_t)b * T + q;
#pragma unroll
            for (int c = 0; c < HD / 64; ++c) {
                const int col = half * (HD / 2) + c * 32;
                uint32_t rr[32];
                tmem_ld32(lane_base + 256 + col, rr);
                tmem_ld_wait();
                if (valid) {
                    uint4* o16 = reinterpret_cast<uint4*>(out + grow_ * ldo + h * HD + col);
                    float4* o32 = reinterpret_cast<float4*>(out32 + grow_ * ldo + h * HD + col);
#pragma unroll
                    for (int v4 = 0; v4 < 4; ++v4) {
                        float f[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            f[e] = __uint_as_float(rr[v4 * 8 + e]) * inv_l;
                            mx = max(mx, abs_bits(bf16r(f[e])));
                        }
                        o16[v4] = make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                                             pack_bf16x2(f[6], f[7]));
                        if (out32) {
                            o32[2 * v4] = make_float4(f[0], f[1], f[2], f[3]);
                            o32[2 * v4 + 1] = make_float4(f[4], f[5], f[6], f[7]);
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(o_empty);  // O drained: the next item's PV(0) may overwrite it
            if (valid && half == 0) lse[((int64_t)b * H + h) * T + q] = m * inv_sqrt_d + logf(lt);
        }
        mx = warp_max_u32(mx);
        if (lane == 0 && amax && mx) atomicMax(amax, mx);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ===========================================================================
// Backward on tcgen05 (reference sdpa_chunked_backward, src/tensorops.cpp:257-303).
//
// Elementwise warps read S (and dP) rows from TMEM, compute
//   P = exp(x - LSE) ,  dS = P (dP - D) / sqrt(hd)
// and write P / dS back as bf16 hi + lo pairs into the TMEM columns they
// have just consumed; the following MMAs take that TMEM region as their A
// operand (kind::f16, A in TMEM).  Column map for one 32-wide chunk c of a
// thread's 64-column half: hi -> [c*32, c*32+16), lo -> [c*32+16, c*32+32)
// (16 bf16 pairs each), so no write ever lands on a column still to be read.
// ===========================================================================
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
// one 32-byte global store (sm_100 256-bit STG); p 32-byte aligned
__device__ __forceinline__ void st_global_v8(void* p, const uint32_t* v) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                 "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// A operand from TMEM
// TMEM column of the bf16 A operand for k-step kk (16 k values) of a 128-wide
// operand laid out by the chunk map above; part 0 = hi, 1 = lo
__device__ __forceinline__ uint32_t a_col(int kk, int part) {
    const int half = kk >> 2, c = (kk >> 1) & 1, sub = kk & 1;
    return (uint32_t)(half * 64 + c * 32 + part * 16 + sub * 8);
}
__device__ __forceinline__ uint32_t cvt_bf16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
// sm_100 paired f32 arithmetic (FFMA2 / FMUL2 / FADD2): each lane is the IEEE
// round-to-nearest scalar operation, so results are bit-identical to fma / mul / sub
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    float2 r;
    asm("{\n\t.reg .b64 a, b, c, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\tmov.b64 c, {%6, %7};\n\t"
        "fma.rn.f32x2 d, a, b, c;\n\tmov.b64 {%0, %1}, d;\n\t}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return r;
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    float2 r;
    asm("{\n\t.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
        "mul.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    float2 r;
    asm("{\n\t.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
        "sub.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}
// v -> bf16 hi + bf16 lo (v - hi), packed pairs; hi is v rounded to nearest
__device__ __forceinline__ void split32(const float (&v)[32], uint32_t (&hi)[16], uint32_t (&lo)[16]) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const uint32_t h = cvt_bf16x2(v[2 * i], v[2 * i + 1]);
        hi[i] = h;
        const float2 d = sub2(make_float2(v[2 * i], v[2 * i + 1]),
                              make_float2(__uint_as_float(h << 16), __uint_as_float(h & 0xffff0000u)));
        lo[i] = cvt_bf16x2(d.x, d.y);
    }
}
// v -> bf16 (round to nearest), packed pairs: the single-part operand of the bf16 P / dS mode
__device__ __forceinline__ void round32(const float (&v)[32], uint32_t (&hi)[16]) {
#pragma unroll
    for (int i = 0; i < 16; ++i) hi[i] = cvt_bf16x2(v[2 * i], v[2 * i + 1]);
}
__device__ __forceinline__ float4 lds4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts2(uint32_t a, float x, float y) {
    asm volatile("st.shared.f32 [%0], %1;\n\tst.shared.f32 [%0+128], %2;" ::"r"(a), "f"(x), "f"(y) : "memory");
}
// P^T / dS^T for 32 query columns of one key row.  sLD holds the columns'
// -LSE*log2e (or -inf past T) and D/sqrt(d); qrel = first column's query - key.
template <bool MASK>
__device__ __forceinline__ void dkdv_elem(const uint32_t (&rs)[32], const uint32_t (&rp)[32], uint32_t sLD,
                                          float c_s, float inv_sqrt_d, int qrel, float (&pv)[32], float (&dsv)[32]) {
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
        const float4 l4 = lds4(sLD + 4 * i);
        const float4 d4 = lds4(sLD + 128 + 4 * i);
        const float nl[4] = {l4.x, l4.y, l4.z, l4.w}, dd[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
        for (int u = 0; u < 4; u += 2) {
            const float2 e = fma2(make_float2(__uint_as_float(rs[i + u]), __uint_as_float(rs[i + u + 1])),
                                  make_float2(c_s, c_s), make_float2(nl[u], nl[u + 1]));
            float p0 = ex2(e.x), p1 = ex2(e.y);
            if (MASK) {
                p0 = qrel + i + u >= 0 ? p0 : 0.0f;
                p1 = qrel + i + u + 1 >= 0 ? p1 : 0.0f;
            }
            pv[i + u] = p0;
            pv[i + u + 1] = p1;
            const float2 dp = fma2(make_float2(__uint_as_float(rp[i + u]), __uint_as_float(rp[i + u + 1])),
                                   make_float2(inv_sqrt_d, inv_sqrt_d), make_float2(-dd[u], -dd[u + 1]));
            const float2 ds = mul2(make_float2(p0, p1), dp);
            dsv[i + u] = ds.x;
            dsv[i + u + 1] = ds.y;
        }
    }
}
// dS for 32 key columns of one query row; keys past `lim` (min(q, T-1)) masked
template <bool MASK>
__device__ __forceinline__ void dq_elem(const uint32_t (&rs)[32], const uint32_t (&rp)[32], float c_s, float nl,
                                        float inv_sqrt_d, float dsc, int k0, int lim, float (&dsv)[32]) {
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
        const float2 e = fma2(make_float2(__uint_as_float(rs[i]), __uint_as_float(rs[i + 1])), make_float2(c_s, c_s),
                              make_float2(nl, nl));
        float p0 = ex2(e.x), p1 = ex2(e.y);
        if (MASK) {
            p0 = k0 + i <= lim ? p0 : 0.0f;
            p1 = k0 + i + 1 <= lim ? p1 : 0.0f;
        }
        const float2 dp = fma2(make_float2(__uint_as_float(rp[i]), __uint_as_float(rp[i + 1])),
                               make_float2(inv_sqrt_d, inv_sqrt_d), make_float2(-dsc, -dsc));
        const float2 ds = mul2(make_float2(p0, p1), dp);
        dsv[i] = ds.x;
        dsv[i + 1] = ds.y;
    }
}

// Batched MMA issue.  The attention MMAs are short (M128 x N64 x K16 = 32 tensor
// cycles), and issuing each through its own elect / uniform-register conversion costs
// more than that, so the MMA warp became the critical path of the backward.  These
// issue a whole group from one elect with the per-k-step operand offsets added inside
// the asm (same MMAs, same order as the per-call loops they replace).
#define QTB_TS(D, A, B, ID, P) "@E tcgen05.mma.cta_group::1.kind::f16 [" D "], [" A "], " B ", " ID ", " P ";\n\t"
#define QTB_SS(D, A, B, ID, P) "@E tcgen05.mma.cta_group::1.kind::f16 [" D "], " A ", " B ", " ID ", " P ";\n\t"
// dV += P^T dO_sub (hi, lo) and dK += dS^T Q_sub (hi, lo) for the 4 k-steps of a 64-query
// sub-tile: A columns a_col(kk, part) of pb (P) / pb + 64 (dS), B = MN-major descriptors
// advancing 16 rows (2048 B) per k-step; acc: accumulate flag of the first k-step.
// operands: %0 dv, %1 dk, %2 pb, %3 bo, %4 bq, %5 idesc, %6 acc
#define QTB_G(DV_A, DK_A, B1, B2) \
    "add.u32 a, %2, " #DV_A ";\n\t" QTB_TS("%0", "a", B1, "%5", "T") \
    "add.u32 a, %2, " #DK_A ";\n\t" QTB_TS("%1", "a", B2, "%5", "T")
__device__ __forceinline__ void mma_g4_hilo(uint32_t dv, uint32_t dk, uint32_t pb, uint64_t bo, uint64_t bq,
                                            uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred E, p, T;\n\t.reg .b32 a;\n\t.reg .b64 o, q;\n\t"
        "elect.sync _|E, 0xffffffff;\n\tsetp.ne.b32 p, %6, 0;\n\tsetp.eq.b32 T, %6, %6;\n\t"
        QTB_TS("%0", "%2", "%3", "%5", "p")
        "add.u32 a, %2, 16;\n\t" QTB_TS("%0", "a", "%3", "%5", "T")
        "add.u32 a, %2, 64;\n\t" QTB_TS("%1", "a", "%4", "%5", "p")
        "add.u32 a, %2, 80;\n\t" QTB_TS("%1", "a", "%4", "%5", "T")
        "add.u64 o, %3, 128;\n\tadd.u64 q, %4, 128;\n\t"
        "add.u32 a, %2, 8;\n\t" QTB_TS("%0", "a", "o", "%5", "T")
        "add.u32 a, %2, 24;\n\t" QTB_TS("%0", "a", "o", "%5", "T")
        "add.u32 a, %2, 72;\n\t" QTB_TS("%1", "a", "q", "%5", "T")
        "add.u32 a, %2, 88;\n\t" QTB_TS("%1", "a", "q", "%5", "T")
        "add.u64 o, %3, 256;\n\tadd.u64 q, %4, 256;\n\t"
        "add.u32 a, %2, 32;\n\t" QTB_TS("%0", "a", "o", "%5", "T")
        "add.u32 a, %2, 48;\n\t" QTB_TS("%0", "a", "o", "%5", "T")
        "add.u32 a, %2, 96;\n\t" QTB_TS("%1", "a", "q", "%5", "T")
        "add.u32 a, %2, 112;\n\t" QTB_TS("%1", "a", "q", "%5", "T")
        "add.u64 o, %3, 384;\n\tadd.u64 q, %4, 384;\n\t"
        "add.u32 a, %2, 40;\n\t" QTB_TS("%0", "a", "o", "%5", "T")
        "add.u32 a, %2, 56;\n\t" QTB_TS("%0", "a", "o", "%5", "T")
        "add.u32 a, %2, 104;\n\t" QTB_TS("%1", "a", "q", "%5", "T")
        "add.u32 a, %2, 120;\n\t" QTB_TS("%1", "a", "q", "%5", "T")
        "}" ::"r"(dv), "r"(dk), "r"(pb), "l"(bo), "l"(bq), "r"(idesc), "r"(acc)
        : "memory");
}
#undef QTB_G
// dQ += dS K_sub (hi, lo) for the 4 k-steps of a 64-key sub-tile
// operands: %0 dq, %1 pb, %2 bk, %3 idesc, %4 acc
__device__ __forceinline__ void mma_dq4_hilo(uint32_t dq, uint32_t pb, uint64_t bk, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred E, p, T;\n\t.reg .b32 a;\n\t.reg .b64 q;\n\t"
        "elect.sync _|E, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 T, %4, %4;\n\t"
        QTB_TS("%0", "%1", "%2", "%3", "p")
        "add.u32 a, %1, 16;\n\t" QTB_TS("%0", "a", "%2", "%3", "T")
        "add.u64 q, %2, 128;\n\t"
        "add.u32 a, %1, 8;\n\t" QTB_TS("%0", "a", "q", "%3", "T")
        "add.u32 a, %1, 24;\n\t" QTB_TS("%0", "a", "q", "%3", "T")
        "add.u64 q, %2, 256;\n\t"
        "add.u32 a, %1, 32;\n\t" QTB_TS("%0", "a", "q", "%3", "T")
        "add.u32 a, %1, 48;\n\t" QTB_TS("%0", "a", "q", "%3", "T")
        "add.u64 q, %2, 384;\n\t"
        "add.u32 a, %1, 40;\n\t" QTB_TS("%0", "a", "q", "%3", "T")
        "add.u32 a, %1, 56;\n\t" QTB_TS("%0", "a", "q", "%3", "T")
        "}" ::"r"(dq), "r"(pb), "l"(bk), "r"(idesc), "r"(acc)
        : "memory");
}
// two SS products over HD/16 k-steps (S = X Y^T and dP = U W^T sharing the k loop): K-major
// SW128 descriptors advance 32 B (2 units) per k-step inside a 64-column atom, atom_stride >> 4
// (1024 units) across.  operands: %0 d0, %1 a0, %2 b0, %3 d1, %4 a1, %5 b1, %6 idesc
#define QTB_SS_STEP(OFF, P)                                                                      \
    "add.u64 x, %1, " #OFF ";\n\tadd.u64 y, %2, " #OFF ";\n\t" QTB_SS("%0", "x", "y", "%6", P) \
    "add.u64 x, %4, " #OFF ";\n\tadd.u64 y, %5, " #OFF ";\n\t" QTB_SS("%3", "x", "y", "%6", P)
template <int HD>
__device__ __forceinline__ void mma_ss2(uint32_t d0, uint64_t a0, uint64_t b0, uint32_t d1, uint64_t a1, uint64_t b1,
                                        uint32_t idesc) {
    static_assert(HD == 64 || HD == 128, "head dim");
    if constexpr (HD == 64) {
        asm volatile("{\n\t.reg .pred E, F, T;\n\t.reg .b64 x, y;\n\t"
                     "elect.sync _|E, 0xffffffff;\n\tsetp.ne.b32 F, %6, %6;\n\tsetp.eq.b32 T, %6, %6;\n\t"
                     QTB_SS_STEP(0, "F") QTB_SS_STEP(2, "T") QTB_SS_STEP(4, "T") QTB_SS_STEP(6, "T")
                     "}" ::"r"(d0), "l"(a0), "l"(b0), "r"(d1), "l"(a1), "l"(b1), "r"(idesc)
                     : "memory");
    } else {
        asm volatile("{\n\t.reg .pred E, F, T;\n\t.reg .b64 x, y;\n\t"
                     "elect.sync _|E, 0xffffffff;\n\tsetp.ne.b32 F, %6, %6;\n\tsetp.eq.b32 T, %6, %6;\n\t"
                     QTB_SS_STEP(0, "F") QTB_SS_STEP(2, "T") QTB_SS_STEP(4, "T") QTB_SS_STEP(6, "T")
                     QTB_SS_STEP(1024, "T") QTB_SS_STEP(1026, "T") QTB_SS_STEP(1028, "T") QTB_SS_STEP(1030, "T")
                     "}" ::"r"(d0), "l"(a0), "l"(b0), "r"(d1), "l"(a1), "l"(b1), "r"(idesc)
                     : "memory");
    }
}
#undef QTB_SS_STEP
// O += P V (hi, lo) over the 8 k-steps of a 128-key tile (forward PV, P from TMEM with the
// a_col chunk map).  operands: %0 o, %1 pa, %2 bv, %3 idesc, %4 acc
#define QTB_PV(OFF_HI, OFF_LO, BOFF)                                                          \
    "add.u64 q, %2, " #BOFF ";\n\t"                                                           \
    "add.u32 a, %1, " #OFF_HI ";\n\t" QTB_TS("%0", "a", "q", "%3", "T")                        \
    "add.u32 a, %1, " #OFF_LO ";\n\t" QTB_TS("%0", "a", "q", "%3", "T")
__device__ __forceinline__ void mma_pv8_hilo(uint32_t o, uint32_t pa, uint64_t bv, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred E, p, T;\n\t.reg .b32 a;\n\t.reg .b64 q;\n\t"
        "elect.sync _|E, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 T, %4, %4;\n\t"
        QTB_TS("%0", "%1", "%2", "%3", "p")
        "add.u32 a, %1, 16;\n\t" QTB_TS("%0", "a", "%2", "%3", "T")
        QTB_PV(8, 24, 128) QTB_PV(32, 48, 256) QTB_PV(40, 56, 384) QTB_PV(64, 80, 512) QTB_PV(72, 88, 640)
        QTB_PV(96, 112, 768) QTB_PV(104, 120, 896)
        "}" ::"r"(o), "r"(pa), "l"(bv), "r"(idesc), "r"(acc)
        : "memory");
}
#undef QTB_PV
// S = Q K^T over HD/16 k-steps (K-major SW128 descriptors, as mma_ss2).  %0 d, %1 a, %2 b, %3 idesc
#define QTB_S1(OFF, P) "add.u64 x, %1, " #OFF ";\n\tadd.u64 y, %2, " #OFF ";\n\t" QTB_SS("%0", "x", "y", "%3", P)
template <int HD>
__device__ __forceinline__ void mma_s1(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    if constexpr (HD == 64) {
        asm volatile("{\n\t.reg .pred E, F, T;\n\t.reg .b64 x, y;\n\t"
                     "elect.sync _|E, 0xffffffff;\n\tsetp.ne.b32 F, %3, %3;\n\tsetp.eq.b32 T, %3, %3;\n\t"
                     QTB_S1(0, "F") QTB_S1(2, "T") QTB_S1(4, "T") QTB_S1(6, "T")
                     "}" ::"r"(d), "l"(a), "l"(b), "r"(idesc)
                     : "memory");
    } else {
        asm volatile("{\n\t.reg .pred E, F, T;\n\t.reg .b64 x, y;\n\t"
                     "elect.sync _|E, 0xffffffff;\n\tsetp.ne.b32 F, %3, %3;\n\tsetp.eq.b32 T, %3, %3;\n\t"
                     QTB_S1(0, "F") QTB_S1(2, "T") QTB_S1(4, "T") QTB_S1(6, "T")
                     QTB_S1(1024, "T") QTB_S1(1026, "T") QTB_S1(1028, "T") QTB_S1(1030, "T")
                     "}" ::"r"(d), "l"(a), "l"(b), "r"(idesc)
                     : "memory");
    }
}
#undef QTB_S1

template <int HD>
struct BwdSmem {
    static constexpr int TILE = 128 * HD * 2;
    static constexpr int NST = HD == 64 ? 4 : 2;  // ring stages of (tile pair)
    static constexpr int QS = HD == 64 ? 2 : 1;   // dQ: Q/dO slots (next head's prefetch)
    static constexpr int OFF_A = 0;               // dK/dV: K tile | dQ: [QS] Q tiles
    static constexpr int OFF_B = QS * TILE;       // dK/dV: V tile | dQ: [QS] dO tiles
    static constexpr int OFF_R = 2 * QS * TILE;   // ring [NST] of (Q_i, dO_i) | (K_j, V_j)
    static constexpr int OFF_BAR = OFF_R + NST * 2 * TILE;
    static constexpr int OFF_LD = OFF_BAR + 512;   // [NSW][64] f32 per-warp LSE / D columns
    static constexpr int BYTES = OFF_LD + NSW * 64 * 4 + 1024;
};

// Backward work is cut into 64-wide sub-tiles (one half of a 128-row Q/dO or
// K/V tile).  Each sub-tile's S and dP (f32, 64 TMEM columns each) live in one
// of NB TMEM buffers, so the MMAs for sub-tile t+1 run while the elementwise
// warps turn sub-tile t into P / dS, and the gradient MMAs of t follow.
template <int HD>
struct BwdPipe {
    static constexpr int NB = (512 - 2 * HD) / 128;  // 3 for hd 64, 2 for hd 128
    static constexpr int ACC = NB * 128;             // accumulator columns
};

// dK / dV for one 128-key tile of one KV head: loops over every query head of
// the GQA group (ascending) and every query tile at or after the diagonal,
// accumulating in TMEM; rounded to bf16 once at the end.
// TMEM: buffers [b*128, +64) S^T -> P^T (hi|lo per 32), [b*128+64, +64) dP^T -> dS^T;
// dV at ACC, dK at ACC + HD.
template <int HD>
__global__ void __launch_bounds__(NT, 1) dkdv_tc_kernel(const __grid_constant__ CUtensorMap tq,
                                                        const __grid_constant__ CUtensorMap tdo, const float* __restrict__ lse,
                                                        const float* __restrict__ Dv, int T, int H, int Hkv,
                                                        int qkv_dim, float inv_sqrt_d, uint16_t* __restrict__ dqkv,
                                                        int plo) {
    using S = BwdSmem<HD>;
    using P = BwdPipe<HD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + S::OFF_BAR);
    uint64_t* kv_full = bar + 0;
    uint64_t* m_done = bar + 1;
    uint64_t* s_full = bar + 2;                   // [NB]
    uint64_t* p_full = bar + 2 + P::NB;           // [NB]
    uint64_t* b_free = bar + 2 + 2 * P::NB;       // [NB]
    uint64_t* r_full = bar + 2 + 3 * P::NB;       // [NST]
    uint64_t* r_empty = r_full + S::NST;          // [NST]
    uint32_t* tslot = reinterpret_cast<uint32_t*>(r_empty + S::NST);

    const int kt = blockIdx.z, kvh = blockIdx.x, b = blockIdx.y;  // tile slowest: longest CTAs first
    const int group = H / Hkv;
    const int d = H * HD;
    const int nq = (T + 127) / 128;
    const int per_head = nq - kt;  // query tiles kt .. nq-1
    const int niter = group * per_head;
    const int nsub = 2 * niter;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tq);
        tma_prefetch(&tdo);
    }
    if (warp == 1 && lane == 0) {
        mbar_init(kv_full, 1);
        mbar_init(m_done, 1);
        for (int i = 0; i < P::NB; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], NSW);
            mbar_init(&b_free[i], 1);
        }
        for (int i = 0; i < S::NST; ++i) {
            mbar_init(&r_full[i], 1);
            mbar_init(&r_empty[i], 1);
        }
        fence_barrier_init();
        fence_async_shared();
    }
    if (warp == 2) tmem_alloc(tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t s_base = smem_u32(sm);

    if (warp == 0 && lane == 0) {
        const int krow = b * T + kt * 128;
        mbar_arrive_expect_tx(kv_full, 2 * S::TILE);
        for (int c = 0; c < HD / 64; ++c) {
            tma_load_2d(&tq, kv_full, sm + S::OFF_A + c * 128 * 128, d + kvh * HD + c * 64, krow);
            tma_load_2d(&tq, kv_full, sm + S::OFF_B + c * 128 * 128, d + Hkv * HD + kvh * HD + c * 64, krow);
        }
        for (int it = 0; it < niter; ++it) {
            const int st = it % S::NST;
            const int h = kvh * group + it / per_head, qi = kt + it % per_head;
            mbar_wait(&r_empty[st], ((it / S::NST) & 1) ^ 1);
            mbar_arrive_expect_tx(&r_full[st], 2 * S::TILE);
            const int qrow = b * T + qi * 128;
            uint8_t* dst = sm + S::OFF_R + st * 2 * S::TILE;
            for (int c = 0; c < HD / 64; ++c) {
                tma_load_2d(&tq, &r_full[st], dst + c * 128 * 128, h * HD + c * 64, qrow);
                tma_load_2d(&tdo, &r_full[st], dst + S::TILE + c * 128 * 128, h * HD + c * 64, qrow);
            }
        }
    } else if (warp == 1) {  // MMA issuer: whole warp, elected lane issues
        const uint32_t idesc_s = make_idesc(1, 1, false, false, 128, 64);  // S^T, dP^T: keys x 64 queries
        const uint32_t idesc_g = make_idesc(1, 1, false, true, 128, HD);   // dV, dK: A TMEM, B MN-major
        const uint32_t ka = s_base + S::OFF_A, va = s_base + S::OFF_B;
        mbar_wait(kv_full, 0);
        auto issue_s = [&](int t) {
            const int it = t >> 1, sub = t & 1, st = it % S::NST, buf = t % P::NB;
            if (sub == 0) mbar_wait(&r_full[st], (it / S::NST) & 1);
            if (t >= P::NB) mbar_wait(&b_free[buf], ((t - P::NB) / P::NB) & 1);
            tc_fence_after();
            const uint32_t qa = s_base + S::OFF_R + st * 2 * S::TILE + sub * 64 * 128, oa = qa + S::TILE;
            mma_ss2<HD>(tmem + buf * 128, kdesc(ka, 0, 128 * 128), kdesc(qa, 0, 128 * 128), tmem + buf * 128 + 64,
                        kdesc(va, 0, 128 * 128), kdesc(oa, 0, 128 * 128), idesc_s);
            tc_commit(&s_full[buf]);
        };
        issue_s(0);
        for (int t = 0; t < nsub; ++t) {
            if (t + 1 < nsub) issue_s(t + 1);
            const int it = t >> 1, sub = t & 1, st = it % S::NST, buf = t % P::NB;
            mbar_wait(&p_full[buf], (t / P::NB) & 1);
            tc_fence_after();
            const uint32_t qa = s_base + S::OFF_R + st * 2 * S::TILE, oa = qa + S::TILE;
            const uint32_t pb = tmem + buf * 128;
            if (plo) {
                mma_g4_hilo(tmem + P::ACC, tmem + P::ACC + HD, pb, mndesc(oa, 4 * sub, 128 * 128),
                            mndesc(qa, 4 * sub, 128 * 128), idesc_g, t != 0);
            } else {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint64_t bo = mndesc(oa, kk + 4 * sub, 128 * 128), bq = mndesc(qa, kk + 4 * sub, 128 * 128);
                    const uint32_t acc = (t | kk) != 0;
                    mma_bf16_ts(tmem + P::ACC, pb + a_col(kk, 0), bo, idesc_g, acc);
                    mma_bf16_ts(tmem + P::ACC + HD, pb + 64 + a_col(kk, 0), bq, idesc_g, acc);
                }
            }
            tc_commit(&b_free[buf]);
            if (sub == 1) tc_commit(&r_empty[st]);
        }
        tc_commit(m_done);
    } else if (warp >= 4) {
        const int wq = warp & 3, half = (warp - 4) >> 2;
        const int r = wq * 32 + lane;
        const int kv = kt * 128 + r;  // key position
        const uint32_t lb = tmem + ((uint32_t)(wq * 32) << 16);
        const float c_s = inv_sqrt_d * LOG2E;
        const uint32_t sLD = s_base + S::OFF_LD + (warp - 4) * 256;
        // raw LSE / D of this warp's 32 query columns of a sub-tile, one per lane;
        // loaded a sub-tile ahead, scaled when stored to shared memory
        int nh = 0, nqi = 0, nsb = 0;  // (head, query tile, sub) of the next sub-tile to load
        float Ln = 0.0f, Dn = 0.0f;
        bool vn = false;
        auto load_ld = [&]() {
            const int ql = (kt + nqi) * 128 + nsb * 64 + half * 32 + lane;
            const int64_t o = ((int64_t)b * H + kvh * group + nh) * T + ql;
            vn = ql < T;
            if (vn) {
                Ln = __ldg(lse + o);
                Dn = __ldg(Dv + o);
            }
            if (++nsb == 2) {
                nsb = 0;
                if (++nqi == per_head) {
                    nqi = 0;
                    ++nh;
                }
            }
        };
        load_ld();
        int buf = 0, ph = 0, qi = kt, sub = 0;
        for (int t = 0; t < nsub; ++t) {
            const int q0 = qi * 128 + sub * 64 + half * 32;
            __syncwarp();
            sts2(sLD + 4 * lane, vn ? -Ln * LOG2E : -INFINITY, vn ? Dn * inv_sqrt_d : 0.0f);
            if (t + 1 < nsub) load_ld();  // consumed next sub-tile: latency hidden
            __syncwarp();
            mbar_wait(&s_full[buf], ph);
            tc_fence_after();
            const uint32_t col = buf * 128 + half * 32;
            uint32_t rs[32], rp[32];
            tmem_ld32(lb + col, rs);
            tmem_ld32(lb + col + 64, rp);
            tmem_ld_wait();
            float pv[32], dsv[32];
            if (q0 >= kt * 128 + 127)  // whole warp above the diagonal
                dkdv_elem<false>(rs, rp, sLD, c_s, inv_sqrt_d, 0, pv, dsv);
            else
                dkdv_elem<true>(rs, rp, sLD, c_s, inv_sqrt_d, q0 - kv, pv, dsv);
            uint32_t hi[16], lo[16];
            if (plo) {
                split32(pv, hi, lo);
                tmem_st16(lb + col, hi);
                tmem_st16(lb + col + 16, lo);
                split32(dsv, hi, lo);
                tmem_st16(lb + col + 64, hi);
                tmem_st16(lb + col + 64 + 16, lo);
            } else {
                round32(pv, hi);
                tmem_st16(lb + col, hi);
                round32(dsv, hi);
                tmem_st16(lb + col + 64, hi);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[buf]);
            if (++buf == P::NB) {
                buf = 0;
                ph ^= 1;
            }
            if (++sub == 2) {
                sub = 0;
                if (++qi == kt + per_head) qi = kt;
            }
        }
        // dV, dK rows (bf16, rounded once): this thread writes HD/2 columns of each
        mbar_wait(m_done, 0);
        tc_fence_after();
        const int64_t grow = (int64_t)b * T + kv;
#pragma unroll
        for (int which = 0; which < 2; ++which) {  // 0 = dV, 1 = dK
#pragma unroll
            for (int c = 0; c < HD / 64; ++c) {
                const int col = half * (HD / 2) + c * 32;
                uint32_t rr[32];
                tmem_ld32(lb + P::ACC + which * HD + col, rr);
                tmem_ld_wait();
                if (kv >= T) continue;
                uint16_t* dst = dqkv + grow * qkv_dim + d + (which ? 0 : Hkv * HD) + kvh * HD + col;
                uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
                for (int v4 = 0; v4 < 4; ++v4)
                    d4[v4] = make_uint4(pack_bf16x2(__uint_as_float(rr[v4 * 8 + 0]), __uint_as_float(rr[v4 * 8 + 1])),
                                        pack_bf16x2(__uint_as_float(rr[v4 * 8 + 2]), __uint_as_float(rr[v4 * 8 + 3])),
                                        pack_bf16x2(__uint_as_float(rr[v4 * 8 + 4]), __uint_as_float(rr[v4 * 8 + 5])),
                                        pack_bf16x2(__uint_as_float(rr[v4 * 8 + 6]), __uint_as_float(rr[v4 * 8 + 7])));
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// dQ for one 128-query tile of every query head of one KV group: items
// (head hh, key tile j <= qt), each two 64-key sub-tiles; the (K_j, V_j) tiles
// stream through a ring, Q/dO of the current head sit in QS slots.  dQ
// accumulates in TMEM over the keys and is written (bf16) per head.
// TMEM: buffers [b*128, +64) S -> dS (hi|lo per 32), [b*128+64, +64) dP; dQ at ACC.
template <int HD>
__global__ void __launch_bounds__(NT, 1) dq_tc_kernel(const __grid_constant__ CUtensorMap tq,
                                                      const __grid_constant__ CUtensorMap tdo, const float* __restrict__ lse,
                                                      const float* __restrict__ Dv, int T, int H, int Hkv, int qkv_dim,
                                                      float inv_sqrt_d, uint16_t* __restrict__ dqkv, int plo) {
    using S = BwdSmem<HD>;
    using P = BwdPipe<HD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + S::OFF_BAR);
    uint64_t* dq_done = bar + 0;
    uint64_t* dq_free = bar + 1;              // epilogue read dQ of the previous head
    uint64_t* qo_full = bar + 2;              // [2]
    uint64_t* qo_empty = bar + 4;             // [2]
    uint64_t* s_full = bar + 6;               // [NB]
    uint64_t* p_full = s_full + P::NB;        // [NB]
    uint64_t* b_free = p_full + P::NB;        // [NB]
    uint64_t* r_full = b_free + P::NB;        // [NST]
    uint64_t* r_empty = r_full + S::NST;      // [NST]
    uint32_t* tslot = reinterpret_cast<uint32_t*>(r_empty + S::NST);

    const int qt = gridDim.z - 1 - blockIdx.z, b = blockIdx.y;  // longest CTAs first
    // blockIdx.x = (kv head, slice of its GQA group): the group's query heads may be
    // split over gridDim.x / Hkv CTAs (dQ of a head needs no cross-head reduction)
    const int hsplit = gridDim.x / Hkv;
    const int kvh = blockIdx.x / hsplit;
    const int group = (H / Hkv) / hsplit;  // query heads handled by this CTA
    const int hbase = kvh * (H / Hkv) + (blockIdx.x % hsplit) * group;
    const int d = H * HD;
    const int per_head = qt + 1;
    const int niter = group * per_head;
    const int nsub = 2 * niter;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tq);
        tma_prefetch(&tdo);
    }
    if (warp == 1 && lane == 0) {
        mbar_init(dq_done, 1);
        mbar_init(dq_free, NSW);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&qo_full[i], 1);
            mbar_init(&qo_empty[i], 1);
        }
        for (int i = 0; i < P::NB; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], NSW);
            mbar_init(&b_free[i], 1);
        }
        for (int i = 0; i < S::NST; ++i) {
            mbar_init(&r_full[i], 1);
            mbar_init(&r_empty[i], 1);
        }
        fence_barrier_init();
        fence_async_shared();
    }
    if (warp == 2) tmem_alloc(tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t s_base = smem_u32(sm);

    if (warp == 0 && lane == 0) {
        const int qrow = b * T + qt * 128;
        for (int it = 0; it < niter; ++it) {
            const int hh = it / per_head, j = it % per_head;
            if (j == 0) {  // this head's Q / dO
                const int slot = hh % S::QS;
                mbar_wait(&qo_empty[slot], ((hh / S::QS) & 1) ^ 1);
                mbar_arrive_expect_tx(&qo_full[slot], 2 * S::TILE);
                const int h = hbase + hh;
                for (int c = 0; c < HD / 64; ++c) {
                    tma_load_2d(&tq, &qo_full[slot], sm + S::OFF_A + slot * S::TILE + c * 128 * 128, h * HD + c * 64, qrow);
                    tma_load_2d(&tdo, &qo_full[slot], sm + S::OFF_B + slot * S::TILE + c * 128 * 128, h * HD + c * 64,
                                qrow);
                }
            }
            const int st = it % S::NST;
            mbar_wait(&r_empty[st], ((it / S::NST) & 1) ^ 1);
            mbar_arrive_expect_tx(&r_full[st], 2 * S::TILE);
            const int krow = b * T + j * 128;
            uint8_t* dst = sm + S::OFF_R + st * 2 * S::TILE;
            for (int c = 0; c < HD / 64; ++c) {
                tma_load_2d(&tq, &r_full[st], dst + c * 128 * 128, d + kvh * HD + c * 64, krow);
                tma_load_2d(&tq, &r_full[st], dst + S::TILE + c * 128 * 128, d + Hkv * HD + kvh * HD + c * 64, krow);
            }
        }
    } else if (warp == 1) {  // MMA issuer: whole warp, elected lane issues
        const uint32_t idesc_s = make_idesc(1, 1, false, false, 128, 64);  // S, dP: queries x 64 keys
        const uint32_t idesc_g = make_idesc(1, 1, false, true, 128, HD);   // dQ: A TMEM, B = K MN-major
        auto issue_s = [&](int t) {
            const int it = t >> 1, sub = t & 1, st = it % S::NST, buf = t % P::NB;
            const int hh = it / per_head, j = it % per_head, slot = hh % S::QS;
            if (sub == 0) {
                if (j == 0) mbar_wait(&qo_full[slot], (hh / S::QS) & 1);
                mbar_wait(&r_full[st], (it / S::NST) & 1);
            }
            if (t >= P::NB) mbar_wait(&b_free[buf], ((t - P::NB) / P::NB) & 1);
            tc_fence_after();
            const uint32_t qa = s_base + S::OFF_A + slot * S::TILE, oa = s_base + S::OFF_B + slot * S::TILE;
            const uint32_t ka = s_base + S::OFF_R + st * 2 * S::TILE + sub * 64 * 128, va = ka + S::TILE;
            mma_ss2<HD>(tmem + buf * 128, kdesc(qa, 0, 128 * 128), kdesc(ka, 0, 128 * 128), tmem + buf * 128 + 64,
                        kdesc(oa, 0, 128 * 128), kdesc(va, 0, 128 * 128), idesc_s);
            tc_commit(&s_full[buf]);
            if (sub == 1 && j == per_head - 1) tc_commit(&qo_empty[slot]);  // last use of this head's Q/dO
        };
        issue_s(0);
        for (int t = 0; t < nsub; ++t) {
            if (t + 1 < nsub) issue_s(t + 1);
            const int it = t >> 1, sub = t & 1, st = it % S::NST, buf = t % P::NB;
            const int hh = it / per_head, j = it % per_head;
            if (j == 0 && sub == 0 && hh > 0) mbar_wait(dq_free, (hh - 1) & 1);  // previous head's dQ read out
            mbar_wait(&p_full[buf], (t / P::NB) & 1);
            tc_fence_after();
            const uint32_t ka = s_base + S::OFF_R + st * 2 * S::TILE;
            const uint32_t pb = tmem + buf * 128;
            if (plo) {
                mma_dq4_hilo(tmem + P::ACC, pb, mndesc(ka, 4 * sub, 128 * 128), idesc_g, (j | sub) != 0);
            } else {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    mma_bf16_ts(tmem + P::ACC, pb + a_col(kk, 0), mndesc(ka, kk + 4 * sub, 128 * 128), idesc_g,
                                (j | sub | kk) != 0);
            }
            tc_commit(&b_free[buf]);
            if (sub == 1) {
                tc_commit(&r_empty[st]);
                if (j == per_head - 1) tc_commit(dq_done);
            }
        }
    } else if (warp >= 4) {
        const int wq = warp & 3, half = (warp - 4) >> 2;
        const int r = wq * 32 + lane;
        const int q = qt * 128 + r;
        const uint32_t lb = tmem + ((uint32_t)(wq * 32) << 16);
        const bool qok = q < T;
        const float c_s = inv_sqrt_d * LOG2E;
        const int64_t grow = (int64_t)b * T + q;
        int t = 0;
        // the row's LSE / D of the next head are loaded one head ahead (their latency otherwise
        // stalls every head switch)
        float Ln = 0.0f, Dn = 0.0f;
        if (qok) {
            Ln = lse[((int64_t)b * H + hbase) * T + q];
            Dn = Dv[((int64_t)b * H + hbase) * T + q];
        }
        for (int hh = 0; hh < group; ++hh) {
            const int h = hbase + hh;
            const float Lq = Ln, Dq = Dn;
            if (qok && hh + 1 < group) {
                Ln = lse[((int64_t)b * H + h + 1) * T + q];
                Dn = Dv[((int64_t)b * H + h + 1) * T + q];
            }
            const float nl = -Lq * LOG2E, dsc = Dq * inv_sqrt_d;
            for (int js = 0; js < 2 * per_head; ++js, ++t) {
                const int buf = t % P::NB;
                mbar_wait(&s_full[buf], (t / P::NB) & 1);
                tc_fence_after();
                const int k0 = js * 64 + half * 32;
                const uint32_t col = buf * 128 + half * 32;
                uint32_t rs[32], rp[32];
                tmem_ld32(lb + col, rs);
                tmem_ld32(lb + col + 64, rp);
                tmem_ld_wait();
                float dsv[32];
                if (k0 + 31 <= qt * 128 + wq * 32 && k0 + 31 < T)  // whole warp below the diagonal
                    dq_elem<false>(rs, rp, c_s, nl, inv_sqrt_d, dsc, k0, 0, dsv);
                else
                    dq_elem<true>(rs, rp, c_s, nl, inv_sqrt_d, dsc, k0, qok ? q : -1, dsv);
                uint32_t hi[16], lo[16];
                if (plo) {
                    split32(dsv, hi, lo);
                    tmem_st16(lb + col, hi);
                    tmem_st16(lb + col + 16, lo);
                } else {
                    round32(dsv, hi);
                    tmem_st16(lb + col, hi);
                }
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&p_full[buf]);
            }
            // this head's dQ: wait for its last MMA, read out, release the TMEM columns
            mbar_wait(dq_done, hh & 1);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < HD / 64; ++c) {
                const int col = half * (HD / 2) + c * 32;
                uint32_t rr[32];
                tmem_ld32(lb + P::ACC + col, rr);
                tmem_ld_wait();
                if (!qok) continue;
                uint4* d4 = reinterpret_cast<uint4*>(dqkv + grow * qkv_dim + h * HD + col);
#pragma unroll
                for (int v4 = 0; v4 < 4; ++v4)
                    d4[v4] = make_uint4(pack_bf16x2(__uint_as_float(rr[v4 * 8 + 0]), __uint_as_float(rr[v4 * 8 + 1])),
                                        pack_bf16x2(__uint_as_float(rr[v4 * 8 + 2]), __uint_as_float(rr[v4 * 8 + 3])),
                                        pack_bf16x2(__uint_as_float(rr[v4 * 8 + 4]), __uint_as_float(rr[v4 * 8 + 5])),
                                        pack_bf16x2(__uint_as_float(rr[v4 * 8 + 6]), __uint_as_float(rr[v4 * 8 + 7])));
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(dq_free);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}


// ===========================================================================
// Forward, two Q tiles per CTA (ping-pong).  A CTA owns the adjacent query tiles
// (2p, 2p+1) of one (head, batch) -- they share every K/V tile but the last --
// and two softmax warpgroups, one per tile, each thread owning a whole row
// (no cross-warp max/sum exchange).  S_X = Q_X K_j^T lands in TMEM; the
// softmax of tile X overwrites its S columns with P (bf16 hi + lo, the
// backward's chunk map) and the MMA warp accumulates O_X += P_X V_j with P as
// the TMEM A operand -- no shared-memory round trip for P.  While one tile's
// softmax runs, the tensor core works on the other tile's S / PV, which is
// what the one-tile kernel cannot do (its softmax and MMAs serialise).
// TMEM: S_A [0,128), S_B [128,256), O_A [256,256+HD), O_B [256+HD,256+2HD).
// Same arithmetic as fwd1p_tc_kernel (online max moved only when it grows by
// > 2^RESCALE, O rescaled in TMEM then, O / l at the end).
// ===========================================================================
template <int HD>
struct Smem2Q {
    static constexpr int Q = BQ * HD * 2;
    static constexpr int K = BKV * HD * 2;
    static constexpr int V = BKV * HD * 2;
    static constexpr int OFF_Q = 0;             // tile A at 0, tile B at Q
    static constexpr int OFF_K = 2 * Q;         // 2 stages
    static constexpr int OFF_V = OFF_K + 2 * K;  // 2 stages
    static constexpr int OFF_BAR = OFF_V + 2 * V;
    static constexpr int BYTES = OFF_BAR + 512 + 1024;
};

template <int HD>
__global__ void __launch_bounds__(NT, 1) fwd2q_tc_kernel(const __grid_constant__ CUtensorMap tm, int T, int H,
                                                         int Hkv, int B, float inv_sqrt_d, uint16_t* __restrict__ out,
                                                         int64_t ldo, float* __restrict__ out32, float* __restrict__ lse,
                                                         uint32_t* __restrict__ amax, int plo, int v8) {
    using S = Smem2Q<HD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + S::OFF_BAR);
    uint64_t* q_full = bar + 0;
    uint64_t* q_empty = bar + 1;
    uint64_t* k_full = bar + 2;    // [2]
    uint64_t* k_empty = bar + 4;   // [2]
    uint64_t* v_full = bar + 6;    // [2]
    uint64_t* v_empty = bar + 8;   // [2]
    uint64_t* s_full = bar + 10;   // [tile]
    uint64_t* p_full = bar + 12;   // [tile]
    uint64_t* pv_done = bar + 14;  // [tile]
    uint64_t* o_full = bar + 16;   // [tile]
    uint64_t* o_empty = bar + 18;  // [tile]
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 20);

    const int nq = (T + BQ - 1) / BQ;
    const int npair = (nq + 1) / 2;
    const int items = npair * H * B;
    const int d = H * HD;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // longest pairs first: pair p = npair-1 .. 0, dealt to the CTAs in snake order
    // (round k runs CTA 0..G-1 when even, G-1..0 when odd) so no CTA collects the
    // longest item of every round
    auto snake = [&](int k) {
        return k * (int)gridDim.x + ((k & 1) ? (int)gridDim.x - 1 - (int)blockIdx.x : (int)blockIdx.x);
    };
    auto decode = [&](int it, int& pr, int& h, int& b) {
        pr = npair - 1 - it / (H * B);
        const int r = it % (H * B);
        h = r % H;
        b = r / H;
    };

    if (warp == 0 && lane == 0) tma_prefetch(&tm);
    if (warp == 1 && lane == 0) {
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&k_empty[i], 1);
            mbar_init(&v_full[i], 1);
            mbar_init(&v_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 4);
            mbar_init(&pv_done[i], 1);
            mbar_init(&o_full[i], 1);
            mbar_init(&o_empty[i], 4);
        }
        fence_barrier_init();
        fence_async_shared();
    }
    if (warp == 2) tmem_alloc(tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t s_base = smem_u32(sm);

    if (warp < 4) setmaxnreg_dec<96>();  // producer / MMA / idle warpgroup
    if (warp == 0 && lane == 0) {
        // ===== TMA producer: Q_A (+ Q_B), then the K/V tiles the pair needs =====
        int ks = 0, vs = 0;
        uint32_t kph = 0, vph = 0;
        int n_it = 0;
        for (int k = 0;; ++k, ++n_it) {
            const int it = snake(k);
            if (it >= items) break;
            int pr, h, b;
            decode(it, pr, h, b);
            const int qa = 2 * pr, qb = 2 * pr + 1;
            const bool hasb = qb < nq;
            const int nj = hasb ? qb + 1 : qa + 1;
            const int kvh = h / (H / Hkv);
            if (n_it > 0) mbar_wait(q_empty, (n_it - 1) & 1);
            mbar_arrive_expect_tx(q_full, (hasb ? 2 : 1) * S::Q);
            for (int c = 0; c < HD / 64; ++c) {
                tma_load_2d(&tm, q_full, sm + S::OFF_Q + c * BQ * 128, h * HD + c * 64, b * T + qa * BQ);
                if (hasb) tma_load_2d(&tm, q_full, sm + S::OFF_Q + S::Q + c * BQ * 128, h * HD + c * 64, b * T + qb * BQ);
            }
            for (int j = 0; j < nj; ++j) {
                const int krow = b * T + j * BKV;
                mbar_wait(&k_empty[ks], kph ^ 1);
                mbar_arrive_expect_tx(&k_full[ks], S::K);
                for (int c = 0; c < HD / 64; ++c)
                    tma_load_2d(&tm, &k_full[ks], sm + S::OFF_K + ks * S::K + c * BKV * 128, d + kvh * HD + c * 64, krow);
                if (++ks == 2) { ks = 0; kph ^= 1; }
                mbar_wait(&v_empty[vs], vph ^ 1);
                mbar_arrive_expect_tx(&v_full[vs], S::V);
                for (int c = 0; c < HD / 64; ++c)
                    tma_load_2d(&tm, &v_full[vs], sm + S::OFF_V + vs * S::V + c * BKV * 128,
                                d + Hkv * HD + kvh * HD + c * 64, krow);
                if (++vs == 2) { vs = 0; vph ^= 1; }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer (one elected thread): PV_A(j), S_A(j+1), PV_B(j), S_B(j+1), ... so the
        // tensor core works on one tile while the other tile's softmax runs =====
        const uint32_t idesc_s = make_idesc(1, 1, false, false, BQ, BKV);
        const uint32_t idesc_o = make_idesc(1, 1, false, true, BQ, HD);
        int ks = 0, vs = 0;
        uint32_t kph = 0, vph = 0;
        uint32_t pcnt[2] = {0, 0}, pvcnt[2] = {0, 0}, ocnt[2] = {0, 0};
        int n_it = 0;
        for (int k = 0;; ++k, ++n_it) {
            const int it = snake(k);
            if (it >= items) break;
            int pr, h, b;
            decode(it, pr, h, b);
            const int qa = 2 * pr, qb = 2 * pr + 1;
            const bool hasb = qb < nq;
            const int nx[2] = {qa + 1, hasb ? qb + 1 : 0};
            const int nj = hasb ? qb + 1 : qa + 1;
            const int last = hasb ? 1 : 0;  // the tile whose range is longest: last user of each K tile
            const int s_total = nx[0] + nx[1];
            int s_issued = 0;
            mbar_wait(q_full, n_it & 1);
            auto s_mma = [&](int x) {
                const uint32_t ka = s_base + S::OFF_K + ks * S::K;
                const uint32_t qa_ = s_base + S::OFF_Q + x * S::Q;
                mma_s1<HD>(tmem + x * 128, kdesc(qa_, 0, BQ * 128), kdesc(ka, 0, BKV * 128), idesc_s);
                tc_commit(&s_full[x]);
                if (++s_issued == s_total) tc_commit(q_empty);  // Q no longer read by this item
            };
            auto k_release = [&]() {
                tc_commit(&k_empty[ks]);
                if (++ks == 2) { ks = 0; kph ^= 1; }
            };
            // S(0) of both tiles
            mbar_wait(&k_full[ks], kph);
            tc_fence_after();
            for (int x = 0; x <= last; ++x) s_mma(x);
            k_release();
            bool k_ready = false;  // K(j+1) waited for
            for (int j = 0; j < nj; ++j) {
                mbar_wait(&v_full[vs], vph);
                const uint32_t va = s_base + S::OFF_V + vs * S::V;
                k_ready = false;
#pragma unroll
                for (int x = 0; x < 2; ++x) {
                    if (j >= nx[x]) continue;
                    mbar_wait(&p_full[x], pcnt[x] & 1);
                    ++pcnt[x];
                    if (j == 0 && ocnt[x] > 0) mbar_wait(&o_empty[x], (ocnt[x] - 1) & 1);  // O_X drained
                    tc_fence_after();
                    const uint32_t pa = tmem + x * 128;
                    const uint32_t od = tmem + 256 + x * HD;
                    if (plo) {
                        mma_pv8_hilo(od, pa, mndesc(va, 0, BKV * 128), idesc_o, j != 0);
                    } else {
#pragma unroll
                        for (int kk = 0; kk < BKV / 16; ++kk)
                            mma_bf16_ts(od, pa + a_col(kk, 0), mndesc(va, kk, BKV * 128), idesc_o, (j | kk) != 0);
                    }
                    tc_commit(&pv_done[x]);
                    ++pvcnt[x];
                    if (j == nx[x] - 1) {
                        tc_commit(&o_full[x]);
                        ++ocnt[x];
                    }
                    if (x == last) tc_commit(&v_empty[vs]);  // V(j) read by both tiles' PV
                    if (j + 1 < nx[x]) {
                        // S_X(j+1) overwrites the columns PV_X(j) reads as P: wait for it first
                        if (!k_ready) {
                            mbar_wait(&k_full[ks], kph);
                            k_ready = true;
                        }
                        mbar_wait(&pv_done[x], (pvcnt[x] - 1) & 1);
                        tc_fence_after();
                        s_mma(x);
                        if (x == last) k_release();
                    }
                }
                if (++vs == 2) { vs = 0; vph ^= 1; }
            }
        }
    } else if (warp >= 4) {
        // ===== softmax: warpgroup x = (warp - 4) / 4 owns tile x; thread = query row =====
        // 200 registers (the producer warpgroup gave its surplus back): the row's 128 scores
        // come out of TMEM in one round trip and stay in registers for the max and exp passes
        setmaxnreg_inc<200>();
        const int x = (warp - 4) >> 2, wq = warp & 3;
        const int r = wq * 32 + lane;
        const uint32_t lane_base = tmem + ((uint32_t)(wq * 32) << 16);
        const uint32_t s_cols = lane_base + x * 128;
        const uint32_t o_cols = lane_base + 256 + x * HD;
        const float a = inv_sqrt_d * LOG2E;
        constexpr float RESCALE = 8.0f;
        uint32_t scnt = 0, ocnt = 0;
        uint32_t mx = 0;
        for (int k = 0;; ++k) {
            const int it = snake(k);
            if (it >= items) break;
            int pr, h, b;
            decode(it, pr, h, b);
            const int qt = 2 * pr + x;
            if (qt >= nq) continue;  // pair without a second tile
            const int nj = qt + 1;
            const int q = qt * BQ + r;
            // l per key half, summed as fwd1p_tc_kernel's two half-row threads do (bitwise equal)
            float m = -INFINITY, l0 = 0.0f, l1 = 0.0f;
            for (int j = 0; j < nj; ++j, ++scnt) {
                mbar_wait(&s_full[x], scnt & 1);
                tc_fence_after();
                uint32_t rr[4][32];
#pragma unroll
                for (int c = 0; c < 4; ++c) tmem_ld32(s_cols + c * 32, rr[c]);
                tmem_ld_wait();
                if (j == qt) {
                    // causal diagonal tile: keys past the row's query become -inf (max unaffected,
                    // exp2 -> +0, exactly the masked value of the one-tile kernel)
                    const int lim = q - j * BKV;
#pragma unroll
                    for (int c = 0; c < 4; ++c)
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (c * 32 + i > lim) rr[c][i] = 0xff800000u;
                }
                // pass 1: the row max over the tile's 128 keys
                float mt = -INFINITY;
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int i = 0; i < 32; ++i) mt = fmaxf(mt, __uint_as_float(rr[c][i]));
                const bool grow = mt > m && (m == -INFINITY || (mt - m) * a > RESCALE);
                if (__any_sync(0xffffffffu, grow && m != -INFINITY)) {
                    // O_X holds PV(..j-1): complete, since the MMA warp waited for it before S(j)
                    const float alpha = (grow && m != -INFINITY) ? ex2((m - mt) * a) : 1.0f;
#pragma unroll 1
                    for (int c = 0; c < HD / 32; ++c) {
                        uint32_t ov[32];
                        tmem_ld32(o_cols + c * 32, ov);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
                        tmem_st32(o_cols + c * 32, ov);
                    }
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                    l0 *= alpha;
                    l1 *= alpha;
                }
                if (grow) m = mt;
                const float nmb = -(m * a);
                // pass 2: p = exp2(x a - m a), written over the chunk as bf16 hi (+ lo)
                float s4[2][4] = {{0.0f, 0.0f, 0.0f, 0.0f}, {0.0f, 0.0f, 0.0f, 0.0f}};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    float pv[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) pv[i] = ex2(__fmaf_rn(__uint_as_float(rr[c][i]), a, nmb));
                    const int hh = c >> 1;
#pragma unroll
                    for (int i = 0; i < 32; i += 2) {
                        const int il = (c & 1) * 32 + i;  // index within the 64-key half
                        s4[hh][(il >> 1) & 3] += pv[i] + pv[i + 1];
                    }
                    uint32_t hi[16], lo[16];
                    if (plo) {
                        split32(pv, hi, lo);
                        tmem_st16(s_cols + c * 32, hi);
                        tmem_st16(s_cols + c * 32 + 16, lo);
                    } else {
                        round32(pv, hi);
                        tmem_st16(s_cols + c * 32, hi);
                    }
                }
                l0 += (s4[0][0] + s4[0][1]) + (s4[0][2] + s4[0][3]);
                l1 += (s4[1][0] + s4[1][1]) + (s4[1][2] + s4[1][3]);
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&p_full[x]);
            }
            const float l = l0 + l1;
            const float inv_l = l > 0.0f ? 1.0f / l : 0.0f;
            mbar_wait(&o_full[x], ocnt & 1);
            ++ocnt;
            tc_fence_after();
            const bool valid = q < T;
            const int64_t grow_ = (int64_t)b * T + q;
            // O_X leaves TMEM in one round trip; the MMA warp may refill it while we store
            uint32_t ro[HD / 32][32];
#pragma unroll
            for (int c = 0; c < HD / 32; ++c) tmem_ld32(o_cols + c * 32, ro[c]);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&o_empty[x]);
            if (valid) {
#pragma unroll
                for (int c = 0; c < HD / 32; ++c) {
                    float f[32];
                    uint32_t pk[16];
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        f[e] = __uint_as_float(ro[c][e]) * inv_l;
                        mx = max(mx, abs_bits(bf16r(f[e])));
                    }
#pragma unroll
                    for (int e = 0; e < 16; ++e) pk[e] = pack_bf16x2(f[2 * e], f[2 * e + 1]);
                    uint16_t* o16 = out + grow_ * ldo + h * HD + c * 32;
                    float* o32 = out32 ? out32 + grow_ * ldo + h * HD + c * 32 : nullptr;
                    if (v8) {  // 32-byte stores: whole sectors per thread-row
                        st_global_v8(o16, pk);
                        st_global_v8(o16 + 16, pk + 8);
                        if (o32)
#pragma unroll
                            for (int v = 0; v < 4; ++v) st_global_v8(o32 + 8 * v, reinterpret_cast<const uint32_t*>(f) + 8 * v);
                    } else {
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            reinterpret_cast<uint4*>(o16)[v] =
                                make_uint4(pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]);
                            if (o32) {
                                reinterpret_cast<float4*>(o32)[2 * v] =
                                    make_float4(f[8 * v], f[8 * v + 1], f[8 * v + 2], f[8 * v + 3]);
                                reinterpret_cast<float4*>(o32)[2 * v + 1] =
                                    make_float4(f[8 * v + 4], f[8 * v + 5], f[8 * v + 6], f[8 * v + 7]);
                            }
                        }
                    }
                }
            }
            if (valid) lse[((int64_t)b * H + h) * T + q] = m * inv_sqrt_d + logf(l);
        }
        mx = warp_max_u32(mx);
        if (lane == 0 && amax && mx) atomicMax(amax, mx);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

}  // namespace attn_tc
}  // namespace qtb

namespace qtb {
namespace gemm {
int make_tmap(CUtensorMap* m, const void* ptr, int elem, uint64_t inner, uint64_t outer, uint64_t row_stride_elems,
              uint32_t box_inner, uint32_t box_outer);
}
}  // namespace qtb

using namespace qtb;

extern "C" int qtk_attn_fwd_tc(const void* qkv, int B, int T, int H, int Hkv, int hd, int qkv_dim, void* out,
                               int64_t ldo, float* out32, float* lse, uint32_t* amax, cudaStream_t s) {
    using namespace qtb::attn_tc;
    if (H % Hkv || (hd != 64 && hd != 128) || (qkv_dim % 8) || (ldo % 8)) return 1;
    CUtensorMap tm;
    int rc = qtb::gemm::make_tmap(&tm, qkv, 2, (uint64_t)qkv_dim, (uint64_t)B * T, (uint64_t)qkv_dim, 64, 128);
    if (rc) return rc;
    const float inv_sqrt_d = 1.0f / sqrtf((float)hd);
    dim3 grid((unsigned)ceil_div(T, BQ), H, B);
    static int two_pass = -1;
    if (two_pass < 0) {
        const char* e = getenv("QTB_ATTN_FWD2");
        two_pass = e ? atoi(e) : 0;  // 1: the two-pass (normalise-first) kernel
    }
#define QTB_FWD(KERNEL, HDV)                                                                                      \
    {                                                                                                            \
        const int smem = Smem<HDV>::BYTES;                                                                       \
        cudaFuncSetAttribute(KERNEL<HDV>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);                    \
        KERNEL<HDV><<<grid, NT, smem, s>>>(tm, T, H, Hkv, inv_sqrt_d, (uint16_t*)out, ldo, out32, lse, amax);   \
    }
    static int persistent = -1;
    if (persistent < 0) {
        const char* e = getenv("QTB_ATTN_PERSIST");
        persistent = e ? atoi(e) : 1;
    }
    if (fwd2q_mode() && !two_pass) {  // two Q tiles per CTA, ping-pong softmax / MMA
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int items = (int)ceil_div(ceil_div(T, BQ), 2) * H * B;
        const unsigned pg = (unsigned)std::min(items, sms);
        const int v8 = ((((uintptr_t)out) | ((uintptr_t)out32)) & 31) == 0 && ldo % 16 == 0;
#define QTB_FWD2Q(HDV)                                                                                           \
        {                                                                                                          \
            const int smem = Smem2Q<HDV>::BYTES;                                                                   \
            cudaFuncSetAttribute(fwd2q_tc_kernel<HDV>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);         \
            fwd2q_tc_kernel<HDV><<<pg, NT, smem, s>>>(tm, T, H, Hkv, B, inv_sqrt_d, (uint16_t*)out, ldo, out32, lse, \
                                                      amax, p_lo_mode(), v8);                                      \
        }
        if (hd == 64) QTB_FWD2Q(64) else QTB_FWD2Q(128)
#undef QTB_FWD2Q
        return (int)cudaGetLastError();
    }
    if (persistent && !two_pass) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int items = (int)ceil_div(T, BQ) * H * B;
        const unsigned pg = (unsigned)std::min(items, sms);
#define QTB_FWDP(HDV)                                                                                            \
        {                                                                                                          \
            const int smem = Smem<HDV>::BYTES;                                                                     \
            cudaFuncSetAttribute(fwd1p_tc_kernel<HDV>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);         \
            fwd1p_tc_kernel<HDV><<<pg, NT, smem, s>>>(tm, T, H, Hkv, B, inv_sqrt_d, (uint16_t*)out, ldo, out32, lse, \
                                                      amax, p_lo_mode());                                          \
        }
        if (hd == 64) QTB_FWDP(64) else QTB_FWDP(128)
#undef QTB_FWDP
        return (int)cudaGetLastError();
    }
    if (hd == 64) {
        if (two_pass) QTB_FWD(fwd_tc_kernel, 64) else QTB_FWD(fwd1_tc_kernel, 64)
    } else {
        if (two_pass) QTB_FWD(fwd_tc_kernel, 128) else QTB_FWD(fwd1_tc_kernel, 128)
    }
#undef QTB_FWD
    return (int)cudaGetLastError();
}

namespace qtb {
namespace attn {
void launch_bwd_dot(const uint16_t* dout, const float* o, int64_t ld, int T, int H, int hd, int64_t rows, float* D,
                    cudaStream_t s);
}  // namespace attn
}  // namespace qtb

// s2 (optional): the dQ kernel runs there, concurrently with dK/dV (they write disjoint
// columns of dqkv); s waits for it before returning
extern "C" int qtk_attn_bwd_tc2(const void* qkv, const float* out32, const void* dout, int64_t ldo, const float* lse,
                                float* Dv, int B, int T, int H, int Hkv, int hd, int qkv_dim, void* dqkv, float* ws,
                                cudaStream_t s, cudaStream_t s2);
extern "C" int qtk_attn_bwd_tc(const void* qkv, const float* out32, const void* dout, int64_t ldo, const float* lse,
                               float* Dv, int B, int T, int H, int Hkv, int hd, int qkv_dim, void* dqkv, float* ws,
                               cudaStream_t s) {
    return qtk_attn_bwd_tc2(qkv, out32, dout, ldo, lse, Dv, B, T, H, Hkv, hd, qkv_dim, dqkv, ws, s, nullptr);
}
extern "C" int qtk_attn_bwd_tc2(const void* qkv, const float* out32, const void* dout, int64_t ldo, const float* lse,
                                float* Dv, int B, int T, int H, int Hkv, int hd, int qkv_dim, void* dqkv, float* ws,
                                cudaStream_t s, cudaStream_t s2) {
    using namespace qtb::attn_tc;
    if (H % Hkv || (hd != 64 && hd != 128) || (qkv_dim % 8) || (ldo % 8)) return 1;
    (void)ws;  // dK/dV accumulate over the GQA group in TMEM: no partials

    const int64_t rows = (int64_t)B * T;
    qtb::attn::launch_bwd_dot((const uint16_t*)dout, out32, ldo, T, H, hd, rows, Dv, s);
    CUtensorMap tq, tdo;
    int rc = qtb::gemm::make_tmap(&tq, qkv, 2, (uint64_t)qkv_dim, (uint64_t)rows, (uint64_t)qkv_dim, 64, 128);
    if (rc) return rc;
    rc = qtb::gemm::make_tmap(&tdo, dout, 2, (uint64_t)ldo, (uint64_t)rows, (uint64_t)ldo, 64, 128);
    if (rc) return rc;
    const float inv_sqrt_d = 1.0f / sqrtf((float)hd);
    dim3 grid(Hkv, B, (unsigned)ceil_div(T, 128));
    static int dq_split = -1;
    if (dq_split < 0) {
        const char* e = getenv("QTB_DQ_SPLIT");
        dq_split = e ? atoi(e) : 0;  // per-head dQ CTAs measured slower (lost K/V tile reuse across the group)
    }
    dim3 gdq(dq_split ? H : Hkv, B, (unsigned)ceil_div(T, 128));  // dQ: one query head per CTA
#define QTB_BWD_TC(HD)                                                                                               \
    {                                                                                                              \
        const int smem = BwdSmem<HD>::BYTES;                                                                       \
        cudaFuncSetAttribute(dkdv_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);               \
        cudaFuncSetAttribute(dq_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);                 \
        cudaStream_t sq = s;                                                                                       \
        if (s2 && s2 != s) {                                                                                       \
            cudaEventRecord(fork_ev(), s);                                                                         \
            cudaStreamWaitEvent(s2, fork_ev(), 0);                                                                 \
            sq = s2;                                                                                               \
        }                                                                                                          \
        dq_tc_kernel<HD><<<gdq, NT, smem, sq>>>(tq, tdo, lse, Dv, T, H, Hkv, qkv_dim, inv_sqrt_d, (uint16_t*)dqkv,   \
                                               p_lo_mode());                                                      \
        dkdv_tc_kernel<HD><<<grid, NT, smem, s>>>(tq, tdo, lse, Dv, T, H, Hkv, qkv_dim, inv_sqrt_d, (uint16_t*)dqkv, \
                                                  p_lo_mode());                                                   \
        if (sq != s) {                                                                                             \
            cudaEventRecord(join_ev(), sq);                                                                        \
            cudaStreamWaitEvent(s, join_ev(), 0);                                                                  \
        }                                                                                                          \
    }
    if (hd == 64)
        QTB_BWD_TC(64)
    else
        QTB_BWD_TC(128)
#undef QTB_BWD_TC
    return (int)cudaGetLastError();
}

extern "C" void qtk_attn_set_plo(int plo) { qtb::attn_tc::g_plo = plo; }
extern "C" void qtk_attn_set_fwd2q(int on) { qtb::attn_tc::g_fwd2q = on; }
