/* qtrain-b200 C ABI — the drop-in boundary for LLMQ's FP8 training step.
 *
 * Everything below is plain C: device pointers, sizes, a cudaStream_t, and an
 * int status (0 ok; 1 invalid_argument; 2 out_of_range; 3 runtime_error; other
 * values are CUDA / driver error codes).  No torch types cross this boundary.
 * Element types: bf16 tensors are passed as uint16_t bit patterns, FP8 codes
 * as uint8_t, absmax slots as the uint32_t bit pattern of a non-negative f32.
 *
 * Two layers:
 *   qtk_*  stateless kernels on caller-owned device memory; each names the
 *          reference primitive it replaces (file:line under
 *          /root/reference/proj).
 *   qt_*   a device-resident training session that owns parameters,
 *          gradients, optimizer state and activations, mirroring the
 *          reference's operator API (include/qtrain/model.hpp,
 *          include/qtrain/optim.hpp).
 */
#ifndef QTRAIN_B200_H
#define QTRAIN_B200_H

#include <cuda_runtime.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------------- */
/* numerics: absmax + FP8 cast                                                */
/* ------------------------------------------------------------------------- */

/* FP8 kinds: 0 = E4M3 (OCP FN), 1 = E5M2 (include/qtrain/numerics.hpp:23). */

/* atomicMax of |x| bits into *amax_bits (caller zeroes it first).  NaN is
 * sticky (reference absmax_or_nan, src/model.cpp:133-140; absmax,
 * src/numerics.cpp:141-148 throws on it, see qt_session error reporting). */
int qtk_absmax_bf16(const void* x, int64_t n, uint32_t* amax_bits, cudaStream_t s);
int qtk_absmax_f32(const float* x, int64_t n, uint32_t* amax_bits, cudaStream_t s);

/* codes[i] = encode(clamp(x[i] * scale)), scale = absmax_scale(amax, kind)
 * written to *scale_out (may be NULL).  Replaces quantize_with_absmax,
 * src/numerics.cpp:160-176. */
int qtk_quantize_bf16(const void* x, int64_t n, int kind, const uint32_t* amax_bits, uint8_t* codes,
                      float* scale_out, cudaStream_t s);

/* x (rows, cols) -> codes_t (cols, rows), and optionally the row-major codes
 * in the same pass.  Replaces transpose_quantize_with_absmax,
 * src/tensorops.cpp:164-182. */
int qtk_quantize_transpose_bf16(const void* x, int64_t rows, int64_t cols, int kind, const uint32_t* amax_bits,
                                uint8_t* codes_t, uint8_t* codes_rm, float* scale_out, cudaStream_t s);

/* ------------------------------------------------------------------------- */
/* GEMM (tcgen05): D[m,n] = sum_k A[m,k] B[n,k]                               */
/* Replaces matmul_tn (src/tensorops.cpp:24-59) and, through the layout      */
/* flags, the transposes in linear_dinput/linear_dweight (src/model.cpp:151-167). */
/* ------------------------------------------------------------------------- */
enum {
    EPI_BF16 = 0,     /* out bf16 = bf16(acc / (sa*sb))                                  */
    EPI_F32 = 1,      /* out f32 = acc                                                   */
    EPI_BF16_RES = 2, /* out bf16 = bf16(bf16(acc/(sa*sb)) + res)                        */
    EPI_BF16_ACC = 3, /* out (bf16 grad buffer) = SR(out + bf16(acc/(sa*sb)))            */
    EPI_F32_ACC = 4   /* out (bf16 grad buffer) = SR(out + acc)                          */
};

typedef struct QtkGemm {
    int kind;           /* 0 = FP8 (kind::f8f6f4), 1 = BF16 (kind::f16)                    */
    int a_fmt, b_fmt;   /* FP8 kinds of A and B (0 E4M3, 1 E5M2); ignored for BF16         */
    int a_mn, b_mn;     /* 0: operand stored [rows][ld] (K contiguous); 1: stored [K][ld]  */
    int64_t M, N, K;
    const void* a;
    int64_t lda;        /* row stride of A's storage, in elements                          */
    const void* b;
    int64_t ldb;
    const float* a_scale; /* device f32 scales (NULL = 1)                                  */
    const float* b_scale;
    int epi;
    void* out;
    int64_t ldo;
    const void* res;    /* EPI_BF16_RES residual (bf16)                                    */
    int64_t ldr;
    uint64_t sr_seed, sr_stream, sr_base; /* EPI_*_ACC stochastic-rounding key           */
    int bn;             /* N tile: 128 or 256 (0 = auto)                                   */
} QtkGemm;

int qtk_gemm(const QtkGemm* g, cudaStream_t s);

#ifdef __cplusplus
}
#endif

#endif /* QTRAIN_B200_H */
