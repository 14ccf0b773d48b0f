/* TEST INFRASTRUCTURE ONLY -- the CPU restatement (plain C) of the LLMQ
 * training-step arithmetic used as the parity checker by tests/, smoke() and
 * bench.py's cpu_baseline leg.  Never linked into libqtrain_b200.so.
 *
 * Every function restates the reference routine named beside it (paths under
 * /root/reference/proj).  Tensors are flat f32 arrays holding values on the
 * bf16 grid where the reference does; FP8 tensors are uint8 codes plus one
 * f32 scale.  All reductions run in the reference's sequential order, so the
 * restatement is bit-identical to the reference compiled with the same libm
 * (checked against oracle/_ref and the golden vectors in tests/).
 */
#ifndef QTRAIN_ORACLE_H
#define QTRAIN_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* numerics (src/numerics.cpp) */
float qto_f8_decode(uint8_t code, int kind);
uint8_t qto_f8_encode(float x, int kind);
float qto_f8_fmax(int kind);
int qto_absmax(const float* x, int64_t n, float* out);                /* -1 on NaN (throws in the reference) */
float qto_absmax_scale(float amax, int kind);
void qto_quantize_with_absmax(const float* x, int64_t n, int kind, float amax, uint8_t* codes, float* scale);
void qto_transpose_quantize_with_absmax(const float* x, int64_t rows, int64_t cols, int kind, float amax,
                                        uint8_t* codes_t, float* scale);
uint64_t qto_fnv1a64(const char* s);
uint32_t qto_rng_uniform(uint64_t seed, uint64_t stream, uint64_t counter);
float qto_rng_uniform_float(uint64_t seed, uint64_t stream, uint64_t counter);
float qto_rng_normal(uint64_t seed, uint64_t stream, uint64_t counter);
float qto_bf16_round(float x);
float qto_sr_bf16(float x, uint64_t seed, uint64_t stream, uint64_t counter);

/* tensorops (src/tensorops.cpp) */
void qto_matmul_fp8(const uint8_t* a, int64_t M, int64_t K, int akind, float ascale, const uint8_t* b, int64_t N,
                    int bkind, float bscale, int round_bf16, float* out);
void qto_matmul_f32(const float* a, int64_t M, int64_t K, const float* b, int64_t N, int round_bf16, float* out);
void qto_rmsnorm_fwd(const float* x, const float* res, const float* gamma, int64_t rows, int64_t d, float eps,
                     float* nr_out, float* normed, float* absmax);
void qto_rmsnorm_bwd(const float* nr, const float* gamma, int64_t rows, int64_t d, float eps, const float* dy,
                     const float* d_extra, float* d_in, float* d_gamma);
void qto_swiglu_fwd(const float* gu, int64_t rows, int64_t two_h, float* h, float* absmax);
void qto_swiglu_bwd(const float* gu, int64_t rows, int64_t two_h, const float* dh, float* dgu);
void qto_sdpa_fwd(const float* q, const float* k, const float* v, int64_t H, int64_t Hkv, int64_t T, int64_t D,
                  float* out);
void qto_sdpa_bwd(const float* q, const float* k, const float* v, const float* go, int64_t H, int64_t Hkv, int64_t T,
                  int64_t D, float* dq, float* dk, float* dv);
int qto_embedding_backward(const int32_t* ids, int64_t n, const float* grad_out, int64_t d, int64_t vocab,
                           float* out);
int qto_cross_entropy(const float* hidden, int64_t N, int64_t d, const float* lm_w, int64_t V, const int32_t* targets,
                      int with_grads, float* loss, float* d_hidden, float* d_lm_w);

/* optimizer / accumulation (src/optim.cpp, src/model.cpp) */
int qto_adamw_range(const char* name, float* p, float* m, float* v, const float* g, int64_t numel, int64_t lo,
                    int64_t hi, float lr, float b1, float b2, float eps, float wd, int bf16_moments, int bf16_params,
                    uint64_t seed, int64_t step, float grad_scale);
double qto_grad_norm_partials(const float* g, int64_t lo, int64_t hi);
void qto_grad_accumulate(const char* name, float* buf, const float* g, int64_t n, int f32_mode, uint64_t seed,
                         uint64_t micro_step);
void qto_init_normal(float* t, int64_t n, float std, uint64_t seed, const char* name);
void qto_shard_layout(int64_t numel, int workers, int64_t* padded, int64_t* per_worker);

#ifdef __cplusplus
}
#endif
#endif
