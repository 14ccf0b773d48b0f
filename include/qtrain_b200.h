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
    EPI_F32_ACC = 4,  /* out (bf16 grad buffer) = SR(out + acc)                          */
    EPI_SWIGLU_BWD = 5 /* acc = dh (bf16(acc/(sa*sb))); res = gate|up (M x 2N bf16);      */
                       /* out (M x 2N) = swiglu_backward(gate|up, dh) (tensorops.cpp:133-153) */
                       /* + absmax of out into amax                                        */
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
    const void* a2;     /* optional split-A operand (same layout/ld as A): D = A.B + A2.B, */
                        /* used for f32-precision operands carried as bf16 hi + lo pairs    */
    void* ws;           /* optional split-K workspace (f32); NULL = no split               */
    int64_t ws_bytes;
    int split_k;        /* 0 = auto (only when the tile grid starves the SMs), 1 = off     */
    uint32_t* amax;     /* EPI_SWIGLU_BWD: absmax (u32 |x| bits) of the output              */
    /* EPI_F32 logits only (all three set or all NULL): per-row softmax statistics of   */
    /* each 128-column block, (max, sum exp(x - max)) as float pairs [M][ceil(N/128)], */
    /* and the logit at column ce_targets[row] -> ce_tgt_logit[row]                     */
    const int32_t* ce_targets;
    float* ce_stats;
    float* ce_tgt_logit;
    /* EPI_*_ACC: when non-NULL, the SR counter base is read on the device as           */
    /* (*sr_micro_step) * M * N instead of sr_base (CUDA-graph replay of the step)       */
    const uint64_t* sr_micro_step;
} QtkGemm;

int qtk_gemm(const QtkGemm* g, cudaStream_t s);
/* workspace bytes the automatic split-K would use for this shape (0 = no split) */
int qtk_gemm_splitk_ws_bytes(int64_t M, int64_t N, int64_t K, int kind);

/* ------------------------------------------------------------------------- */
/* fused block ops (src/tensorops.cpp, src/model.cpp)                          */
/* ------------------------------------------------------------------------- */

/* embedding gather + (inputs, targets) split of B*(T+1) token ids
 * (src/model.cpp:316-331); *err = 2 on an out-of-range id. */
int qtk_embed_fwd(const int32_t* tokens, int B, int T, const void* embed, int d, int64_t V, void* r, int32_t* inputs,
                  int32_t* targets, int* err, cudaStream_t s);

/* rmsnorm_residual_fused (src/tensorops.cpp:61-86): nr = x ? bf16(x+res) : res;
 * normed = bf16((nr*inv)*gamma); absmax(normed) -> *amax (may be NULL).
 * Sequential per-row f32 sum of squares == the reference bitwise. */
int qtk_rmsnorm_fwd(const void* x, const void* res, const void* gamma, int64_t rows, int d, float eps, void* nr_out,
                    void* normed, float* inv_out, uint32_t* amax, cudaStream_t s);

/* rmsnorm_residual_backward (src/tensorops.cpp:88-112).  dgamma_part needs
 * qtk_rmsnorm_bwd_partials(rows, d) x d floats; dgamma (d floats) is their
 * fixed-order column sum. */
int qtk_rmsnorm_bwd_partials(int64_t rows, int d);
int qtk_rmsnorm_bwd(const void* nr, const void* gamma, int64_t rows, int d, float eps, const void* dy,
                    const void* d_extra, void* d_in, float* dgamma_part, float* dgamma, uint32_t* amax,
                    cudaStream_t s);

/* rope_apply (src/model.cpp:171-191) in place over the first n_rot_heads heads
 * of each (rows, qkv_dim) row; cs_tab = T x hd/2 float2 {cos, sin} built on the
 * host with the reference's powf/cosf/sinf.  amax (optional) covers the whole
 * row (d_qkv quantization). */
int qtk_rope(void* qkv, int64_t rows, int T, int n_rot_heads, int hd, int qkv_dim, const void* cs_tab, int backward,
             uint32_t* amax, cudaStream_t s);

/* swiglu_fused / swiglu_backward (src/tensorops.cpp:114-153) + fused absmax. */
int qtk_swiglu_fwd(const void* gu, int64_t rows, int H, void* h, uint32_t* amax, cudaStream_t s);
int qtk_swiglu_bwd(const void* gu, const void* dh, int64_t rows, int H, void* dgu, uint32_t* amax, cudaStream_t s);
/* Test infrastructure: counts[0..2] = mismatches of the SwiGLU kernels' fast
 * x/(1+e) and 1/(1+e) against div.rn / rcp.rn over all 65536 bf16 gate
 * values, and how many took the fast path; counts[3..5] = a failing gate's
 * bf16 bits and both f32 quotients (device counters, 6 x u32). */
int qtk_swiglu_selfcheck(uint32_t* counts, cudaStream_t s);

/* GradAccumulator::accumulate for an f32 gradient (src/model.cpp:455-462). */
/* *_ms variants: base = (*micro_step_dev) * n (device-resident counter, graph replay) */
int qtk_sr_accumulate_f32_ms(void* buf, const float* g, int64_t n, uint64_t seed, uint64_t stream,
                             const uint64_t* micro_step_dev, cudaStream_t s);
int qtk_embed_bwd_ms(const int32_t* sorted_pos, const int32_t* seg_off, const int32_t* seg_tok, const int* nseg_dev,
                     int max_seg, const void* d_r, int d, int64_t numel, void* grad, uint64_t seed, uint64_t stream,
                     const uint64_t* micro_step_dev, cudaStream_t s);
int qtk_sr_accumulate_f32(void* buf, const float* g, int64_t n, uint64_t seed, uint64_t stream, uint64_t base,
                          cudaStream_t s);

/* embedding_backward_sorted (src/tensorops.cpp:317-342) + bf16 round + accumulate. */
size_t qtk_embed_sort_scratch_bytes(int n, int64_t V);
int qtk_embed_sort(const int32_t* ids, int n, int64_t V, void* scratch, size_t scratch_bytes, int32_t* sorted_pos,
                   int32_t* seg_tok, int32_t* seg_off, int* nseg, cudaStream_t s);
int qtk_embed_bwd(const int32_t* sorted_pos, const int32_t* seg_off, const int32_t* seg_tok, const int* nseg_dev,
                  int max_seg, const void* d_r, int d, void* grad, uint64_t seed, uint64_t stream, uint64_t base,
                  cudaStream_t s);

/* causal GQA attention (sdpa_chunked / sdpa_chunked_backward,
 * src/tensorops.cpp:191-303) on the (B*T, qkv_dim) RoPE'd tensor. */
/* attention MMA operand precision: 1 = P (and dS) as bf16 hi + lo (f32-faithful
 * products), 0 = bf16 (default from QTB_ATTN_PLO) */
void qtk_attn_set_plo(int plo);
/* attention forward kernel: 1 = two query tiles per CTA (softmax / MMA ping-pong), 0 = one */
void qtk_attn_set_fwd2q(int on);
/* RMSNorm path: 0 by shape, 1 split-role chain kernel on the streaming path, 2 split-role chain + row
 * kernels everywhere, 3 (default) forward as 2 and backward as 1; all bit-identical outputs */
void qtk_rms_set_path(int mode);
/* RoPE kernel: 1 (default) head-looped (table chunk loaded once per row), 0 per-item; bitwise equal */
void qtk_rope_set_heads(int on);
int qtk_attn_fwd(const void* qkv, int B, int T, int H, int Hkv, int hd, int qkv_dim, void* out, int64_t ldo,
                 float* out32, float* lse, uint32_t* amax, cudaStream_t s);
/* precision mode (process-wide): fast_exp = __expf for exp(); bwd_split = P and
 * dS carried as bf16 hi+lo in the backward MMAs (default 0, 1) */
void qtk_attn_set_mode(int fast_exp, int bwd_split);
/* ws: qtk_attn_bwd_ws_bytes(...) of f32 scratch for the GQA per-head dK/dV partials */
size_t qtk_attn_bwd_ws_bytes(int B, int T, int H, int Hkv, int hd);
int qtk_attn_bwd(const void* qkv, const float* out32, const void* dout, int64_t ldo, const float* lse, float* Dv, int B,
                 int T, int H, int Hkv, int hd, int qkv_dim, void* dqkv, float* ws, cudaStream_t s);
/* as qtk_attn_bwd; the tcgen05 path runs its dQ kernel on s2 concurrently with dK/dV on s
 * (disjoint columns of dqkv) and joins s2 into s before returning */
int qtk_attn_bwd2(const void* qkv, const float* out32, const void* dout, int64_t ldo, const float* lse, float* Dv,
                  int B, int T, int H, int Hkv, int hd, int qkv_dim, void* dqkv, float* ws, cudaStream_t s,
                  cudaStream_t s2);

/* fused_cross_entropy_chunked softmax stage (src/tensorops.cpp:367-393):
 * per-row loss and dlogits from f32 logits; dlogits (f32 in the reference) is
 * written as bf16 hi + lo parts (either may be NULL). */
int qtk_ce_softmax(const float* logits, int64_t ldl, int64_t rows, int V, const int32_t* targets, float inv_n,
                   void* dlogits, void* dlogits_lo, int64_t ldd, float* loss_rows, cudaStream_t s);
/* same, with the per-row statistics the logits GEMM produced (QtkGemm.ce_*): one
 * pass over the logits instead of two */
int qtk_ce_softmax_stats(const float* logits, int64_t ldl, int64_t rows, int V, const int32_t* targets,
                         const float* stats, const float* tgt_logit, float inv_n, void* dlogits, void* dlogits_lo,
                         int64_t ldd, float* loss_rows, cudaStream_t s);
/* the target-exact CE backward (DESIGN.md §2 A15): as qtk_ce_softmax_stats, but
 * dlogits (bf16) has the target entry zeroed and dl_tgt[row] = (p_t - 1) / N
 * (f32) holds it; no lo part */
int qtk_ce_softmax_stats_tx(const float* logits, int64_t ldl, int64_t rows, int V, const int32_t* targets,
                            const float* stats, const float* tgt_logit, float inv_n, void* dlogits, int64_t ldd,
                            float* loss_rows, float* dl_tgt, cudaStream_t s);
/* d_hidden = bf16(acc + dl_tgt[m] * lm_w[targets[m]])   (acc: f32 M x d, the
 * split-K sum of bf16(dlogits) . lm_w) */
int qtk_lm_dgrad_finish(const float* acc, int64_t M, int d, const float* dl_tgt, const int32_t* targets,
                        const void* lm_w, void* d_hidden, cudaStream_t s);
/* acc[v] += sum_{m: targets[m] = v} dl_tgt[m] * hidden[m], ascending m, over the
 * segments of qtk_embed_sort(targets) (acc: f32 V x d) */
int qtk_lm_wgrad_targets(float* acc, int d, const int32_t* sorted_pos, const int32_t* seg_tok, const int32_t* seg_off,
                         const int* nseg, int64_t max_segs, const float* dl_tgt, const void* hidden, cudaStream_t s);
int qtk_loss_reduce(const float* loss_rows, int64_t n, float inv_n, float* out, float* accum, cudaStream_t s);

/* optimizer (src/optim.cpp:37-110).  segs: device array of per-tensor segment
 * records (size qtk_seg_size()). */
int qtk_seg_size(void);
int qtk_grad_sumsq(const void* grad, int grad_f32, const void* segs, int nseg, int64_t nblk, double* partials,
                   double* scratch, double* out, cudaStream_t s);
/* One shard of reduce_scatter_copy / reduce_scatter_oracle (src/comms.cpp:185-254,
 * include/qtrain/comms.hpp:113-132): acc (f32, n) += the W bf16 chunks of this
 * shard (device pointers indexed by source worker), own chunk first then ascending
 * sources, each add stochastically rounded to bf16 with stream
 * fnv1a64("rs/<step>/<layer>/<src>") and counter = element index (stochastic = 0:
 * plain f32 adds).  The trainer's own gradient exchange is the ascending-rank f32
 * sum of the session (src/trainer.cpp:90-103); this is the SR protocol's arithmetic. */
int qtk_reduce_scatter_sr(float* acc, const void* const* srcs, int W, int self, int64_t n, int stochastic,
                          uint64_t seed, uint64_t step, uint64_t layer, cudaStream_t s);
int qtk_adamw_chunk_size(void);
int qtk_adamw_chunk_entry_size(void);
int qtk_adamw_dev(void* p, float* m, float* v, void* m16, void* v16, const void* grad, int grad_f32, const void* segs,
                  const void* chunks, int nchunks, float lr, float b1, float b2, float eps, float wd, float bc1,
                  float bc2, const float* grad_scale_dev, uint64_t seed, int64_t step, int bf16_moments, int* err,
                  uint32_t* seg_amax, cudaStream_t s);
/* same, with step / bc1 / bc2 read on the device from step_dev = {int64 step; f32 bc1;
 * f32 bc2} (CUDA-graph replay; bc1/bc2 still computed on the host with powf) */
int qtk_adamw_dev_sd(void* p, float* m, float* v, void* m16, void* v16, const void* grad, int grad_f32,
                     const void* segs, const void* chunks, int nchunks, float lr, float b1, float b2, float eps,
                     float wd, float bc1, float bc2, const float* grad_scale_dev, uint64_t seed, int64_t step,
                     int bf16_moments, int* err, uint32_t* seg_amax, const void* step_dev, cudaStream_t s);

/* ------------------------------------------------------------------------- */
/* device-resident session: the reference operator API                        */
/* ------------------------------------------------------------------------- */

/* ModelConfig (include/qtrain/model.hpp:24-39) */
typedef struct QtModelConfig {
    int n_layers, d_model, d_ff, n_heads, n_kv_heads;
    int64_t vocab;
    int seq_len;
} QtModelConfig;

/* PrecisionMap (model.hpp:47-57): block_matmuls 0 = FP8_E4M3, 1 = BF16;
 * backward_grads 0 = E4M3, 1 = E5M2.  The device path runs FP8 only. */
typedef struct QtPrecisionMap {
    int block_matmuls, backward_grads, f32_debug;
} QtPrecisionMap;

/* RunPlan subset (include/qtrain/memplan.hpp:54-67) + ChunkSpec (model.hpp:158-161).
 * recompute_bits: RecomputeSet bits (model.hpp:59-80). */
typedef struct QtRunPlan {
    int micro_batch, ga_steps, recompute_bits;
    int64_t lmhead_chunk_tokens, attn_chunk_rows;
    int shard_weights, shard_grads, bf16_moments;
    /* OffloadSet bits (memplan.hpp:34-42): 1 x (residuals), 2 m, 4 v, 8 master,
     * 16 weights, 32 grads; transfer_policy: QT_XFER_* (memplan.hpp:44) */
    int offload_bits, transfer_policy;
} QtRunPlan;
enum { QT_OFF_X = 1, QT_OFF_M = 2, QT_OFF_V = 4, QT_OFF_MASTER = 8, QT_OFF_WEIGHTS = 16, QT_OFF_GRADS = 32 };
enum { QT_XFER_ZERO_COPY = 0, QT_XFER_DOUBLE_BUFFER = 1 };

/* AdamWHyper (include/qtrain/optim.hpp:20-26) + RunManifest::max_grad_norm */
typedef struct QtAdamW {
    float lr, beta1, beta2, eps, weight_decay, max_grad_norm;
} QtAdamW;

typedef struct qt_session qt_session;

const char* qt_last_error(void);
int qt_nccl_unique_id(void* out128);
int qt_session_create(const QtModelConfig* cfg, const QtPrecisionMap* prec, const QtRunPlan* plan, const QtAdamW* hyper,
                      uint64_t seed, int rank, int world, const void* nccl_id, int device, qt_session** out);
void qt_session_destroy(qt_session* s);

/* In-process worker group (the reference's WorkerGroup, include/qtrain/comms.hpp:51-78,
 * src/comms.cpp:19-38): `world` sessions, one per host thread, on one GPU or several,
 * created with qt_session_create_in_group(..., group, rank, device, ...).  Their
 * collectives are copy-engine pulls between the sessions' arenas (cudaMemcpyAsync,
 * no SM work, src/comms.cpp:185-293) ordered by CUDA events and a
 * host barrier; every rank must enter the same collectives in the same order (as
 * in the reference).  The group must outlive its sessions. */
typedef struct qt_group qt_group;
int qt_group_create(int world, qt_group** out);
void qt_group_destroy(qt_group* g);
int qt_session_create_in_group(const QtModelConfig* cfg, const QtPrecisionMap* prec, const QtRunPlan* plan,
                               const QtAdamW* hyper, uint64_t seed, qt_group* group, int rank, int device,
                               qt_session** out);
/* "none" (world 1), "nccl" or "peer-copy" */
const char* qt_session_transport(qt_session* s);
void* qt_session_stream(qt_session* s);
size_t qt_session_bytes(qt_session* s);
int qt_num_params(qt_session* s);
int qt_param_info(qt_session* s, int i, const char** name, int64_t* numel);
int qt_param_upload(qt_session* s, int i, const float* host);
int qt_param_download(qt_session* s, int i, float* host);
int qt_grad_download(qt_session* s, int i, float* host);
/* world > 1: the cross-rank reduced f32 gradient of tensor i (all ranks' shards gathered) */
int qt_reduced_grad_download(qt_session* s, int i, float* host);
int qt_moments_download(qt_session* s, int i, float* m, float* v);
/* m, v: the full tensor; each rank stores its ZeRO-1 slice (bf16-SR moments: values on the bf16 grid) */
int qt_moments_upload(qt_session* s, int i, const float* m, const float* v, int64_t step_count);
/* the slice [lo, lo + n) of tensor i that qt_moments_download returns on this rank */
int qt_moments_slice(qt_session* s, int i, int64_t* lo, int64_t* n);
int qt_step_count(qt_session* s, int64_t* out);
/* per-micro-batch losses of the last qt_train_step on this rank (ga_steps floats) */
int qt_step_losses(qt_session* s, float* out);
int qt_session_rank(qt_session* s, int* rank, int* world);
int qt_init_params(qt_session* s, uint64_t seed);                 /* init_params, model.cpp:67-86   */
int qt_build_step_context(qt_session* s);                          /* build_step_context, :88-107    */
int qt_forward(qt_session* s, const int32_t* tokens_dev, int64_t n_tokens, int64_t batch, int with_grads,
               float* loss_host);                                  /* model_forward, :297-352        */
int qt_backward(qt_session* s, uint64_t micro_step);               /* model_backward + accumulate    */
int qt_zero_grads(qt_session* s);
int qt_grad_norm(qt_session* s, double* norm_host);                /* global_grad_norm, optim.cpp:87-105 */
int qt_adamw_step(qt_session* s, float grad_scale);                /* (sharded_)adamw_step           */
int qt_train_step(qt_session* s, const int32_t* tokens_dev, int64_t tokens_per_mb, int64_t batch, int64_t step,
                  float max_grad_norm, float* loss_host, float* norm_host); /* trainer.cpp:64-110 */
int qt_upload_tokens(qt_session* s, const int32_t* host, int64_t n, int32_t** dev_out);
int qt_sync(qt_session* s);
int qt_forward_stats(qt_session* s, float* out);
int qt_saved_raw(qt_session* s, int layer, const char* site, void* host, int64_t* bytes, int* dtype);
int qt_scales(qt_session* s, int which, float* out);
int qt_weight_codes(qt_session* s, int layer, int which, uint8_t* host);
int qt_set_profile(qt_session* s, int on);
int qt_profile_read(qt_session* s, int ncat, double* ms, int64_t* launches, double* work);
int qt_shard_layout(int64_t numel, int workers, int64_t* padded, int64_t* per_worker);
uint64_t qt_fnv1a64(const char* s);
/* the RoPE {cos, sin} table the session builds (T x hd/2 float pairs, the
 * reference's powf/cosf/sinf, src/model.cpp:178-183) -> host_out (T*hd floats) */
int qt_rope_table(int T, int hd, float* host_out);
/* which instantiation qtk_gemm launches for *g (no launch): cta_group, BN,
 * split-K factor, grid, output tiles per CTA of the persistent loop */
int qtk_gemm_plan(const QtkGemm* g, int* cg, int* bn, int* splits, int* grid, int* tiles_per_cta);
/* whether qtk_gemm runs *g as a tail split (head launch of *m_head rows + a split-K launch
 * of the remaining rows split *s_tail ways): 1 yes, 0 no (then *m_head = M, *s_tail = 1) */
int qtk_gemm_tail_plan(const QtkGemm* g, int64_t* m_head, int* s_tail);
int qt_count_step_kernels(qt_session* s, const int32_t* tokens_dev, int64_t tokens_per_mb, int64_t batch,
                          int64_t* kernels, int64_t* other_nodes);
/* diagnostic: one trainer step captured into a CUDA graph and replayed `iters` times
 * (same step counters each replay); mean device ms per replay -> *ms */
int qt_time_graph_step(qt_session* s, const int32_t* tokens_dev, int64_t tokens_per_mb, int64_t batch, int64_t step,
                       int iters, float* ms);

/* ------------------------------------------------------------------------- */
/* planner (csrc/planner.cpp; src/memplan.cpp, src/profiles.cpp,              */
/* src/offload.cpp).  Status codes as above; message in qt_plan_last_error(). */
/* ------------------------------------------------------------------------- */
/* HardwareProfile (include/qtrain/profiles.hpp:14-33) */
typedef struct QtHardwareProfile {
    char name[32];
    uint64_t device_bytes, host_bytes;
    double peak_flops_fp8, peak_flops_bf16, peak_flops_f32; /* dense FLOP/s */
    double mem_bandwidth, link_bandwidth;                   /* bytes/s     */
    int p2p;
    double attainable_fraction, zero_copy_efficiency, double_buffer_efficiency;
} QtHardwareProfile;
/* MemoryBreakdown::Tier (include/qtrain/memplan.hpp:100-116) */
typedef struct QtMemTier {
    uint64_t params_fp8, params_bf16_master, moments_m, moments_v, grads, residuals, activations, logits_workspace,
        attn_workspace;
} QtMemTier;
/* FlopBreakdown (memplan.hpp:148-160): per token, forward + backward */
typedef struct QtFlops {
    double linear, lmhead, attention, recompute;
} QtFlops;
/* TimeBreakdown (memplan.hpp:176-185) */
typedef struct QtStepTime {
    double compute, transfer, exposed_transfer, optimizer, total;
    int feasible_in_time;
    double tokens_per_second;
} QtStepTime;
const char* qt_plan_last_error(void);
/* model_presets (src/memplan.cpp:98-108): toy, 0.5b, 1.5b, 3b, 7b, 14b, 32b */
int qt_model_preset(const char* name, QtModelConfig* cfg, int* tied);
/* builtins of src/profiles.cpp:21-39 plus "b200" */
int qt_profile_by_name(const char* name, QtHardwareProfile* out);
int qt_profile_load(const char* name_or_path, QtHardwareProfile* out); /* profiles.cpp:82-93 */
int qt_profile_from_json(const char* text, QtHardwareProfile* out);
/* text outputs: *needed = bytes incl. NUL; buf may be NULL to query the size */
int qt_profile_to_json(const QtHardwareProfile* p, char* buf, size_t cap, size_t* needed);
int qt_param_counts(const QtModelConfig* cfg, int tied, uint64_t* total, uint64_t* block_linear,
                    uint64_t* per_layer_linear, uint64_t* lmhead, uint64_t* embed, uint64_t* norms);
/* memory_breakdown (memplan.cpp:177-268): per worker */
int qt_memory_breakdown(const QtModelConfig* cfg, const QtPrecisionMap* prec, const QtRunPlan* plan, int workers,
                        int tied, QtMemTier* device, QtMemTier* host);
int qt_flop_breakdown(const QtModelConfig* cfg, int recompute_bits, int tied, QtFlops* out);
int qt_lower_bound_seconds_per_token(const QtFlops* f, const QtPrecisionMap* prec, const QtHardwareProfile* hw,
                                     int attainable, int include_recompute, double* out);
int qt_mfu(double measured_tps, const QtModelConfig* cfg, const QtPrecisionMap* prec, const QtHardwareProfile* hw,
           int tied, double* out);
int qt_fp8_speedup_ceiling(const QtModelConfig* cfg, const QtHardwareProfile* hw, int tied, double* out);
int qt_estimate_step_time(const QtModelConfig* cfg, const QtPrecisionMap* prec, const QtRunPlan* plan,
                          const QtHardwareProfile* hw, int workers, int tied, QtStepTime* out);
/* search_plan (memplan.cpp:471-551) -> JSON {"feasible": [...], "n_feasible", "no_fit_reason"?};
 * max_results <= 0: all */
int qt_search_plan(const QtModelConfig* cfg, const QtHardwareProfile* hw, int workers, int64_t target_batch_tokens,
                   int block_matmuls, int exhaustive, int tied, int max_results, char* json_out, size_t cap,
                   size_t* needed);
/* plan_residency (offload.cpp:40-163) -> JSON {"events": [...], "high_water_*", "feasible", "report"?} */
int qt_plan_residency(const QtModelConfig* cfg, const QtPrecisionMap* prec, const QtRunPlan* plan,
                      uint64_t device_budget, int tied, char* json_out, size_t cap, size_t* needed);
/* transfer_time (offload.cpp:165-171) */
int qt_transfer_time(uint64_t bytes, const QtHardwareProfile* hw, int policy, double* out);

/* ------------------------------------------------------------------------- */
/* trainer, corpora, checkpoints (csrc/trainer.cpp; src/trainer.cpp,          */
/* src/manifest.cpp, src/corpus.cpp, src/checkpoint.cpp).  Errors: status as  */
/* above, message in qt_train_last_error().                                  */
/* ------------------------------------------------------------------------- */
const char* qt_train_last_error(void);
/* make_corpus (corpus.cpp:58-69): kind "perm-walk" | "uniform"; train_out n_train*(seq_len+1),
 * val_out n_val*(seq_len+1) ids */
int qt_make_corpus(const char* kind, int64_t vocab, int seq_len, int n_train, int n_val, uint64_t seed,
                   int32_t* train_out, int32_t* val_out);
/* manifest_to_json(manifest_from_json(text or path)) (manifest.cpp:45-188) */
int qt_manifest_normalize(const char* manifest, char* json_out, size_t cap, size_t* needed);
/* run_training_to_files (trainer.cpp:35-171) on the device: metrics CSV and the QTCKPT01
 * checkpoint per the manifest's outputs; "resume_from": <checkpoint> continues a run;
 * W workers = W sessions of one peer group on device w % device_count (0 = all visible).
 * result_json: {"metrics": [...], "initial_train_loss", "final_train_loss", "final_val_loss"} */
int qt_run_training(const char* manifest, int device_count, char* result_json, size_t cap, size_t* needed);
/* QTCKPT01 (checkpoint.cpp:19-80) of the params (for_each_param order), optional optimizer
 * moments ("optim.m.<name>", "optim.v.<name>", name order) and "optim.step" */
int qt_checkpoint_save(qt_session* const* sessions, int n_sessions, const QtModelConfig* cfg, const char* path,
                       int with_optimizer);
int qt_checkpoint_load(qt_session* const* sessions, int n_sessions, const char* path, int64_t* step_out);

#ifdef __cplusplus
}
#endif

#endif /* QTRAIN_B200_H */
