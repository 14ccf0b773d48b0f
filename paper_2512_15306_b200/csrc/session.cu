// Device-resident training session: the B200 implementation of the
// reference's model/optimizer entry points (include/qtrain/model.hpp:125-211,
// include/qtrain/optim.hpp:55-77) and of one trainer step
// (src/trainer.cpp:64-131), driving the qtk_* kernels on one CUDA stream.
//
// HBM layout (one arena, allocated once at creation):
//   params   bf16, every tensor in for_each_param order (model.hpp:107-121),
//            each padded to W*pw elements (ZeRO-1 shard layout, comms.cpp:69-73)
//   grads    bf16 GradAccumulator buffers, same layout (SR-accumulated by the
//            wgrad GEMM epilogues)
//   m, v     f32 (or bf16-SR) AdamW moments for this rank's shard only
//   wcodes   E4M3 codes of the four block weights per layer (StepContext)
//   per layer saved activations (kept sites) + shared scratch (dropped sites)
//   CE       f32 logits and bf16 dlogits for the whole micro-batch
#include "common.cuh"
#include "kernels.h"
#include "nccl_dl.h"
#include "transport.cuh"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "hostjson.h"
namespace qtb {
namespace plan {
using DeviceBytesFn = uint64_t (*)(const QtModelConfig&, const QtPrecisionMap&, const QtRunPlan&, int, bool,
                                   const QtMemTier&);
json::Value search_with(const QtModelConfig& c, const QtHardwareProfile& hw, int W, int64_t target_tokens, int matmuls,
                        bool exhaustive, bool tied, DeviceBytesFn fn, int max_results);
}  // namespace plan
}  // namespace qtb
namespace qtb {

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
thread_local std::string g_last_error;

struct QtError : std::runtime_error {
    int code;
    QtError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
#define QT_CHECK_CUDA(x)                                                                              \
    do {                                                                                              \
        cudaError_t e_ = (x);                                                                         \
        if (e_ != cudaSuccess) throw QtError(3, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                                    " at " #x);                                       \
    } while (0)
#define QT_CHECK_K(x)                                                                                 \
    do {                                                                                              \
        int rc_ = (x);                                                                                \
        if (rc_ != 0) throw QtError(rc_ == 1 ? 1 : 3, std::string("kernel launch failed (") +        \
                                                          std::to_string(rc_) + "): " #x);            \
    } while (0)

uint64_t fnv1a64(const std::string& s) {
    uint64_t h = 0xCBF29CE484222325ull;
    for (unsigned char c : s) {
        h ^= c;
        h *= 0x100000001B3ull;
    }
    return h;
}

// layout-compatible with qtb::Seg in ce_optim.cu (size checked at runtime)
struct SegH {
    int64_t off, n, gstart, gnumel;
    uint64_t sm, sv, sw;
    int64_t blk0, poff;
};

// ---------------------------------------------------------------------------
// small session kernels
// ---------------------------------------------------------------------------
// normal_init (src/model.cpp:56-65) with rng_normal (src/numerics.cpp:216-226)
__global__ void init_normal_kernel(uint16_t* t, int64_t n, float std_, uint64_t seed, uint64_t stream, int64_t base) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t c = (uint64_t)(base + i);
        const double u1 = ((double)rng_uniform(seed, stream, 2 * c) + 1.0) * 0x1.0p-32;
        const double u2 = (double)rng_uniform(seed, stream, 2 * c + 1) * 0x1.0p-32;
        const double r = sqrt(-2.0 * log(u1));
        const float z = (float)(r * cos(2.0 * 3.14159265358979323846 * u2));
        t[i] = f2bfbits(__fmul_rn(std_, z));
    }
}
__global__ void fill_bf16_kernel(uint16_t* t, int64_t n, float v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        t[i] = f2bfbits(v);
}
__global__ void f32_to_bf16_kernel(const float* in, uint16_t* out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = f2bfbits(in[i]);
}
__global__ void bf16_to_f32_kernel(const uint16_t* in, float* out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = bfbits2f(in[i]);
}
// trainer.cpp:105-107 + optim.cpp:107-110: norm = sqrt(ssq)*mean_scale,
// clip = min(1, max/norm), grad_scale = mean_scale*clip
__global__ void finalize_scale_kernel(const double* ssq, float mean_scale, float max_norm, float* grad_scale,
                                      double* norm_out, int* err) {
    if (!isfinite(*ssq) && *err == 0) *err = 3;
    const double norm = sqrt(*ssq) * (double)mean_scale;
    float clip = 1.0f;
    if (!(max_norm <= 0.0f || norm <= (double)max_norm)) clip = (float)((double)max_norm / norm);
    *grad_scale = __fmul_rn(mean_scale, clip);
    *norm_out = norm;
}
__global__ void set_scale_kernel(float* p, float v) { *p = v; }
// Update gate (the reference throws before any update, model.cpp:125-129, 324-325):
// an out-of-range token, a non-finite forward statistic or loss poisons the local
// sum of squares with NaN before the cross-rank all-reduce, so every rank sees the
// same non-finite norm and skips AdamW (adamw_kernel returns when *err != 0).
__global__ void poison_ssq_kernel(double* ssq, const int* err, const uint32_t* act_amax, int n_act,
                                  const uint32_t* fin_amax, const float* losses, int n_loss) {
    bool bad = *err != 0 || *fin_amax >= 0x7F800000u;
    for (int i = 0; i < n_act; ++i) bad |= act_amax[i] >= 0x7F800000u;
    for (int i = 0; i < n_loss; ++i) bad |= !isfinite(losses[i]);
    if (bad) *ssq = __longlong_as_double(0x7FF8000000000000ll);
}
// non-finite global norm -> err = 3 (adamw_step: non-finite gradient) unless already set
__global__ void gate_kernel(const double* ssq, int* err) {
    if (!isfinite(*ssq) && *err == 0) *err = 3;
}
// w_amax[l*4 + k] = seg_amax[param index of block weight k of layer l] (k: qkv, o, gate_up, down)
__global__ void gather_wamax_kernel(const uint32_t* __restrict__ seg_amax, uint32_t* __restrict__ w_amax, int L) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= L * 4) return;
    const int l = i / 4, k = i % 4;
    const int off[4] = {1, 2, 4, 5};
    w_amax[i] = seg_amax[1 + 6 * l + off[k]];
}
// E4M3 scales of n tensors from their absmax bit patterns (absmax_scale, src/numerics.cpp:150-158)
__global__ void weight_scale_kernel(const uint32_t* __restrict__ amax, float* __restrict__ scale, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) scale[i] = absmax_scale(__uint_as_float(amax[i]), kE4M3);
}
// cross-worker sum in ascending worker order, plain f32 (src/trainer.cpp:95-102)
// recv holds W rank blocks of `stride` elements; sums elements [0, n) of each
__global__ void ordered_sum_kernel(const uint16_t* __restrict__ recv, int W, int64_t n, int64_t stride,
                                   float* __restrict__ out, int acc) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float s = bfbits2f(recv[i]);
        for (int w = 1; w < W; ++w) s = __fadd_rn(s, bfbits2f(recv[(int64_t)w * stride + i]));
        out[i] = acc ? __fadd_rn(out[i], s) : s;
    }
}

// reduce_scatter_copy's arithmetic (src/comms.cpp:136-146, 233-254) for one shard:
// acc += own chunk first, then the other sources in ascending order, each add
// SR-rounded to bf16 with stream fnv1a64("rs/<step>/<layer>/<src>"), counter = i
// (stochastic = 0: plain f32 adds).  Source chunks are bf16.
struct RsArgs {
    const uint16_t* src[16];
    uint64_t key[16];
};
__global__ void reduce_scatter_sr_kernel(float* __restrict__ acc, RsArgs a, int W, int self, int64_t n,
                                         int stochastic) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float v = acc[i];
        for (int t = 0; t < W; ++t) {
            const int src = t == 0 ? self : (t - 1 < self ? t - 1 : t);
            v = __fadd_rn(v, bfbits2f(a.src[src][i]));
            if (stochastic) v = sr_bf16k(v, a.key[src], (uint64_t)i);
        }
        acc[i] = v;
    }
}

// rope_apply angles (src/model.cpp:178-183) with the reference's own float libm
// calls (std::pow / std::cos / std::sin on float): T x hd/2 {cos, sin}
void rope_table_host(int T, int hd, float2* tab) {
    const int half = hd / 2;
    for (int t = 0; t < T; ++t) {
        for (int i = 0; i < half; ++i) {
            const float freq = std::pow(10000.0f, -2.0f * static_cast<float>(i) / static_cast<float>(hd));
            const float angle = static_cast<float>(t) * freq;
            tab[(size_t)t * half + i] = make_float2(std::cos(angle), std::sin(angle));
        }
    }
}

inline int grid_for(int64_t n, int per = 256) { return (int)std::min<int64_t>(std::max<int64_t>(ceil_div(n, per), 1), 16 * kNumSMs); }

// ---------------------------------------------------------------------------
// session
// ---------------------------------------------------------------------------
enum Site { S_N1 = 0, S_ATT = 1, S_N2 = 2, S_H = 3 };
enum GSite { G_DR = 0, G_DGU = 1, G_DAO = 2, G_DQKV = 3 };
enum WIdx { W_QKV = 0, W_O = 1, W_GU = 2, W_DOWN = 3 };

struct ParamT {
    std::string name;
    std::vector<int64_t> shape;
    int64_t numel = 0, off = 0, padded = 0, pw = 0;
    // storage: params hold [lo, lo + store) of the tensor at `off` (shard_weights keeps only the
    // rank's ZeRO-1 slice of a block weight); the gradient accumulator sits at `goff` in the full
    // buffer, or (shard_grads, layer tensors) at `loff` in the per-layer buffer
    int64_t lo = 0, store = 0, goff = -1, loff = -1;
    bool sharded = false;
    uint64_t s_acc = 0, s_m = 0, s_v = 0, s_w = 0, s_init = 0;
};

struct LayerBufs {
    uint16_t* r_in = nullptr;
    uint8_t* n1c = nullptr;
    uint16_t* qkv = nullptr;
    uint16_t* att = nullptr;
    float* att32 = nullptr;  // unrounded attention output (sdpa backward's orow, tensorops.cpp:278-281)
    uint8_t* attc = nullptr;
    float* lse = nullptr;
    uint16_t* r_mid = nullptr;
    uint8_t* n2c = nullptr;
    uint16_t* gu = nullptr;
    uint8_t* hc = nullptr;
    bool keep_all = true;
};

struct ProfRec {
    int cat;
    cudaEvent_t a, b;
    double work;
};

class Session {
   public:
    QtModelConfig cfg;
    QtPrecisionMap prec;
    QtRunPlan plan;
    QtAdamW hyper;
    uint64_t seed;
    int rank, world;
    cudaStream_t st = nullptr;
    cudaStream_t cst = nullptr;  // communication stream (per-layer gradient exchange, shard_grads)
    cudaEvent_t ev_grad = nullptr, ev_comm = nullptr;
    std::vector<int64_t> soff_of;  // offset of each tensor's shard in the W x shard_total exchange layout
    bool comm_pending = false;
    bool exchange_in_backward = false;  // shard_grads: per-layer exchange during this backward
    // CUDA-graph replay of the trainer step: per-step values live in a device block the
    // host rewrites before each launch; kernels read them there while use_dev_ctr is set
    struct StepBlockH {
        int64_t step;  // AdamW step being applied (1-based)
        float bc1, bc2;
    };
    uint8_t* step_blk = nullptr;  // StepBlockH, then ga_steps uint64 micro-steps
    bool use_dev_ctr = false;
    int cur_ga = 0;
    cudaGraphExec_t gexec = nullptr;
    // pinned staging ring for the step block (pageable H2D copies would synchronise the
    // stream); slot i is reused only after its copy has executed (event)
    static constexpr int kBlkRing = 8;
    uint8_t* blk_host = nullptr;
    cudaEvent_t blk_ev[kBlkRing] = {};
    int blk_slot = 0;
    int64_t g_tpm = -1, g_batch = -1;
    float g_max_norm = 0.0f;
    const uint64_t* ms_dev(int ga) const { return reinterpret_cast<const uint64_t*>(step_blk + 16) + ga; }
    std::unique_ptr<Transport> tr;  // world > 1: NCCL or the in-process copy-engine peer group

    int L, d, F, Hh, H, Hkv, hd, q, T;
    int64_t V, Mmax;
    std::vector<ParamT> P;
    std::map<std::string, int> pidx;
    int64_t p_total = 0;   // padded elements of all tensors (the unsharded layout)
    int64_t shard_total = 0;
    int64_t step_count = 0;  // completed optimizer steps (OptimState::step_count)

    // arena
    uint8_t* arena = nullptr;
    size_t arena_bytes = 0;
    uint16_t* params = nullptr;
    uint16_t* grads = nullptr;
    float* m32 = nullptr;
    float* v32 = nullptr;
    uint16_t* m16 = nullptr;
    uint16_t* v16 = nullptr;
    float* gshard = nullptr;      // f32 reduced grads of this rank's shard (W>1)
    uint16_t* recvbuf = nullptr;  // W x shard_total bf16 (W x the non-layer shards under shard_grads)
    int64_t p_store = 0, g_store = 0;  // params / full gradient buffer elements
    // shard_grads: per-layer gradient buffers (double-buffered: layer l is exchanged on the
    // communication stream while layer l-1's backward writes the other) and their receive areas
    uint16_t* lgrad[2] = {nullptr, nullptr};
    uint16_t* lrecv[2] = {nullptr, nullptr};
    int64_t layer_g = 0, layer_shard = 0;  // elements of one layer's 6 tensors, padded / per rank
    cudaEvent_t ev_lfree[2] = {nullptr, nullptr};
    // streamed FP8 weight codes (shard_weights and/or offloaded weights): the rank's slice
    // codes, two layer slots filled one layer ahead on the communication stream, and the
    // pinned host copy (offload.weights; the paper's host weight cache under shard_weights)
    std::vector<uint8_t*> wown;      // L*4 (shard_weights)
    uint8_t* wslot[2][4] = {};
    uint8_t* whost = nullptr;        // L x layer codes (pinned)
    // offload tiers (RunPlan::offload, memplan.hpp:34-52): pinned host region holding the
    // offloaded optimizer moments (m, v), bf16 master block weights and/or gradient buffer.
    // Zero-copy: kernels address it directly (UVA).  Double-buffer (m, v): AdamW streams the
    // moments through two device slots group by group on the copy engines.
    uint8_t* harena = nullptr;
    size_t harena_bytes = 0;
    int64_t p_master = 0;            // elements of the host master region (offload.master)
    uint16_t* hmaster = nullptr;
    float* mstage[2][2] = {};        // [slot][m|v] f32 (or bf16) staging of the double buffer
    int64_t mstage_elems = 0;
    struct MGroup {
        int c0, c1;                  // chunk-table range
        int64_t e0, e1;              // moment element range
    };
    std::vector<MGroup> mgroups;
    cudaEvent_t ev_mready[2] = {}, ev_mdone[2] = {}, ev_mfree[2] = {};
    // offload.x: the layer inputs r_in[0..L-1] live in pinned host memory; two device slots
    // (layer l in slot l%2) are written back after the forward produces them and refilled
    // one layer ahead of the backward
    uint16_t* xslot[2] = {nullptr, nullptr};
    uint16_t* xhost = nullptr;
    int xslot_layer[2] = {-1, -1};
    cudaEvent_t ev_xready[2] = {}, ev_xfree[2] = {};
    int64_t wl_off[4] = {}, wl_total = 0;  // a layer's 4 tensors inside a slot / whost entry
    int slot_layer[2] = {-1, -1};    // which layer's codes each slot holds (this step)
    std::vector<char> published;     // whost[l] holds this step's codes
    cudaEvent_t ev_wfree[2] = {nullptr, nullptr}, ev_wready[2] = {nullptr, nullptr}, ev_codes = nullptr;
    std::vector<uint8_t*> wcodes;  // L*4
    std::vector<LayerBufs> lb;
    uint16_t *s_n1 = nullptr, *s_attn_out = nullptr, *s_n2 = nullptr, *s_h = nullptr, *normed_final = nullptr;
    uint16_t *d_r = nullptr, *d_h = nullptr, *d_gu = nullptr, *d_n = nullptr, *d_ao = nullptr, *d_att = nullptr,
             *d_qkv = nullptr, *d_hidden = nullptr;
    uint8_t* gcodes = nullptr;  // grad-kind codes scratch (M x max(F, q))
    // weight-gradient GEMMs on a side stream (QTB_WGRAD_SIDE): the wgrad of a d_out overlaps its
    // dgrad and the elementwise work after it; the grad-kind codes alternate between two
    // buffers so the next cast need not wait for the previous wgrad
    uint8_t* gcodes2 = nullptr;
    cudaStream_t wst = nullptr;
    cudaEvent_t ev_qready = nullptr, ev_wdone[2] = {nullptr, nullptr}, ev_wjoin = nullptr;
    float* gemm_ws = nullptr;   // split-K partials for the small-grid weight-gradient GEMMs
    float* gemm_ws2 = nullptr;  // the side stream's
    int64_t gemm_ws_bytes = 0;
    float* logits = nullptr;
    uint16_t* dlogits = nullptr;
    uint16_t* dlogits_lo = nullptr;  // hi/lo CE backward only (lm_tx() off)
    // target-exact CE backward (lm_tx()): f32 target terms, the LM-head split-K partials,
    // the f32 sum buffer (d_hidden before rounding, then d_lm_w) and the targets' stable sort
    float* dl_tgt = nullptr;
    float* lm_ws = nullptr;
    int64_t lm_ws_bytes = 0;
    int lm_splits = 1;
    float* lm_acc = nullptr;
    int32_t *t_sorted_pos = nullptr, *t_seg_tok = nullptr, *t_seg_off = nullptr;
    int* t_nseg = nullptr;
    float* loss_rows = nullptr;
    float* ce_stats = nullptr;   // [M][ceil(V/128)] (max, sum exp) pairs from the logits GEMM
    float* ce_tgt = nullptr;     // [M] logit of the target
    float* dgamma_part = nullptr;
    float* dgamma = nullptr;
    float* rms_inv = nullptr;  // per-row 1/rms scratch of the forward norms
    float* Dv = nullptr;
    float* attn_ws = nullptr;  // GQA per-head dK/dV partials
    float2* rope_tab = nullptr;
    int32_t *tok_buf = nullptr, *inputs = nullptr, *targets = nullptr, *sorted_pos = nullptr, *seg_tok = nullptr,
            *seg_off = nullptr;
    int* nseg = nullptr;
    void* sort_scratch = nullptr;
    size_t sort_scratch_bytes = 0;
    double* norm_partials = nullptr;
    double* norm_scratch = nullptr;
    int64_t norm_blocks = 0;
    SegH* segs_dev = nullptr;
    int nsegs = 0;
    void* chunks_dev = nullptr;  // AdamW per-CTA chunk table
    int nchunks = 0;
    // device scalars
    uint32_t* act_amax = nullptr;  // L*4
    float* act_scale = nullptr;    // L*4
    uint32_t* w_amax = nullptr;    // L*4
    float* w_scale = nullptr;      // L*4
    uint32_t* g_amax = nullptr;    // L*4
    float* g_scale = nullptr;      // L*4
    uint32_t* fin_amax = nullptr;
    uint32_t* seg_amax = nullptr;  // per-parameter |w| max of the weights AdamW just wrote
    bool amax_cached = false;      // seg_amax describes the current params (next build_step_context skips absmax)
    float* loss_dev = nullptr;     // per micro-batch losses (ga_steps)
    double* ssq_dev = nullptr;
    double* norm_dev = nullptr;
    float* gscale_dev = nullptr;
    int* err_dev = nullptr;
    float* scratch_f32 = nullptr;  // param download staging

    // current micro-batch
    int curB = 0, curT = 0;
    int64_t curM = 0;
    bool have_fwd = false, fwd_with_grads = false;
    bool in_step = false;          // inside train_step_body (per-micro-batch losses in loss_dev[1..GA])
    int64_t pre_step_count = -1;   // step_count before the last train_step (restored when it is gated)

    // profiling
    bool prof_on = false;
    std::vector<ProfRec> prof;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;

    Session(const QtModelConfig& c, const QtPrecisionMap& p, const QtRunPlan& pl, const QtAdamW& h, uint64_t sd, int rk,
            int ws, const void* nccl_id, int device, std::shared_ptr<PeerGroup> group = nullptr)
        : cfg(c), prec(p), plan(pl), hyper(h), seed(sd), rank(rk), world(ws) {
        validate();
        QT_CHECK_CUDA(cudaSetDevice(device));
        QT_CHECK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        L = c.n_layers;
        d = c.d_model;
        F = c.d_ff;
        Hh = c.d_ff / 2;
        H = c.n_heads;
        Hkv = c.n_kv_heads;
        hd = d / H;
        q = d + 2 * Hkv * hd;
        V = c.vocab;
        T = c.seq_len;
        Mmax = (int64_t)std::max(1, pl.micro_batch) * T;
        build_params();
        allocate();
        build_segments();
        build_rope_table();
        if (world > 1) {
            try {
                if (group) {
                    if (group->world != world) throw QtError(1, "peer group size != world");
                    tr = std::make_unique<PeerTransport>(group, rank, device, arena, arena_bytes, harena, harena_bytes);
                } else {
                    if (!nccl_id) throw QtError(1, "world > 1 needs an NCCL unique id (or a peer group)");
                    if (harena && !shard_weights() && offload_master())
                        throw QtError(1, "offload.master over NCCL needs shard_weights (NCCL gathers device memory)");
                    tr = std::make_unique<NcclTransport>(rank, world, nccl_id);
                }
            } catch (const TransportError& e) {
                throw QtError(3, e.what());
            }
        }
        if (world > 1 || stream_codes()) {
            QT_CHECK_CUDA(cudaStreamCreateWithFlags(&cst, cudaStreamNonBlocking));
            for (cudaEvent_t* e : {&ev_grad, &ev_comm, &ev_codes, &ev_lfree[0], &ev_lfree[1], &ev_wfree[0], &ev_wfree[1],
                                   &ev_wready[0], &ev_wready[1]})
                QT_CHECK_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        }
        if (stream_codes() && offload_weights())
            QT_CHECK_CUDA(cudaMallocHost(&whost, std::max<size_t>((size_t)L * wl_total, 1)));
        if (wgrad_side()) {
            QT_CHECK_CUDA(cudaStreamCreateWithFlags(&wst, cudaStreamNonBlocking));
            for (cudaEvent_t* e : {&ev_qready, &ev_wdone[0], &ev_wdone[1], &ev_wjoin})
                QT_CHECK_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        }
        if (offload_x()) {
            if (!cst) QT_CHECK_CUDA(cudaStreamCreateWithFlags(&cst, cudaStreamNonBlocking));
            for (cudaEvent_t* e : {&ev_xready[0], &ev_xready[1], &ev_xfree[0], &ev_xfree[1]})
                QT_CHECK_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        }
        if (stream_moments()) {
            if (!cst) QT_CHECK_CUDA(cudaStreamCreateWithFlags(&cst, cudaStreamNonBlocking));
            for (cudaEvent_t* e : {&ev_mready[0], &ev_mready[1], &ev_mdone[0], &ev_mdone[1], &ev_mfree[0], &ev_mfree[1]})
                QT_CHECK_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        }
        QT_CHECK_CUDA(cudaStreamSynchronize(st));
    }

    // Dry layout: the arena (and pinned host) bytes a session of this shape allocates,
    // computed by the same allocate() without touching a device (qt_session_footprint)
    struct DryRun {};
    bool dry = false;
    size_t host_bytes = 0;
    Session(DryRun, const QtModelConfig& c, const QtPrecisionMap& p, const QtRunPlan& pl, int ws)
        : cfg(c), prec(p), plan(pl), hyper{}, seed(0), rank(0), world(ws), dry(true) {
        validate();
        L = c.n_layers;
        d = c.d_model;
        F = c.d_ff;
        Hh = c.d_ff / 2;
        H = c.n_heads;
        Hkv = c.n_kv_heads;
        hd = d / H;
        q = d + 2 * Hkv * hd;
        V = c.vocab;
        T = c.seq_len;
        Mmax = (int64_t)std::max(1, pl.micro_batch) * T;
        build_params();
        allocate();
    }

    ~Session() {
        tr.reset();
        for (auto e : ev_pool) cudaEventDestroy(e);
        for (cudaEvent_t e : {ev_grad, ev_comm, ev_codes, ev_lfree[0], ev_lfree[1], ev_wfree[0], ev_wfree[1], ev_wready[0],
                              ev_wready[1]})
            if (e) cudaEventDestroy(e);
        if (cst) cudaStreamDestroy(cst);
        for (cudaEvent_t e : {ev_qready, ev_wdone[0], ev_wdone[1], ev_wjoin})
            if (e) cudaEventDestroy(e);
        if (wst) cudaStreamDestroy(wst);
        if (whost) cudaFreeHost(whost);
        if (harena) cudaFreeHost(harena);
        for (cudaEvent_t e : {ev_mready[0], ev_mready[1], ev_mdone[0], ev_mdone[1], ev_mfree[0], ev_mfree[1],
                              ev_xready[0], ev_xready[1], ev_xfree[0], ev_xfree[1]})
            if (e) cudaEventDestroy(e);
        if (gexec) cudaGraphExecDestroy(gexec);
        for (auto& e : blk_ev)
            if (e) cudaEventDestroy(e);
        if (blk_host) cudaFreeHost(blk_host);
        if (arena) cudaFree(arena);
        if (st) cudaStreamDestroy(st);
    }

    void validate() {
        // ModelConfig::validate (src/model.cpp:12-17)
        if (cfg.d_model % cfg.n_heads != 0) throw QtError(1, "ModelConfig: d_model % n_heads != 0");
        if (cfg.n_heads % cfg.n_kv_heads != 0) throw QtError(1, "ModelConfig: n_heads % n_kv_heads != 0");
        if (cfg.d_ff % 2 != 0) throw QtError(1, "ModelConfig: d_ff must be even (gate | up halves)");
        if (cfg.n_layers < 1 || cfg.vocab < 2 || cfg.seq_len < 1) throw QtError(1, "ModelConfig: degenerate");
        if (prec.block_matmuls != 0 || prec.f32_debug)
            throw QtError(1, "qtrain-b200 runs the FP8 block-matmul path only (BF16 / f32_debug modes are oracle-only)");
        const int hd_ = cfg.d_model / cfg.n_heads;
        if (hd_ != 32 && hd_ != 64 && hd_ != 128) throw QtError(1, "head_dim must be 32, 64 or 128");
        if (cfg.d_model % 16 || cfg.d_ff % 32) throw QtError(1, "d_model % 16 and d_ff % 32 must be 0 (TMA/vector alignment)");
        if (cfg.vocab % 8) throw QtError(1, "vocab % 8 must be 0 (TMA row alignment of the bf16 dlogits)");
        if (plan.micro_batch < 1 || plan.ga_steps < 1) throw QtError(1, "RunPlan: micro_batch/ga_steps must be >= 1");
        if (world < 1 || rank < 0 || rank >= world) throw QtError(1, "bad rank/world");
    }

    void add_param(const std::string& name, std::vector<int64_t> shape) {
        ParamT t;
        t.name = name;
        t.shape = shape;
        t.numel = 1;
        for (auto s : shape) t.numel *= s;
        const int64_t unit = 256 * (int64_t)world;  // shard_layout (src/comms.cpp:69-73)
        t.padded = ceil_div(t.numel, unit) * unit;
        t.pw = t.padded / world;
        t.off = p_total;
        p_total += t.padded;
        t.s_acc = fnv1a64("gradaccum/" + name);
        t.s_m = fnv1a64("adamw/" + name + "/m");
        t.s_v = fnv1a64("adamw/" + name + "/v");
        t.s_w = fnv1a64("adamw/" + name + "/w");
        t.s_init = fnv1a64("init/" + name);
        pidx[name] = (int)P.size();
        P.push_back(t);
    }

    void build_params() {
        add_param("embed", {V, d});
        for (int l = 0; l < L; ++l) {
            const std::string pre = "layers." + std::to_string(l) + ".";
            add_param(pre + "ln1_g", {d});
            add_param(pre + "w_qkv", {q, d});
            add_param(pre + "w_o", {d, d});
            add_param(pre + "ln2_g", {d});
            add_param(pre + "w_gate_up", {F, d});
            add_param(pre + "w_down", {d, Hh});
        }
        add_param("final_g", {d});
        add_param("lm_head", {V, d});
        shard_total = 0;
        soff_of.clear();
        for (auto& t : P) {
            soff_of.push_back(shard_total);
            shard_total += t.pw;
        }
        // storage layout (world 1: offsets == the unsharded layout, params and grads alike)
        p_store = g_store = layer_g = p_master = 0;
        for (int i = 0; i < (int)P.size(); ++i) {
            ParamT& t = P[i];
            t.sharded = shard_weights() && is_block_weight(i);
            t.lo = t.sharded ? (int64_t)rank * t.pw : 0;
            t.store = t.sharded ? t.pw : t.padded;
            if (offload_master() && is_block_weight(i)) {  // placed in the host region (allocate)
                t.off = p_master;
                p_master += t.store;
            } else {
                t.off = p_store;
                p_store += t.store;
            }
            if (shard_grads() && i >= 1 && i <= 6 * L) {
                const int k = (i - 1) % 6;
                if (k == 0) layer_g = 0;
                t.loff = layer_g;
                layer_g += t.padded;
            } else {
                t.goff = g_store;
                g_store += t.padded;
            }
        }
        layer_shard = layer_g / std::max(world, 1);
    }
    // elements of tensor t stored on this rank ([lo, lo + n) of the tensor)
    int64_t stored(const ParamT& t) const { return std::max<int64_t>(0, std::min(t.store, t.numel - t.lo)); }
    // the gradient accumulator of tensor i (layer l's slot under shard_grads)
    uint16_t* gbuf(const ParamT& t) {
        if (t.goff >= 0) return grads + t.goff;
        const int pi = (int)(&t - P.data());
        return lgrad[((pi - 1) / 6) % 2] + t.loff;
    }
    const ParamT& par(const std::string& n) const { return P.at(pidx.at(n)); }
    uint16_t* pptr(const std::string& n) { return params + par(n).off; }
    uint16_t* gptr(const std::string& n) { return gbuf(par(n)); }
    int lp(int l, int k) const { return 1 + 6 * l + k; }  // k: 0 ln1 1 qkv 2 o 3 ln2 4 gu 5 down

    bool keep(int site) const {
        // KeepMask::from (src/model.cpp:221-235); RecomputeSite bits: 0 SwiGLU 1 RMSNorm 2 Attention 3 QKV 4 FFN 5 Block
        const int b = plan.recompute_bits;
        const bool block = b & (1 << 5);
        if (block) return false;
        switch (site) {
            case 0: return !(b & (1 << 1));                     // n1
            case 1: return !(b & (1 << 3));                     // qkv
            case 2: return !(b & (1 << 2));                     // att
            case 3: return true;                                // r_mid
            case 4: return !(b & (1 << 1));                     // n2
            case 5: return !(b & (1 << 4));                     // gate_up
            case 6: return !(b & (1 << 4)) && !(b & (1 << 0));  // h
        }
        return true;
    }

    void allocate() {
        struct Req {
            void** p;
            size_t bytes;
        };
        std::vector<Req> reqs, hreqs;
        auto req = [&](auto** p, size_t bytes) { reqs.push_back({reinterpret_cast<void**>(p), bytes}); };
        auto hreq = [&](auto** p, size_t bytes) { hreqs.push_back({reinterpret_cast<void**>(p), bytes}); };
        const int64_t M = Mmax;
        req(&params, p_store * 2);
        if (offload_master()) hreq(&hmaster, std::max<int64_t>(p_master, 1) * 2);
        if (offload_grads()) hreq(&grads, std::max<int64_t>(g_store, 1) * 2);
        else req(&grads, std::max<int64_t>(g_store, 1) * 2);
        {
            const size_t mb = plan.bf16_moments ? 2 : 4;
            auto mreq = [&](bool host, void** p) {
                if (host) hreqs.push_back({p, (size_t)shard_total * mb});
                else reqs.push_back({p, (size_t)shard_total * mb});
            };
            mreq(offload_m(), plan.bf16_moments ? (void**)&m16 : (void**)&m32);
            mreq(offload_v(), plan.bf16_moments ? (void**)&v16 : (void**)&v32);
            if (stream_moments()) {
                // groups of whole AdamW chunks, <= 32 Mi elements, streamed through 2 slots
                build_mgroups();
                for (int sl = 0; sl < 2; ++sl)
                    for (int k = 0; k < 2; ++k)
                        if ((k == 0 && offload_m()) || (k == 1 && offload_v()))
                            req(&mstage[sl][k], (size_t)mstage_elems * mb);
            }
        }
        if (world > 1) {
            req(&gshard, shard_total * 4);
            if (shard_grads()) {
                // the non-layer tensors (embed, final_g, lm_head) exchange through recvbuf at
                // the end; each layer through its own double-buffered receive area
                int64_t rest = 0;
                for (auto& t : P)
                    if (t.goff >= 0) rest += t.pw;
                req(&recvbuf, (size_t)world * rest * 2);
                for (int k = 0; k < 2; ++k) {
                    req(&lgrad[k], layer_g * 2);
                    req(&lrecv[k], (size_t)world * layer_shard * 2);
                }
            } else {
                req(&recvbuf, (size_t)world * shard_total * 2);
            }
        }
        wcodes.assign((size_t)L * 4, nullptr);
        {
            const int wk[4] = {1, 2, 4, 5};
            wl_total = 0;
            for (int k = 0; k < 4; ++k) {
                wl_off[k] = wl_total;
                wl_total += ceil_div(P[lp(0, wk[k])].padded, 128) * 128;
            }
        }
        if (!stream_codes()) {
            for (int l = 0; l < L; ++l) {
                req(&wcodes[l * 4 + W_QKV], (size_t)P[lp(l, 1)].padded);
                req(&wcodes[l * 4 + W_O], (size_t)P[lp(l, 2)].padded);
                req(&wcodes[l * 4 + W_GU], (size_t)P[lp(l, 4)].padded);
                req(&wcodes[l * 4 + W_DOWN], (size_t)P[lp(l, 5)].padded);
            }
        } else {
            for (int sl = 0; sl < 2; ++sl) req(&wslot[sl][0], (size_t)wl_total);
            if (shard_weights()) {
                wown.assign((size_t)L * 4, nullptr);
                const int wk[4] = {1, 2, 4, 5};
                for (int l = 0; l < L; ++l)
                    for (int k = 0; k < 4; ++k) req(&wown[l * 4 + k], (size_t)P[lp(l, wk[k])].pw);
            }
            if (offload_weights()) host_bytes += (size_t)L * wl_total;
        }
        lb.assign(L + 1, LayerBufs());
        // shared scratch for dropped sites
        LayerBufs sc;
        req(&sc.n1c, M * d);
        req(&sc.qkv, M * q * 2);
        req(&sc.att, M * d * 2);
        req(&sc.att32, M * d * 4);
        req(&sc.attc, M * d);
        req(&sc.lse, (size_t)plan.micro_batch * H * T * 4);
        req(&sc.r_mid, M * d * 2);
        req(&sc.n2c, M * d);
        req(&sc.gu, M * F * 2);
        req(&sc.hc, M * Hh);
        if (offload_x()) {  // two device slots + the host copy of r_in[0..L-1]
            req(&xslot[0], M * d * 2);
            req(&xslot[1], M * d * 2);
            req(&lb[L].r_in, M * d * 2);
            hreq(&xhost, (size_t)L * M * d * 2);
        } else {
            for (int l = 0; l <= L; ++l) req(&lb[l].r_in, M * d * 2);  // r_in[L] = r_final
        }
        std::vector<LayerBufs> own(L);
        for (int l = 0; l < L; ++l) {
            if (keep(0)) req(&own[l].n1c, M * d);
            if (keep(1)) req(&own[l].qkv, M * q * 2);
            if (keep(2)) {
                req(&own[l].att, M * d * 2);
                req(&own[l].att32, M * d * 4);
                req(&own[l].attc, M * d);
                req(&own[l].lse, (size_t)plan.micro_batch * H * T * 4);
            }
            if (keep(3)) req(&own[l].r_mid, M * d * 2);
            if (keep(4)) req(&own[l].n2c, M * d);
            if (keep(5)) req(&own[l].gu, M * F * 2);
            if (keep(6)) req(&own[l].hc, M * Hh);
        }
        req(&s_n1, M * d * 2);
        req(&s_attn_out, M * d * 2);
        req(&s_n2, M * d * 2);
        req(&s_h, M * Hh * 2);
        req(&normed_final, M * d * 2);
        req(&d_r, M * d * 2);
        req(&d_h, M * Hh * 2);
        req(&d_gu, M * F * 2);
        req(&d_n, M * d * 2);
        req(&d_ao, M * d * 2);
        req(&d_att, M * d * 2);
        req(&d_qkv, M * q * 2);
        req(&d_hidden, M * d * 2);
        req(&gcodes, M * std::max(F, q));
        if (wgrad_side()) req(&gcodes2, M * std::max(F, q));
        {
            // wgrad shapes (out, in, K = tokens) and small fwd/dgrad shapes
            const int64_t shapes[][3] = {{q, d, M}, {d, d, M}, {F, d, M}, {d, Hh, M}, {M, q, d}, {M, d, d},
                                         {M, F, d}, {M, d, Hh}, {M, Hh, d}, {M, d, F}, {M, d, q}};
            for (auto& sh : shapes)
                gemm_ws_bytes = std::max<int64_t>(gemm_ws_bytes, qtk_gemm_splitk_ws_bytes(sh[0], sh[1], sh[2], 0));
            if (gemm_ws_bytes > 0) req(&gemm_ws, gemm_ws_bytes);
            if (gemm_ws_bytes > 0 && wgrad_side()) req(&gemm_ws2, gemm_ws_bytes);
        }
        req(&logits, (size_t)M * V * 4);
        req(&dlogits, (size_t)M * V * 2);
        if (lm_tx()) {
            // split-K over the vocabulary keeps each tensor-core f32 accumulation chain short
            // (~19k terms): the chain's truncating adds drift by ~1e-4 relative over 152k terms
            lm_splits = (int)std::min<int64_t>(8, std::max<int64_t>(1, ceil_div(V, 16384)));
            lm_ws_bytes = lm_splits > 1 ? (int64_t)lm_splits * M * d * 4 : 0;
            if (lm_ws_bytes) req(&lm_ws, lm_ws_bytes);
            req(&lm_acc, (size_t)std::max<int64_t>(V, M) * d * 4);
            req(&dl_tgt, M * 4);
            req(&t_sorted_pos, M * 4);
            req(&t_seg_tok, M * 4);
            req(&t_seg_off, (M + 1) * 4);
            req(&t_nseg, 16);
        } else {
            req(&dlogits_lo, (size_t)M * V * 2);
        }
        req(&loss_rows, M * 4);
        req(&ce_stats, (size_t)M * ceil_div(V, 128) * 8);
        req(&ce_tgt, M * 4);
        // the fused and streaming backward paths need different scratch; size for the worst row count
        int nblk = 0;
        for (int64_t r = 1; r <= M; ++r) nblk = std::max(nblk, qtk_rmsnorm_bwd_partials(r, d));
        req(&dgamma_part, (size_t)nblk * d * 4);
        req(&dgamma, d * 4);
        req(&rms_inv, M * 4);
        req(&Dv, (size_t)plan.micro_batch * H * T * 4);
        {
            const size_t wb = qtk_attn_bwd_ws_bytes(plan.micro_batch, T, H, Hkv, hd);
            if (wb) req(&attn_ws, wb);
        }
        req(&rope_tab, (size_t)T * (hd / 2) * 8);
        req(&tok_buf, (size_t)plan.ga_steps * plan.micro_batch * (T + 1) * 4);
        req(&inputs, M * 4);
        req(&targets, M * 4);
        req(&sorted_pos, M * 4);
        req(&seg_tok, M * 4);
        req(&seg_off, (M + 1) * 4);
        req(&nseg, 16);
        sort_scratch_bytes = qtk_embed_sort_scratch_bytes((int)M, V);
        req(&sort_scratch, sort_scratch_bytes);
        // norm partials sized for the largest buffer the norm runs over
        norm_blocks = 0;
        for (auto& t : P) norm_blocks += ceil_div(world > 1 ? t.pw : t.numel, 256);
        req(&norm_partials, norm_blocks * 8);
        req(&norm_scratch, 1024 * 8);
        req(&segs_dev, P.size() * sizeof(SegH));
        {
            int64_t nch = 0;
            const int64_t cs = qtk_adamw_chunk_size();
            for (auto& t : P) nch += ceil_div(world > 1 ? t.pw : t.numel, cs);
            req(&chunks_dev, nch * qtk_adamw_chunk_entry_size());
        }
        req(&act_amax, L * 16);
        req(&act_scale, L * 16);
        req(&w_amax, L * 16);
        req(&w_scale, L * 16);
        req(&g_amax, L * 16);
        req(&g_scale, L * 16);
        req(&fin_amax, 16);
        req(&seg_amax, P.size() * 4);
        req(&step_blk, 16 + 8 * (size_t)std::max(plan.ga_steps, 1));
        req(&loss_dev, std::max(plan.ga_steps, 1) * 4 + 16);
        req(&ssq_dev, 16);
        req(&norm_dev, 16);
        req(&gscale_dev, 16);
        req(&err_dev, 16);
        int64_t maxp = 0;
        for (auto& t : P) maxp = std::max(maxp, t.padded);
        req(&scratch_f32, maxp * 4);

        size_t total = 0;
        for (auto& r : reqs) total += (r.bytes + 255) & ~size_t(255);
        size_t htotal = 0;
        for (auto& r : hreqs) htotal += (r.bytes + 4095) & ~size_t(4095);
        host_bytes += htotal;
        if (dry) {
            arena_bytes = total;
            return;
        }
        if (htotal) {
            QT_CHECK_CUDA(cudaMallocHost(&harena, htotal));
            std::memset(harena, 0, htotal);
            harena_bytes = htotal;
            size_t ho = 0;
            for (auto& r : hreqs) {
                *r.p = harena + ho;
                ho += (r.bytes + 4095) & ~size_t(4095);
            }
        }
        QT_CHECK_CUDA(cudaMalloc(&arena, total));
        arena_bytes = total;
        QT_CHECK_CUDA(cudaMemsetAsync(arena, 0, total, st));
        size_t off = 0;
        for (auto& r : reqs) {
            *r.p = arena + off;
            off += (r.bytes + 255) & ~size_t(255);
        }
        if (offload_x())
            for (int l = 0; l < L; ++l) lb[l].r_in = xslot[l % 2];
        if (offload_master())  // block weights in the host region, addressed from the params base (UVA)
            for (int i = 0; i < (int)P.size(); ++i)
                if (is_block_weight(i)) P[i].off += (int64_t)(hmaster - params);
        for (int l = 0; l < L; ++l) {
            LayerBufs& b = lb[l];
            b.n1c = own[l].n1c ? own[l].n1c : sc.n1c;
            b.qkv = own[l].qkv ? own[l].qkv : sc.qkv;
            b.att = own[l].att ? own[l].att : sc.att;
            b.att32 = own[l].att32 ? own[l].att32 : sc.att32;
            b.attc = own[l].attc ? own[l].attc : sc.attc;
            b.lse = own[l].lse ? own[l].lse : sc.lse;
            b.r_mid = own[l].r_mid ? own[l].r_mid : sc.r_mid;
            b.gu = own[l].gu ? own[l].gu : sc.gu;
            b.n2c = own[l].n2c ? own[l].n2c : sc.n2c;
            b.hc = own[l].hc ? own[l].hc : sc.hc;
            b.keep_all = keep(0) && keep(1) && keep(2) && keep(3) && keep(4) && keep(5) && keep(6);
        }
    }

    // AdamW / norm segments for this rank (ZeRO-1 slices when world > 1)
    struct ChunkH {
        int32_t seg, pad;
        int64_t start;
    };
    std::vector<SegH> segs_h;
    std::vector<ChunkH> chunks_h;
    // the AdamW / norm segments and chunk table on the host (params offsets final: after allocate)
    void make_segments() {
        std::vector<SegH>& segs = segs_h;
        segs.clear();
        int64_t blk = 0, soff = 0;
        for (auto& t : P) {
            SegH s{};
            if (world == 1) {
                s.off = t.goff;  // gradient and moment offset (== the params offset unless offloaded)
                s.n = t.numel;
                s.gstart = 0;
                s.poff = t.off;
            } else {
                const int64_t lo = std::min<int64_t>((int64_t)rank * t.pw, t.numel);
                const int64_t hi = std::min<int64_t>((int64_t)(rank + 1) * t.pw, t.numel);
                s.off = soff;
                s.n = hi - lo;
                s.gstart = (int64_t)rank * t.pw;
                s.poff = t.sharded ? t.off : t.off + (int64_t)rank * t.pw;
                soff += t.pw;
            }
            s.gnumel = t.numel;
            s.sm = t.s_m;
            s.sv = t.s_v;
            s.sw = t.s_w;
            s.blk0 = blk;
            blk += ceil_div(s.n, 256);
            segs.push_back(s);
        }
        // norm blocks in name (std::map) order are not needed for the tree sum; layout order is used
        norm_blocks = blk;
        nsegs = (int)segs.size();
        chunks_h.clear();
        const int64_t cs = qtk_adamw_chunk_size();
        for (int i = 0; i < nsegs; ++i)
            for (int64_t s0 = 0; s0 < segs[i].n; s0 += cs) chunks_h.push_back({i, 0, s0});
        nchunks = (int)chunks_h.size();
    }
    // double-buffered moments: consecutive chunks grouped to <= 32 Mi moment elements
    void build_mgroups() {
        make_segments();
        mgroups.clear();
        // groups of <= 32 Mi moment elements, and at least 8 groups for small models (the two
        // device slots then hold a quarter of the moments at most)
        const int64_t cs = qtk_adamw_chunk_size();
        int64_t tot = 0;
        for (const SegH& sg : segs_h) tot += sg.n;
        const int64_t cap = std::max<int64_t>(std::min<int64_t>(int64_t(32) << 20, ceil_div(tot, 8)), cs);
        mstage_elems = 0;
        int c0 = 0;
        while (c0 < nchunks) {
            const int64_t e0 = segs_h[chunks_h[c0].seg].off + chunks_h[c0].start;
            int c1 = c0;
            int64_t e1 = e0;
            while (c1 < nchunks) {
                const SegH& sg = segs_h[chunks_h[c1].seg];
                const int64_t end = sg.off + std::min(chunks_h[c1].start + cs, sg.n);
                if (c1 > c0 && end - e0 > cap) break;
                e1 = end;
                ++c1;
            }
            mgroups.push_back({c0, c1, e0, e1});
            mstage_elems = std::max(mstage_elems, ceil_div(e1 - e0, 4) * 4 + 4);
            c0 = c1;
        }
    }
    void build_segments() {
        if ((int)sizeof(SegH) != qtk_seg_size()) throw QtError(3, "Seg layout mismatch");
        if ((int)sizeof(ChunkH) != qtk_adamw_chunk_entry_size()) throw QtError(3, "AdamW chunk layout mismatch");
        make_segments();
        if (stream_moments()) build_mgroups();
        QT_CHECK_CUDA(cudaMemcpyAsync(segs_dev, segs_h.data(), segs_h.size() * sizeof(SegH), cudaMemcpyHostToDevice,
                                      st));
        QT_CHECK_CUDA(cudaMemcpyAsync(chunks_dev, chunks_h.data(), chunks_h.size() * sizeof(ChunkH),
                                      cudaMemcpyHostToDevice, st));
        QT_CHECK_CUDA(cudaStreamSynchronize(st));
    }

    void build_rope_table() {
        std::vector<float2> tab((size_t)T * (hd / 2));
        rope_table_host(T, hd, tab.data());
        QT_CHECK_CUDA(cudaMemcpyAsync(rope_tab, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice, st));
        QT_CHECK_CUDA(cudaStreamSynchronize(st));
    }

    // ---------------- profiling ----------------
    int prof_begin() { return prof_begin_on(st); }
    int prof_begin_on(cudaStream_t ss) {
        if (!prof_on) return -1;
        if (ev_used + 2 > ev_pool.size()) {
            for (int i = 0; i < 256; ++i) {
                cudaEvent_t e;
                cudaEventCreate(&e);
                ev_pool.push_back(e);
            }
        }
        cudaEvent_t a = ev_pool[ev_used++], b = ev_pool[ev_used++];
        cudaEventRecord(a, ss);
        prof.push_back({0, a, b, 0.0});
        return (int)prof.size() - 1;
    }
    void prof_end(int h, int cat, double work) { prof_end_on(h, cat, work, st); }
    void prof_end_on(int h, int cat, double work, cudaStream_t ss) {
        if (h < 0) return;
        prof[h].cat = cat;
        prof[h].work = work;
        cudaEventRecord(prof[h].b, ss);
    }

    // ---------------- GEMM helper ----------------
    void gemm(int kind, int afmt, int bfmt, bool a_mn, bool b_mn, int64_t M, int64_t N, int64_t K, const void* a,
              int64_t lda, const void* b, int64_t ldb, const float* as, const float* bs, int epi, void* out,
              int64_t ldo, const void* res = nullptr, int64_t ldr = 0, uint64_t sr_seed = 0, uint64_t sr_stream = 0,
              uint64_t sr_base = 0, const void* a2 = nullptr, uint32_t* amax = nullptr, const int32_t* ce_targets = nullptr,
              float* ce_st = nullptr, float* ce_tl = nullptr, float* ws = nullptr, int64_t ws_bytes = 0,
              int split_k = 0, cudaStream_t on = nullptr) {
        QtkGemm g{};
        g.kind = kind;
        g.a_fmt = afmt;
        g.b_fmt = bfmt;
        g.a_mn = a_mn;
        g.b_mn = b_mn;
        g.M = M;
        g.N = N;
        g.K = K;
        g.a = a;
        g.lda = lda;
        g.b = b;
        g.ldb = ldb;
        g.a_scale = as;
        g.b_scale = bs;
        g.epi = epi;
        g.out = out;
        g.ldo = ldo;
        g.res = res;
        g.ldr = ldr;
        g.sr_seed = sr_seed;
        g.sr_stream = sr_stream;
        g.sr_base = sr_base;
        g.bn = 0;
        g.a2 = a2;
        g.ws = ws ? ws : (on && on == wst ? gemm_ws2 : gemm_ws);  // each stream its own split-K workspace
        g.ws_bytes = ws ? ws_bytes : gemm_ws_bytes;
        g.split_k = ws ? split_k : 0;
        g.amax = amax;
        if (use_dev_ctr && (epi == EPI_BF16_ACC || epi == EPI_F32_ACC)) g.sr_micro_step = ms_dev(cur_ga);
        g.ce_targets = ce_targets;
        g.ce_stats = ce_st;
        g.ce_tgt_logit = ce_tl;
        cudaStream_t gs_ = on ? on : st;
        const int h = prof_begin_on(gs_);
        QT_CHECK_K(qtk_gemm(&g, gs_));
        prof_end_on(h, kind == 0 ? 0 : 1, 2.0 * M * N * K * (a2 ? 2 : 1), gs_);
    }

    int gkind() const { return prec.backward_grads == 0 ? kE4M3 : kE5M2; }
    // a collective through the transport; its failures surface as runtime_error (status 3)
    template <typename F>
    void coll(F&& f) {
        try {
            f();
        } catch (const TransportError& e) {
            throw QtError(3, e.what());
        }
    }
    bool ce_stats_on() const {
        static int f = -1;
        if (f < 0) {
            const char* e = getenv("QTB_CE_STATS");
            f = e ? atoi(e) : 1;
        }
        return f != 0 && V % 4 == 0;  // TMA-stored f32 logits rows
    }
    // target-exact CE backward: bf16 dlogits without the target entry + the exact f32 target
    // term (QTB_LM_TX=0: the bf16 hi + lo split-A path)
    // attention backward: dQ on the side stream next to dK/dV (QTB_ATTN_2S)
    static bool attn_two_streams() {
        static int f = -1;
        if (f < 0) {
            const char* e = getenv("QTB_ATTN_2S");
            f = e ? atoi(e) : 1;
        }
        return f != 0 && wgrad_side();
    }
    static bool wgrad_side() {
        static int f = -1;
        if (f < 0) {
            const char* e = getenv("QTB_WGRAD_SIDE");
            f = e ? atoi(e) : 1;
        }
        return f != 0;
    }
    // side stream in use for this backward (not while profiling: the per-class event brackets
    // time kernels one at a time)
    bool side_on() const { return wgrad_side() && wst && !prof_on; }
    bool lm_tx() const {
        static int f = -1;
        if (f < 0) {
            const char* e = getenv("QTB_LM_TX");
            f = e ? atoi(e) : 1;
        }
        return f != 0 && ce_stats_on() && d % 4 == 0;
    }
    bool fuse_swiglu_bwd() const {
        static int f = -1;
        if (f < 0) {
            // off by default: the sigmoid/exp math concentrated in 8 epilogue warps per SM costs
            // more than the d_h round trip it saves (measured +70 us/layer at 0.5B)
            const char* e = getenv("QTB_FUSE_SWIGLU_BWD");
            f = e ? atoi(e) : 0;
        }
        return f && Hh % 64 == 0;
    }

    // ---------------- StepContext (src/model.cpp:88-107) ----------------
    bool shard_weights() const { return plan.shard_weights && world > 1; }
    // RunPlan::offload.weights: the FP8 codes live in pinned host memory, two layer slots on
    // the device (memplan.hpp:34-52; with shard_weights this is the paper's host weight cache)
    bool offload_weights() const { return (plan.offload_bits & QT_OFF_WEIGHTS) != 0; }
    bool offload_master() const { return (plan.offload_bits & QT_OFF_MASTER) != 0; }
    bool offload_m() const { return (plan.offload_bits & QT_OFF_M) != 0; }
    bool offload_v() const { return (plan.offload_bits & QT_OFF_V) != 0; }
    bool offload_grads() const { return (plan.offload_bits & QT_OFF_GRADS) != 0; }
    bool offload_x() const { return (plan.offload_bits & QT_OFF_X) != 0; }
    bool zero_copy() const { return plan.transfer_policy == QT_XFER_ZERO_COPY; }
    // moments streamed through device slots (double-buffer policy)
    bool stream_moments() const { return (offload_m() || offload_v()) && !zero_copy(); }
    // the block weights' codes are streamed per layer (not all resident)
    bool stream_codes() const { return shard_weights() || offload_weights(); }
    // the codes of weight k (W_QKV, W_O, W_GU, W_DOWN) of layer l
    const uint8_t* wc(int l, int k) const {
        if (!stream_codes()) return wcodes[l * 4 + k];
        return wslot[l % 2][0] + wl_off[k];
    }
    bool shard_grads() const { return plan.shard_grads && world > 1; }
    // w_qkv, w_o, w_gate_up, w_down of some layer (for_each_param order, model.hpp:107-121)
    bool is_block_weight(int pi) const {
        if (pi < 1 || pi > 6 * L) return false;
        const int k = (pi - 1) % 6;
        return k == 1 || k == 2 || k == 4 || k == 5;
    }

    void build_step_context() {
        QT_CHECK_CUDA(cudaMemsetAsync(w_amax, 0, L * 16, st));
        slot_layer[0] = slot_layer[1] = -1;  // last step's codes are stale
        if (stream_codes()) published.assign((size_t)L, 0);
        if (shard_weights()) {
            // RunPlan::shard_weights: each rank holds only its ZeRO-1 slice of the block
            // weights.  Per-tensor absmax = max over the ranks' slice maxima (all-reduce MAX of
            // the u32 |x| patterns), each rank casts its slice with that scale into its own
            // slice codes; the forward/backward all-gather the E4M3 codes (1 B/param) one layer
            // ahead (fetch_layer).  Codes equal a cast of the full tensor bit for bit.
            for (int l = 0; l < L; ++l) {
                const int widx[4] = {lp(l, 1), lp(l, 2), lp(l, 4), lp(l, 5)};
                for (int k = 0; k < 4; ++k) {
                    const ParamT& t = P[widx[k]];
                    const int64_t n = stored(t);
                    if (n > 0) QT_CHECK_K(qtk_absmax_bf16(params + t.off, n, w_amax + l * 4 + k, st));
                }
            }
            coll([&] { tr->allreduce_max_u32(w_amax, (size_t)L * 4, st); });
            weight_scale_kernel<<<(unsigned)ceil_div(L * 4, 128), 128, 0, st>>>(w_amax, w_scale, L * 4);  // ranks with an empty slice
            QT_CHECK_CUDA(cudaGetLastError());
            for (int l = 0; l < L; ++l) {
                const int widx[4] = {lp(l, 1), lp(l, 2), lp(l, 4), lp(l, 5)};
                for (int k = 0; k < 4; ++k) {
                    const ParamT& t = P[widx[k]];
                    const int64_t n = stored(t);
                    const int h = prof_begin();
                    if (n > 0)
                        QT_CHECK_K(qtk_quantize_bf16(params + t.off, n, kE4M3, w_amax + l * 4 + k, wown[l * 4 + k],
                                                     w_scale + l * 4 + k, st));
                    prof_end(h, 3, 3.0 * n);
                }
            }
            QT_CHECK_CUDA(cudaEventRecord(ev_codes, st));  // the slice codes are ready
            return;
        }
        if (amax_cached) {  // the absmax AdamW folded in while writing these weights
            gather_wamax_kernel<<<(unsigned)ceil_div(L * 4, 128), 128, 0, st>>>(seg_amax, w_amax, L);
            QT_CHECK_CUDA(cudaGetLastError());
        }
        for (int l = 0; l < L; ++l) {
            const int widx[4] = {lp(l, 1), lp(l, 2), lp(l, 4), lp(l, 5)};
            for (int k = 0; k < 4; ++k) {
                const ParamT& t = P[widx[k]];
                const int h = prof_begin();
                if (!amax_cached) QT_CHECK_K(qtk_absmax_bf16(params + t.off, t.numel, w_amax + l * 4 + k, st));
                // offload.weights: cast into a device slot, then publish to the host cache
                uint8_t* dst = offload_weights() ? wslot[l % 2][0] + wl_off[k] : wcodes[l * 4 + k];
                QT_CHECK_K(qtk_quantize_bf16(params + t.off, t.numel, kE4M3, w_amax + l * 4 + k, dst,
                                             w_scale + l * 4 + k, st));
                prof_end(h, 3, 3.0 * t.numel);
            }
            if (offload_weights()) {
                QT_CHECK_CUDA(cudaMemcpyAsync(whost + (size_t)l * wl_total, wslot[l % 2][0], (size_t)wl_total,
                                              cudaMemcpyDeviceToHost, st));
                QT_CHECK_CUDA(cudaEventRecord(ev_wready[l % 2], st));
                published[(size_t)l] = 1;
                slot_layer[l % 2] = l;
            }
        }
        if (stream_codes()) QT_CHECK_CUDA(cudaEventRecord(ev_codes, st));  // codes (and slots) written
    }

    // ---------------- streamed weight codes (shard_weights / offload.weights) ----------------
    // fetch_layer(l) fills slot l%2 with layer l's codes on the communication stream once the
    // slot's previous user finished (ev_wfree), and records ev_wready.  Source: the peers'
    // slices (all-gather; with offload.weights also published to the host cache, so later
    // passes of this step read the host copy), or the host cache.  Every rank takes the same
    // decisions, so the collectives line up.
    void fetch_layer(int l) {
        const int sl = l % 2;
        if (slot_layer[sl] == l) return;
        QT_CHECK_CUDA(cudaStreamWaitEvent(cst, ev_wfree[sl], 0));
        QT_CHECK_CUDA(cudaStreamWaitEvent(cst, ev_codes, 0));  // this step's codes exist
        const int h = prof_begin_on(cst);
        if (shard_weights() && !published[(size_t)l]) {
            const int widx[4] = {lp(l, 1), lp(l, 2), lp(l, 4), lp(l, 5)};
            std::vector<GatherItem> items;
            for (int k = 0; k < 4; ++k)
                items.push_back({wown[l * 4 + k], wslot[sl][0] + wl_off[k], (size_t)P[widx[k]].pw});
            coll([&] { tr->allgather_to(items, cst); });
            if (offload_weights()) {
                QT_CHECK_CUDA(cudaMemcpyAsync(whost + (size_t)l * wl_total, wslot[sl][0], (size_t)wl_total,
                                              cudaMemcpyDeviceToHost, cst));
                published[(size_t)l] = 1;
            }
        } else {
            QT_CHECK_CUDA(cudaMemcpyAsync(wslot[sl][0], whost + (size_t)l * wl_total, (size_t)wl_total,
                                          cudaMemcpyHostToDevice, cst));
        }
        prof_end_on(h, 9, (double)wl_total, cst);
        QT_CHECK_CUDA(cudaEventRecord(ev_wready[sl], cst));
        slot_layer[sl] = l;
    }
    // before layer l's compute: its codes are in the slot (prefetching l+dir meanwhile)
    void codes_acquire(int l, int next) {
        if (!stream_codes()) return;
        fetch_layer(l);
        if (next >= 0 && next < L) fetch_layer(next);
        QT_CHECK_CUDA(cudaStreamWaitEvent(st, ev_wready[l % 2], 0));
    }
    // after layer l's compute: its slot may be refilled
    void codes_release(int l) {
        if (!stream_codes()) return;
        QT_CHECK_CUDA(cudaEventRecord(ev_wfree[l % 2], st));
    }

    // ---------------- offloaded residuals (offload.x) ----------------
    // before the compute stream writes r_in[l] into its slot: the slot's previous content is
    // on the host (forward write-back) or no longer read (backward)
    void x_before_write(int l) { QT_CHECK_CUDA(cudaStreamWaitEvent(st, ev_xfree[l % 2], 0)); }
    // r_in[l] was just produced in its slot: copy it to the host on the copy engine
    void x_publish(int l) {
        const int sl = l % 2;
        const size_t bytes = (size_t)curM * d * 2;
        QT_CHECK_CUDA(cudaEventRecord(ev_xready[sl], st));
        QT_CHECK_CUDA(cudaStreamWaitEvent(cst, ev_xready[sl], 0));
        QT_CHECK_CUDA(cudaMemcpyAsync(xhost + (size_t)l * Mmax * d, xslot[sl], bytes, cudaMemcpyDeviceToHost, cst));
        QT_CHECK_CUDA(cudaEventRecord(ev_xfree[sl], cst));
        xslot_layer[sl] = l;
    }
    void x_fetch(int l) {
        const int sl = l % 2;
        if (xslot_layer[sl] == l) return;
        QT_CHECK_CUDA(cudaStreamWaitEvent(cst, ev_xfree[sl], 0));
        QT_CHECK_CUDA(cudaMemcpyAsync(xslot[sl], xhost + (size_t)l * Mmax * d, (size_t)curM * d * 2,
                                      cudaMemcpyHostToDevice, cst));
        QT_CHECK_CUDA(cudaEventRecord(ev_xready[sl], cst));
        xslot_layer[sl] = l;
    }
    // backward of layer l: r_in[l] in its slot (r_in[next] prefetched)
    void x_acquire(int l, int next) {
        x_fetch(l);
        if (next >= 0) x_fetch(next);
        QT_CHECK_CUDA(cudaStreamWaitEvent(st, ev_xready[l % 2], 0));
    }

    // ---------------- block forward (src/model.cpp:239-293) ----------------
    void block_forward(int l, bool record) {
        LayerBufs& b = lb[l];
        const int64_t M = curM;
        uint32_t* am = act_amax + l * 4;
        float* sc = act_scale + l * 4;
        const float* ws = w_scale + l * 4;
        const ParamT& ln1 = P[lp(l, 0)];
        const ParamT& ln2 = P[lp(l, 3)];
        int h;
        // rmsnorm1 (pass-through residual) + N1 absmax
        h = prof_begin();
        QT_CHECK_K(qtk_rmsnorm_fwd(nullptr, b.r_in, params + ln1.off, M, d, 1e-6f, nullptr, s_n1, rms_inv,
                                   record ? am + S_N1 : nullptr, st));
        prof_end(h, 4, 4.0 * M * d);
        h = prof_begin();
        QT_CHECK_K(qtk_quantize_bf16(s_n1, M * d, kE4M3, am + S_N1, b.n1c, sc + S_N1, st));
        prof_end(h, 3, 3.0 * M * d);
        gemm(0, kE4M3, kE4M3, false, false, M, q, d, b.n1c, d, wc(l, W_QKV), d, sc + S_N1, ws + W_QKV, EPI_BF16,
             b.qkv, q);
        h = prof_begin();
        QT_CHECK_K(qtk_rope(b.qkv, M, curT, H + Hkv, hd, q, rope_tab, 0, nullptr, st));
        prof_end(h, 5, 4.0 * M * (d + Hkv * hd));
        h = prof_begin();
        QT_CHECK_K(qtk_attn_fwd(b.qkv, curB, curT, H, Hkv, hd, q, b.att, d, b.att32, b.lse,
                                record ? am + S_ATT : nullptr, st));
        prof_end(h, 6, 4.0 * curB * H * (double)curT * curT / 2 * hd);
        h = prof_begin();
        QT_CHECK_K(qtk_quantize_bf16(b.att, M * d, kE4M3, am + S_ATT, b.attc, sc + S_ATT, st));
        prof_end(h, 3, 3.0 * M * d);
        gemm(0, kE4M3, kE4M3, false, false, M, d, d, b.attc, d, wc(l, W_O), d, sc + S_ATT, ws + W_O, EPI_BF16,
             s_attn_out, d);
        h = prof_begin();
        QT_CHECK_K(qtk_rmsnorm_fwd(s_attn_out, b.r_in, params + ln2.off, M, d, 1e-6f, b.r_mid, s_n2, rms_inv,
                                   record ? am + S_N2 : nullptr, st));
        prof_end(h, 4, 8.0 * M * d);
        h = prof_begin();
        QT_CHECK_K(qtk_quantize_bf16(s_n2, M * d, kE4M3, am + S_N2, b.n2c, sc + S_N2, st));
        prof_end(h, 3, 3.0 * M * d);
        gemm(0, kE4M3, kE4M3, false, false, M, F, d, b.n2c, d, wc(l, W_GU), d, sc + S_N2, ws + W_GU, EPI_BF16,
             b.gu, F);
        h = prof_begin();
        QT_CHECK_K(qtk_swiglu_fwd(b.gu, M, Hh, s_h, record ? am + S_H : nullptr, st));
        prof_end(h, 5, 2.0 * M * F + 2.0 * M * Hh);
        h = prof_begin();
        QT_CHECK_K(qtk_quantize_bf16(s_h, M * Hh, kE4M3, am + S_H, b.hc, sc + S_H, st));
        prof_end(h, 3, 3.0 * M * Hh);
        // r_out = bf16(bf16(h . Wdown^T) + r_mid)  (model.cpp:281-283) -> next layer's r_in
        gemm(0, kE4M3, kE4M3, false, false, M, d, Hh, b.hc, Hh, wc(l, W_DOWN), Hh, sc + S_H, ws + W_DOWN,
             EPI_BF16_RES, lb[l + 1].r_in, d, b.r_mid, d);
    }

    // Backward-time recompute of the dropped sites of layer l only (KeepMask, model.cpp:221-235,
    // replay with the forward's cached statistics, :374-378): each dropped site is rebuilt from
    // the nearest kept (or rebuilt) input; kept sites are not touched and the block output
    // (the next layer's residual) is never recomputed.  Bitwise the forward's values.
    void block_replay(int l) {
        LayerBufs& b = lb[l];
        const int64_t M = curM;
        uint32_t* am = act_amax + l * 4;
        float* sc = act_scale + l * 4;
        const float* ws = w_scale + l * 4;
        const ParamT& ln1 = P[lp(l, 0)];
        const ParamT& ln2 = P[lp(l, 3)];
        int h;
        if (!keep(0)) {  // n1 codes (qkv wgrad, qkv recompute)
            h = prof_begin();
            QT_CHECK_K(qtk_rmsnorm_fwd(nullptr, b.r_in, params + ln1.off, M, d, 1e-6f, nullptr, s_n1, rms_inv, nullptr,
                                       st));
            prof_end(h, 4, 4.0 * M * d);
            h = prof_begin();
            QT_CHECK_K(qtk_quantize_bf16(s_n1, M * d, kE4M3, am + S_N1, b.n1c, sc + S_N1, st));
            prof_end(h, 3, 3.0 * M * d);
        }
        if (!keep(1)) {  // post-RoPE qkv
            gemm(0, kE4M3, kE4M3, false, false, M, q, d, b.n1c, d, wc(l, W_QKV), d, sc + S_N1, ws + W_QKV, EPI_BF16,
                 b.qkv, q);
            h = prof_begin();
            QT_CHECK_K(qtk_rope(b.qkv, M, curT, H + Hkv, hd, q, rope_tab, 0, nullptr, st));
            prof_end(h, 5, 4.0 * M * (d + Hkv * hd));
        }
        if (!keep(2)) {  // attention output (bf16, f32, codes) + LSE
            h = prof_begin();
            QT_CHECK_K(qtk_attn_fwd(b.qkv, curB, curT, H, Hkv, hd, q, b.att, d, b.att32, b.lse, nullptr, st));
            prof_end(h, 6, 4.0 * curB * H * (double)curT * curT / 2 * hd);
            h = prof_begin();
            QT_CHECK_K(qtk_quantize_bf16(b.att, M * d, kE4M3, am + S_ATT, b.attc, sc + S_ATT, st));
            prof_end(h, 3, 3.0 * M * d);
        }
        if (!keep(3)) {  // r_mid (block recompute): out-projection + fused residual rmsnorm
            gemm(0, kE4M3, kE4M3, false, false, M, d, d, b.attc, d, wc(l, W_O), d, sc + S_ATT, ws + W_O, EPI_BF16,
                 s_attn_out, d);
            h = prof_begin();
            QT_CHECK_K(qtk_rmsnorm_fwd(s_attn_out, b.r_in, params + ln2.off, M, d, 1e-6f, b.r_mid, s_n2, rms_inv,
                                       nullptr, st));
            prof_end(h, 4, 8.0 * M * d);
        } else if (!keep(4)) {  // n2 from the kept r_mid (pass-through residual: same bits)
            h = prof_begin();
            QT_CHECK_K(qtk_rmsnorm_fwd(nullptr, b.r_mid, params + ln2.off, M, d, 1e-6f, nullptr, s_n2, rms_inv,
                                       nullptr, st));
            prof_end(h, 4, 4.0 * M * d);
        }
        if (!keep(4)) {
            h = prof_begin();
            QT_CHECK_K(qtk_quantize_bf16(s_n2, M * d, kE4M3, am + S_N2, b.n2c, sc + S_N2, st));
            prof_end(h, 3, 3.0 * M * d);
        }
        if (!keep(5))
            gemm(0, kE4M3, kE4M3, false, false, M, F, d, b.n2c, d, wc(l, W_GU), d, sc + S_N2, ws + W_GU, EPI_BF16,
                 b.gu, F);
        if (!keep(6)) {
            h = prof_begin();
            QT_CHECK_K(qtk_swiglu_fwd(b.gu, M, Hh, s_h, nullptr, st));
            prof_end(h, 5, 2.0 * M * F + 2.0 * M * Hh);
            h = prof_begin();
            QT_CHECK_K(qtk_quantize_bf16(s_h, M * Hh, kE4M3, am + S_H, b.hc, sc + S_H, st));
            prof_end(h, 3, 3.0 * M * Hh);
        }
    }

    // ---------------- model_forward (src/model.cpp:297-352) ----------------
    void forward(const int32_t* tokens, int64_t n_tokens, int64_t batch, bool with_grads) {
        if (batch < 1 || n_tokens % batch != 0) throw QtError(1, "model_forward: token count not divisible by batch");
        const int64_t seq = n_tokens / batch - 1;
        if (seq < 1 || seq > cfg.seq_len) throw QtError(1, "model_forward: bad sequence length");
        if (batch * seq > Mmax) throw QtError(1, "model_forward: batch exceeds the session's micro_batch");
        curB = (int)batch;
        curT = (int)seq;
        curM = batch * seq;
        const int64_t M = curM;
        QT_CHECK_CUDA(cudaMemsetAsync(act_amax, 0, L * 16, st));
        QT_CHECK_CUDA(cudaMemsetAsync(fin_amax, 0, 4, st));
        int h = prof_begin();
        if (offload_x()) x_before_write(0);
        QT_CHECK_K(qtk_embed_fwd(tokens, curB, curT, params + par("embed").off, d, V, lb[0].r_in, inputs, targets,
                                 err_dev, st));
        prof_end(h, 5, 4.0 * M * d);
        if (offload_x()) x_publish(0);
        if (with_grads) QT_CHECK_K(qtk_embed_sort(inputs, (int)M, V, sort_scratch, sort_scratch_bytes, sorted_pos,
                                                  seg_tok, seg_off, nseg, st));
        for (int l = 0; l < L; ++l) {
            codes_acquire(l, l + 1);
            if (offload_x() && l + 1 < L) x_before_write(l + 1);
            block_forward(l, true);
            codes_release(l);
            if (offload_x() && l + 1 < L) x_publish(l + 1);
        }
        h = prof_begin();
        QT_CHECK_K(qtk_rmsnorm_fwd(nullptr, lb[L].r_in, pptr("final_g"), M, d, 1e-6f, nullptr, normed_final, rms_inv,
                                   fin_amax, st));
        prof_end(h, 4, 4.0 * M * d);
        // fused CE forward (+ dlogits for the backward): logits in f32 (tensorops.cpp:372-376)
        if (ce_stats_on()) {
            // the logits GEMM also emits per-row (max, sum exp) of each 128-column block and the
            // target logit, so the softmax stage reads the logits once
            gemm(1, 0, 0, false, false, M, V, d, normed_final, d, pptr("lm_head"), d, nullptr, nullptr, EPI_F32, logits,
                 V, nullptr, 0, 0, 0, 0, nullptr, nullptr, targets, ce_stats, ce_tgt);
            h = prof_begin();
            if (lm_tx() && with_grads) {
                QT_CHECK_K(qtk_ce_softmax_stats_tx(logits, V, M, (int)V, targets, ce_stats, ce_tgt, 1.0f / (float)M,
                                                   dlogits, V, loss_rows, dl_tgt, st));
                prof_end(h, 7, 6.0 * M * V);
                // positions grouped by target (stable: ascending within a target) for d_lm_w's target terms
                h = prof_begin();
                QT_CHECK_K(qtk_embed_sort(targets, (int)M, V, sort_scratch, sort_scratch_bytes, t_sorted_pos,
                                          t_seg_tok, t_seg_off, t_nseg, st));
                prof_end(h, 5, 0.0);
            } else {
                QT_CHECK_K(qtk_ce_softmax_stats(logits, V, M, (int)V, targets, ce_stats, ce_tgt, 1.0f / (float)M,
                                                with_grads ? dlogits : nullptr, with_grads ? dlogits_lo : nullptr, V,
                                                loss_rows, st));
                prof_end(h, 7, (with_grads ? 8.0 : 0.0) * M * V);
            }
        } else {
            gemm(1, 0, 0, false, false, M, V, d, normed_final, d, pptr("lm_head"), d, nullptr, nullptr, EPI_F32, logits,
                 V);
            h = prof_begin();
            QT_CHECK_K(qtk_ce_softmax(logits, V, M, (int)V, targets, 1.0f / (float)M, with_grads ? dlogits : nullptr,
                                      with_grads ? dlogits_lo : nullptr, V, loss_rows, st));
            prof_end(h, 7, (with_grads ? 10.0 : 4.0) * M * V);
        }
        QT_CHECK_K(qtk_loss_reduce(loss_rows, M, 1.0f / (float)M, loss_dev, nullptr, st));
        have_fwd = true;
        fwd_with_grads = with_grads;
    }

    // ---------------- grad-kind casts and weight gradients (side stream) ----------------
    int gbuf_i = 0;
    bool wdone_valid[2] = {false, false};  // ev_wdone[k] recorded in this backward
    // the full gradient buffer is all zeros (zeroed and not yet accumulated into)
    bool grads_fresh = false;
    // absmax-scaled cast of a d_out into the next grad-codes buffer (waiting for the wgrad that
    // read that buffer two casts ago); the side stream may read it after this
    uint8_t* quant_grad(const uint16_t* src, int64_t n, int gk_, uint32_t* amax, float* scale) {
        uint8_t* buf = gcodes;
        if (side_on()) {
            buf = gbuf_i ? gcodes2 : gcodes;
            if (wdone_valid[gbuf_i]) QT_CHECK_CUDA(cudaStreamWaitEvent(st, ev_wdone[gbuf_i], 0));
        }
        const int h = prof_begin();
        QT_CHECK_K(qtk_quantize_bf16(src, n, gk_, amax, buf, scale, st));
        prof_end(h, 3, 3.0 * n);
        if (side_on()) {
            QT_CHECK_CUDA(cudaEventRecord(ev_qready, st));
            QT_CHECK_CUDA(cudaStreamWaitEvent(wst, ev_qready, 0));
        }
        return buf;
    }
    // GradAccumulator SR-accumulate wgrad of tensor t from the codes `gc` (model.cpp:160-167,
    // 448-464): on the side stream, which then marks the codes buffer free
    void wgrad(int64_t Mo, int64_t No, int64_t K, const uint8_t* gc, int64_t lda, const uint8_t* act, int64_t ldb,
               const float* gsc, const float* asc, const ParamT& t, uint64_t micro_step) {
        const uint64_t aseed = seed + (uint64_t)rank;
        // GradAccumulator into a zero buffer: SR(0 + bf16(acc/(sa*sb))) returns the bf16 value
        // unchanged (a representable value passes through, numerics.cpp:240-250), so the first
        // accumulation is the plain rounded store: no read of the buffer, no RNG (same bits)
        const bool fresh = t.goff < 0 || grads_fresh;
        gemm(0, gkind(), kE4M3, true, true, Mo, No, K, gc, lda, act, ldb, gsc, asc, fresh ? EPI_BF16 : EPI_BF16_ACC,
             gbuf(t), No, nullptr,
             0, aseed, t.s_acc, micro_step * (uint64_t)t.numel, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0,
             0, side_on() ? wst : nullptr);
        if (side_on()) {
            QT_CHECK_CUDA(cudaEventRecord(ev_wdone[gbuf_i], wst));
            wdone_valid[gbuf_i] = true;
            gbuf_i ^= 1;
        }
    }
    // the compute stream waits for every weight gradient issued so far
    void wgrad_join() {
        if (!side_on()) return;
        QT_CHECK_CUDA(cudaEventRecord(ev_wjoin, wst));
        QT_CHECK_CUDA(cudaStreamWaitEvent(st, ev_wjoin, 0));
    }

    // ---------------- model_backward + GradAccumulator (src/model.cpp:354-464) ----------------
    void backward(uint64_t micro_step) {
        if (!have_fwd || !fwd_with_grads) throw QtError(1, "model_backward: no forward with grads to differentiate");
        gbuf_i = 0;
        wdone_valid[0] = wdone_valid[1] = false;
        const int64_t M = curM;
        const uint64_t aseed = seed + (uint64_t)rank;  // trainer.cpp:68-70: worker w accumulates with seed+w
        const int gk = gkind();
        int h;
        // CE backward matmuls: d_hidden = dlogits . lm_w ; d_lm_w = dlogits^T . hidden
        if (lm_tx()) {
            // dlogits = bf16 non-target entries + the exact f32 target term (tensorops.cpp:372-405)
            const ParamT& t = par("lm_head");
            gemm(1, 0, 0, false, true, M, d, V, dlogits, V, pptr("lm_head"), d, nullptr, nullptr, EPI_F32, lm_acc, d,
                 nullptr, 0, 0, 0, 0, nullptr, nullptr, nullptr, nullptr, nullptr, lm_ws, lm_ws_bytes, lm_splits);
            h = prof_begin();
            QT_CHECK_K(qtk_lm_dgrad_finish(lm_acc, M, d, dl_tgt, targets, pptr("lm_head"), d_hidden, st));
            prof_end(h, 5, 8.0 * M * d);
            gemm(1, 0, 0, true, true, V, d, M, dlogits, V, normed_final, d, nullptr, nullptr, EPI_F32, lm_acc, d);
            h = prof_begin();
            QT_CHECK_K(qtk_lm_wgrad_targets(lm_acc, d, t_sorted_pos, t_seg_tok, t_seg_off, t_nseg, M, dl_tgt,
                                            normed_final, st));
            prof_end(h, 5, 2.0 * M * d);
            h = prof_begin();
            accumulate_f32(t, lm_acc, micro_step);
            prof_end(h, 5, 8.0 * (double)t.numel);
        } else {
        // (dlogits is f32 in the reference: hi + lo bf16 parts through the split-A GEMM)
        gemm(1, 0, 0, false, true, M, d, V, dlogits, V, pptr("lm_head"), d, nullptr, nullptr, EPI_BF16, d_hidden, d,
             nullptr, 0, 0, 0, 0, dlogits_lo);
        {
            const ParamT& t = par("lm_head");
            gemm(1, 0, 0, true, true, V, d, M, dlogits, V, normed_final, d, nullptr, nullptr, EPI_F32_ACC,
                 gbuf(t), d, nullptr, 0, aseed, t.s_acc, micro_step * (uint64_t)t.numel, dlogits_lo);
        }
        }
        // final norm backward (model.cpp:359-363)
        h = prof_begin();
        QT_CHECK_CUDA(cudaMemsetAsync(g_amax, 0, L * 16, st));
        QT_CHECK_K(qtk_rmsnorm_bwd(lb[L].r_in, pptr("final_g"), M, d, 1e-6f, d_hidden, nullptr, d_r, dgamma_part,
                                   dgamma, g_amax + (L - 1) * 4 + G_DR, st));
        accumulate_f32(par("final_g"), dgamma, micro_step);
        prof_end(h, 4, 8.0 * M * d);
        for (int l = L - 1; l >= 0; --l) {
            LayerBufs& b = lb[l];
            codes_acquire(l, l - 1);
            if (offload_x()) x_acquire(l, l - 1);
            if (exchange_in_backward) {  // the layer's gradient slot: free (exchange done) and zeroed
                QT_CHECK_CUDA(cudaStreamWaitEvent(st, ev_lfree[l % 2], 0));
                QT_CHECK_CUDA(cudaMemsetAsync(lgrad[l % 2], 0, layer_g * 2, st));
            }
            if (!b.keep_all) block_replay(l);  // dropped sites only, cached stats (model.cpp:374-378)
            uint32_t* ga = g_amax + l * 4;
            float* gs = g_scale + l * 4;
            const float* as = act_scale + l * 4;
            const float* ws = w_scale + l * 4;
            const ParamT& pq = P[lp(l, 1)];
            const ParamT& po = P[lp(l, 2)];
            const ParamT& pg = P[lp(l, 4)];
            const ParamT& pd = P[lp(l, 5)];
            // ---- FFN down: dY = d_r
            uint8_t* gc = quant_grad(d_r, M * d, gk, ga + G_DR, gs + G_DR);
            wgrad(d, Hh, M, gc, d, b.hc, Hh, gs + G_DR, as + S_H, pd, micro_step);
            if (fuse_swiglu_bwd()) {
                // d_h = down-proj dgrad, consumed in the GEMM epilogue by swiglu_backward:
                // d_gate|d_up + their absmax written directly (d_h never reaches HBM)
                gemm(0, gk, kE4M3, false, true, M, Hh, d, gc, d, wc(l, W_DOWN), Hh, gs + G_DR,
                     ws + W_DOWN, EPI_SWIGLU_BWD, d_gu, F, b.gu, F, 0, 0, 0, nullptr, ga + G_DGU);
            } else {
                gemm(0, gk, kE4M3, false, true, M, Hh, d, gc, d, wc(l, W_DOWN), Hh, gs + G_DR,
                     ws + W_DOWN, EPI_BF16, d_h, Hh);
                h = prof_begin();
                QT_CHECK_K(qtk_swiglu_bwd(b.gu, d_h, M, Hh, d_gu, ga + G_DGU, st));
                prof_end(h, 5, 2.0 * M * F * 2 + 2.0 * M * Hh);
            }
            // ---- gate_up
            gc = quant_grad(d_gu, M * F, gk, ga + G_DGU, gs + G_DGU);
            wgrad(F, d, M, gc, F, b.n2c, d, gs + G_DGU, as + S_N2, pg, micro_step);
            gemm(0, gk, kE4M3, false, true, M, d, F, gc, F, wc(l, W_GU), d, gs + G_DGU, ws + W_GU, EPI_BF16,
                 d_n, d);
            // ---- rmsnorm2 backward: d_attn_out = ... + d_r (model.cpp:393-399)
            h = prof_begin();
            QT_CHECK_K(qtk_rmsnorm_bwd(b.r_mid, params + P[lp(l, 3)].off, M, d, 1e-6f, d_n, d_r, d_ao, dgamma_part,
                                       dgamma, ga + G_DAO, st));
            accumulate_f32(P[lp(l, 3)], dgamma, micro_step);
            prof_end(h, 4, 10.0 * M * d);
            // ---- attention output projection
            gc = quant_grad(d_ao, M * d, gk, ga + G_DAO, gs + G_DAO);
            wgrad(d, d, M, gc, d, b.attc, d, gs + G_DAO, as + S_ATT, po, micro_step);
            gemm(0, gk, kE4M3, false, true, M, d, d, gc, d, wc(l, W_O), d, gs + G_DAO, ws + W_O, EPI_BF16,
                 d_att, d);
            // ---- attention backward + inverse RoPE
            h = prof_begin();
            QT_CHECK_K(qtk_attn_bwd2(b.qkv, b.att32, d_att, d, b.lse, Dv, curB, curT, H, Hkv, hd, q, d_qkv, attn_ws, st,
                                     attn_two_streams() && side_on() ? wst : nullptr));
            prof_end(h, 8, 10.0 * curB * H * (double)curT * curT / 2 * hd);
            h = prof_begin();
            QT_CHECK_K(qtk_rope(d_qkv, M, curT, H + Hkv, hd, q, rope_tab, 1, ga + G_DQKV, st));
            prof_end(h, 5, 4.0 * M * q);
            // ---- qkv projection
            gc = quant_grad(d_qkv, M * q, gk, ga + G_DQKV, gs + G_DQKV);
            wgrad(q, d, M, gc, q, b.n1c, d, gs + G_DQKV, as + S_N1, pq, micro_step);
            gemm(0, gk, kE4M3, false, true, M, d, q, gc, q, wc(l, W_QKV), d, gs + G_DQKV, ws + W_QKV,
                 EPI_BF16, d_n, d);
            // ---- rmsnorm1 backward: d_r = ... + d_attn_out (model.cpp:433-439)
            h = prof_begin();
            QT_CHECK_K(qtk_rmsnorm_bwd(b.r_in, params + P[lp(l, 0)].off, M, d, 1e-6f, d_n, d_ao, d_r, dgamma_part,
                                       dgamma, l > 0 ? g_amax + (l - 1) * 4 + G_DR : nullptr, st));
            accumulate_f32(P[lp(l, 0)], dgamma, micro_step);
            prof_end(h, 4, 10.0 * M * d);
            codes_release(l);
            if (offload_x()) QT_CHECK_CUDA(cudaEventRecord(ev_xfree[l % 2], st));
            if (exchange_in_backward) {
                wgrad_join();  // the layer's weight gradients are final
                reduce_layer_async(l);
            }
        }
        wgrad_join();
        // ordered embedding backward, bf16 round, accumulate (model.cpp:442-444)
        {
            const ParamT& t = par("embed");
            h = prof_begin();
            if (use_dev_ctr)
                QT_CHECK_K(qtk_embed_bwd_ms(sorted_pos, seg_off, seg_tok, nseg, (int)M, d_r, d, t.numel, gbuf(t),
                                            aseed, t.s_acc, ms_dev(cur_ga), st));
            else
                QT_CHECK_K(qtk_embed_bwd(sorted_pos, seg_off, seg_tok, nseg, (int)M, d_r, d, gbuf(t), aseed,
                                         t.s_acc, micro_step * (uint64_t)t.numel, st));
            prof_end(h, 5, 4.0 * M * d);
        }
        grads_fresh = false;  // this micro-batch's gradients are in the buffer now
    }

    void accumulate_f32(const ParamT& t, const float* g, uint64_t micro_step) {
        if (use_dev_ctr)
            QT_CHECK_K(qtk_sr_accumulate_f32_ms(gbuf(t), g, t.numel, seed + (uint64_t)rank, t.s_acc,
                                                ms_dev(cur_ga), st));
        else
            QT_CHECK_K(qtk_sr_accumulate_f32(gbuf(t), g, t.numel, seed + (uint64_t)rank, t.s_acc,
                                             micro_step * (uint64_t)t.numel, st));
    }

    // ---------------- cross-rank gradient reduction (ZeRO-1) ----------------
    // all-to-all of bf16 shards + ascending-rank f32 sum == trainer.cpp:90-103 bitwise, for
    // the tensors [i0, i1) (contiguous shards); rank r's chunk of tensor i lands at
    // rbuf + r*rstride + (soff_of[i] - soff_of[i0]); acc: add onto the shard (shard_grads, GA > 1)
    void exchange(int i0, int i1, cudaStream_t s, uint16_t* rbuf, int64_t rstride, bool acc) {
        std::vector<AllToAllItem> items;
        for (int i = i0; i < i1; ++i) {
            const ParamT& t = P[i];
            items.push_back({gbuf(t), (size_t)t.pw * 2, rbuf + (soff_of[i] - soff_of[i0]), (size_t)rstride * 2,
                             (size_t)t.pw * 2});
        }
        coll([&] { tr->alltoall(items, s); });
        const int64_t n = soff_of[i1 - 1] + P[i1 - 1].pw - soff_of[i0];
        ordered_sum_kernel<<<grid_for(n), 256, 0, s>>>(rbuf, world, n, rstride, gshard + soff_of[i0], acc ? 1 : 0);
        QT_CHECK_CUDA(cudaGetLastError());
    }
    void reduce_grads() {
        const int h = prof_begin();
        exchange(0, (int)P.size(), st, recvbuf, shard_total, false);
        prof_end(h, 9, 2.0 * shard_total * (world - 1) * 2);
    }
    // RunPlan::shard_grads: layer l's gradients (this micro-batch) are final once its backward
    // is done: exchange them on the communication stream while layers l-1..0 run, into the
    // rank's f32 shard; the layer's slot is then free for layer l-2
    void reduce_layer_async(int l) {
        QT_CHECK_CUDA(cudaEventRecord(ev_grad, st));
        QT_CHECK_CUDA(cudaStreamWaitEvent(cst, ev_grad, 0));
        const int h = prof_begin_on(cst);
        exchange(lp(l, 0), lp(l, 5) + 1, cst, lrecv[l % 2], layer_shard, cur_ga > 0);
        prof_end_on(h, 9, 2.0 * layer_shard * (world - 1) * 2, cst);
        QT_CHECK_CUDA(cudaEventRecord(ev_lfree[l % 2], cst));
        comm_pending = true;
    }
    void reduce_rest_and_join() {
        // embed (index 0) and final_g / lm_head (the last two), accumulated locally over the
        // micro-batches, on the comm stream; then join
        QT_CHECK_CUDA(cudaEventRecord(ev_grad, st));
        QT_CHECK_CUDA(cudaStreamWaitEvent(cst, ev_grad, 0));
        const int np = (int)P.size();
        const int64_t rest = P[0].pw + P[np - 2].pw + P[np - 1].pw;
        exchange(0, 1, cst, recvbuf, rest, false);
        exchange(np - 2, np, cst, recvbuf + P[0].pw, rest, false);
        QT_CHECK_CUDA(cudaEventRecord(ev_comm, cst));
        QT_CHECK_CUDA(cudaStreamWaitEvent(st, ev_comm, 0));
        comm_pending = false;
    }

    void grad_sumsq() {
        const void* g = world > 1 ? (const void*)gshard : (const void*)grads;
        QT_CHECK_K(qtk_grad_sumsq(g, world > 1, segs_dev, nsegs, norm_blocks, norm_partials, norm_scratch, ssq_dev, st));
        poison_ssq_kernel<<<1, 1, 0, st>>>(ssq_dev, err_dev, act_amax, have_fwd ? L * 4 : 0, fin_amax, loss_dev + 1,
                                          in_step ? plan.ga_steps : 0);
        QT_CHECK_CUDA(cudaGetLastError());
        if (world > 1) coll([&] { tr->allreduce_sum_f64(ssq_dev, 1, st); });
    }

    // AdamW on this rank's shard + all-gather of the updated bf16 params (optim.cpp:112-176)
    void adamw(const float* grad_scale_dev) {
        const int64_t step = step_count + 1;
        const float bc1 = 1.0f - std::pow(hyper.beta1, static_cast<float>(step));
        const float bc2 = 1.0f - std::pow(hyper.beta2, static_cast<float>(step));
        const void* g = world > 1 ? (const void*)gshard : (const void*)grads;
        const int64_t total = world > 1 ? shard_total : p_total;
        int h = prof_begin();
        QT_CHECK_CUDA(cudaMemsetAsync(seg_amax, 0, P.size() * 4, st));
        auto launch = [&](float* m, float* v, uint16_t* mh, uint16_t* vh, const uint8_t* chunks, int n) {
            QT_CHECK_K(qtk_adamw_dev_sd(params, m, v, mh, vh, g, world > 1, segs_dev, chunks, n, hyper.lr, hyper.beta1,
                                        hyper.beta2, hyper.eps, hyper.weight_decay, bc1, bc2, grad_scale_dev, seed, step,
                                        plan.bf16_moments, err_dev, seg_amax, use_dev_ctr ? step_blk : nullptr, st));
        };
        if (!stream_moments()) {
            launch(m32, v32, m16, v16, static_cast<const uint8_t*>(chunks_dev), nchunks);
        } else {
            // offload (double-buffer policy): each group's offloaded moments go host -> slot on
            // the copy engine (one group ahead), AdamW updates them in the slot, and they go back
            const size_t mb = plan.bf16_moments ? 2 : 4;
            uint8_t* hm = plan.bf16_moments ? (uint8_t*)m16 : (uint8_t*)m32;
            uint8_t* hv = plan.bf16_moments ? (uint8_t*)v16 : (uint8_t*)v32;
            auto h2d = [&](int gi) {
                const MGroup& gp = mgroups[(size_t)gi];
                const int sl = gi % 2;
                const size_t bytes = (size_t)(gp.e1 - gp.e0) * mb;
                if (offload_m())
                    QT_CHECK_CUDA(cudaMemcpyAsync(mstage[sl][0], hm + gp.e0 * mb, bytes, cudaMemcpyHostToDevice, cst));
                if (offload_v())
                    QT_CHECK_CUDA(cudaMemcpyAsync(mstage[sl][1], hv + gp.e0 * mb, bytes, cudaMemcpyHostToDevice, cst));
                QT_CHECK_CUDA(cudaEventRecord(ev_mready[sl], cst));
            };
            QT_CHECK_CUDA(cudaEventRecord(ev_mdone[0], st));  // the grads of this step are final
            QT_CHECK_CUDA(cudaStreamWaitEvent(cst, ev_mdone[0], 0));
            const int ng = (int)mgroups.size();
            if (ng) h2d(0);
            for (int gi = 0; gi < ng; ++gi) {
                const MGroup& gp = mgroups[(size_t)gi];
                const int sl = gi % 2;
                if (gi + 1 < ng) h2d(gi + 1);
                QT_CHECK_CUDA(cudaStreamWaitEvent(st, ev_mready[sl], 0));
                // moment pointers rebased so that element e0 of the group sits at the slot start
                auto base = [&](int k, uint8_t* hostp) -> uint8_t* {
                    const bool off = k == 0 ? offload_m() : offload_v();
                    return off ? reinterpret_cast<uint8_t*>(mstage[sl][k]) - gp.e0 * (int64_t)mb : hostp;
                };
                uint8_t* mp = base(0, hm);
                uint8_t* vp = base(1, hv);
                launch(plan.bf16_moments ? nullptr : (float*)mp, plan.bf16_moments ? nullptr : (float*)vp,
                       plan.bf16_moments ? (uint16_t*)mp : nullptr, plan.bf16_moments ? (uint16_t*)vp : nullptr,
                       static_cast<const uint8_t*>(chunks_dev) + (size_t)gp.c0 * sizeof(ChunkH), gp.c1 - gp.c0);
                QT_CHECK_CUDA(cudaEventRecord(ev_mdone[sl], st));
                QT_CHECK_CUDA(cudaStreamWaitEvent(cst, ev_mdone[sl], 0));
                const size_t bytes = (size_t)(gp.e1 - gp.e0) * mb;
                if (offload_m())
                    QT_CHECK_CUDA(cudaMemcpyAsync(hm + gp.e0 * mb, mstage[sl][0], bytes, cudaMemcpyDeviceToHost, cst));
                if (offload_v())
                    QT_CHECK_CUDA(cudaMemcpyAsync(hv + gp.e0 * mb, mstage[sl][1], bytes, cudaMemcpyDeviceToHost, cst));
            }
            QT_CHECK_CUDA(cudaEventRecord(ev_mfree[0], cst));  // every moment is back on the host
            QT_CHECK_CUDA(cudaStreamWaitEvent(st, ev_mfree[0], 0));
        }
        prof_end(h, 10, (double)total * (plan.bf16_moments ? 14.0 : 22.0));
        amax_cached = !shard_weights();
        if (world > 1 && amax_cached)  // slice maxima -> tensor maxima
            coll([&] { tr->allreduce_max_u32(seg_amax, P.size(), st); });
        if (world > 1) {
            h = prof_begin();
            std::vector<AllGatherItem> items;
            for (int i = 0; i < (int)P.size(); ++i) {
                if (shard_weights() && is_block_weight(i)) continue;  // gathered as FP8 codes next step
                const ParamT& t = P[i];
                items.push_back({params + t.off, (size_t)t.pw * 2});
            }
            coll([&] { tr->allgather(items, st); });
            prof_end(h, 9, 2.0 * shard_total * (world - 1));
        }
        step_count += 1;
    }

    // ---------------- one trainer step (src/trainer.cpp:64-110) ----------------
    static bool graph_enabled() {
        static int f = -1;
        if (f < 0) {
            const char* e = getenv("QTB_GRAPH");
            f = e ? atoi(e) : 1;
        }
        return f != 0;
    }

    // One trainer step.  Steady state (weight absmax cached by the previous AdamW, no
    // profiling): the step is captured once into a CUDA graph reading its per-step values
    // (micro-steps, AdamW step and bias corrections) from step_blk, then replayed.
    void train_step(const int32_t* tokens, int64_t tokens_per_mb, int64_t batch, int64_t step, float max_norm) {
        const int GA = plan.ga_steps;
        pre_step_count = step_count;
        // world > 1 stays stream-launched: the NCCL exchange inside a captured graph has
        // not been exercised on hardware this round (gpurun boxes have one GPU)
        if (!graph_enabled() || prof_on || !amax_cached || world > 1 || stream_codes() || stream_moments() ||
            offload_x()) {
            train_step_body(tokens, tokens_per_mb, batch, step, max_norm);
            return;
        }
        const int64_t ntok = (int64_t)GA * tokens_per_mb;
        if (ntok > (int64_t)GA * plan.micro_batch * (T + 1)) throw QtError(1, "train_step: token buffer too small");
        if (tokens != tok_buf)
            QT_CHECK_CUDA(cudaMemcpyAsync(tok_buf, tokens, ntok * 4, cudaMemcpyDeviceToDevice, st));
        const size_t bsz = 16 + 8 * (size_t)GA, bstride = (bsz + 63) & ~size_t(63);
        if (!blk_host) {
            QT_CHECK_CUDA(cudaMallocHost(&blk_host, bstride * kBlkRing));
            for (auto& e : blk_ev) QT_CHECK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        const int slot = blk_slot;
        blk_slot = (blk_slot + 1) % kBlkRing;
        QT_CHECK_CUDA(cudaEventSynchronize(blk_ev[slot]));  // its previous copy has executed
        uint8_t* blk = blk_host + slot * bstride;
        StepBlockH h{step + 1, 1.0f - std::pow(hyper.beta1, static_cast<float>(step + 1)),
                     1.0f - std::pow(hyper.beta2, static_cast<float>(step + 1))};
        std::memcpy(blk, &h, sizeof(h));
        for (int ga = 0; ga < GA; ++ga) {
            const uint64_t ms = (uint64_t)step * GA + ga;
            std::memcpy(blk + 16 + 8 * ga, &ms, 8);
        }
        QT_CHECK_CUDA(cudaMemcpyAsync(step_blk, blk, bsz, cudaMemcpyHostToDevice, st));
        QT_CHECK_CUDA(cudaEventRecord(blk_ev[slot], st));
        if (!gexec || g_tpm != tokens_per_mb || g_batch != batch || g_max_norm != max_norm) {
            if (gexec) cudaGraphExecDestroy(gexec);
            gexec = nullptr;
            cudaGraph_t g = nullptr;
            QT_CHECK_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
            use_dev_ctr = true;
            try {
                train_step_body(tok_buf, tokens_per_mb, batch, step, max_norm);
            } catch (...) {
                use_dev_ctr = false;
                cudaStreamEndCapture(st, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            use_dev_ctr = false;
            QT_CHECK_CUDA(cudaStreamEndCapture(st, &g));
            QT_CHECK_CUDA(cudaGraphInstantiate(&gexec, g, 0));
            cudaGraphDestroy(g);
            g_tpm = tokens_per_mb;
            g_batch = batch;
            g_max_norm = max_norm;
        } else {
            // host-side effects of the body (forward/backward bookkeeping, optimizer step count)
            curB = (int)batch;
            curT = (int)(tokens_per_mb / batch - 1);
            curM = (int64_t)curB * curT;
            have_fwd = true;
            fwd_with_grads = true;
            step_count = step + 1;
            amax_cached = !shard_weights();
        }
        QT_CHECK_CUDA(cudaGraphLaunch(gexec, st));
    }

    void train_step_body(const int32_t* tokens, int64_t tokens_per_mb, int64_t batch, int64_t step, float max_norm) {
        const int GA = plan.ga_steps;
        struct InStep {
            bool& f;
            InStep(bool& x) : f(x) { f = true; }
            ~InStep() { f = false; }
        } in_step_guard(in_step);
        build_step_context();
        QT_CHECK_CUDA(cudaMemsetAsync(grads, 0, g_store * 2, st));
        grads_fresh = true;
        for (int ga = 0; ga < GA; ++ga) {
            forward(tokens + (int64_t)ga * tokens_per_mb, tokens_per_mb, batch, true);
            QT_CHECK_CUDA(cudaMemcpyAsync(loss_dev + 1 + ga, loss_dev, 4, cudaMemcpyDeviceToDevice, st));
            // shard_grads: each micro-batch's gradients of layer l are exchanged into the rank's
            // shard while layers < l run backward (GA = 1: the order of trainer.cpp:90-103)
            exchange_in_backward = shard_grads();
            cur_ga = ga;
            backward((uint64_t)step * GA + ga);
            exchange_in_backward = false;
        }
        if (world > 1) {
            if (shard_grads()) reduce_rest_and_join();
            else reduce_grads();
        }
        grad_sumsq();
        const float mean_scale = 1.0f / (static_cast<float>(GA) * world);
        finalize_scale_kernel<<<1, 1, 0, st>>>(ssq_dev, mean_scale, max_norm, gscale_dev, norm_dev, err_dev);
        QT_CHECK_CUDA(cudaGetLastError());
        step_count = step;
        adamw(gscale_dev);
    }

    // non-finite diagnostics (model.cpp:125-129, trainer.cpp:113-115)
    void check_errors(bool after_forward) {
        int err = 0;
        QT_CHECK_CUDA(cudaMemcpyAsync(&err, err_dev, 4, cudaMemcpyDeviceToHost, st));
        std::vector<uint32_t> am((size_t)L * 4);
        uint32_t fa = 0;
        float loss = 0;
        QT_CHECK_CUDA(cudaMemcpyAsync(am.data(), act_amax, L * 16, cudaMemcpyDeviceToHost, st));
        QT_CHECK_CUDA(cudaMemcpyAsync(&fa, fin_amax, 4, cudaMemcpyDeviceToHost, st));
        QT_CHECK_CUDA(cudaMemcpyAsync(&loss, loss_dev, 4, cudaMemcpyDeviceToHost, st));
        QT_CHECK_CUDA(cudaStreamSynchronize(st));
        if (err == 2) {
            cudaMemsetAsync(err_dev, 0, 4, st);
            throw QtError(2, "model_forward: token id out of range");
        }
        if (after_forward) {
            static const char* names[4] = {"rmsnorm1", "attention", "rmsnorm2", "swiglu"};
            for (int l = 0; l < L; ++l)
                for (int s = 0; s < 4; ++s)
                    if (am[l * 4 + s] >= 0x7F800000u)
                        throw QtError(3, std::string("non-finite value at ") + names[s] + " (layer " +
                                             std::to_string(l) + ")");
            if (fa >= 0x7F800000u) throw QtError(3, "non-finite value at final rmsnorm");
            if (!std::isfinite(loss)) throw QtError(3, "non-finite value at cross entropy");
        }
        if (err == 3) {
            cudaMemsetAsync(err_dev, 0, 4, st);
            throw QtError(3, "adamw_step: non-finite gradient" + nonfinite_grad_name());
        }
    }
    // a gated step left params and moments untouched: undo its host-side bookkeeping
    void on_gated_step() {
        if (pre_step_count >= 0) step_count = pre_step_count;
        amax_cached = false;
    }
    // " in <name>": the first tensor in update order (NamedTensors, optim.cpp:66-74) whose
    // norm partials are non-finite (src/optim.cpp:47 names the tensor)
    std::string nonfinite_grad_name() {
        std::vector<double> part((size_t)norm_blocks);
        std::vector<SegH> segs((size_t)nsegs);
        if (norm_blocks <= 0) return "";
        if (cudaMemcpy(part.data(), norm_partials, part.size() * 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
            cudaMemcpy(segs.data(), segs_dev, segs.size() * sizeof(SegH), cudaMemcpyDeviceToHost) != cudaSuccess)
            return "";
        for (int i = 0; i < nsegs; ++i) {
            const int64_t nb = ceil_div(segs[i].n, 256);
            for (int64_t b = 0; b < nb; ++b)
                if (!std::isfinite(part[(size_t)(segs[i].blk0 + b)])) return " in " + P[i].name;
        }
        return world > 1 ? " (on another rank)" : "";
    }
};

}  // namespace qtb

// ===========================================================================
// C ABI
// ===========================================================================
using namespace qtb;

struct qt_session {
    std::unique_ptr<Session> s;
};
struct qt_group {
    std::shared_ptr<PeerGroup> g;  // each member session holds a reference too
};

template <typename F>
static int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const QtError& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return 3;
    }
}

extern "C" {

const char* qt_last_error(void) { return g_last_error.c_str(); }

int qt_nccl_unique_id(void* out128) {
    return guard([&] {
        auto& api = NcclApi::get();
        if (!api.ok) throw QtError(3, "NCCL not loadable");
        ncclUniqueId id;
        ncclResult_t r = api.GetUniqueId(&id);
        if (r != ncclSuccess) throw QtError(3, api.GetErrorString(r));
        std::memcpy(out128, &id, sizeof(id));
    });
}

int qt_session_create(const QtModelConfig* cfg, const QtPrecisionMap* prec, const QtRunPlan* plan, const QtAdamW* hyper,
                      uint64_t seed, int rank, int world, const void* nccl_id, int device, qt_session** out) {
    *out = nullptr;
    return guard([&] {
        auto* h = new qt_session();
        try {
            h->s = std::make_unique<Session>(*cfg, *prec, *plan, *hyper, seed, rank, world, nccl_id, device);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

void qt_session_destroy(qt_session* s) { delete s; }

// In-process worker group (the reference's WorkerGroup, src/comms.cpp:19-38):
// W sessions, one per host thread, on one device or several, whose collectives
// are copy-engine pulls between their arenas (transport.cuh PeerTransport).
int qt_group_create(int world, qt_group** out) {
    *out = nullptr;
    return guard([&] {
        if (world < 1 || world > 64) throw QtError(1, "qt_group_create: world must be in [1, 64]");
        auto* g = new qt_group();
        g->g = std::make_shared<PeerGroup>(world);
        *out = g;
    });
}
void qt_group_destroy(qt_group* g) { delete g; }

int qt_session_create_in_group(const QtModelConfig* cfg, const QtPrecisionMap* prec, const QtRunPlan* plan,
                               const QtAdamW* hyper, uint64_t seed, qt_group* group, int rank, int device,
                               qt_session** out) {
    *out = nullptr;
    return guard([&] {
        if (!group) throw QtError(1, "qt_session_create_in_group: null group");
        auto* h = new qt_session();
        try {
            h->s = std::make_unique<Session>(*cfg, *prec, *plan, *hyper, seed, rank, group->g->world, nullptr, device,
                                             group->g);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

// which transport a session's collectives use: "none" (world 1), "nccl", "peer-copy"
const char* qt_session_transport(qt_session* s) { return s->s->tr ? s->s->tr->kind() : "none"; }

void* qt_session_stream(qt_session* s) { return (void*)s->s->st; }
size_t qt_session_bytes(qt_session* s) { return s->s->arena_bytes; }

int qt_num_params(qt_session* s) { return (int)s->s->P.size(); }

int qt_param_info(qt_session* s, int i, const char** name, int64_t* numel) {
    return guard([&] {
        if (i < 0 || i >= (int)s->s->P.size()) throw QtError(2, "param index out of range");
        *name = s->s->P[i].name.c_str();
        *numel = s->s->P[i].numel;
    });
}

int qt_param_upload(qt_session* h, int i, const float* host) {
    return guard([&] {
        Session& s = *h->s;
        const ParamT& t = s.P.at(i);
        s.amax_cached = false;
        const int64_t n = s.stored(t);  // shard_weights: the rank keeps its slice only
        if (n > 0) {
            QT_CHECK_CUDA(cudaMemcpyAsync(s.scratch_f32, host + t.lo, n * 4, cudaMemcpyHostToDevice, s.st));
            f32_to_bf16_kernel<<<grid_for(n), 256, 0, s.st>>>(s.scratch_f32, s.params + t.off, n);
        }
        QT_CHECK_CUDA(cudaStreamSynchronize(s.st));
    });
}

static void download_bf16(Session& s, const uint16_t* src, int64_t n, float* host) {
    bf16_to_f32_kernel<<<grid_for(n), 256, 0, s.st>>>(src, s.scratch_f32, n);
    QT_CHECK_CUDA(cudaMemcpyAsync(host, s.scratch_f32, n * 4, cudaMemcpyDeviceToHost, s.st));
    QT_CHECK_CUDA(cudaStreamSynchronize(s.st));
}

// With shard_weights each rank keeps only its ZeRO-1 slice of a block weight
// current: the download gathers the owners' slices (peer group: direct reads of
// the idle peers' arenas; NCCL: a collective every rank must enter).
int qt_param_download(qt_session* h, int i, float* host) {
    return guard([&] {
        Session& s = *h->s;
        const ParamT& t = s.P.at(i);
        if (t.sharded) {  // the ranks' slices, read from the peers (NCCL: a collective)
            uint16_t* stage = reinterpret_cast<uint16_t*>(s.scratch_f32);
            s.coll([&] { s.tr->gather_idle(s.params + t.off, (size_t)t.pw * 2, stage, s.st); });
            std::vector<uint16_t> b((size_t)t.numel);
            QT_CHECK_CUDA(cudaMemcpy(b.data(), stage, t.numel * 2, cudaMemcpyDeviceToHost));
            for (int64_t e = 0; e < t.numel; ++e) {
                const uint32_t u = (uint32_t)b[(size_t)e] << 16;
                std::memcpy(host + e, &u, 4);
            }
            return;
        }
        download_bf16(s, s.params + t.off, t.numel, host);
    });
}

int qt_grad_download(qt_session* h, int i, float* host) {
    return guard([&] {
        Session& s = *h->s;
        const ParamT& t = s.P.at(i);
        if (t.goff < 0)
            throw QtError(1, "shard_grads keeps no local accumulator for layer tensors (qt_reduced_grad_download)");
        download_bf16(s, s.grads + t.goff, t.numel, host);
    });
}
// the cross-rank reduced f32 gradient of tensor i (world > 1): every rank's shard, gathered
int qt_reduced_grad_download(qt_session* h, int i, float* host) {
    return guard([&] {
        Session& s = *h->s;
        if (s.world < 2) throw QtError(1, "qt_reduced_grad_download: world > 1 only");
        const ParamT& t = s.P.at(i);
        s.coll([&] { s.tr->gather_idle(s.gshard + s.soff_of[i], (size_t)t.pw * 4, s.scratch_f32, s.st); });
        QT_CHECK_CUDA(cudaMemcpy(host, s.scratch_f32, t.numel * 4, cudaMemcpyDeviceToHost));
    });
}

// f32 moments of this rank's slice of tensor i (world == 1: the whole tensor)
int qt_moments_download(qt_session* h, int i, float* m, float* v) {
    return guard([&] {
        Session& s = *h->s;
        const ParamT& t = s.P.at(i);
        std::vector<SegH> segs(s.nsegs);
        QT_CHECK_CUDA(cudaMemcpy(segs.data(), s.segs_dev, segs.size() * sizeof(SegH), cudaMemcpyDefault));
        const SegH& sg = segs[i];
        const int64_t off = sg.off;  // moment offset (world 1: the gradient layout)
        if (s.plan.bf16_moments) {  // bf16-SR moments, widened to f32 (exact)
            download_bf16(s, s.m16 + off, sg.n, m);
            download_bf16(s, s.v16 + off, sg.n, v);
            return;
        }
        QT_CHECK_CUDA(cudaMemcpy(m, s.m32 + off, sg.n * 4, cudaMemcpyDefault));
        QT_CHECK_CUDA(cudaMemcpy(v, s.v32 + off, sg.n * 4, cudaMemcpyDefault));
    });
}

// m, v: the full tensor (numel floats); each rank keeps its ZeRO-1 slice.  bf16-SR moments
// take values on the bf16 grid (as a checkpoint of such moments holds) and store them exactly.
int qt_moments_upload(qt_session* h, int i, const float* m, const float* v, int64_t step_count) {
    return guard([&] {
        Session& s = *h->s;
        const ParamT& t = s.P.at(i);
        std::vector<SegH> segs(s.nsegs);
        QT_CHECK_CUDA(cudaMemcpy(segs.data(), s.segs_dev, segs.size() * sizeof(SegH), cudaMemcpyDefault));
        const SegH& sg = segs[i];
        const int64_t off = sg.off;  // moment offset (world 1: the gradient layout)
        const int64_t lo = s.world > 1 ? std::min<int64_t>((int64_t)s.rank * t.pw, t.numel) : 0;
        if (sg.n > 0) {
            if (s.plan.bf16_moments) {
                for (int k = 0; k < 2; ++k) {
                    QT_CHECK_CUDA(cudaMemcpyAsync(s.scratch_f32, (k ? v : m) + lo, sg.n * 4, cudaMemcpyDefault,
                                                  s.st));
                    f32_to_bf16_kernel<<<grid_for(sg.n), 256, 0, s.st>>>(s.scratch_f32, (k ? s.v16 : s.m16) + off,
                                                                           sg.n);
                }
            } else {
                QT_CHECK_CUDA(cudaMemcpyAsync(s.m32 + off, m + lo, sg.n * 4, cudaMemcpyDefault, s.st));
                QT_CHECK_CUDA(cudaMemcpyAsync(s.v32 + off, v + lo, sg.n * 4, cudaMemcpyDefault, s.st));
            }
            QT_CHECK_CUDA(cudaStreamSynchronize(s.st));
        }
        s.step_count = step_count;
    });
}

int qt_step_count(qt_session* h, int64_t* out) {
    return guard([&] { *out = h->s->step_count; });
}

// per-micro-batch losses of the last qt_train_step on this rank (ga_steps floats)
int qt_step_losses(qt_session* h, float* out) {
    return guard([&] {
        Session& s = *h->s;
        QT_CHECK_CUDA(cudaMemcpyAsync(out, s.loss_dev + 1, 4 * (size_t)s.plan.ga_steps, cudaMemcpyDeviceToHost, s.st));
        QT_CHECK_CUDA(cudaStreamSynchronize(s.st));
    });
}

int qt_session_rank(qt_session* h, int* rank, int* world) {
    return guard([&] {
        *rank = h->s->rank;
        *world = h->s->world;
    });
}

// ZeRO-1 slice [lo, lo + n) of tensor i this rank's optimizer state covers
int qt_moments_slice(qt_session* h, int i, int64_t* lo, int64_t* n) {
    return guard([&] {
        Session& s = *h->s;
        const ParamT& t = s.P.at(i);
        *lo = s.world > 1 ? std::min<int64_t>((int64_t)s.rank * t.pw, t.numel) : 0;
        *n = s.world > 1 ? std::min<int64_t>(t.pw, t.numel - *lo) : t.numel;
        if (*n < 0) *n = 0;
    });
}

// init_params (src/model.cpp:67-86) on device
int qt_init_params(qt_session* h, uint64_t seed) {
    return guard([&] {
        Session& s = *h->s;
        s.amax_cached = false;
        const float std_ = 1.0f / std::sqrt(static_cast<float>(s.d));
        for (auto& t : s.P) {
            const bool gamma = t.shape.size() == 1;
            const int64_t n = s.stored(t);  // shard_weights: the rank's slice [lo, lo + n)
            if (n <= 0) continue;
            if (gamma)
                fill_bf16_kernel<<<grid_for(n), 256, 0, s.st>>>(s.params + t.off, n, 1.0f);
            else
                init_normal_kernel<<<grid_for(n), 256, 0, s.st>>>(s.params + t.off, n, std_, seed, t.s_init, t.lo);
        }
        QT_CHECK_CUDA(cudaGetLastError());
        QT_CHECK_CUDA(cudaStreamSynchronize(s.st));
    });
}

int qt_build_step_context(qt_session* h) {
    return guard([&] { h->s->build_step_context(); });
}

int qt_forward(qt_session* h, const int32_t* tokens_dev, int64_t n_tokens, int64_t batch, int with_grads,
               float* loss_host) {
    return guard([&] {
        Session& s = *h->s;
        s.forward(tokens_dev, n_tokens, batch, with_grads != 0);
        if (loss_host) {
            s.check_errors(true);
            QT_CHECK_CUDA(cudaMemcpy(loss_host, s.loss_dev, 4, cudaMemcpyDeviceToHost));
        }
    });
}

int qt_backward(qt_session* h, uint64_t micro_step) {
    return guard([&] { h->s->backward(micro_step); });
}

int qt_zero_grads(qt_session* h) {
    return guard([&] {
        QT_CHECK_CUDA(cudaMemsetAsync(h->s->grads, 0, h->s->g_store * 2, h->s->st));
        h->s->grads_fresh = true;
    });
}

int qt_grad_norm(qt_session* h, double* norm_host) {
    return guard([&] {
        Session& s = *h->s;
        if (s.world > 1) s.reduce_grads();
        s.grad_sumsq();
        double ssq = 0;
        QT_CHECK_CUDA(cudaMemcpyAsync(&ssq, s.ssq_dev, 8, cudaMemcpyDeviceToHost, s.st));
        QT_CHECK_CUDA(cudaStreamSynchronize(s.st));
        *norm_host = std::sqrt(ssq);
    });
}

// adamw_step(st, params, grads, grad_scale) (src/optim.cpp:153-164); sharded when world > 1
int qt_adamw_step(qt_session* h, float grad_scale) {
    return guard([&] {
        Session& s = *h->s;
        // g * inf (or NaN) is non-finite for every element: the reference throws on the
        // first tensor it visits (src/optim.cpp:46-47) before changing anything
        if (!std::isfinite(grad_scale)) throw QtError(3, "adamw_step: non-finite gradient in " + s.P[0].name);
        set_scale_kernel<<<1, 1, 0, s.st>>>(s.gscale_dev, grad_scale);
        // gate the whole update on finite gradients (the reference throws on the first
        // non-finite one, src/optim.cpp:47): one norm pass, then AdamW skips if *err != 0
        s.grad_sumsq();
        gate_kernel<<<1, 1, 0, s.st>>>(s.ssq_dev, s.err_dev);
        QT_CHECK_CUDA(cudaGetLastError());
        s.pre_step_count = s.step_count;
        s.adamw(s.gscale_dev);
        try {
            s.check_errors(false);
        } catch (...) {
            s.on_gated_step();
            throw;
        }
    });
}

// full trainer step; tokens_dev holds ga_steps micro-batches of batch*(seq+1) ids
int qt_train_step(qt_session* h, const int32_t* tokens_dev, int64_t tokens_per_mb, int64_t batch, int64_t step,
                  float max_grad_norm, float* loss_host, float* norm_host) {
    return guard([&] {
        Session& s = *h->s;
        s.train_step(tokens_dev, tokens_per_mb, batch, step, max_grad_norm);
        // always checked: a gated step (bad token, non-finite activation or gradient)
        // left params and moments untouched; report it before the caller moves on
        try {
            s.check_errors(true);
        } catch (...) {
            s.on_gated_step();
            throw;
        }
        if (loss_host || norm_host) {
            std::vector<float> l(s.plan.ga_steps);
            double nrm = 0;
            QT_CHECK_CUDA(cudaMemcpyAsync(l.data(), s.loss_dev + 1, 4 * l.size(), cudaMemcpyDeviceToHost, s.st));
            QT_CHECK_CUDA(cudaMemcpyAsync(&nrm, s.norm_dev, 8, cudaMemcpyDeviceToHost, s.st));
            QT_CHECK_CUDA(cudaStreamSynchronize(s.st));
            double sum = 0;
            for (float x : l) sum += x;
            if (loss_host) *loss_host = (float)(sum / s.plan.ga_steps);  // per-rank mean; callers average over ranks
            if (norm_host) *norm_host = (float)nrm;
        }
    });
}

// staging copy for the end-to-end path: host tokens -> the session's token buffer
int qt_upload_tokens(qt_session* h, const int32_t* host, int64_t n, int32_t** dev_out) {
    return guard([&] {
        Session& s = *h->s;
        const int64_t cap = (int64_t)s.plan.ga_steps * s.plan.micro_batch * (s.T + 1);
        if (n > cap) throw QtError(1, "too many tokens for the session's token buffer");
        QT_CHECK_CUDA(cudaMemcpyAsync(s.tok_buf, host, n * 4, cudaMemcpyHostToDevice, s.st));
        *dev_out = s.tok_buf;
    });
}

int qt_sync(qt_session* h) {
    return guard([&] { QT_CHECK_CUDA(cudaStreamSynchronize(h->s->st)); });
}

// absmax statistics {N1, ATT, N2, H} per layer (ForwardStats, model.hpp:148-151)
int qt_forward_stats(qt_session* h, float* out) {
    return guard([&] {
        Session& s = *h->s;
        QT_CHECK_CUDA(cudaMemcpy(out, s.act_amax, s.L * 16, cudaMemcpyDeviceToHost));
    });
}

// raw bytes of a saved site of the last forward: dtype 0 = bf16, 1 = fp8 codes, 2 = f32
int qt_saved_raw(qt_session* h, int layer, const char* site, void* host, int64_t* bytes, int* dtype) {
    return guard([&] {
        Session& s = *h->s;
        const std::string n(site);
        const int64_t M = s.curM;
        const void* src = nullptr;
        int64_t nb = 0;
        int dt = 0;
        if (layer < 0 || layer > s.L) throw QtError(2, "layer out of range");
        LayerBufs& b = s.lb[layer];
        if (n == "r_in") {
            src = (s.offload_x() && layer < s.L) ? s.xhost + (size_t)layer * s.Mmax * s.d : b.r_in;
            nb = M * s.d * 2;
        }
        else if (n == "normed_final") { src = s.normed_final; nb = M * s.d * 2; }
        else if (n == "dlogits") { src = s.dlogits; nb = M * s.V * 2; }
        else if (n == "dlogits_lo") { src = s.dlogits_lo; nb = M * s.V * 2; }
        else if (n == "d_hidden") { src = s.d_hidden; nb = M * s.d * 2; }
        else if (n == "dl_tgt") { src = s.dl_tgt; nb = M * 4; dt = 2; }
        else if (n == "logits") { src = s.logits; nb = M * s.V * 4; dt = 2; }
        else if (layer == s.L) throw QtError(1, "only r_in exists for layer L (r_final)");
        else if (n == "n1c") { src = b.n1c; nb = M * s.d; dt = 1; }
        else if (n == "qkv") { src = b.qkv; nb = M * s.q * 2; }
        else if (n == "att") { src = b.att; nb = M * s.d * 2; }
        else if (n == "attc") { src = b.attc; nb = M * s.d; dt = 1; }
        else if (n == "r_mid") { src = b.r_mid; nb = M * s.d * 2; }
        else if (n == "n2c") { src = b.n2c; nb = M * s.d; dt = 1; }
        else if (n == "gate_up") { src = b.gu; nb = M * s.F * 2; }
        else if (n == "hc") { src = b.hc; nb = M * s.Hh; dt = 1; }
        else if (n == "lse") { src = b.lse; nb = (int64_t)s.curB * s.H * s.curT * 4; dt = 2; }
        else throw QtError(1, "unknown site " + n);
        if (!src) throw QtError(1, "site " + n + " is not kept in this CE backward mode");
        *bytes = nb;
        *dtype = dt;
        if (host) QT_CHECK_CUDA(cudaMemcpy(host, src, nb, cudaMemcpyDefault));
    });
}

// device scalars: which = 0 act scales (L*4), 1 weight scales (L*4), 2 grad scales (L*4), 3 weight amax (L*4)
int qt_scales(qt_session* h, int which, float* out) {
    return guard([&] {
        Session& s = *h->s;
        const void* src = which == 0 ? (void*)s.act_scale : which == 1 ? (void*)s.w_scale
                        : which == 2 ? (void*)s.g_scale : (void*)s.w_amax;
        QT_CHECK_CUDA(cudaMemcpy(out, src, s.L * 16, cudaMemcpyDeviceToHost));
    });
}

int qt_weight_codes(qt_session* h, int layer, int which, uint8_t* host) {
    return guard([&] {
        Session& s = *h->s;
        const int64_t n[4] = {(int64_t)s.q * s.d, (int64_t)s.d * s.d, (int64_t)s.F * s.d, (int64_t)s.d * s.Hh};
        if (layer < 0 || layer >= s.L || which < 0 || which > 3) throw QtError(2, "layer/weight out of range");
        if (!s.stream_codes()) {
            QT_CHECK_CUDA(cudaMemcpy(host, s.wcodes[layer * 4 + which], n[which], cudaMemcpyDeviceToHost));
        } else if (s.offload_weights() && !s.published.empty() && s.published[(size_t)layer]) {
            std::memcpy(host, s.whost + (size_t)layer * s.wl_total + s.wl_off[which], (size_t)n[which]);
        } else if (s.shard_weights()) {
            const int widx[4] = {1, 2, 4, 5};
            const ParamT& t = s.P[s.lp(layer, widx[which])];
            uint8_t* stage = reinterpret_cast<uint8_t*>(s.scratch_f32);
            s.coll([&] { s.tr->gather_idle(s.wown[layer * 4 + which], (size_t)t.pw, stage, s.st); });
            QT_CHECK_CUDA(cudaMemcpy(host, stage, n[which], cudaMemcpyDeviceToHost));
        } else {
            throw QtError(1, "weight codes are not built yet (build_step_context)");
        }
    });
}

int qt_set_profile(qt_session* h, int on) {
    return guard([&] {
        Session& s = *h->s;
        s.prof_on = on != 0;
        s.prof.clear();
        s.ev_used = 0;
    });
}

// per-category totals since qt_set_profile: ms[ncat], launches[ncat], work[ncat] (flops or bytes)
int qt_profile_read(qt_session* h, int ncat, double* ms, int64_t* launches, double* work) {
    return guard([&] {
        Session& s = *h->s;
        QT_CHECK_CUDA(cudaStreamSynchronize(s.st));
        for (int c = 0; c < ncat; ++c) {
            ms[c] = 0;
            launches[c] = 0;
            work[c] = 0;
        }
        for (auto& r : s.prof) {
            if (r.cat < 0 || r.cat >= ncat) continue;
            float t = 0;
            cudaEventElapsedTime(&t, r.a, r.b);
            ms[r.cat] += t;
            launches[r.cat] += 1;
            work[r.cat] += r.work;
        }
    });
}

int qt_session_footprint(const QtModelConfig* cfg, const QtPrecisionMap* prec, const QtRunPlan* plan, int world,
                         uint64_t* device_bytes, uint64_t* host_bytes) {
    return guard([&] {
        if (world < 1) throw QtError(1, "qt_session_footprint: world must be >= 1");
        Session s(Session::DryRun{}, *cfg, *prec, *plan, world);
        *device_bytes = s.arena_bytes;
        *host_bytes = s.host_bytes + Session::kBlkRing * 64;  // + the step-block staging ring
    });
}

int qt_search_plan_session(const QtModelConfig* cfg, const QtHardwareProfile* hw, int workers,
                           int64_t target_batch_tokens, int exhaustive, int max_results, char* json_out, size_t cap,
                           size_t* needed) {
    int rc = 0;
    const int g = guard([&] {
        // the search ladder of the reference, filtered by the session's real arena: plans whose
        // recompute/offload/sharding the session does not run, or that its kernels reject, fail
        // the footprint and drop out
        auto fn = [](const QtModelConfig& c, const QtPrecisionMap& p, const QtRunPlan& pl, int W, bool,
                     const QtMemTier&) -> uint64_t {
            QtPrecisionMap pr = p;
            pr.backward_grads = 1;
            try {
                Session s(Session::DryRun{}, c, pr, pl, W);
                return s.arena_bytes;
            } catch (const std::exception&) {
                return ~uint64_t(0);
            }
        };
        const std::string text =
            qtb::plan::search_with(*cfg, *hw, workers, target_batch_tokens, 0, exhaustive != 0, false, fn, max_results)
                .dump();
        if (needed) *needed = text.size() + 1;
        if (json_out && cap >= text.size() + 1) std::memcpy(json_out, text.c_str(), text.size() + 1);
        else if (json_out) rc = 1;
    });
    return g ? g : rc;
}

// host-side ZeRO-1 layout (src/comms.cpp:69-73), exported for the gloo tests
int qt_shard_layout(int64_t numel, int workers, int64_t* padded, int64_t* per_worker) {
    if (workers < 1) return 1;
    const int64_t unit = 256 * (int64_t)workers;
    *padded = ceil_div(numel, unit) * unit;
    *per_worker = *padded / workers;
    return 0;
}

uint64_t qt_fnv1a64(const char* s) { return fnv1a64(s); }

// the session's RoPE table (T x hd/2 {cos, sin} float pairs) into host memory
int qt_rope_table(int T, int hd, float* host_out) {
    if (T < 1 || hd < 2 || (hd & 1) || !host_out) return 1;
    rope_table_host(T, hd, reinterpret_cast<float2*>(host_out));
    return 0;
}

// one shard of reduce_scatter_copy / reduce_scatter_oracle (src/comms.cpp:185-254):
// srcs = W device pointers (bf16 chunks of this shard, indexed by source worker)
int qtk_reduce_scatter_sr(float* acc, const void* const* srcs, int W, int self, int64_t n, int stochastic,
                          uint64_t seed, uint64_t step, uint64_t layer, cudaStream_t s) {
    if (W < 1 || W > 16 || self < 0 || self >= W || n < 0 || !acc || !srcs) return 1;
    if (n == 0) return 0;
    qtb::RsArgs a{};
    for (int w = 0; w < W; ++w) {
        if (!srcs[w]) return 1;
        a.src[w] = static_cast<const uint16_t*>(srcs[w]);
        const std::string name = "rs/" + std::to_string(step) + "/" + std::to_string(layer) + "/" + std::to_string(w);
        a.key[w] = qtb::rng_key(seed, qtb::fnv1a64(name));
    }
    qtb::reduce_scatter_sr_kernel<<<qtb::grid_for(n), 256, 0, s>>>(acc, a, W, self, n, stochastic);
    return (int)cudaGetLastError();
}

// Exact count of this library's kernel launches in one trainer step: the
// step is captured into a CUDA graph (not executed) and its kernel nodes are
// counted.  Collective nodes (NCCL) are counted separately.
// Diagnostic: one trainer step captured into a CUDA graph and replayed `iters`
// times (the same step counters each replay, so the math repeats step `step`);
// returns the mean device time per replay.  Measures what graph launch would
// save over stream launch; not a training entry point.
int qt_time_graph_step(qt_session* h, const int32_t* tokens_dev, int64_t tokens_per_mb, int64_t batch, int64_t step,
                       int iters, float* ms_out) {
    return guard([&] {
        Session& s = *h->s;
        const int64_t saved_step = s.step_count;
        const bool saved_amax = s.amax_cached;
        cudaGraph_t g = nullptr;
        QT_CHECK_CUDA(cudaStreamBeginCapture(s.st, cudaStreamCaptureModeRelaxed));
        try {
            s.train_step_body(tokens_dev, tokens_per_mb, batch, step, s.hyper.max_grad_norm);
        } catch (...) {
            cudaStreamEndCapture(s.st, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        QT_CHECK_CUDA(cudaStreamEndCapture(s.st, &g));
        s.step_count = saved_step;
        s.amax_cached = saved_amax;
        cudaGraphExec_t ge = nullptr;
        QT_CHECK_CUDA(cudaGraphInstantiate(&ge, g, 0));
        QT_CHECK_CUDA(cudaGraphLaunch(ge, s.st));  // warm-up
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, s.st);
        for (int i = 0; i < iters; ++i) QT_CHECK_CUDA(cudaGraphLaunch(ge, s.st));
        cudaEventRecord(b, s.st);
        QT_CHECK_CUDA(cudaEventSynchronize(b));
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, a, b);
        *ms_out = ms / iters;
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
    });
}

int qt_count_step_kernels(qt_session* h, const int32_t* tokens_dev, int64_t tokens_per_mb, int64_t batch,
                          int64_t* kernels, int64_t* other_nodes) {
    return guard([&] {
        Session& s = *h->s;
        const int64_t saved_step = s.step_count;
        const bool saved_amax = s.amax_cached;  // the captured step is not executed
        cudaGraph_t g = nullptr;
        QT_CHECK_CUDA(cudaStreamBeginCapture(s.st, cudaStreamCaptureModeRelaxed));
        try {
            s.train_step_body(tokens_dev, tokens_per_mb, batch, saved_step, s.hyper.max_grad_norm);
        } catch (...) {
            cudaStreamEndCapture(s.st, &g);
            if (g) cudaGraphDestroy(g);
            s.step_count = saved_step;
            s.amax_cached = saved_amax;
            throw;
        }
        QT_CHECK_CUDA(cudaStreamEndCapture(s.st, &g));
        s.step_count = saved_step;
        s.amax_cached = saved_amax;
        size_t n = 0;
        QT_CHECK_CUDA(cudaGraphGetNodes(g, nullptr, &n));
        std::vector<cudaGraphNode_t> nodes(n);
        QT_CHECK_CUDA(cudaGraphGetNodes(g, nodes.data(), &n));
        int64_t k = 0, o = 0;
        for (auto nd : nodes) {
            cudaGraphNodeType t;
            cudaGraphNodeGetType(nd, &t);
            if (t == cudaGraphNodeTypeKernel) ++k;
            else if (t != cudaGraphNodeTypeEmpty) ++o;
        }
        cudaGraphDestroy(g);
        *kernels = k;
        *other_nodes = o;
    });
}

}  // extern "C"
