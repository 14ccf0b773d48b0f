// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" wrapper over the UNMODIFIED reference implementation (qtrain,
// compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libqtrain_ref.so).  It exposes plain pointer/size entry points
// so Python tests and bench.py's cpu_baseline leg can call the reference's
// own code through ctypes.  Every function names the reference routine it
// forwards to (file:line under /root/reference/proj).
//
// Status codes mirror the product C-ABI: 0 ok, 1 std::invalid_argument,
// 2 std::out_of_range, 3 std::runtime_error (message in ref_last_error()).

#include "qtrain/model.hpp"
#include "qtrain/numerics.hpp"
#include "qtrain/optim.hpp"
#include "qtrain/tensorops.hpp"
#include "qtrain/trainer.hpp"
#include "qtrain/corpus.hpp"
#include "qtrain/memplan.hpp"
#include "qtrain/comms.hpp"
#include "qtrain/offload.hpp"
#include "qtrain/profiles.hpp"
#include "qtrain/manifest.hpp"
#include "qtrain/checkpoint.hpp"

#include <json.hpp>

#include <chrono>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

using namespace qtrain;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

F8Kind kind_of(int k) { return k == 0 ? F8Kind::E4M3 : F8Kind::E5M2; }

Tensor make_tensor(const float* p, std::vector<std::int64_t> shape) {
    const auto n = Tensor::numel_of(shape);
    return Tensor{std::move(shape), std::vector<float>(p, p + n)};
}

void put(const Tensor& t, float* out) { std::memcpy(out, t.data.data(), t.data.size() * sizeof(float)); }

ScaledQuant make_quant(const std::uint8_t* codes, std::int64_t rows, std::int64_t cols, int kind,
                       float scale) {
    ScaledQuant q;
    q.shape = {rows, cols};
    q.codes.assign(codes, codes + rows * cols);
    q.kind = kind_of(kind);
    q.scale = scale;
    return q;
}

ModelConfig cfg_of(const int* c) {
    // c = {n_layers, d_model, d_ff, n_heads, n_kv_heads, vocab, seq_len}
    ModelConfig m;
    m.n_layers = c[0];
    m.d_model = c[1];
    m.d_ff = c[2];
    m.n_heads = c[3];
    m.n_kv_heads = c[4];
    m.vocab = c[5];
    m.seq_len = c[6];
    return m;
}

PrecisionMap prec_of(int matmuls, int grads, int f32_debug) {
    PrecisionMap p;
    p.block_matmuls = matmuls == 0 ? MatmulPrecision::FP8_E4M3 : MatmulPrecision::BF16;
    p.backward_grads = grads == 0 ? GradPrecision::E4M3 : GradPrecision::E5M2;
    p.f32_debug = f32_debug != 0;
    return p;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- numerics (src/numerics.cpp) -------------------------------------------

// src/numerics.cpp:129
int ref_f8_encode(const float* x, std::int64_t n, int kind, std::uint8_t* out) {
    return guard([&] {
        for (std::int64_t i = 0; i < n; ++i) out[i] = f8_encode(x[i], kind_of(kind));
    });
}
// src/numerics.cpp:127
int ref_f8_decode_table(int kind, float* out256) {
    return guard([&] {
        const auto t = f8_decode_table(kind_of(kind));
        for (int i = 0; i < 256; ++i) out256[i] = t[static_cast<std::size_t>(i)];
    });
}
float ref_f8_fmax(int kind) { return f8_fmax(kind_of(kind)); }
// src/numerics.cpp:141-148
int ref_absmax(const float* x, std::int64_t n, float* out) {
    return guard([&] { *out = absmax(std::span<const float>(x, static_cast<std::size_t>(n))); });
}
// src/numerics.cpp:150-158
float ref_absmax_scale(float a, int kind) { return absmax_scale(a, kind_of(kind)); }
// src/numerics.cpp:160-176
int ref_quantize_with_absmax(const float* x, std::int64_t n, int kind, float amax, std::uint8_t* codes,
                             float* scale) {
    return guard([&] {
        const auto q = quantize_with_absmax(std::span<const float>(x, static_cast<std::size_t>(n)), {n},
                                            kind_of(kind), amax);
        std::memcpy(codes, q.codes.data(), q.codes.size());
        *scale = q.scale;
    });
}
// src/tensorops.cpp:164-182
int ref_transpose_quantize_with_absmax(const float* x, std::int64_t rows, std::int64_t cols, int kind,
                                       float amax, std::uint8_t* codes, float* scale) {
    return guard([&] {
        const auto q = transpose_quantize_with_absmax(make_tensor(x, {rows, cols}), kind_of(kind), amax);
        std::memcpy(codes, q.codes.data(), q.codes.size());
        *scale = q.scale;
    });
}
// src/numerics.cpp:203-210
std::uint32_t ref_rng_uniform(std::uint64_t seed, std::uint64_t stream, std::uint64_t counter) {
    return rng_uniform({seed, stream, counter});
}
float ref_rng_normal(std::uint64_t seed, std::uint64_t stream, std::uint64_t counter) {
    return rng_normal({seed, stream, counter});
}
std::uint64_t ref_fnv1a64(const char* s) { return fnv1a64(s); }
float ref_bf16_round(float x) { return bf16_round(x); }
float ref_stochastic_round_bf16(float x, std::uint64_t seed, std::uint64_t stream, std::uint64_t counter) {
    return stochastic_round_bf16(x, {seed, stream, counter});
}

// ---- tensorops (src/tensorops.cpp) ------------------------------------------

// src/tensorops.cpp:41-59
int ref_matmul_fp8(const std::uint8_t* a, std::int64_t M, std::int64_t K, int akind, float ascale,
                   const std::uint8_t* b, std::int64_t N, int bkind, float bscale, int round_bf16,
                   float* out) {
    return guard([&] {
        const auto r = matmul_tn(make_quant(a, M, K, akind, ascale), make_quant(b, N, K, bkind, bscale),
                                 round_bf16 ? OutRound::Bf16 : OutRound::None);
        put(r, out);
    });
}
// src/tensorops.cpp:24-39
int ref_matmul_f32(const float* a, std::int64_t M, std::int64_t K, const float* b, std::int64_t N,
                   int round_bf16, float* out) {
    return guard([&] {
        put(matmul_tn(make_tensor(a, {M, K}), make_tensor(b, {N, K}),
                      round_bf16 ? OutRound::Bf16 : OutRound::None),
            out);
    });
}
// src/tensorops.cpp:61-86
int ref_rmsnorm_residual_fused(const float* x, const float* res, const float* gamma, std::int64_t rows,
                               std::int64_t d, float eps, float* nr_out, float* normed_out,
                               float* absmax_out) {
    return guard([&] {
        Tensor xt;
        if (x) xt = make_tensor(x, {rows, d});
        auto [nr, nf] = rmsnorm_residual_fused(x ? &xt : nullptr, make_tensor(res, {rows, d}),
                                               make_tensor(gamma, {d}), eps, OutRound::Bf16);
        put(nr, nr_out);
        put(nf.value, normed_out);
        *absmax_out = nf.absmax;
    });
}
// src/tensorops.cpp:88-112
int ref_rmsnorm_residual_backward(const float* nr, const float* gamma, std::int64_t rows, std::int64_t d,
                                  float eps, const float* dy, const float* d_extra, float* d_in,
                                  float* d_gamma) {
    return guard([&] {
        Tensor de;
        if (d_extra) de = make_tensor(d_extra, {rows, d});
        auto g = rmsnorm_residual_backward(make_tensor(nr, {rows, d}), make_tensor(gamma, {d}), eps,
                                           make_tensor(dy, {rows, d}), d_extra ? &de : nullptr,
                                           OutRound::Bf16);
        put(g.d_input, d_in);
        put(g.d_gamma, d_gamma);
    });
}
// src/tensorops.cpp:114-132
int ref_swiglu_fused(const float* gu, std::int64_t rows, std::int64_t two_h, float* h, float* absmax_out) {
    return guard([&] {
        auto r = swiglu_fused(make_tensor(gu, {rows, two_h}), OutRound::Bf16);
        put(r.value, h);
        *absmax_out = r.absmax;
    });
}
// src/tensorops.cpp:134-153
int ref_swiglu_backward(const float* gu, std::int64_t rows, std::int64_t two_h, const float* dh,
                        float* dgu) {
    return guard([&] {
        put(swiglu_backward(make_tensor(gu, {rows, two_h}), make_tensor(dh, {rows, two_h / 2}),
                            OutRound::Bf16),
            dgu);
    });
}
// src/tensorops.cpp:227-255
int ref_sdpa(const float* q, const float* k, const float* v, std::int64_t H, std::int64_t Hkv,
             std::int64_t T, std::int64_t D, std::int64_t chunk_rows, float* out) {
    return guard([&] {
        put(sdpa_chunked(make_tensor(q, {H, T, D}), make_tensor(k, {Hkv, T, D}),
                         make_tensor(v, {Hkv, T, D}), chunk_rows, OutRound::Bf16),
            out);
    });
}
// src/tensorops.cpp:257-303
int ref_sdpa_backward(const float* q, const float* k, const float* v, const float* go, std::int64_t H,
                      std::int64_t Hkv, std::int64_t T, std::int64_t D, std::int64_t chunk_rows,
                      float* dq, float* dk, float* dv) {
    return guard([&] {
        auto g = sdpa_chunked_backward(make_tensor(q, {H, T, D}), make_tensor(k, {Hkv, T, D}),
                                       make_tensor(v, {Hkv, T, D}), make_tensor(go, {H, T, D}),
                                       chunk_rows, OutRound::Bf16);
        put(g.dq, dq);
        put(g.dk, dk);
        put(g.dv, dv);
    });
}
// src/tensorops.cpp:317-342
int ref_embedding_backward(const std::int32_t* ids, std::int64_t n, const float* grad_out, std::int64_t d,
                           std::int64_t vocab, float* out) {
    return guard([&] {
        put(embedding_backward_sorted(std::span<const std::int32_t>(ids, static_cast<std::size_t>(n)),
                                      make_tensor(grad_out, {n, d}), vocab),
            out);
    });
}
// src/tensorops.cpp:344-410
int ref_cross_entropy(const float* hidden, std::int64_t N, std::int64_t d, const float* lm_w,
                      std::int64_t V, const std::int32_t* targets, std::int64_t chunk, int with_grads,
                      float* loss, float* d_hidden, float* d_lm_w) {
    return guard([&] {
        auto r = fused_cross_entropy_chunked(make_tensor(hidden, {N, d}), make_tensor(lm_w, {V, d}),
                                             std::span<const std::int32_t>(targets, static_cast<std::size_t>(N)),
                                             chunk, with_grads != 0, OutRound::Bf16);
        *loss = r.loss;
        if (with_grads) {
            put(r.d_hidden, d_hidden);
            put(r.d_lm_w, d_lm_w);
        }
    });
}

// ---- optimizer primitives (src/optim.cpp) -----------------------------------

// src/optim.cpp:153-164 on a single named tensor; m/v/p updated in place
int ref_adamw_tensor(const char* name, float* p, float* m, float* v, const float* g, std::int64_t n,
                     float lr, float b1, float b2, float eps, float wd, int bf16_moments, int bf16_params,
                     std::uint64_t seed, std::int64_t step_count, float grad_scale) {
    return guard([&] {
        OptimState st;
        st.hyper = AdamWHyper{lr, b1, b2, eps, wd};
        st.moments = bf16_moments ? MomentPrecision::BF16_SR : MomentPrecision::F32;
        st.params = bf16_params ? ParamPrecision::BF16_SR : ParamPrecision::F32;
        st.seed = seed;
        st.step_count = step_count;
        Tensor pt = make_tensor(p, {n});
        st.slots.emplace(name, std::make_pair(make_tensor(m, {n}), make_tensor(v, {n})));
        GradMap gm;
        gm.emplace(name, make_tensor(g, {n}));
        NamedTensors nt{{name, &pt}};
        adamw_step(st, nt, gm, grad_scale);
        put(pt, p);
        put(st.slots.at(name).first, m);
        put(st.slots.at(name).second, v);
    });
}
// src/optim.cpp:87-105
double ref_grad_norm_partials(const float* g, std::int64_t n) {
    return grad_norm_block_partials(make_tensor(g, {n}), 0, n);
}
// src/model.cpp:448-464 on one named tensor.  GradAccumulator has no buffer
// setter, so the update line model.cpp:455-462 is applied through the
// reference's own stochastic_round_bf16 / fnv1a64 on an existing buffer.
int ref_grad_accumulate(const char* name, float* buf, const float* g, std::int64_t n, int f32_mode,
                        std::uint64_t seed, std::uint64_t micro_step) {
    return guard([&] {
        const std::uint64_t stream = fnv1a64(std::string("gradaccum/") + name);
        const std::uint64_t base = micro_step * static_cast<std::uint64_t>(n);
        for (std::int64_t i = 0; i < n; ++i) {
            const float s = buf[i] + g[i];
            buf[i] = f32_mode ? s
                              : stochastic_round_bf16(s, {seed, stream, base + static_cast<std::uint64_t>(i)});
        }
    });
}

// ---- model-level handle (src/model.cpp, src/optim.cpp, src/trainer.cpp) ------

struct RefModel {
    ModelConfig cfg;
    ModelParams params;
    OptimState opt;
    PrecisionMap prec;
    ChunkSpec chunks;
    RecomputeSet recompute;
    std::uint64_t seed = 0;
    // last forward / backward, kept for inspection by tests
    std::unique_ptr<ForwardResult> fwd;
    GradMap grads;     // raw model_backward output
    GradMap acc_grads; // after GradAccumulator + cross-worker sum (trainer.cpp:90-103)
    double last_norm = 0.0;
    std::vector<std::pair<std::string, Tensor*>> named;
    void rebuild_names() {
        named.clear();
        for_each_param(params, [&](const std::string& n, Tensor& t) { named.emplace_back(n, &t); });
    }
};

// init_params: src/model.cpp:67-86
void* ref_model_new(const int* cfg7, std::uint64_t seed, int matmuls, int grads, int f32_debug) {
    auto* m = new RefModel();
    if (guard([&] {
            m->cfg = cfg_of(cfg7);
            m->params = init_params(m->cfg, seed);
            m->prec = prec_of(matmuls, grads, f32_debug);
            m->seed = seed;
            m->opt.seed = seed;
            m->opt.params = m->prec.f32_debug ? ParamPrecision::F32 : ParamPrecision::BF16_SR;
            m->rebuild_names();
        }) != 0) {
        delete m;
        return nullptr;
    }
    return m;
}
void ref_model_free(void* h) { delete static_cast<RefModel*>(h); }

int ref_model_set_options(void* h, int recompute_bits, std::int64_t lmhead_chunk, std::int64_t attn_chunk,
                          float lr, float b1, float b2, float eps, float wd, int bf16_moments) {
    auto* m = static_cast<RefModel*>(h);
    return guard([&] {
        m->recompute.bits = static_cast<std::uint8_t>(recompute_bits);
        m->chunks = ChunkSpec{lmhead_chunk, attn_chunk};
        m->opt.hyper = AdamWHyper{lr, b1, b2, eps, wd};
        m->opt.moments = bf16_moments ? MomentPrecision::BF16_SR : MomentPrecision::F32;
    });
}

int ref_model_num_params(void* h) { return static_cast<int>(static_cast<RefModel*>(h)->named.size()); }
const char* ref_model_param_name(void* h, int i) {
    return static_cast<RefModel*>(h)->named[static_cast<std::size_t>(i)].first.c_str();
}
std::int64_t ref_model_param_numel(void* h, int i) {
    return static_cast<RefModel*>(h)->named[static_cast<std::size_t>(i)].second->numel();
}
void ref_model_get_param(void* h, int i, float* out) {
    put(*static_cast<RefModel*>(h)->named[static_cast<std::size_t>(i)].second, out);
}
void ref_model_set_param(void* h, int i, const float* in) {
    auto* t = static_cast<RefModel*>(h)->named[static_cast<std::size_t>(i)].second;
    std::memcpy(t->data.data(), in, t->data.size() * sizeof(float));
}
// optimizer moments by param index (zeros until the first step)
int ref_model_get_moments(void* h, int i, float* m_out, float* v_out) {
    auto* m = static_cast<RefModel*>(h);
    return guard([&] {
        m->opt.ensure_slots(m->named);
        const auto& [mm, vv] = m->opt.slots.at(m->named[static_cast<std::size_t>(i)].first);
        put(mm, m_out);
        put(vv, v_out);
    });
}
int ref_model_set_moments(void* h, int i, const float* m_in, const float* v_in, std::int64_t step_count) {
    auto* m = static_cast<RefModel*>(h);
    return guard([&] {
        m->opt.ensure_slots(m->named);
        auto& [mm, vv] = m->opt.slots.at(m->named[static_cast<std::size_t>(i)].first);
        std::memcpy(mm.data.data(), m_in, mm.data.size() * sizeof(float));
        std::memcpy(vv.data.data(), v_in, vv.data.size() * sizeof(float));
        m->opt.step_count = step_count;
    });
}

// model_forward + model_backward on one micro-batch (src/model.cpp:297-446)
int ref_model_fwd_bwd(void* h, const std::int32_t* tokens, std::int64_t n_tokens, std::int64_t batch,
                      int with_grads, float* loss) {
    auto* m = static_cast<RefModel*>(h);
    return guard([&] {
        const StepContext sc = build_step_context(m->cfg, m->params, m->prec);
        m->fwd = std::make_unique<ForwardResult>(
            model_forward(m->cfg, m->params, sc, std::span<const std::int32_t>(tokens, n_tokens), batch,
                          m->recompute, m->prec, m->chunks, with_grads != 0));
        *loss = m->fwd->loss;
        if (with_grads) m->grads = model_backward(m->cfg, m->params, sc, *m->fwd, m->recompute, m->prec, m->chunks);
    });
}

// forward stats {N1, ATT, N2, H} per layer (include/qtrain/model.hpp:148-151)
void ref_model_forward_stats(void* h, float* out) {
    auto* m = static_cast<RefModel*>(h);
    for (std::size_t l = 0; l < m->fwd->stats.per_layer.size(); ++l)
        for (int s = 0; s < 4; ++s) out[l * 4 + s] = m->fwd->stats.per_layer[l][static_cast<std::size_t>(s)];
}

// saved activation by site name: r_in n1 qkv att r_mid n2 gate_up h; r_final;
// returns numel or -1 when the site was not kept
std::int64_t ref_model_saved(void* h, int layer, const char* site, float* out) {
    auto* m = static_cast<RefModel*>(h);
    const std::string s(site);
    if (s == "r_final") {
        if (out) put(m->fwd->r_final, out);
        return m->fwd->r_final.numel();
    }
    if (s == "d_hidden") {
        if (out) put(m->fwd->d_hidden, out);
        return m->fwd->d_hidden.numel();
    }
    auto& L = m->fwd->layers[static_cast<std::size_t>(layer)];
    const std::optional<Tensor>* opt = nullptr;
    if (s == "r_in") {
        if (out) put(L.r_in, out);
        return L.r_in.numel();
    }
    if (s == "n1") opt = &L.n1;
    else if (s == "qkv") opt = &L.qkv;
    else if (s == "att") opt = &L.att;
    else if (s == "r_mid") opt = &L.r_mid;
    else if (s == "n2") opt = &L.n2;
    else if (s == "gate_up") opt = &L.gate_up;
    else if (s == "h") opt = &L.h;
    if (!opt || !opt->has_value()) return -1;
    if (out) put(**opt, out);
    return (*opt)->numel();
}

// raw gradient of one parameter from the last ref_model_fwd_bwd
int ref_model_grad(void* h, const char* name, float* out) {
    auto* m = static_cast<RefModel*>(h);
    return guard([&] { put(m->grads.at(name), out); });
}
int ref_model_acc_grad(void* h, const char* name, float* out) {
    auto* m = static_cast<RefModel*>(h);
    return guard([&] { put(m->acc_grads.at(name), out); });
}

// One optimizer step exactly as run_training does (src/trainer.cpp:64-110):
// build the step context, GA x W micro-batches (worker w uses seed+w for SR),
// ascending-worker f32 sum, global norm * mean_scale, clip, (sharded) AdamW.
// tokens: GA*W micro-batches back to back, each batch*(seq+1) ids, ordered
// (ga, w) as trainer.cpp:75-76 derives mb_index.
int ref_model_train_step(void* h, const std::int32_t* tokens, std::int64_t tokens_per_mb, std::int64_t batch,
                         int ga_steps, int workers, std::int64_t step, float max_grad_norm,
                         float* train_loss, float* grad_norm) {
    auto* m = static_cast<RefModel*>(h);
    return guard([&] {
        const StepContext sc = build_step_context(m->cfg, m->params, m->prec);
        const int W = workers;
        std::vector<GradAccumulator> accs;
        for (int w = 0; w < W; ++w) accs.emplace_back(m->prec.f32_debug, m->seed + static_cast<std::uint64_t>(w));
        double loss_sum = 0.0;
        for (int ga = 0; ga < ga_steps; ++ga) {
            for (int w = 0; w < W; ++w) {
                const std::int32_t* mb = tokens + (static_cast<std::int64_t>(ga) * W + w) * tokens_per_mb;
                auto fwd = model_forward(m->cfg, m->params, sc, std::span<const std::int32_t>(mb, tokens_per_mb),
                                         batch, m->recompute, m->prec, m->chunks);
                loss_sum += fwd.loss;
                auto g = model_backward(m->cfg, m->params, sc, fwd, m->recompute, m->prec, m->chunks);
                accs[static_cast<std::size_t>(w)].accumulate(g, static_cast<std::uint64_t>(step) * ga_steps + ga);
            }
        }
        GradMap grads = accs[0].take();
        for (int w = 1; w < W; ++w) {
            const auto other = accs[static_cast<std::size_t>(w)].take();
            for (auto& [name, g] : grads) {
                const auto& o = other.at(name);
                for (std::size_t i = 0; i < g.data.size(); ++i) g.data[i] += o.data[i];
            }
        }
        const float mean_scale = 1.0f / (static_cast<float>(ga_steps) * W);
        const double norm = global_grad_norm(grads) * mean_scale;
        const float clip = clip_scale(norm, max_grad_norm);
        const float scale = mean_scale * clip;
        m->opt.step_count = step;
        if (W == 1) {
            adamw_step(m->opt, m->named, grads, scale);
        } else {
            WorkerGroup group(W);
            sharded_adamw_step(group, m->opt, m->named, grads, scale, /*threaded=*/false);
        }
        m->acc_grads = std::move(grads);
        m->last_norm = norm;
        *train_loss = static_cast<float>(loss_sum / (ga_steps * W));
        *grad_norm = static_cast<float>(norm);
    });
}

// timing helper for bench.py's cpu_baseline leg: one full step (as above) on
// the calling thread, returns seconds
double ref_model_time_step(void* h, const std::int32_t* tokens, std::int64_t tokens_per_mb, std::int64_t batch,
                           std::int64_t step) {
    float loss = 0.0f, norm = 0.0f;
    const auto t0 = std::chrono::steady_clock::now();
    const int rc = ref_model_train_step(h, tokens, tokens_per_mb, batch, 1, 1, step, 1.0f, &loss, &norm);
    const auto t1 = std::chrono::steady_clock::now();
    if (rc != 0) return -1.0;
    return std::chrono::duration<double>(t1 - t0).count();
}

// corpus (src/corpus.cpp:58-69)
int ref_make_corpus(int uniform, std::int64_t vocab, int seq_len, int n_train, int n_val, std::uint64_t seed,
                    std::int32_t* train_out, std::int32_t* val_out) {
    return guard([&] {
        CorpusSpec s;
        s.kind = uniform ? "uniform" : "perm-walk";
        s.vocab = vocab;
        s.seq_len = seq_len;
        s.n_train = n_train;
        s.n_val = n_val;
        s.seed = seed;
        const Corpus c = make_corpus(s);
        std::memcpy(train_out, c.train.data(), c.train.size() * sizeof(std::int32_t));
        std::memcpy(val_out, c.val.data(), c.val.size() * sizeof(std::int32_t));
    });
}

// MFU accounting (src/memplan.cpp:264-312): per-token FP8 and BF16 FLOPs
void ref_flops_per_token(const int* cfg7, double* fp8_flops, double* bf16_flops) {
    const auto fb = flop_breakdown(cfg_of(cfg7), RecomputeSet::none(), false);
    *fp8_flops = fb.linear;
    *bf16_flops = fb.lmhead + fb.attention;
}

// reduce_scatter_oracle / reduce_scatter_copy (src/comms.cpp:185-254): chunks is
// W x W x n (chunks[i][j] = worker i's chunk for shard j), acc W x n in/out
static int rs_common(const float* chunks, float* acc, int W, std::int64_t n, int stochastic, std::uint64_t seed,
                     std::uint64_t step, std::uint64_t layer, int protocol) {
    return guard([&] {
        std::vector<std::vector<Tensor>> ch((std::size_t)W);
        std::vector<Tensor> ac;
        for (int i = 0; i < W; ++i) {
            for (int j = 0; j < W; ++j) ch[(std::size_t)i].push_back(make_tensor(chunks + ((std::int64_t)i * W + j) * n, {n}));
            ac.push_back(make_tensor(acc + (std::int64_t)i * n, {n}));
        }
        SrSpec sr;
        sr.stochastic = stochastic != 0;
        sr.seed = seed;
        sr.step = step;
        sr.layer = layer;
        std::vector<Tensor> out;
        if (protocol) {
            WorkerGroup g(W);
            out = reduce_scatter_copy(g, ch, ac, sr, false, 0);
        } else {
            out = reduce_scatter_oracle(ch, ac, sr);
        }
        for (int i = 0; i < W; ++i) put(out[(std::size_t)i], acc + (std::int64_t)i * n);
    });
}
int ref_reduce_scatter_oracle(const float* chunks, float* acc, int W, std::int64_t n, int stochastic,
                              std::uint64_t seed, std::uint64_t step, std::uint64_t layer) {
    return rs_common(chunks, acc, W, n, stochastic, seed, step, layer, 0);
}
int ref_reduce_scatter_copy(const float* chunks, float* acc, int W, std::int64_t n, int stochastic,
                            std::uint64_t seed, std::uint64_t step, std::uint64_t layer) {
    return rs_common(chunks, acc, W, n, stochastic, seed, step, layer, 1);
}

// ---- planner (src/memplan.cpp, src/profiles.cpp, src/offload.cpp) ---------
// plan10 = {micro_batch, ga_steps, recompute_bits, offload_bits, shard_weights, shard_grads,
//           block_matmuls (0 fp8 / 1 bf16), bf16_moments, lmhead_chunk_tokens, attn_chunk_rows}
static RunPlan plan_of(const std::int64_t* p) {
    RunPlan r;
    r.micro_batch = (int)p[0];
    r.ga_steps = (int)p[1];
    r.recompute.bits = (std::uint8_t)p[2];
    const int ob = (int)p[3];
    r.offload.x = ob & 1;
    r.offload.m = ob & 2;
    r.offload.v = ob & 4;
    r.offload.master = ob & 8;
    r.offload.weights = ob & 16;
    r.offload.grads = ob & 32;
    r.shard_weights = p[4] != 0;
    r.shard_grads = p[5] != 0;
    r.precision.block_matmuls = p[6] == 0 ? MatmulPrecision::FP8_E4M3 : MatmulPrecision::BF16;
    r.moments = p[7] ? MomentPrecision::BF16_SR : MomentPrecision::F32;
    r.lmhead_chunk_tokens = p[8];
    r.attn_chunk_rows = p[9];
    return r;
}
static void put_tier(const MemoryBreakdown::Tier& t, std::uint64_t* o) {
    o[0] = t.params_fp8;
    o[1] = t.params_bf16_master;
    o[2] = t.moments_m;
    o[3] = t.moments_v;
    o[4] = t.grads;
    o[5] = t.residuals;
    o[6] = t.activations;
    o[7] = t.logits_workspace;
    o[8] = t.attn_workspace;
}
static int put_str(const std::string& s, char* out, std::size_t cap) {
    if (s.size() + 1 > cap) throw std::invalid_argument("output buffer too small: " + std::to_string(s.size() + 1));
    std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
}
static HardwareProfile prof_from(const char* name_or_json) {
    const std::string s(name_or_json);
    if (!s.empty() && s[0] == '{') return profile_from_json(s);
    return profile_by_name(s);
}

// memory_breakdown (src/memplan.cpp:263-268): out = device tier[9], host tier[9]
int ref_memory_breakdown(const int* cfg7, int tied, const std::int64_t* plan10, int workers, std::uint64_t* out18) {
    return guard([&] {
        const auto mb = memory_breakdown(cfg_of(cfg7), plan_of(plan10), workers, tied != 0);
        put_tier(mb.device, out18);
        put_tier(mb.host, out18 + 9);
    });
}
// flop_breakdown (src/memplan.cpp:274-290): {linear, lmhead, attention, recompute}
int ref_flop_breakdown(const int* cfg7, int recompute_bits, int tied, double* out4) {
    return guard([&] {
        RecomputeSet rc;
        rc.bits = (std::uint8_t)recompute_bits;
        const auto fb = flop_breakdown(cfg_of(cfg7), rc, tied != 0);
        out4[0] = fb.linear;
        out4[1] = fb.lmhead;
        out4[2] = fb.attention;
        out4[3] = fb.recompute;
    });
}
// mfu (src/memplan.cpp:315-320)
int ref_mfu(double tps, const int* cfg7, int matmuls, const char* profile, int tied, double* out) {
    return guard([&] { *out = mfu(tps, cfg_of(cfg7), prec_of(matmuls, 0, 0), prof_from(profile), tied != 0); });
}
int ref_fp8_speedup_ceiling(const int* cfg7, const char* profile, int tied, double* out) {
    return guard([&] { *out = fp8_speedup_ceiling(cfg_of(cfg7), prof_from(profile), tied != 0); });
}
// estimate_step_time (src/memplan.cpp:331-406): {compute, transfer, exposed, optimizer, total, feasible, tps}
int ref_estimate_step_time(const int* cfg7, const std::int64_t* plan10, const char* profile, int workers, int tied,
                           double* out7) {
    return guard([&] {
        const auto t = estimate_step_time(cfg_of(cfg7), plan_of(plan10), prof_from(profile), workers, tied != 0);
        out7[0] = t.compute;
        out7[1] = t.transfer;
        out7[2] = t.exposed_transfer;
        out7[3] = t.optimizer;
        out7[4] = t.total;
        out7[5] = t.feasible_in_time ? 1.0 : 0.0;
        out7[6] = t.tokens_per_second;
    });
}
// search_plan (src/memplan.cpp:471-551) -> JSON {"feasible": [{"str", "tps", "device"}], "no_fit_reason"}
int ref_search_plan(const int* cfg7, const char* profile, int workers, std::int64_t target, int matmuls,
                    int exhaustive, int tied, char* out, std::size_t cap) {
    return guard([&] {
        const auto r = search_plan(cfg_of(cfg7), prof_from(profile), workers, target,
                                   matmuls == 0 ? MatmulPrecision::FP8_E4M3 : MatmulPrecision::BF16, exhaustive != 0,
                                   tied != 0);
        nlohmann::json j;
        j["feasible"] = nlohmann::json::array();
        for (const auto& v : r.feasible)
            j["feasible"].push_back({{"str", v.plan.str()},
                                     {"tps", v.time.tokens_per_second},
                                     {"device", v.memory.device.total()},
                                     {"host", v.memory.host.total()}});
        if (r.no_fit_reason) j["no_fit_reason"] = *r.no_fit_reason;
        put_str(j.dump(), out, cap);
    });
}
// plan_residency (src/offload.cpp:40-163) -> {"jsonl", "high_water", "hw_weights", "hw_grads", "hw_residuals", "feasible"}
int ref_plan_residency(const int* cfg7, const std::int64_t* plan10, std::uint64_t budget, int tied, char* out,
                       std::size_t cap) {
    return guard([&] {
        TierBudget b;
        b.device_bytes = budget;
        const auto r = plan_residency(cfg_of(cfg7), plan_of(plan10), b, tied != 0);
        nlohmann::json j;
        j["jsonl"] = r.to_jsonl();
        j["high_water"] = r.high_water_device;
        j["hw_weights"] = r.high_water_by_category_weights;
        j["hw_grads"] = r.high_water_by_category_grads;
        j["hw_residuals"] = r.high_water_by_category_residuals;
        j["feasible"] = r.feasible;
        j["report"] = r.report;
        put_str(j.dump(), out, cap);
    });
}
int ref_profile_json(const char* name, char* out, std::size_t cap) {
    return guard([&] { put_str(profile_to_json(profile_by_name(name)), out, cap); });
}
int ref_transfer_time(std::uint64_t bytes, const char* profile, int policy, double* out) {
    return guard([&] {
        *out = transfer_time(bytes, prof_from(profile), policy == 0 ? TransferPolicy::ZeroCopy : TransferPolicy::DoubleBuffer);
    });
}

// ---- manifest / trainer / checkpoint (src/manifest.cpp, src/trainer.cpp, src/checkpoint.cpp)
int ref_manifest_normalize(const char* text, char* out, std::size_t cap) {
    return guard([&] { put_str(manifest_to_json(manifest_from_json(text)), out, cap); });
}
// run_training_to_files (src/trainer.cpp:152-171): metrics CSV + checkpoint per the manifest
int ref_run_training(const char* text, char* csv_out, std::size_t cap) {
    return guard([&] {
        const auto r = run_training_to_files(manifest_from_json(text));
        put_str(metrics_to_csv(r), csv_out, cap);
    });
}

} // extern "C"
