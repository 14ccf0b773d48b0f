// The reference's trainer step (src/trainer.cpp:64-110) written with the
// reference's free-function signatures (qtrain::build_step_context,
// model_forward, model_backward, global_grad_norm, clip_scale, adamw_step),
// namespace swapped to qtrain_b200, plus a QTCKPT01 checkpoint round trip.
// Build:
//   g++ -std=c++17 -O2 examples/reference_signatures.cpp -Iinclude -I/usr/local/cuda/include \
//       -Lpaper_2512_15306_b200 -lqtrain_b200 -Wl,-rpath,$PWD/paper_2512_15306_b200 -o build/ref_sig
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "qtrain_b200/qtrain.hpp"

namespace qt = qtrain_b200;

int main(int argc, char** argv) {
    const std::string ckpt = argc > 1 ? argv[1] : "/tmp/ref_sig.ckpt";
    qt::ModelConfig cfg;
    cfg.n_layers = 2;
    cfg.d_model = 128;
    cfg.d_ff = 256;
    cfg.n_heads = 4;
    cfg.n_kv_heads = 2;
    cfg.vocab = 512;
    cfg.seq_len = 64;
    qt::PrecisionMap prec;
    prec.backward_grads = qt::GradPrecision::E5M2;
    qt::RunPlan plan;
    plan.micro_batch = 2;
    plan.ga_steps = 2;
    qt::Session params(cfg, prec, plan, qt::AdamWHyper{}, /*seed=*/99);
    params.init_params(99);
    const int GA = 2, batch = 2;
    const float max_grad_norm = 1.0f;
    std::vector<std::int32_t> toks(batch * (cfg.seq_len + 1));
    float first = 0.0f, last = 0.0f;
    for (int step = 0; step < 8; ++step) {
        const auto sc = qt::build_step_context(cfg, params, prec);  // trainer.cpp:65
        params.zero_grads();
        double loss_sum = 0.0;
        for (int ga = 0; ga < GA; ++ga) {
            for (std::size_t i = 0; i < toks.size(); ++i)  // a learnable walk over 64 ids
                toks[i] = static_cast<std::int32_t>((i * 7 + step * 3 + ga) % 64);
            auto fwd = qt::model_forward(cfg, params, sc, toks, batch, qt::RecomputeSet::none(), prec);
            loss_sum += fwd.loss;
            qt::model_backward(cfg, params, sc, fwd, qt::RecomputeSet::none(), prec, {},
                               static_cast<std::uint64_t>(step) * GA + ga);
        }
        const float mean_scale = 1.0f / GA;
        const double norm = qt::global_grad_norm(params) * mean_scale;  // trainer.cpp:105
        const float clip = qt::clip_scale(norm, max_grad_norm);
        qt::adamw_step(params, mean_scale * clip);
        const float train_loss = static_cast<float>(loss_sum / GA);
        if (step == 0) first = train_loss;
        last = train_loss;
        std::printf("step %d loss %.5f norm %.5f\n", step, train_loss, norm);
    }
    // checkpoint round trip: a fresh session restores params and optimizer state bit for bit
    qt::save_checkpoint(ckpt, params, cfg);
    qt::Session other(cfg, prec, plan, qt::AdamWHyper{}, 99);
    const std::int64_t step = qt::load_checkpoint(ckpt, other);
    bool same = step == 8;
    for (int i = 0; i < static_cast<int>(params.params().size()); ++i) {
        const auto a = params.get_param(i), b = other.get_param(i);
        same = same && std::memcmp(a.data(), b.data(), a.size() * sizeof(float)) == 0;
    }
    // errors keep the reference's exception types and messages
    bool threw = false;
    try {
        params.adamw_step(INFINITY);
    } catch (const std::runtime_error& e) {
        threw = std::strstr(e.what(), "adamw_step: non-finite gradient in") != nullptr;
    }
    // a per-call recompute set other than the session's is rejected (invalid_argument)
    bool rejected = false;
    try {
        const auto sc = qt::build_step_context(cfg, params, prec);
        qt::model_forward(cfg, params, sc, toks, batch, qt::RecomputeSet::block(), prec);
    } catch (const std::invalid_argument& e) {
        rejected = std::strstr(e.what(), "recompute set differs") != nullptr;
    }
    threw = threw && rejected;
    std::printf("%s first %.5f last %.5f checkpoint %s errors %s\n", last < first && same && threw ? "OK" : "FAIL",
                first, last, same ? "bitwise" : "DIFFERS", threw ? "ok" : "WRONG");
    return last < first && same && threw ? 0 : 1;
}
