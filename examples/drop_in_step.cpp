// Drop-in usage of the reference's operator API (qtrain::model_forward /
// model_backward / global_grad_norm / clip / adamw_step, src/trainer.cpp:64-110)
// from plain C++ over libqtrain_b200.so.  Build:
//   g++ -std=c++17 -O2 examples/drop_in_step.cpp -Iinclude -I/usr/local/cuda/include \
//       -Lpaper_2512_15306_b200 -lqtrain_b200 -Wl,-rpath,$PWD/paper_2512_15306_b200 -o build/drop_in_step
#include <cmath>
#include <cstdio>
#include <random>

#include "qtrain_b200/qtrain.hpp"

int main() {
    using namespace qtrain_b200;
    ModelConfig cfg;
    cfg.n_layers = 2;
    cfg.d_model = 256;
    cfg.d_ff = 1536;
    cfg.n_heads = 4;
    cfg.n_kv_heads = 4;
    cfg.vocab = 512;
    cfg.seq_len = 256;
    PrecisionMap prec;
    prec.backward_grads = GradPrecision::E5M2;
    RunPlan plan;
    plan.micro_batch = 4;
    AdamWHyper hyper;
    Session s(cfg, prec, plan, hyper, /*seed=*/1234);
    s.init_params(1234);
    std::mt19937 gen(7);
    std::vector<std::int32_t> toks(4 * (cfg.seq_len + 1));
    float first = 0.f, last = 0.f;
    for (int step = 0; step < 20; ++step) {
        for (auto& t : toks) t = static_cast<std::int32_t>(gen() % 64);  // small alphabet: learnable
        // the reference's step, spelled out through the operator API
        s.build_step_context();
        s.zero_grads();
        const float loss = s.model_forward(toks, 4);
        s.model_backward(static_cast<std::uint64_t>(step));
        const double norm = s.global_grad_norm();
        const float clip = (norm <= 1.0) ? 1.0f : static_cast<float>(1.0 / norm);
        s.adamw_step(clip);
        if (step == 0) first = loss;
        last = loss;
        std::printf("step %2d loss %.5f grad_norm %.4f\n", step, loss, norm);
    }
    // error behaviour mirrors the reference: out-of-range ids throw std::out_of_range
    toks[5] = 100000;
    try {
        s.model_forward(toks, 4);
        std::printf("FAIL: no exception\n");
        return 1;
    } catch (const std::out_of_range& e) {
        std::printf("out_of_range: %s\n", e.what());
    }
    return (std::isfinite(last) && last < first) ? 0 : 1;
}
