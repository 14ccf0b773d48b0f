// TEST INFRASTRUCTURE (checker only, never shipped).
//
// The reference's model.cpp keeps rope_apply (src/model.cpp:169-191) inside an
// anonymous namespace, so no header exposes it.  This translation unit compiles
// the UNMODIFIED src/model.cpp where it lies under /root/reference (#include,
// nothing copied) and adds one extern "C" entry that calls that internal
// function, so the device RoPE can be pinned against the reference itself
// instead of a restatement.  oracle/Makefile links this TU in place of
// model.o: every other model.cpp symbol keeps its single definition.
#include "model.cpp"

namespace {
qtrain::ModelConfig cfg_from(const int* c) {
    qtrain::ModelConfig m;
    m.n_layers = c[0];
    m.d_model = c[1];
    m.d_ff = c[2];
    m.n_heads = c[3];
    m.n_kv_heads = c[4];
    m.vocab = c[5];
    m.seq_len = c[6];
    return m;
}
}  // namespace

extern "C" int ref_rope_apply(const int* cfg7, float* qkv, std::int64_t batch, std::int64_t seq, int backward) {
    try {
        using namespace qtrain;
        const ModelConfig cfg = cfg_from(cfg7);
        const ModelParams params;
        const StepContext step;
        const PrecisionMap prec;
        Ctx c{cfg, params, step, prec, ChunkSpec{}, batch, seq, OutRound::Bf16, 0};
        const std::int64_t rows = batch * seq, qd = cfg.qkv_dim();
        Tensor t({rows, qd}, std::vector<float>(qkv, qkv + rows * qd));
        rope_apply(c, t, backward != 0);
        std::copy(t.data.begin(), t.data.end(), qkv);
        return 0;
    } catch (...) {
        return 3;
    }
}
