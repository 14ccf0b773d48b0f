// Manifest-driven trainer, synthetic corpora and QTCKPT01 checkpoints with
// resume, on the device session.
//
// Reference: src/trainer.cpp:35-171 (run_training, metrics CSV,
// run_training_to_files), src/manifest.cpp:45-188 (RunManifest JSON),
// src/corpus.cpp:15-69 (perm-walk / uniform corpora), src/checkpoint.cpp:19-80
// (QTCKPT01 container).  Differences, all additions:
//   * the step runs on the B200 session (qt_train_step): W workers are W
//     sessions of one in-process peer group (copy-engine collectives), on as
//     many GPUs as are visible (rank w on device w % ndev);
//   * resume: a checkpoint carries the optimizer moments (as the reference's
//     does) plus "optim.step", and a run started from it continues bit for bit
//     where the saved run left off (same micro-batch indices, SR and AdamW
//     keys, step counter);
//   * a checkpoint can be written every k steps ("outputs.checkpoint_every").
// Host code only: every kernel runs inside the session.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <mutex>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "hostjson.h"
#include "qtrain_b200.h"

namespace qtb {
namespace trainer {

using json::Value;

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void invalid(const std::string& m) { throw Error(1, m); }

// ---------------------------------------------------------------- numerics (host)
// rng_uniform / fnv1a64 (src/numerics.cpp:192-235), as the session's device copies
inline uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}
inline uint32_t rng_uniform(uint64_t seed, uint64_t stream, uint64_t counter) {
    uint64_t z = mix64(mix64(mix64(0x9E3779B97F4A7C15ull ^ seed) ^ stream) ^ counter);
    z = mix64(z);
    return (uint32_t)(z >> 32) ^ (uint32_t)z;
}
inline uint64_t fnv1a64(const std::string& s) {
    uint64_t h = 0xCBF29CE484222325ull;
    for (unsigned char c : s) {
        h ^= c;
        h *= 0x100000001B3ull;
    }
    return h;
}

// ---------------------------------------------------------------- corpus
struct CorpusSpec {
    std::string kind = "perm-walk";
    int64_t vocab = 512;
    int seq_len = 128, n_train = 256, n_val = 16;
    uint64_t seed = 0;
};
struct Corpus {
    std::vector<int32_t> train, val;
    int stride = 0;
    size_t train_sequences() const { return train.size() / (size_t)stride; }
};

// perm-walk: token t+1 = perm[token t] from a seeded start; uniform: iid ids
void fill(std::vector<int32_t>& out, const CorpusSpec& c, const std::vector<int32_t>& perm, uint64_t stream, int count) {
    const int stride = c.seq_len + 1;
    out.assign((size_t)count * stride, 0);
    const bool walk = c.kind == "perm-walk";
    for (int s = 0; s < count; ++s) {
        int32_t tok = walk ? (int32_t)(rng_uniform(c.seed, stream, (uint64_t)s) % (uint32_t)c.vocab) : 0;
        int32_t* row = out.data() + (size_t)s * stride;
        for (int t = 0; t < stride; ++t) {
            if (walk) {
                row[t] = tok;
                tok = perm[(size_t)tok];
            } else {
                row[t] = (int32_t)(rng_uniform(c.seed, stream + 1, (uint64_t)s * (uint64_t)stride + (uint64_t)t) %
                                   (uint32_t)c.vocab);
            }
        }
    }
}

Corpus make_corpus(const CorpusSpec& c) {
    if (c.kind != "perm-walk" && c.kind != "uniform") invalid("unknown corpus kind: " + c.kind);
    if (c.vocab < 2 || c.seq_len < 1 || c.n_train < 1) invalid("degenerate corpus spec");
    std::vector<int32_t> perm((size_t)c.vocab);
    for (int64_t i = 0; i < c.vocab; ++i) perm[(size_t)i] = (int32_t)i;
    const uint64_t ps = fnv1a64("corpus/perm");
    for (int64_t i = c.vocab - 1; i > 0; --i) {  // seeded Fisher-Yates
        const int64_t j = (int64_t)(rng_uniform(c.seed, ps, (uint64_t)i) % (uint32_t)(i + 1));
        std::swap(perm[(size_t)i], perm[(size_t)j]);
    }
    Corpus out;
    out.stride = c.seq_len + 1;
    fill(out.train, c, perm, fnv1a64("corpus/train"), c.n_train);
    fill(out.val, c, perm, fnv1a64("corpus/val"), c.n_val);
    return out;
}

// ---------------------------------------------------------------- manifest
struct Manifest {
    uint64_t seed = 0;
    std::string model_preset;
    QtModelConfig model{2, 64, 256, 4, 2, 512, 128};
    bool tied = false;
    // RunPlan (memplan.hpp:54-67); precision map FP8/E4M3 by default
    int micro_batch = 1, ga_steps = 1, recompute_bits = 0, offload_bits = 0;
    bool shard_weights = false, shard_grads = false;
    int64_t lmhead_chunk_tokens = 512, attn_chunk_rows = 256;
    int matmuls = 0, grads = 0, f32_debug = 0;
    bool bf16_moments = true;  // RunPlan::moments defaults to BF16_SR (memplan.hpp:62)
    QtAdamW optim{1e-3f, 0.9f, 0.95f, 1e-8f, 0.0f, 1.0f};
    CorpusSpec corpus;
    int steps = 100, eval_every = 1, workers = 1;
    std::string hardware = "rtx4090";
    std::string metrics_csv = "metrics.csv", checkpoint_out;
    // additions
    std::string resume_from;
    int checkpoint_every = 0;
};

std::vector<std::string> names_of(const Value& j) {
    std::vector<std::string> out;
    if (j.is_string()) {
        out.push_back(j.as_string());
    } else {
        for (const Value& x : j.items()) out.push_back(x.as_string());
    }
    return out;
}

int recompute_bits(const std::vector<std::string>& names) {  // recompute_set_from_names (src/model.cpp:31-44)
    static const char* site[6] = {"swiglu", "rmsnorm", "attention", "qkv", "ffn", "block"};
    int bits = 0;
    for (std::string n : names) {
        if (n == "none" || n.empty()) continue;
        if (n == "att") n = "attention";
        int k = -1;
        for (int i = 0; i < 6; ++i)
            if (n == site[i]) k = i;
        if (k < 0) invalid("unknown recompute site: " + n);
        bits |= 1 << k;
    }
    return bits;
}

int offload_bits(const std::vector<std::string>& names) {  // offload_set_from_names (src/memplan.cpp:47-60)
    int bits = 0;
    for (const std::string& n : names) {
        if (n == "x" || n == "residuals") bits |= QT_OFF_X;
        else if (n == "m") bits |= QT_OFF_M;
        else if (n == "v") bits |= QT_OFF_V;
        else if (n == "master" || n == "theta*") bits |= QT_OFF_MASTER;
        else if (n == "weights" || n == "theta") bits |= QT_OFF_WEIGHTS;
        else if (n == "grads" || n == "g") bits |= QT_OFF_GRADS;
        else if (n == "none" || n.empty()) continue;
        else invalid("unknown offload category: " + n);
    }
    return bits;
}

void validate_model(const QtModelConfig& c) {  // ModelConfig::validate (src/model.cpp:12-17)
    if (c.n_layers < 1 || c.d_model < 1 || c.n_heads < 1 || c.n_kv_heads < 1 || c.vocab < 2 || c.seq_len < 1)
        invalid("ModelConfig: degenerate dimensions");
    if (c.d_model % c.n_heads) invalid("ModelConfig: d_model % n_heads != 0");
    if (c.n_heads % c.n_kv_heads) invalid("ModelConfig: n_heads % n_kv_heads != 0");
    if (c.d_ff % 2) invalid("ModelConfig: d_ff must be even");
}

// manifest_from_json (src/manifest.cpp:45-129)
Manifest parse_manifest(const std::string& text) {
    Value j;
    try {
        j = Value::parse(text);
    } catch (const json::ParseError& e) {
        invalid(std::string("manifest: ") + e.what());
    }
    Manifest m;
    m.seed = j.get_or<uint64_t>("seed", 0);
    if (j.contains("model")) {
        const Value& jm = j.at("model");
        if (jm.is_string()) {
            m.model_preset = jm.as_string();
            int tied = 0;
            if (qt_model_preset(m.model_preset.c_str(), &m.model, &tied) != 0) invalid(qt_plan_last_error());
            m.tied = tied != 0;
        } else {
            m.model.n_layers = (int)jm.at("n_layers").as_int();
            m.model.d_model = (int)jm.at("d_model").as_int();
            m.model.d_ff = (int)jm.at("d_ff").as_int();
            m.model.n_heads = (int)jm.at("n_heads").as_int();
            m.model.n_kv_heads = (int)jm.at("n_kv_heads").as_int();
            m.model.vocab = jm.at("vocab").as_int();
            m.model.seq_len = (int)jm.at("seq_len").as_int();
            m.tied = jm.get_or<bool>("tied_embeddings", false);
        }
        validate_model(m.model);
    }
    if (j.contains("precision")) {
        const Value& jp = j.at("precision");
        const std::string mm = jp.get_or<std::string>("matmuls", "fp8-e4m3");
        if (mm == "fp8-e4m3" || mm == "fp8") m.matmuls = 0;
        else if (mm == "bf16") m.matmuls = 1;
        else invalid("manifest: unknown matmul precision " + mm);
        const std::string bg = jp.get_or<std::string>("backward_grads", "e4m3");
        if (bg == "e4m3") m.grads = 0;
        else if (bg == "e5m2") m.grads = 1;
        else invalid("manifest: unknown backward grad kind " + bg);
        m.f32_debug = jp.get_or<bool>("f32_debug", false);
    }
    if (j.contains("plan")) {
        const Value& jp = j.at("plan");
        m.micro_batch = jp.get_or<int>("micro_batch", 1);
        m.ga_steps = jp.get_or<int>("ga_steps", 1);
        if (jp.contains("recompute")) m.recompute_bits = recompute_bits(names_of(jp.at("recompute")));
        if (jp.contains("offload")) m.offload_bits = offload_bits(names_of(jp.at("offload")));
        m.shard_weights = jp.get_or<bool>("shard_weights", false);
        m.shard_grads = jp.get_or<bool>("shard_grads", false);
        m.lmhead_chunk_tokens = jp.get_or<int64_t>("lmhead_chunk_tokens", 512);
        m.attn_chunk_rows = jp.get_or<int64_t>("attn_chunk_rows", 256);
    }
    if (j.contains("optimizer")) {
        const Value& jo = j.at("optimizer");
        m.optim.lr = jo.get_or<float>("lr", 1e-3f);
        m.optim.beta1 = jo.get_or<float>("beta1", 0.9f);
        m.optim.beta2 = jo.get_or<float>("beta2", 0.95f);
        m.optim.eps = jo.get_or<float>("eps", 1e-8f);
        m.optim.weight_decay = jo.get_or<float>("weight_decay", 0.0f);
        m.optim.max_grad_norm = jo.get_or<float>("max_grad_norm", 1.0f);
        const std::string mom = jo.get_or<std::string>("moments", "f32");
        if (mom == "f32") m.bf16_moments = false;
        else if (mom == "bf16") m.bf16_moments = true;
        else invalid("manifest: unknown moment precision " + mom);
    }
    if (j.contains("corpus")) {
        const Value& jc = j.at("corpus");
        m.corpus.kind = jc.get_or<std::string>("kind", "perm-walk");
        m.corpus.vocab = jc.get_or<int64_t>("vocab", m.model.vocab);
        m.corpus.seq_len = jc.get_or<int>("seq_len", m.model.seq_len);
        m.corpus.n_train = jc.get_or<int>("n_train", 256);
        m.corpus.n_val = jc.get_or<int>("n_val", 16);
        m.corpus.seed = jc.get_or<uint64_t>("seed", m.seed);
    } else {
        m.corpus.vocab = m.model.vocab;
        m.corpus.seq_len = m.model.seq_len;
        m.corpus.seed = m.seed;
    }
    m.steps = j.get_or<int>("steps", 100);
    m.eval_every = j.get_or<int>("eval_every", 1);
    m.hardware = j.get_or<std::string>("hardware", "rtx4090");
    m.workers = j.get_or<int>("workers", 1);
    if (j.contains("outputs")) {
        const Value& jo = j.at("outputs");
        m.metrics_csv = jo.get_or<std::string>("metrics_csv", "metrics.csv");
        m.checkpoint_out = jo.get_or<std::string>("checkpoint", "");
        m.checkpoint_every = jo.get_or<int>("checkpoint_every", 0);
    }
    m.resume_from = j.get_or<std::string>("resume_from", "");
    if (m.corpus.vocab != m.model.vocab) invalid("manifest: corpus vocab must match model vocab");
    if (m.corpus.seq_len > m.model.seq_len) invalid("manifest: corpus sequences longer than the model context");
    return m;
}

// manifest_to_json (src/manifest.cpp:131-181)
Value manifest_json(const Manifest& m) {
    Value j = Value::object();
    j["seed"] = (unsigned long long)m.seed;
    if (!m.model_preset.empty()) {
        j["model"] = m.model_preset;
    } else {
        Value jm = Value::object();
        jm["n_layers"] = m.model.n_layers;
        jm["d_model"] = m.model.d_model;
        jm["d_ff"] = m.model.d_ff;
        jm["n_heads"] = m.model.n_heads;
        jm["n_kv_heads"] = m.model.n_kv_heads;
        jm["vocab"] = (long long)m.model.vocab;
        jm["seq_len"] = m.model.seq_len;
        jm["tied_embeddings"] = m.tied;
        j["model"] = jm;
    }
    Value jp = Value::object();
    jp["matmuls"] = m.matmuls == 0 ? "fp8-e4m3" : "bf16";
    jp["backward_grads"] = m.grads == 0 ? "e4m3" : "e5m2";
    jp["f32_debug"] = m.f32_debug != 0;
    j["precision"] = jp;
    // recompute names: a site is listed when all its bits are set (manifest.cpp:148-152)
    static const char* rc_names[6] = {"swiglu", "rmsnorm", "attention", "qkv", "ffn", "block"};
    Value rc = Value::array();
    for (int i = 0; i < 6; ++i)
        if (m.recompute_bits & (1 << i)) rc.push_back(rc_names[i]);
    static const char* off_names[6] = {"x", "m", "v", "master", "weights", "grads"};
    Value off = Value::array();
    for (int i = 0; i < 6; ++i)
        if (m.offload_bits & (1 << i)) off.push_back(off_names[i]);
    Value pl = Value::object();
    pl["micro_batch"] = m.micro_batch;
    pl["ga_steps"] = m.ga_steps;
    pl["recompute"] = rc;
    pl["offload"] = off;
    pl["shard_weights"] = m.shard_weights;
    pl["shard_grads"] = m.shard_grads;
    pl["lmhead_chunk_tokens"] = (long long)m.lmhead_chunk_tokens;
    pl["attn_chunk_rows"] = (long long)m.attn_chunk_rows;
    j["plan"] = pl;
    Value jo = Value::object();
    jo["lr"] = m.optim.lr;
    jo["beta1"] = m.optim.beta1;
    jo["beta2"] = m.optim.beta2;
    jo["eps"] = m.optim.eps;
    jo["weight_decay"] = m.optim.weight_decay;
    jo["max_grad_norm"] = m.optim.max_grad_norm;
    jo["moments"] = m.bf16_moments ? "bf16" : "f32";
    j["optimizer"] = jo;
    Value jc = Value::object();
    jc["kind"] = m.corpus.kind;
    jc["vocab"] = (long long)m.corpus.vocab;
    jc["seq_len"] = m.corpus.seq_len;
    jc["n_train"] = m.corpus.n_train;
    jc["n_val"] = m.corpus.n_val;
    jc["seed"] = (unsigned long long)m.corpus.seed;
    j["corpus"] = jc;
    j["steps"] = m.steps;
    j["eval_every"] = m.eval_every;
    j["hardware"] = m.hardware;
    j["workers"] = m.workers;
    Value out = Value::object();
    out["metrics_csv"] = m.metrics_csv;
    out["checkpoint"] = m.checkpoint_out;
    if (m.checkpoint_every) out["checkpoint_every"] = m.checkpoint_every;
    j["outputs"] = out;
    if (!m.resume_from.empty()) j["resume_from"] = m.resume_from;
    return j;
}

std::string read_file(const std::string& path, const char* what) {
    std::ifstream in(path, std::ios::binary);
    if (!in.good()) throw Error(3, std::string("cannot open ") + what + ": " + path);
    std::ostringstream buf;
    buf << in.rdbuf();
    return buf.str();
}

Manifest load_manifest(const std::string& path_or_text) {
    const bool text = !path_or_text.empty() && path_or_text.find('{') != std::string::npos;
    return parse_manifest(text ? path_or_text : read_file(path_or_text, "manifest"));
}

// ---------------------------------------------------------------- QTCKPT01 (src/checkpoint.cpp:19-80)
const char kMagic[8] = {'Q', 'T', 'C', 'K', 'P', 'T', '0', '1'};

struct CkptTensor {
    std::string name;
    std::vector<int64_t> shape;
    std::vector<float> data;
};

void save_checkpoint(const std::string& path, const std::vector<CkptTensor>& ts) {
    Value man = Value::object();
    man["byte_order"] = "little";
    man["dtype"] = "f32";
    Value list = Value::array();
    uint64_t off = 0;
    for (const CkptTensor& t : ts) {
        Value e = Value::object();
        e["name"] = t.name;
        Value sh = Value::array();
        for (int64_t x : t.shape) sh.push_back((long long)x);
        e["shape"] = sh;
        e["dtype"] = "f32";
        e["offset_elems"] = (unsigned long long)off;
        e["numel"] = (long long)t.data.size();
        list.push_back(e);
        off += t.data.size();
    }
    man["tensors"] = list;
    const std::string text = man.dump();
    const std::string tmp = path + ".tmp";
    {
        std::ofstream out(tmp, std::ios::binary | std::ios::trunc);
        if (!out.good()) throw Error(3, "cannot open checkpoint for writing: " + path);
        out.write(kMagic, 8);
        const uint64_t len = text.size();
        out.write(reinterpret_cast<const char*>(&len), 8);
        out.write(text.data(), (std::streamsize)text.size());
        for (const CkptTensor& t : ts)
            out.write(reinterpret_cast<const char*>(t.data.data()), (std::streamsize)(t.data.size() * 4));
        if (!out.good()) throw Error(3, "checkpoint write failed: " + path);
    }
    if (std::rename(tmp.c_str(), path.c_str()) != 0) throw Error(3, "checkpoint rename failed: " + path);
}

std::vector<CkptTensor> load_checkpoint(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in.good()) throw Error(3, "cannot open checkpoint: " + path);
    char magic[8];
    in.read(magic, 8);
    if (!in.good() || std::memcmp(magic, kMagic, 8) != 0) throw Error(3, "not a checkpoint file: " + path);
    uint64_t len = 0;
    in.read(reinterpret_cast<char*>(&len), 8);
    std::string text(len, '\0');
    in.read(text.data(), (std::streamsize)len);
    if (!in.good()) throw Error(3, "truncated checkpoint: " + path);
    const Value man = Value::parse(text);
    if (man.at("byte_order").as_string() != "little" || man.at("dtype").as_string() != "f32")
        throw Error(3, "unsupported checkpoint layout: " + path);
    const std::streampos base = in.tellg();
    std::vector<CkptTensor> out;
    for (const Value& e : man.at("tensors").items()) {
        CkptTensor t;
        t.name = e.at("name").as_string();
        int64_t n = 1;
        for (const Value& x : e.at("shape").items()) {
            t.shape.push_back(x.as_int());
            n *= x.as_int();
        }
        t.data.resize((size_t)n);
        in.seekg(base + (std::streamoff)(e.at("offset_elems").as_uint() * 4));
        in.read(reinterpret_cast<char*>(t.data.data()), (std::streamsize)(n * 4));
        if (!in.good()) throw Error(3, "truncated checkpoint: " + path);
        out.push_back(std::move(t));
    }
    return out;
}

void chk(int rc) {
    if (rc != 0) throw Error(rc == 1 || rc == 2 ? rc : 3, qt_last_error());
}

// the param shapes in for_each_param order (model.hpp:107-121)
std::vector<int64_t> param_shape(const QtModelConfig& c, const std::string& name) {
    const int64_t d = c.d_model, hd = c.d_model / c.n_heads, q = d + 2 * (int64_t)c.n_kv_heads * hd;
    auto ends = [&](const char* suf) {
        const size_t n = std::strlen(suf);
        return name.size() >= n && name.compare(name.size() - n, n, suf) == 0;
    };
    if (name == "embed" || name == "lm_head") return {c.vocab, d};
    if (name == "final_g" || ends(".ln1_g") || ends(".ln2_g")) return {d};
    if (ends(".w_qkv")) return {q, d};
    if (ends(".w_o")) return {d, d};
    if (ends(".w_gate_up")) return {c.d_ff, d};
    if (ends(".w_down")) return {d, c.d_ff / 2};
    throw Error(3, "unknown parameter " + name);
}

// The sessions of a run (one per worker): params + optimizer state -> tensors in the
// reference's container order: params (for_each_param), then optim.m./optim.v. per name in
// OptimState::slots order (std::map: lexicographic), then optim.step (addition).
std::vector<CkptTensor> snapshot(const QtModelConfig& cfg, const std::vector<qt_session*>& ss, bool with_optim,
                                 const float* last_val = nullptr) {
    qt_session* s0 = ss[0];
    const int np = qt_num_params(s0);
    std::vector<CkptTensor> out;
    std::vector<std::string> names;
    for (int i = 0; i < np; ++i) {
        const char* nm = nullptr;
        int64_t n = 0;
        chk(qt_param_info(s0, i, &nm, &n));
        CkptTensor t;
        t.name = nm;
        t.shape = param_shape(cfg, t.name);
        t.data.resize((size_t)n);
        chk(qt_param_download(s0, i, t.data.data()));
        names.push_back(t.name);
        out.push_back(std::move(t));
    }
    if (!with_optim) return out;
    std::vector<int> order(np);
    for (int i = 0; i < np; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int a, int b) { return names[a] < names[b]; });
    for (int i : order) {
        CkptTensor m, v;
        m.name = "optim.m." + names[i];
        v.name = "optim.v." + names[i];
        m.shape = v.shape = out[(size_t)i].shape;
        m.data.assign(out[(size_t)i].data.size(), 0.0f);
        v.data.assign(m.data.size(), 0.0f);
        for (qt_session* s : ss) {  // each rank's ZeRO-1 slice
            int64_t lo = 0, n = 0;
            chk(qt_moments_slice(s, i, &lo, &n));
            if (n <= 0) continue;
            std::vector<float> a((size_t)n), b((size_t)n);
            chk(qt_moments_download(s, i, a.data(), b.data()));
            std::copy(a.begin(), a.end(), m.data.begin() + lo);
            std::copy(b.begin(), b.end(), v.data.begin() + lo);
        }
        out.push_back(std::move(m));
        out.push_back(std::move(v));
    }
    int64_t step = 0;
    chk(qt_step_count(s0, &step));
    CkptTensor st;
    st.name = "optim.step";
    st.shape = {1};
    st.data = {(float)step};
    out.push_back(std::move(st));
    if (last_val) {  // the trainer's last eval loss, so a resumed run's CSV continues exactly
        CkptTensor lv;
        lv.name = "trainer.val_loss";
        lv.shape = {1};
        lv.data = {*last_val};
        out.push_back(std::move(lv));
    }
    return out;
}

// params (and, when present, moments + step) into every session of the run
int64_t restore(const std::vector<CkptTensor>& ts, const std::vector<qt_session*>& ss, float* last_val = nullptr) {
    qt_session* s0 = ss[0];
    const int np = qt_num_params(s0);
    auto find = [&](const std::string& n) -> const CkptTensor* {
        for (const CkptTensor& t : ts)
            if (t.name == n) return &t;
        return nullptr;
    };
    const CkptTensor* st = find("optim.step");
    if (const CkptTensor* lv = find("trainer.val_loss"); lv && last_val) *last_val = lv->data.at(0);
    const int64_t step = st ? (int64_t)st->data.at(0) : 0;
    for (int i = 0; i < np; ++i) {
        const char* nm = nullptr;
        int64_t n = 0;
        chk(qt_param_info(s0, i, &nm, &n));
        const CkptTensor* p = find(nm);
        if (!p) throw Error(3, std::string("checkpoint lacks parameter ") + nm);
        if ((int64_t)p->data.size() != n) throw Error(1, std::string("checkpoint shape mismatch for ") + nm);
        const CkptTensor* m = find(std::string("optim.m.") + nm);
        const CkptTensor* v = find(std::string("optim.v.") + nm);
        for (qt_session* s : ss) {
            chk(qt_param_upload(s, i, p->data.data()));
            if (m && v) chk(qt_moments_upload(s, i, m->data.data(), v->data.data(), step));
        }
    }
    return step;
}

// ---------------------------------------------------------------- run_training (src/trainer.cpp:35-137)
struct StepMetrics {
    int step;
    int64_t tokens;
    float train_loss, val_loss, grad_norm;
    double sim_time;
};

std::string metrics_csv(const std::vector<StepMetrics>& ms) {  // metrics_to_csv (trainer.cpp:139-150)
    std::string out = "step,tokens,train_loss,val_loss,grad_norm,sim_time\n";
    char line[256];
    for (const StepMetrics& m : ms) {
        std::snprintf(line, sizeof(line), "%d,%lld,%.9g,%.9g,%.9g,%.6e\n", m.step, (long long)m.tokens,
                      m.train_loss, m.val_loss, m.grad_norm, m.sim_time);
        out += line;
    }
    return out;
}

struct Run {
    Manifest m;
    Corpus corpus;
    qt_group* group = nullptr;
    std::vector<qt_session*> ss;
    ~Run() {
        for (qt_session* s : ss)
            if (s) qt_session_destroy(s);
        if (group) qt_group_destroy(group);
    }
};

// take_batch (trainer.cpp:19-31): micro_batch sequences starting at microbatch_index*micro_batch
void take_batch(const Corpus& c, uint64_t mb_index, int micro_batch, int32_t* out) {
    const size_t n_seq = c.train_sequences();
    for (int k = 0; k < micro_batch; ++k) {
        const size_t s = (size_t)((mb_index * (uint64_t)micro_batch + (uint64_t)k) % n_seq);
        std::memcpy(out + (size_t)k * c.stride, c.train.data() + s * c.stride, (size_t)c.stride * 4);
    }
}

Value run_training(const Manifest& m, int device_count) {
    validate_model(m.model);
    if (m.workers < 1) invalid("manifest: workers must be >= 1");
    if (m.steps < 0) invalid("manifest: steps must be >= 0");
    Run run;
    run.m = m;
    run.corpus = make_corpus(m.corpus);
    const int W = m.workers, GA = m.ga_steps, MB = m.micro_batch;
    const int eval_seqs = std::min(m.corpus.n_val, 4);
    QtPrecisionMap prec{m.matmuls, m.grads, m.f32_debug};
    // the session's activation arena also holds the fixed eval batch
    QtRunPlan plan{std::max(MB, eval_seqs), GA, m.recompute_bits, m.lmhead_chunk_tokens, m.attn_chunk_rows,
                   m.shard_weights ? 1 : 0, m.shard_grads ? 1 : 0, m.bf16_moments ? 1 : 0, m.offload_bits,
                   QT_XFER_DOUBLE_BUFFER};
    QtAdamW hyper = m.optim;
    if (device_count < 1) {
        if (cudaGetDeviceCount(&device_count) != cudaSuccess || device_count < 1)
            throw Error(3, "run_training: no CUDA device");
    }
    run.ss.assign((size_t)W, nullptr);
    if (W == 1) {
        chk(qt_session_create(&m.model, &prec, &plan, &hyper, m.seed, 0, 1, nullptr, 0, &run.ss[0]));
    } else {
        chk(qt_group_create(W, &run.group));
        for (int w = 0; w < W; ++w)
            chk(qt_session_create_in_group(&m.model, &prec, &plan, &hyper, m.seed, run.group, w, w % device_count,
                                           &run.ss[(size_t)w]));
    }
    int start = 0;
    float last_val = 0.0f, initial = 0.0f;
    if (!m.resume_from.empty()) {
        start = (int)restore(load_checkpoint(m.resume_from), run.ss, &last_val);
    } else {
        for (qt_session* s : run.ss) chk(qt_init_params(s, m.seed));  // init_params (model.cpp:67-86)
    }
    if (start > m.steps) invalid("resume_from: checkpoint step beyond manifest steps");

    // simulated wall clock of the reference trainer (trainer.cpp:50)
    QtHardwareProfile hw{};
    if (qt_profile_load(m.hardware.c_str(), &hw) != 0) throw Error(1, qt_plan_last_error());
    QtRunPlan est_plan = plan;
    est_plan.micro_batch = MB;
    QtStepTime tb{};
    if (qt_estimate_step_time(&m.model, &prec, &est_plan, &hw, W, m.tied ? 1 : 0, &tb) != 0)
        throw Error(1, qt_plan_last_error());

    const int stride = run.corpus.stride;
    std::vector<int32_t> eval_batch(run.corpus.val.begin(), run.corpus.val.begin() + (size_t)eval_seqs * stride);
    std::vector<StepMetrics> metrics;
    int64_t tokens_seen = (int64_t)start * GA * W * MB * m.corpus.seq_len;
    std::vector<std::vector<int32_t>> toks((size_t)W, std::vector<int32_t>((size_t)GA * MB * stride));
    std::vector<std::vector<float>> losses((size_t)W, std::vector<float>((size_t)GA));
    std::vector<float> norms((size_t)W);
    std::vector<int> rcs((size_t)W);
    std::vector<std::string> errs((size_t)W);
    for (int step = start; step < m.steps; ++step) {
        for (int w = 0; w < W; ++w)
            for (int ga = 0; ga < GA; ++ga)
                take_batch(run.corpus, ((uint64_t)step * GA + ga) * W + (uint64_t)w, MB,
                           toks[(size_t)w].data() + (size_t)ga * MB * stride);
        auto body = [&](int w) {
            qt_session* s = run.ss[(size_t)w];
            int32_t* dev = nullptr;
            rcs[(size_t)w] = qt_upload_tokens(s, toks[(size_t)w].data(), (int64_t)toks[(size_t)w].size(), &dev);
            if (!rcs[(size_t)w])
                rcs[(size_t)w] = qt_train_step(s, dev, (int64_t)MB * stride, MB, step, m.optim.max_grad_norm, nullptr,
                                               &norms[(size_t)w]);
            if (!rcs[(size_t)w]) rcs[(size_t)w] = qt_step_losses(s, losses[(size_t)w].data());
            if (rcs[(size_t)w]) errs[(size_t)w] = qt_last_error();
        };
        if (W == 1) {
            body(0);
        } else {  // one host thread per worker (WorkerGroup::run, comms.cpp:19-36)
            std::vector<std::thread> th;
            for (int w = 0; w < W; ++w) th.emplace_back(body, w);
            for (auto& t : th) t.join();
        }
        for (int w = 0; w < W; ++w)
            if (rcs[(size_t)w]) throw Error(rcs[(size_t)w] <= 3 ? rcs[(size_t)w] : 3, errs[(size_t)w]);
        double loss_sum = 0.0;  // (ga, w) order of trainer.cpp:75-86
        for (int ga = 0; ga < GA; ++ga)
            for (int w = 0; w < W; ++w) loss_sum += losses[(size_t)w][(size_t)ga];
        tokens_seen += (int64_t)GA * W * MB * m.corpus.seq_len;
        const float train_loss = (float)(loss_sum / (GA * W));
        if (!std::isfinite(train_loss))
            throw Error(3, "training diverged: non-finite loss at step " + std::to_string(step));
        if (step % std::max(1, m.eval_every) == 0) {
            // eval forward with the step context built before this step's update (trainer.cpp:117)
            float vl = 0.0f;
            auto ev = [&](int w) {
                qt_session* s = run.ss[(size_t)w];
                int32_t* dev = nullptr;
                rcs[(size_t)w] = qt_upload_tokens(s, eval_batch.data(), (int64_t)eval_batch.size(), &dev);
                if (!rcs[(size_t)w])
                    rcs[(size_t)w] = qt_forward(s, dev, (int64_t)eval_batch.size(), eval_seqs, 0, w == 0 ? &vl : nullptr);
                if (rcs[(size_t)w]) errs[(size_t)w] = qt_last_error();
            };
            // every rank runs it (with shard_weights the forward gathers weights per layer)
            if (W == 1) {
                ev(0);
            } else {
                std::vector<std::thread> th;
                for (int w = 0; w < W; ++w) th.emplace_back(ev, w);
                for (auto& t : th) t.join();
            }
            for (int w = 0; w < W; ++w)
                if (rcs[(size_t)w]) throw Error(rcs[(size_t)w] <= 3 ? rcs[(size_t)w] : 3, errs[(size_t)w]);
            last_val = vl;
        }
        StepMetrics sm{step, tokens_seen, train_loss, last_val, norms[0], tb.total * (step + 1)};
        metrics.push_back(sm);
        if (step == start) initial = train_loss;
        if (m.checkpoint_every > 0 && !m.checkpoint_out.empty() && (step + 1) % m.checkpoint_every == 0 &&
            step + 1 < m.steps)
            save_checkpoint(m.checkpoint_out + ".step" + std::to_string(step + 1),
                            snapshot(m.model, run.ss, true, &last_val));
    }
    {
        std::ofstream csv(m.metrics_csv, std::ios::binary | std::ios::trunc);
        if (!csv.good()) throw Error(3, "cannot write metrics csv: " + m.metrics_csv);
        const std::string text = metrics_csv(metrics);
        csv.write(text.data(), (std::streamsize)text.size());
    }
    if (!m.checkpoint_out.empty()) save_checkpoint(m.checkpoint_out, snapshot(m.model, run.ss, true, &last_val));
    Value res = Value::object();
    res["initial_train_loss"] = initial;
    res["final_train_loss"] = metrics.empty() ? 0.0f : metrics.back().train_loss;
    res["final_val_loss"] = last_val;
    res["start_step"] = start;
    Value rows = Value::array();
    for (const StepMetrics& s : metrics) {
        Value r = Value::object();
        r["step"] = s.step;
        r["tokens"] = (long long)s.tokens;
        r["train_loss"] = s.train_loss;
        r["val_loss"] = s.val_loss;
        r["grad_norm"] = s.grad_norm;
        r["sim_time"] = s.sim_time;
        rows.push_back(r);
    }
    res["metrics"] = rows;
    return res;
}

}  // namespace trainer
}  // namespace qtb

// ---------------------------------------------------------------- C ABI
namespace {
thread_local std::string g_train_err;

template <typename F>
int train_guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const qtb::trainer::Error& e) {
        g_train_err = e.what();
        return e.code;
    } catch (const std::invalid_argument& e) {
        g_train_err = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        g_train_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_train_err = e.what();
        return 3;
    }
}

int put_text(const std::string& s, char* buf, size_t cap, size_t* needed) {
    if (needed) *needed = s.size() + 1;
    if (!buf) return 0;
    if (cap < s.size() + 1) return 1;
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return 0;
}
}  // namespace

extern "C" {

const char* qt_train_last_error(void) { return g_train_err.c_str(); }

int qt_make_corpus(const char* kind, int64_t vocab, int seq_len, int n_train, int n_val, uint64_t seed,
                   int32_t* train_out, int32_t* val_out) {
    return train_guard([&] {
        qtb::trainer::CorpusSpec c;
        c.kind = kind ? kind : "perm-walk";
        c.vocab = vocab;
        c.seq_len = seq_len;
        c.n_train = n_train;
        c.n_val = n_val;
        c.seed = seed;
        const auto co = qtb::trainer::make_corpus(c);
        std::memcpy(train_out, co.train.data(), co.train.size() * 4);
        if (val_out) std::memcpy(val_out, co.val.data(), co.val.size() * 4);
    });
}

int qt_manifest_normalize(const char* manifest, char* json_out, size_t cap, size_t* needed) {
    int rc = 0;
    const int g = train_guard([&] {
        rc = put_text(qtb::trainer::manifest_json(qtb::trainer::load_manifest(manifest ? manifest : "")).dump(2),
                      json_out, cap, needed);
    });
    return g ? g : rc;
}

int qt_run_training(const char* manifest, int device_count, char* result_json, size_t cap, size_t* needed) {
    int rc = 0;
    const int g = train_guard([&] {
        const auto m = qtb::trainer::load_manifest(manifest ? manifest : "");
        rc = put_text(qtb::trainer::run_training(m, device_count).dump(), result_json, cap, needed);
    });
    return g ? g : rc;
}

int qt_checkpoint_save(qt_session* const* sessions, int n_sessions, const QtModelConfig* cfg, const char* path,
                       int with_optimizer) {
    return train_guard([&] {
        if (n_sessions < 1) throw qtb::trainer::Error(1, "checkpoint_save: no sessions");
        std::vector<qt_session*> ss(sessions, sessions + n_sessions);
        qtb::trainer::save_checkpoint(path, qtb::trainer::snapshot(*cfg, ss, with_optimizer != 0));
    });
}

int qt_checkpoint_load(qt_session* const* sessions, int n_sessions, const char* path, int64_t* step_out) {
    return train_guard([&] {
        if (n_sessions < 1) throw qtb::trainer::Error(1, "checkpoint_load: no sessions");
        std::vector<qt_session*> ss(sessions, sessions + n_sessions);
        const int64_t st = qtb::trainer::restore(qtb::trainer::load_checkpoint(path), ss);
        if (step_out) *step_out = st;
    });
}

}  // extern "C"
