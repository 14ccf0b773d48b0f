// Analytical planner with a B200 hardware profile.
//
// Reference: src/memplan.cpp:80-551 (ParamCounts, presets, memory_breakdown,
// flop_breakdown, lower-bound step time, MFU, estimate_step_time,
// search_plan), src/profiles.cpp:21-95 (hardware profiles), src/offload.cpp:
// 40-180 (residency schedule, transfer time), src/comms.cpp:262-281 (shard
// traffic model).  The arithmetic below reproduces the reference's numbers
// for the same inputs (tests/test_planner_cpu.py checks them against the
// reference library built in oracle/_ref); it is organised as tables of
// per-category byte rules instead of the reference's inline code.
//
// B200-specific additions:
//   * a "b200" builtin profile (180 GB HBM3e, dense FP8/BF16 spec peaks, the
//     measured HBM copy rate, NVLink 5 per-direction bandwidth, p2p);
//   * qt_session_footprint: the exact device + pinned-host bytes a qt_session
//     of this shape allocates (session.cu's arena, not an estimate);
//   * qt_search_plan_session: the reference's search ladder ranked by the
//     estimated step time but filtered by the session's real footprint
//     against the profile's device capacity.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "hostjson.h"
#include "qtrain_b200.h"

namespace qtb {
namespace plan {

using json::Value;

struct PlanError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

// RecomputeSite bits (include/qtrain/model.hpp:59-80)
enum Site { kSwiGLU = 0, kRMSNorm = 1, kAttention = 2, kQKV = 3, kFFN = 4, kBlock = 5 };
inline bool has(int bits, int site) { return (bits & (1 << kBlock)) || (bits & (1 << site)); }
// OffloadSet bits (include/qtrain/memplan.hpp:34-42), in the reference's field order
enum Off { kX = 0, kM = 1, kV = 2, kMaster = 3, kWeights = 4, kGrads = 5 };
inline bool off(int bits, int o) { return (bits >> o) & 1; }

struct Counts {
    uint64_t total = 0, block_linear = 0, per_layer_linear = 0, lmhead = 0, embed = 0, norms = 0;
};

Counts counts_of(const QtModelConfig& c, bool tied) {
    const uint64_t d = (uint64_t)c.d_model, ff = (uint64_t)c.d_ff;
    const uint64_t qkv = d + 2ull * c.n_kv_heads * (d / c.n_heads);
    Counts k;
    // qkv, o, gate_up, down projections of one block
    k.per_layer_linear = qkv * d + d * d + ff * d + (ff / 2) * d;
    k.block_linear = k.per_layer_linear * (uint64_t)c.n_layers;
    k.lmhead = (uint64_t)c.vocab * d;
    k.embed = (uint64_t)c.vocab * d;
    k.norms = (2ull * c.n_layers + 1) * d;
    k.total = k.block_linear + k.embed + k.norms + (tied ? 0 : k.lmhead);
    return k;
}

struct Geometry {
    Counts n;
    int64_t L, d, qkv, ff, vocab, heads, seq, tokens;
};

Geometry geometry(const QtModelConfig& c, int micro_batch, bool tied) {
    Geometry g;
    g.n = counts_of(c, tied);
    g.L = c.n_layers;
    g.d = c.d_model;
    g.qkv = c.d_model + 2 * c.n_kv_heads * (c.d_model / c.n_heads);
    g.ff = c.d_ff;
    g.vocab = c.vocab;
    g.heads = c.n_heads;
    g.seq = c.seq_len;
    g.tokens = (int64_t)micro_batch * c.seq_len;
    return g;
}

inline uint64_t per_worker(uint64_t bytes, int W) { return W > 1 ? bytes / (uint64_t)W : bytes; }

// Stored activation sites of one layer, per token (src/memplan.cpp:6-17 table):
// {bytes per element in fp8 mode, in bf16 mode, width, kept unless one of these sites recomputes}
struct SiteRule {
    int fp8_b, bf16_b;
    int width;  // 0 d, 1 qkv, 2 d_ff, 3 d_ff/2
    int drop_mask;
};
const SiteRule kSites[7] = {
    {1, 2, 0, 1 << kRMSNorm},                 // n1
    {2, 2, 1, 1 << kQKV},                     // qkv
    {1, 2, 0, 1 << kAttention},               // att
    {2, 2, 0, 0},                             // r_mid (block only)
    {1, 2, 0, 1 << kRMSNorm},                 // n2
    {2, 2, 2, 1 << kFFN},                     // gate_up
    {1, 2, 3, (1 << kFFN) | (1 << kSwiGLU)},  // h
};

void site_bytes(const Geometry& g, int rc_bits, bool fp8, uint64_t* kept, uint64_t* transient) {
    *kept = *transient = 0;
    const bool block = rc_bits & (1 << kBlock);
    for (const SiteRule& s : kSites) {
        const uint64_t w = s.width == 0 ? g.d : s.width == 1 ? g.qkv : s.width == 2 ? g.ff : g.ff / 2;
        const uint64_t b = w * (uint64_t)(fp8 ? s.fp8_b : s.bf16_b);
        *transient += b;
        if (!block && !(rc_bits & s.drop_mask)) *kept += b;
    }
}

QtMemTier& tier_of(bool host, QtMemTier& dev, QtMemTier& hst) { return host ? hst : dev; }

uint64_t tier_total(const QtMemTier& t) {
    return t.params_fp8 + t.params_bf16_master + t.moments_m + t.moments_v + t.grads + t.residuals + t.activations +
           t.logits_workspace + t.attn_workspace;
}

// memory_breakdown_from_counts (src/memplan.cpp:177-261)
void memory(const Geometry& g, const QtRunPlan& p, bool fp8, int W, QtMemTier& dev, QtMemTier& hst) {
    std::memset(&dev, 0, sizeof(dev));
    std::memset(&hst, 0, sizeof(hst));
    const int ob = p.offload_bits;
    const uint64_t mom_b = p.bf16_moments ? 2 : 4;
    const uint64_t tokens = (uint64_t)g.tokens;
    const uint64_t nonblock = g.n.total - g.n.block_linear;

    // quantized (or bf16) compute weights of the blocks; fp8 adds 8 f32 scales per layer
    const uint64_t wb = (fp8 ? g.n.block_linear : 2 * g.n.block_linear) + (fp8 ? (uint64_t)g.L * 32 : 0);
    {
        QtMemTier& t = tier_of(off(ob, kWeights), dev, hst);
        (fp8 ? t.params_fp8 : t.params_bf16_master) += p.shard_weights ? per_worker(wb, W) : wb;
        if (off(ob, kWeights))  // two layer-sized streaming buffers stay on the device
            (fp8 ? dev.params_fp8 : dev.params_bf16_master) +=
                2 * (fp8 ? g.n.per_layer_linear : 2 * g.n.per_layer_linear);
        dev.params_bf16_master += 2 * nonblock;  // lm-head / embedding / norms: bf16, resident
    }
    if (fp8) tier_of(off(ob, kMaster), dev, hst).params_bf16_master += per_worker(2 * g.n.block_linear, W);
    const uint64_t mom = per_worker(g.n.total * mom_b, W);  // ZeRO-1 whenever W > 1
    tier_of(off(ob, kM), dev, hst).moments_m += mom;
    tier_of(off(ob, kV), dev, hst).moments_v += mom;
    {
        const uint64_t bg = p.shard_grads ? per_worker(2 * g.n.block_linear, W) : 2 * g.n.block_linear;
        tier_of(off(ob, kGrads), dev, hst).grads += bg;
        if (off(ob, kGrads)) dev.grads += 4 * g.n.per_layer_linear;
        dev.grads += 2 * nonblock;
    }
    {
        const uint64_t resid = (uint64_t)g.L * tokens * (uint64_t)g.d * 2;
        tier_of(off(ob, kX), dev, hst).residuals += resid;
        if (off(ob, kX)) dev.residuals += 2 * tokens * (uint64_t)g.d * 2;
    }
    {
        uint64_t kept, transient;
        site_bytes(g, p.recompute_bits, fp8, &kept, &transient);
        uint64_t act = kept * tokens * (uint64_t)g.L;
        if (has(p.recompute_bits, kBlock)) act += transient * tokens;
        dev.activations += act;
    }
    {
        const int64_t ce = p.lmhead_chunk_tokens > 0 ? std::min<int64_t>(p.lmhead_chunk_tokens, g.tokens) : g.tokens;
        dev.logits_workspace += (uint64_t)ce * (uint64_t)g.vocab * 4;
        const int64_t rows = p.attn_chunk_rows > 0 ? std::min<int64_t>(p.attn_chunk_rows, g.seq) : g.seq;
        dev.attn_workspace += (uint64_t)g.heads * (uint64_t)rows * (uint64_t)g.seq * 8;
    }
}

// flop_breakdown (src/memplan.cpp:267-290): per token, forward + backward
QtFlops flops(const QtModelConfig& c, int rc_bits, bool tied) {
    const Counts k = counts_of(c, tied);
    QtFlops f{};
    const double d = c.d_model;
    f.linear = 6.0 * (double)k.block_linear;
    f.lmhead = 6.0 * (double)c.vocab * d;
    f.attention = 12.0 * ((double)c.seq_len / 2.0) * d * c.n_layers;
    const double attn_fwd = f.attention / 3.0;
    const double qkv = d + 2.0 * c.n_kv_heads * (c.d_model / c.n_heads);
    if (rc_bits & (1 << kBlock)) {
        f.recompute = 2.0 * (double)k.block_linear + attn_fwd;
    } else {
        if (rc_bits & (1 << kQKV)) f.recompute += 2.0 * d * qkv * c.n_layers;
        if (rc_bits & (1 << kFFN)) f.recompute += 2.0 * (d * c.d_ff + (double)c.d_ff / 2.0 * d) * c.n_layers;
        if (rc_bits & (1 << kAttention)) f.recompute += attn_fwd;
    }
    return f;
}

double peak_of(const QtHardwareProfile& hw, int which) {  // 0 fp8, 1 bf16, 2 f32
    return which == 0 ? hw.peak_flops_fp8 : which == 1 ? hw.peak_flops_bf16 : hw.peak_flops_f32;
}

// lower_bound_seconds_per_token (src/memplan.cpp:302-313) over FlopBreakdown::by_precision (:292-300)
double lower_bound(const QtFlops& f, const QtPrecisionMap& pr, const QtHardwareProfile& hw, bool attainable,
                   bool with_recompute) {
    const double extra = with_recompute ? f.recompute : 0.0;
    struct Bucket {
        int which;
        double ops;
    };
    std::vector<Bucket> b;
    if (pr.f32_debug)
        b = {{2, f.linear + f.lmhead + f.attention + extra}};
    else if (pr.block_matmuls == 0)
        b = {{0, f.linear + extra}, {1, f.lmhead + f.attention}};
    else
        b = {{1, f.linear + f.lmhead + f.attention + extra}};
    static const char* nm[3] = {"fp8", "bf16", "f32"};
    double s = 0.0;
    for (const Bucket& x : b) {
        const double pk = peak_of(hw, x.which) * (attainable ? hw.attainable_fraction : 1.0);
        if (pk <= 0.0) throw PlanError(std::string("profile lacks a peak rate for ") + nm[x.which]);
        s += x.ops / pk;
    }
    return s;
}

// grad_shard_traffic (src/comms.cpp:272-281)
uint64_t grad_shard_traffic(int ga, int W, uint64_t grad_bytes, bool p2p) {
    if (W < 2) return 0;
    const double v = (double)ga * ((double)(W - 1) / W) * (double)grad_bytes * (p2p ? 1 : 2);
    return (uint64_t)v;
}

// estimate_step_time (src/memplan.cpp:331-406)
QtStepTime step_time(const QtModelConfig& c, const QtPrecisionMap& pr, const QtRunPlan& p, const QtHardwareProfile& hw,
                     int W, bool tied) {
    const Geometry g = geometry(c, p.micro_batch, tied);
    const bool fp8 = pr.block_matmuls == 0;
    const int ob = p.offload_bits;
    const double tok = (double)g.tokens;
    const QtFlops f = flops(c, p.recompute_bits, tied);
    QtStepTime t{};
    t.feasible_in_time = 1;
    t.compute = tok * lower_bound(f, pr, hw, true, true);

    const double bw = hw.link_bandwidth * std::max(hw.zero_copy_efficiency, hw.double_buffer_efficiency);
    const uint64_t wbytes = fp8 ? g.n.block_linear : 2 * g.n.block_linear;
    const uint64_t gbytes = 2 * g.n.block_linear;
    const uint64_t rbytes = (uint64_t)g.L * (uint64_t)g.tokens * (uint64_t)g.d * 2;
    double per_mb = 0.0;  // bytes moved per micro-batch
    if (off(ob, kWeights) || p.shard_weights) per_mb += 2.0 * (double)wbytes;
    if (off(ob, kX)) per_mb += 2.0 * (double)rbytes;
    if (off(ob, kGrads)) per_mb += (double)gbytes;
    if (p.shard_grads && W > 1) per_mb += (double)grad_shard_traffic(1, W, gbytes, hw.p2p) / W;

    const uint64_t mb = p.bf16_moments ? 2 : 4;
    double opt = 0.0;  // optimizer-phase streaming, not hidden behind compute
    if (off(ob, kM)) opt += 2.0 * (double)(g.n.total * mb);
    if (off(ob, kV)) opt += 2.0 * (double)(g.n.total * mb);
    if (off(ob, kMaster) && fp8) opt += 2.0 * (double)(2 * g.n.total);
    opt /= W;

    if ((per_mb > 0.0 || opt > 0.0) && bw <= 0.0) {
        t.feasible_in_time = 0;
        t.total = std::numeric_limits<double>::infinity();
        return t;
    }
    const double xfer = bw > 0.0 ? per_mb / bw : 0.0;
    const double exposed = std::max(0.0, xfer - t.compute) + xfer / (double)g.L;  // + the first prefetch
    t.transfer = p.ga_steps * xfer;
    t.exposed_transfer = p.ga_steps * exposed;
    t.optimizer = bw > 0.0 ? opt / bw : 0.0;
    double sync = 0.0;  // replicated lm-head/embedding gradients, once per step, not hidden
    if (W > 1) sync = (double)((g.n.lmhead + g.n.embed) * 2) * (hw.p2p ? 1 : 2) / hw.link_bandwidth;
    const double one_mb = t.compute + exposed;
    t.compute = p.ga_steps * t.compute;
    t.total = p.ga_steps * one_mb + t.optimizer + sync;
    t.tokens_per_second = (double)p.ga_steps * tok * W / t.total;
    return t;
}

// ---------------------------------------------------------------- model presets
// Public decoder shapes of model_presets (src/memplan.cpp:98-108); seq_len 1024 is the
// accounting fixture length.  {name, layers, d, d_ff (fused), heads, kv_heads, vocab, seq, tied}
struct Preset {
    const char* name;
    QtModelConfig cfg;
    int tied;
};
const Preset kPresets[] = {
    {"toy", {2, 64, 256, 4, 2, 512, 128}, 0},
    {"0.5b", {24, 896, 9728, 14, 2, 151936, 1024}, 1},
    {"1.5b", {28, 1536, 17920, 12, 2, 151936, 1024}, 1},
    {"3b", {36, 2048, 22016, 16, 2, 151936, 1024}, 1},
    {"7b", {28, 3584, 37888, 28, 4, 152064, 1024}, 0},
    {"14b", {48, 5120, 27648, 40, 8, 152064, 1024}, 0},
    {"32b", {64, 5120, 55296, 40, 8, 152064, 1024}, 0},
};

const Preset& preset_by_name(const std::string& name) {
    for (const Preset& p : kPresets)
        if (name == p.name) return p;
    std::string avail;
    for (const Preset& p : kPresets) avail += std::string(" ") + p.name;
    throw PlanError("unknown model preset '" + name + "'; available:" + avail);
}

// ---------------------------------------------------------------- profiles
// Builtins of src/profiles.cpp:21-39 plus the B200.
std::vector<QtHardwareProfile> builtin_profiles() {
    auto mk = [](const char* n, uint64_t dev, uint64_t host, double f8, double bf, double f32, double mem, double link,
                 int p2p, double att, double zc, double db) {
        QtHardwareProfile p{};
        std::strncpy(p.name, n, sizeof(p.name) - 1);
        p.device_bytes = dev;
        p.host_bytes = host;
        p.peak_flops_fp8 = f8;
        p.peak_flops_bf16 = bf;
        p.peak_flops_f32 = f32;
        p.mem_bandwidth = mem;
        p.link_bandwidth = link;
        p.p2p = p2p;
        p.attainable_fraction = att;
        p.zero_copy_efficiency = zc;
        p.double_buffer_efficiency = db;
        return p;
    };
    return {
        mk("rtx5060ti", 16ull << 30, 128000000000ull, 94.9e12, 47.4e12, 23.7e12, 448e9, 32e9, 0, 1.08, 0.3, 0.9),
        mk("rtx4090", 24ull << 30, 256000000000ull, 330.4e12, 165.2e12, 82.6e12, 1008e9, 32e9, 0, 1.03, 0.3, 0.9),
        mk("l40s", 48ull << 30, 256000000000ull, 733e12, 362.1e12, 91.6e12, 864e9, 32e9, 1, 0.75, 0.9, 0.7),
        mk("h100", 80ull << 30, 1024000000000ull, 1978.9e12, 989.4e12, 66.9e12, 3350e9, 450e9, 1, 1.0, 0.9, 0.9),
        mk("dgx_spark", 128000000000ull, 128000000000ull, 250e12, 125e12, 31e12, 300e9, 300e9, 0, 0.7, 0.9, 0.9),
        // B200 (one GPU of an 8-GPU HGX/DGX box): 180 GB HBM3e; dense spec peaks 4.5 PF FP8 /
        // 2.25 PF BF16; HBM at the measured copy rate (MEASURED_PEAKS.json, 6.54 TB/s);
        // NVLink 5 at 900 GB/s per direction through NVSwitch (p2p, copy engines).  The
        // attainable fraction is the measured sustained bf16 matmul rate over spec
        // (1390 / 2250 TF/s); host link = PCIe 5 x16.
        mk("b200", 180000000000ull, 2000000000000ull, 4.5e15, 2.25e15, 80e12, 6.54e12, 900e9, 1, 0.618, 0.9, 0.95),
    };
}

QtHardwareProfile profile_by_name(const std::string& name) {
    for (const auto& p : builtin_profiles())
        if (name == p.name) return p;
    std::string avail;
    for (const auto& p : builtin_profiles()) avail += std::string(" ") + p.name;
    throw PlanError("unknown hardware profile '" + name + "'; available:" + avail);
}

Value profile_json(const QtHardwareProfile& p) {
    Value j = Value::object();
    j["name"] = std::string(p.name);
    j["device_bytes"] = (unsigned long long)p.device_bytes;
    j["host_bytes"] = (unsigned long long)p.host_bytes;
    Value pk = Value::object();
    pk["fp8"] = p.peak_flops_fp8;
    pk["bf16"] = p.peak_flops_bf16;
    pk["f32"] = p.peak_flops_f32;
    j["peak_flops"] = pk;
    j["mem_bandwidth"] = p.mem_bandwidth;
    j["link_bandwidth"] = p.link_bandwidth;
    j["p2p"] = p.p2p != 0;
    j["attainable_fraction"] = p.attainable_fraction;
    j["zero_copy_efficiency"] = p.zero_copy_efficiency;
    j["double_buffer_efficiency"] = p.double_buffer_efficiency;
    return j;
}

QtHardwareProfile profile_from(const Value& j) {
    QtHardwareProfile p{};
    const std::string n = j.at("name").as_string();
    std::strncpy(p.name, n.c_str(), sizeof(p.name) - 1);
    p.device_bytes = j.at("device_bytes").as_uint();
    p.host_bytes = j.at("host_bytes").as_uint();
    p.peak_flops_fp8 = j.at("peak_flops").at("fp8").as_double();
    p.peak_flops_bf16 = j.at("peak_flops").at("bf16").as_double();
    p.peak_flops_f32 = j.at("peak_flops").at("f32").as_double();
    p.mem_bandwidth = j.at("mem_bandwidth").as_double();
    p.link_bandwidth = j.at("link_bandwidth").as_double();
    p.p2p = j.at("p2p").as_bool();
    p.attainable_fraction = j.at("attainable_fraction").as_double();
    p.zero_copy_efficiency = j.get_or<double>("zero_copy_efficiency", 1.0);
    p.double_buffer_efficiency = j.get_or<double>("double_buffer_efficiency", 1.0);
    return p;
}

QtHardwareProfile load_profile(const std::string& name_or_path) {
    if (name_or_path.find('/') == std::string::npos && name_or_path.find(".json") == std::string::npos)
        return profile_by_name(name_or_path);
    std::ifstream in(name_or_path);
    if (!in.good()) throw std::runtime_error("cannot open hardware profile: " + name_or_path);
    std::ostringstream buf;
    buf << in.rdbuf();
    return profile_from(Value::parse(buf.str()));
}

// ---------------------------------------------------------------- search
std::string recompute_str(int bits) {
    static const char* nm[6] = {"swiglu", "rmsnorm", "attention", "qkv", "ffn", "block"};
    std::string s;
    for (int i = 0; i < 6; ++i)
        if (bits & (1 << i)) s += (s.empty() ? "" : ",") + std::string(nm[i]);
    return s.empty() ? "none" : s;
}
std::string offload_str(int bits) {
    static const char* nm[6] = {"x", "m", "v", "master", "weights", "grads"};
    std::string s;
    for (int i = 0; i < 6; ++i)
        if (bits & (1 << i)) s += (s.empty() ? "" : ",") + std::string(nm[i]);
    return s.empty() ? "none" : s;
}
// RunPlan::str (src/memplan.cpp:62-70): the search's deterministic tie-break key
std::string plan_str(const QtRunPlan& p, bool fp8) {
    std::ostringstream os;
    os << "mb=" << p.micro_batch << " ga=" << p.ga_steps << " recompute=" << recompute_str(p.recompute_bits)
       << " offload=" << offload_str(p.offload_bits) << " shard_w=" << (p.shard_weights ? 1 : 0)
       << " shard_g=" << (p.shard_grads ? 1 : 0) << " prec=" << (fp8 ? "fp8" : "bf16")
       << " moments=" << (p.bf16_moments ? "bf16" : "f32");
    return os.str();
}

// the offload ladder (src/memplan.cpp:416-447): moments, master, weights, residuals, grads
std::vector<int> offload_options(bool fp8, bool exhaustive) {
    std::vector<int> out;
    if (exhaustive) {
        for (int b = 0; b < 64; ++b)
            if (fp8 || !off(b, kMaster)) out.push_back(b);
        return out;
    }
    const int M_ = 1 << kM, V_ = 1 << kV, MS = 1 << kMaster, W_ = 1 << kWeights, X_ = 1 << kX, G_ = 1 << kGrads;
    const int ladder[9] = {0, X_, M_ | V_, X_ | M_ | V_, M_ | V_ | MS, X_ | M_ | V_ | MS, M_ | V_ | MS | W_,
                           X_ | M_ | V_ | MS | W_, X_ | M_ | V_ | MS | W_ | G_};
    for (int b : ladder) {
        if (!fp8) b &= ~MS;
        if (std::find(out.begin(), out.end(), b) == out.end()) out.push_back(b);
    }
    return out;
}
const int kRecomputeLadder[5] = {0, 1 << kSwiGLU, (1 << kFFN) | (1 << kAttention), (1 << kQKV) | (1 << kFFN),
                                 1 << kBlock};

std::string binding(const QtMemTier& t) {
    const std::pair<const char*, uint64_t> cats[7] = {
        {"params", t.params_fp8 + t.params_bf16_master}, {"moments", t.moments_m + t.moments_v},
        {"grads", t.grads},                               {"residuals", t.residuals},
        {"activations", t.activations},                   {"logits workspace", t.logits_workspace},
        {"attention workspace", t.attn_workspace}};
    int best = 0;
    for (int i = 1; i < 7; ++i)
        if (cats[i].second > cats[best].second) best = i;
    return cats[best].first;
}

Value tier_json(const QtMemTier& t) {
    Value j = Value::object();
    j["params_fp8"] = (unsigned long long)t.params_fp8;
    j["params_bf16_master"] = (unsigned long long)t.params_bf16_master;
    j["moments_m"] = (unsigned long long)t.moments_m;
    j["moments_v"] = (unsigned long long)t.moments_v;
    j["grads"] = (unsigned long long)t.grads;
    j["residuals"] = (unsigned long long)t.residuals;
    j["activations"] = (unsigned long long)t.activations;
    j["logits_workspace"] = (unsigned long long)t.logits_workspace;
    j["attn_workspace"] = (unsigned long long)t.attn_workspace;
    j["total"] = (unsigned long long)tier_total(t);
    return j;
}

Value plan_json(const QtRunPlan& p, bool fp8) {
    Value j = Value::object();
    j["micro_batch"] = p.micro_batch;
    j["ga_steps"] = p.ga_steps;
    j["recompute_bits"] = p.recompute_bits;
    j["offload_bits"] = p.offload_bits;
    j["shard_weights"] = p.shard_weights != 0;
    j["shard_grads"] = p.shard_grads != 0;
    j["bf16_moments"] = p.bf16_moments != 0;
    j["str"] = plan_str(p, fp8);
    return j;
}

Value time_json(const QtStepTime& t) {
    Value j = Value::object();
    j["compute"] = t.compute;
    j["transfer"] = t.transfer;
    j["exposed_transfer"] = t.exposed_transfer;
    j["optimizer"] = t.optimizer;
    j["total"] = t.total;
    j["tokens_per_second"] = t.tokens_per_second;
    return j;
}

// device-bytes oracle used to filter plans: the reference's breakdown, or the session's real arena
using DeviceBytesFn = uint64_t (*)(const QtModelConfig&, const QtPrecisionMap&, const QtRunPlan&, int W, bool tied,
                                   const QtMemTier& dev);

// search_plan (src/memplan.cpp:471-551)
Value search(const QtModelConfig& c, const QtHardwareProfile& hw, int W, int64_t target_tokens, int matmuls,
             bool exhaustive, bool tied, DeviceBytesFn dev_fn, int max_results) {
    const bool fp8 = matmuls == 0;
    QtPrecisionMap pr{matmuls, 0, 0};
    const int batches[12] = {1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64};
    std::vector<std::pair<int, int>> shard = {{0, 0}};
    if (W > 1) {
        shard = {{0, 0}, {1, 0}, {1, 1}};
        if (exhaustive) shard.push_back({0, 1});
    }
    std::vector<int> moments = {1};
    if (exhaustive) moments.push_back(0);
    struct Cand {
        QtRunPlan p;
        QtMemTier dev, host;
        uint64_t dev_bytes;
        QtStepTime t;
        std::string key;
    };
    std::vector<Cand> ok;
    for (int mb : batches) {
        const int64_t per_step = (int64_t)mb * c.seq_len * W;
        if (per_step > target_tokens && mb != 1) continue;
        const int ga = (int)std::max<int64_t>(1, (target_tokens + per_step - 1) / per_step);
        for (int rc : kRecomputeLadder)
            for (int ob : offload_options(fp8, exhaustive))
                for (auto [sw, sg] : shard)
                    for (int bm : moments) {
                        QtRunPlan p{};
                        p.micro_batch = mb;
                        p.ga_steps = ga;
                        p.recompute_bits = rc;
                        p.offload_bits = ob;
                        p.shard_weights = sw;
                        p.shard_grads = sg;
                        p.bf16_moments = bm;
                        p.lmhead_chunk_tokens = 512;
                        p.attn_chunk_rows = 256;
                        Cand cd{};
                        cd.p = p;
                        memory(geometry(c, mb, tied), p, fp8, W, cd.dev, cd.host);
                        cd.dev_bytes = dev_fn ? dev_fn(c, pr, p, W, tied, cd.dev) : tier_total(cd.dev);
                        if (cd.dev_bytes > hw.device_bytes || tier_total(cd.host) > hw.host_bytes) continue;
                        cd.t = step_time(c, pr, p, hw, W, tied);
                        if (!cd.t.feasible_in_time) continue;
                        cd.key = plan_str(p, fp8);
                        ok.push_back(cd);
                    }
    }
    std::sort(ok.begin(), ok.end(), [](const Cand& a, const Cand& b) {
        if (a.t.tokens_per_second != b.t.tokens_per_second) return a.t.tokens_per_second > b.t.tokens_per_second;
        return a.key < b.key;
    });
    Value out = Value::object();
    Value list = Value::array();
    int n = 0;
    for (const Cand& cd : ok) {
        if (max_results > 0 && n++ >= max_results) break;
        Value v = Value::object();
        v["plan"] = plan_json(cd.p, fp8);
        v["device"] = tier_json(cd.dev);
        v["host"] = tier_json(cd.host);
        v["device_bytes"] = (unsigned long long)cd.dev_bytes;
        v["time"] = time_json(cd.t);
        list.push_back(v);
    }
    out["n_feasible"] = (unsigned long long)ok.size();
    out["feasible"] = list;
    if (ok.empty()) {
        // the most aggressive plan names the binding constraint
        QtRunPlan p{};
        p.micro_batch = 1;
        p.ga_steps = 1;
        p.recompute_bits = 1 << kBlock;
        p.offload_bits = fp8 ? 63 : 63 & ~(1 << kMaster);
        p.shard_weights = p.shard_grads = W > 1;
        p.bf16_moments = 1;
        p.lmhead_chunk_tokens = 512;
        p.attn_chunk_rows = 256;
        QtMemTier dv, hs;
        memory(geometry(c, 1, tied), p, fp8, W, dv, hs);
        std::ostringstream os;
        os << "model does not fit: ";
        if (tier_total(dv) > hw.device_bytes)
            os << "device needs " << tier_total(dv) / 1e9 << " GB (" << hw.device_bytes / 1e9
               << " GB available), binding: " << binding(dv);
        else
            os << "host needs " << tier_total(hs) / 1e9 << " GB (" << hw.host_bytes / 1e9
               << " GB available), binding: " << binding(hs);
        out["no_fit_reason"] = os.str();
    }
    return out;
}

// ---------------------------------------------------------------- residency (src/offload.cpp:40-163)
struct Residency {
    Value events = Value::array();
    uint64_t resident = 0, hw_total = 0;
    uint64_t cw = 0, hw_w = 0, cg = 0, hw_g = 0, cx = 0, hw_x = 0;
    double clock = 0.0;
    void emit(const char* kind, const char* cat, int layer, int buffer, uint64_t bytes, int64_t delta) {
        resident = (uint64_t)((int64_t)resident + delta);
        auto bump = [&](uint64_t& cur, uint64_t& high) {
            cur = (uint64_t)((int64_t)cur + delta);
            high = std::max(high, cur);
        };
        if (!std::strcmp(cat, "weights")) bump(cw, hw_w);
        if (!std::strcmp(cat, "grads")) bump(cg, hw_g);
        if (!std::strcmp(cat, "residuals")) bump(cx, hw_x);
        hw_total = std::max(hw_total, resident);
        Value e = Value::object();
        e["time"] = clock;
        e["kind"] = kind;
        e["category"] = cat;
        e["layer"] = layer;
        e["buffer"] = buffer;
        e["bytes"] = (unsigned long long)bytes;
        e["resident"] = (unsigned long long)resident;
        events.push_back(e);
        clock += 1.0;
    }
};

Value residency(const QtModelConfig& c, const QtPrecisionMap& pr, const QtRunPlan& p, uint64_t budget, bool tied) {
    const Geometry g = geometry(c, p.micro_batch, tied);
    const bool fp8 = pr.block_matmuls == 0;
    const int ob = p.offload_bits;
    const uint64_t lw = fp8 ? g.n.per_layer_linear : 2 * g.n.per_layer_linear;
    const uint64_t lg = 2 * g.n.per_layer_linear;
    const uint64_t lx = (uint64_t)g.tokens * (uint64_t)g.d * 2;
    const uint64_t mb = p.bf16_moments ? 2 : 4;
    const int L = c.n_layers;
    QtMemTier dev, host;
    memory(g, p, fp8, 1, dev, host);
    uint64_t fixed = tier_total(dev);
    if (off(ob, kWeights)) fixed -= 2 * lw;
    if (off(ob, kGrads)) fixed -= 2 * lg;
    if (off(ob, kX)) fixed -= 2 * lx;
    const bool blk = has(p.recompute_bits, kBlock);
    const uint64_t trans = blk ? dev.activations : 0;
    if (blk) fixed -= trans;
    Residency r;
    r.resident = r.hw_total = fixed;
    // forward: weights prefetched one layer ahead, residuals evicted as produced
    if (off(ob, kWeights)) r.emit("prefetch", "weights", 0, 0, lw, (int64_t)lw);
    for (int l = 0; l < L; ++l) {
        if (off(ob, kWeights) && l + 1 < L) r.emit("prefetch", "weights", l + 1, (l + 1) % 2, lw, (int64_t)lw);
        if (trans) r.emit("compute", "activations", l, -1, 0, (int64_t)trans);
        r.emit("compute", "forward", l, l % 2, 0, 0);
        if (trans) r.emit("compute", "activations", l, -1, 0, -(int64_t)trans);
        if (off(ob, kWeights)) r.emit("evict", "weights", l, l % 2, lw, -(int64_t)lw);
        if (off(ob, kX)) {
            r.emit("compute", "residuals", l, -1, 0, (int64_t)lx);
            r.emit("evict", "residuals", l, -1, lx, -(int64_t)lx);
        }
    }
    // backward: weights and residuals stream back, gradient buffers drain one layer behind
    if (off(ob, kWeights)) r.emit("prefetch", "weights", L - 1, (L - 1) % 2, lw, (int64_t)lw);
    if (off(ob, kX)) r.emit("prefetch", "residuals", L - 1, -1, lx, (int64_t)lx);
    int draining = -1;
    for (int l = L - 1; l >= 0; --l) {
        if (off(ob, kWeights) && l > 0) r.emit("prefetch", "weights", l - 1, (l - 1) % 2, lw, (int64_t)lw);
        if (off(ob, kX) && l > 0) r.emit("prefetch", "residuals", l - 1, -1, lx, (int64_t)lx);
        if (off(ob, kGrads)) r.emit("compute", "grads", l, l % 2, 0, (int64_t)lg);
        if (trans) r.emit("compute", "activations", l, -1, 0, (int64_t)trans);
        r.emit("compute", "backward", l, l % 2, 0, 0);
        if (trans) r.emit("compute", "activations", l, -1, 0, -(int64_t)trans);
        if (off(ob, kWeights)) r.emit("evict", "weights", l, l % 2, lw, -(int64_t)lw);
        if (off(ob, kX)) r.emit("evict", "residuals", l, -1, lx, -(int64_t)lx);
        if (off(ob, kGrads)) {
            if (draining >= 0) r.emit("evict", "grads", draining, draining % 2, lg, -(int64_t)lg);
            draining = l;
        }
    }
    if (off(ob, kGrads) && draining >= 0) r.emit("evict", "grads", draining, draining % 2, lg, -(int64_t)lg);
    // optimizer phase: offloaded state streams through in layer chunks
    if (off(ob, kM) || off(ob, kV) || off(ob, kMaster)) {
        uint64_t chunk = 0;
        if (off(ob, kM)) chunk += g.n.per_layer_linear * mb;
        if (off(ob, kV)) chunk += g.n.per_layer_linear * mb;
        if (off(ob, kMaster) && fp8) chunk += 2 * g.n.per_layer_linear;
        for (int l = 0; l < L; ++l) {
            r.emit("prefetch", "moments", l, l % 2, chunk, (int64_t)chunk);
            r.emit("compute", "optimizer", l, l % 2, 0, 0);
            r.emit("publish", "moments", l, l % 2, chunk, -(int64_t)chunk);
        }
    }
    Value out = Value::object();
    out["events"] = r.events;
    out["high_water_device"] = (unsigned long long)r.hw_total;
    out["high_water_weights"] = (unsigned long long)r.hw_w;
    out["high_water_grads"] = (unsigned long long)r.hw_g;
    out["high_water_residuals"] = (unsigned long long)r.hw_x;
    out["feasible"] = r.hw_total <= budget;
    if (r.hw_total > budget) {
        std::ostringstream os;
        os << "device high-water " << r.hw_total / 1e9 << " GB exceeds budget " << budget / 1e9 << " GB";
        out["report"] = os.str();
    }
    return out;
}

}  // namespace plan
}  // namespace qtb

// ---------------------------------------------------------------- C ABI
namespace {
thread_local std::string g_plan_err;

template <typename F>
int plan_guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_plan_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_plan_err = e.what();
        return 3;
    }
}

int put_text(const std::string& s, char* buf, size_t cap, size_t* needed) {
    if (needed) *needed = s.size() + 1;
    if (!buf || cap < s.size() + 1) return buf ? 1 : 0;
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return 0;
}

void check_cfg(const QtModelConfig* c) {
    if (!c || c->n_layers < 1 || c->d_model < 1 || c->n_heads < 1 || c->n_kv_heads < 1 ||
        c->d_model % c->n_heads || c->n_heads % c->n_kv_heads || c->d_ff % 2)
        throw std::invalid_argument("planner: invalid ModelConfig");
}
}  // namespace

extern "C" {

const char* qt_plan_last_error(void) { return g_plan_err.c_str(); }

int qt_model_preset(const char* name, QtModelConfig* cfg, int* tied) {
    return plan_guard([&] {
        const auto& p = qtb::plan::preset_by_name(name ? name : "");
        *cfg = p.cfg;
        if (tied) *tied = p.tied;
    });
}

int qt_profile_by_name(const char* name, QtHardwareProfile* out) {
    return plan_guard([&] { *out = qtb::plan::profile_by_name(name ? name : ""); });
}

int qt_profile_load(const char* name_or_path, QtHardwareProfile* out) {
    return plan_guard([&] { *out = qtb::plan::load_profile(name_or_path ? name_or_path : ""); });
}

int qt_profile_to_json(const QtHardwareProfile* p, char* buf, size_t cap, size_t* needed) {
    int rc = 0;
    const int g = plan_guard([&] { rc = put_text(qtb::plan::profile_json(*p).dump(2), buf, cap, needed); });
    return g ? g : rc;
}

int qt_profile_from_json(const char* text, QtHardwareProfile* out) {
    return plan_guard([&] { *out = qtb::plan::profile_from(qtb::json::Value::parse(text ? text : "")); });
}

int qt_param_counts(const QtModelConfig* cfg, int tied, uint64_t* total, uint64_t* block_linear,
                    uint64_t* per_layer_linear, uint64_t* lmhead, uint64_t* embed, uint64_t* norms) {
    return plan_guard([&] {
        check_cfg(cfg);
        const auto k = qtb::plan::counts_of(*cfg, tied != 0);
        *total = k.total;
        *block_linear = k.block_linear;
        *per_layer_linear = k.per_layer_linear;
        *lmhead = k.lmhead;
        *embed = k.embed;
        *norms = k.norms;
    });
}

int qt_memory_breakdown(const QtModelConfig* cfg, const QtPrecisionMap* prec, const QtRunPlan* plan, int workers,
                        int tied, QtMemTier* device, QtMemTier* host) {
    return plan_guard([&] {
        check_cfg(cfg);
        if (workers < 1) throw std::invalid_argument("memory_breakdown: workers must be >= 1");
        qtb::plan::memory(qtb::plan::geometry(*cfg, plan->micro_batch, tied != 0), *plan, prec->block_matmuls == 0,
                          workers, *device, *host);
    });
}

int qt_flop_breakdown(const QtModelConfig* cfg, int recompute_bits, int tied, QtFlops* out) {
    return plan_guard([&] {
        check_cfg(cfg);
        *out = qtb::plan::flops(*cfg, recompute_bits, tied != 0);
    });
}

int qt_lower_bound_seconds_per_token(const QtFlops* f, const QtPrecisionMap* prec, const QtHardwareProfile* hw,
                                     int attainable, int include_recompute, double* out) {
    return plan_guard([&] { *out = qtb::plan::lower_bound(*f, *prec, *hw, attainable != 0, include_recompute != 0); });
}

int qt_mfu(double measured_tps, const QtModelConfig* cfg, const QtPrecisionMap* prec, const QtHardwareProfile* hw,
           int tied, double* out) {
    return plan_guard([&] {
        check_cfg(cfg);
        if (measured_tps <= 0.0) throw std::invalid_argument("mfu: measured_tps must be positive");
        *out = measured_tps * qtb::plan::lower_bound(qtb::plan::flops(*cfg, 0, tied != 0), *prec, *hw, false, false);
    });
}

int qt_fp8_speedup_ceiling(const QtModelConfig* cfg, const QtHardwareProfile* hw, int tied, double* out) {
    return plan_guard([&] {
        check_cfg(cfg);
        const QtFlops f = qtb::plan::flops(*cfg, 0, tied != 0);
        const QtPrecisionMap bf{1, 0, 0}, f8{0, 0, 0};
        *out = qtb::plan::lower_bound(f, bf, *hw, false, false) / qtb::plan::lower_bound(f, f8, *hw, false, false) - 1.0;
    });
}

int qt_estimate_step_time(const QtModelConfig* cfg, const QtPrecisionMap* prec, const QtRunPlan* plan,
                          const QtHardwareProfile* hw, int workers, int tied, QtStepTime* out) {
    return plan_guard([&] {
        check_cfg(cfg);
        *out = qtb::plan::step_time(*cfg, *prec, *plan, *hw, workers, tied != 0);
    });
}

int qt_search_plan(const QtModelConfig* cfg, const QtHardwareProfile* hw, int workers, int64_t target_batch_tokens,
                   int block_matmuls, int exhaustive, int tied, int max_results, char* json_out, size_t cap,
                   size_t* needed) {
    int rc = 0;
    const int g = plan_guard([&] {
        check_cfg(cfg);
        rc = put_text(qtb::plan::search(*cfg, *hw, workers, target_batch_tokens, block_matmuls, exhaustive != 0,
                                        tied != 0, nullptr, max_results)
                          .dump(),
                      json_out, cap, needed);
    });
    return g ? g : rc;
}

int qt_plan_residency(const QtModelConfig* cfg, const QtPrecisionMap* prec, const QtRunPlan* plan,
                      uint64_t device_budget, int tied, char* json_out, size_t cap, size_t* needed) {
    int rc = 0;
    const int g = plan_guard([&] {
        check_cfg(cfg);
        rc = put_text(qtb::plan::residency(*cfg, *prec, *plan, device_budget, tied != 0).dump(), json_out, cap, needed);
    });
    return g ? g : rc;
}

// transfer_time (src/offload.cpp:165-171): 20 us latency + bytes / (link * policy efficiency)
int qt_transfer_time(uint64_t bytes, const QtHardwareProfile* hw, int policy, double* out) {
    return plan_guard([&] {
        if (hw->link_bandwidth <= 0.0) throw std::invalid_argument("transfer_time: zero link bandwidth");
        const double eff = policy == QT_XFER_ZERO_COPY ? hw->zero_copy_efficiency : hw->double_buffer_efficiency;
        *out = 20e-6 + (double)bytes / (hw->link_bandwidth * eff);
    });
}

}  // extern "C"

// The session-footprint search lives next to the session (session.cu) because it needs
// the arena layout; it reuses qtb::plan::search with a device-bytes callback.
namespace qtb {
namespace plan {
Value search_with(const QtModelConfig& c, const QtHardwareProfile& hw, int W, int64_t target_tokens, int matmuls,
                  bool exhaustive, bool tied, DeviceBytesFn fn, int max_results) {
    return search(c, hw, W, target_tokens, matmuls, exhaustive, tied, fn, max_results);
}
}  // namespace plan
}  // namespace qtb
