/* TEST INFRASTRUCTURE ONLY -- plain-C restatement of the reference arithmetic
 * (see qtrain_oracle.h).  Compiled by oracle/Makefile with -ffp-contract=off so
 * no FMA contraction changes a rounding; reductions run in the reference's
 * sequential order.  Used as the checker, never as the thing measured.
 */
#include "qtrain_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* FP8 tables: src/numerics.cpp:17-119                                        */
/* ------------------------------------------------------------------------- */
typedef struct {
    float decode[256];
    float pos_values[128]; /* finite non-negative values, ascending */
    uint8_t pos_codes[128];
    int npos;
    float fmax;
    uint8_t nan_code, inf_code;
} F8Tab;

static F8Tab g_tab[2];
static int g_tab_ready = 0;

/* decode_raw, src/numerics.cpp:28-48 */
static float decode_raw(uint8_t code, int kind) {
    const int exp_bits = kind == 0 ? 4 : 5, man_bits = kind == 0 ? 3 : 2, bias = kind == 0 ? 7 : 15;
    const int ieee = kind != 0;
    const int sign = (code >> 7) ? -1 : 1;
    const int exp_mask = (1 << exp_bits) - 1, man_mask = (1 << man_bits) - 1;
    const int e = (code >> man_bits) & exp_mask, m = code & man_mask;
    if (ieee && e == exp_mask) return m == 0 ? (float)sign * INFINITY : NAN;
    if (!ieee && e == exp_mask && m == man_mask) return NAN;
    const float man_scale = 1.0f / (float)(1 << man_bits);
    if (e == 0) return (float)sign * (float)m * man_scale * exp2f((float)(1 - bias));
    return (float)sign * (1.0f + (float)m * man_scale) * exp2f((float)(e - bias));
}

static void build_tables(void) {
    for (int kind = 0; kind < 2; ++kind) {
        F8Tab* t = &g_tab[kind];
        t->npos = 0;
        t->fmax = 0.0f;
        t->nan_code = 0x7F;
        t->inf_code = 0;
        for (int c = 0; c < 256; ++c) t->decode[c] = decode_raw((uint8_t)c, kind);
        for (int c = 0; c < 128; ++c) {
            const float v = t->decode[c];
            if (isfinite(v)) {
                /* insertion sort by value (codes are already monotone, numerics.cpp:71-72) */
                int j = t->npos++;
                while (j > 0 && t->pos_values[j - 1] > v) {
                    t->pos_values[j] = t->pos_values[j - 1];
                    t->pos_codes[j] = t->pos_codes[j - 1];
                    --j;
                }
                t->pos_values[j] = v;
                t->pos_codes[j] = (uint8_t)c;
                if (v > t->fmax) t->fmax = v;
            } else if (isinf(v)) {
                t->inf_code = (uint8_t)c;
            }
        }
    }
    g_tab_ready = 1;
}

static const F8Tab* tab(int kind) {
    if (!g_tab_ready) build_tables();
    return &g_tab[kind ? 1 : 0];
}

float qto_f8_decode(uint8_t code, int kind) { return tab(kind)->decode[code]; }
float qto_f8_fmax(int kind) { return tab(kind)->fmax; }

/* F8Tables::encode, src/numerics.cpp:87-112: RNE over the finite values,
 * ties to the even code, saturating, NaN -> nan_code, E5M2 keeps +-inf */
uint8_t qto_f8_encode(float x, int kind) {
    const F8Tab* t = tab(kind);
    if (isnan(x)) return t->nan_code;
    const int neg = signbit(x) != 0;
    const float a = fabsf(x);
    uint8_t code;
    if (isinf(x) && t->inf_code != 0) {
        code = t->inf_code;
    } else if (a >= t->pos_values[t->npos - 1]) {
        code = t->pos_codes[t->npos - 1];
    } else {
        int lo = 0, hi = t->npos; /* lower_bound: first value >= a */
        while (lo < hi) {
            const int mid = (lo + hi) / 2;
            if (t->pos_values[mid] < a) lo = mid + 1;
            else hi = mid;
        }
        const int h = lo;
        if (t->pos_values[h] == a || h == 0) {
            code = t->pos_codes[h];
        } else {
            const int l = h - 1;
            const float mid = 0.5f * (t->pos_values[l] + t->pos_values[h]);
            if (a < mid) code = t->pos_codes[l];
            else if (a > mid) code = t->pos_codes[h];
            else code = (t->pos_codes[l] & 1u) == 0 ? t->pos_codes[l] : t->pos_codes[h];
        }
    }
    return neg ? (uint8_t)(code | 0x80u) : code;
}

/* absmax, src/numerics.cpp:141-148 */
int qto_absmax(const float* x, int64_t n, float* out) {
    float m = 0.0f;
    for (int64_t i = 0; i < n; ++i) {
        if (isnan(x[i])) return -1;
        const float a = fabsf(x[i]);
        m = m < a ? a : m;
    }
    *out = m;
    return 0;
}

/* absmax_scale, src/numerics.cpp:150-158 */
float qto_absmax_scale(float amax, int kind) {
    if (amax == 0.0f) return 1.0f;
    const double exact = (double)qto_f8_fmax(kind) / (double)amax;
    float s = (float)exact;
    if ((double)s < exact) s = nextafterf(s, INFINITY);
    return s;
}

static float clampf(float v, float lo, float hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* quantize_with_absmax, src/numerics.cpp:160-176 */
void qto_quantize_with_absmax(const float* x, int64_t n, int kind, float amax, uint8_t* codes, float* scale) {
    const float s = qto_absmax_scale(amax, kind), fmax = qto_f8_fmax(kind);
    for (int64_t i = 0; i < n; ++i) codes[i] = qto_f8_encode(clampf(x[i] * s, -fmax, fmax), kind);
    *scale = s;
}

/* transpose_quantize_with_absmax, src/tensorops.cpp:164-182 */
void qto_transpose_quantize_with_absmax(const float* x, int64_t rows, int64_t cols, int kind, float amax,
                                        uint8_t* codes_t, float* scale) {
    const float s = qto_absmax_scale(amax, kind), fmax = qto_f8_fmax(kind);
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c)
            codes_t[c * rows + r] = qto_f8_encode(clampf(x[r * cols + c] * s, -fmax, fmax), kind);
    *scale = s;
}

/* ------------------------------------------------------------------------- */
/* counter RNG, FNV-1a, bf16 rounding: src/numerics.cpp:192-258               */
/* ------------------------------------------------------------------------- */
static uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

uint32_t qto_rng_uniform(uint64_t seed, uint64_t stream, uint64_t counter) {
    uint64_t z = 0x9E3779B97F4A7C15ull;
    z = mix64(z ^ seed);
    z = mix64(z ^ stream);
    z = mix64(z ^ counter);
    z = mix64(z);
    return (uint32_t)(z >> 32) ^ (uint32_t)z;
}

float qto_rng_uniform_float(uint64_t seed, uint64_t stream, uint64_t counter) {
    return (float)(qto_rng_uniform(seed, stream, counter) >> 8) * 0x1.0p-24f;
}

float qto_rng_normal(uint64_t seed, uint64_t stream, uint64_t counter) {
    const double u1 = ((double)qto_rng_uniform(seed, stream, 2 * counter) + 1.0) * 0x1.0p-32;
    const double u2 = (double)qto_rng_uniform(seed, stream, 2 * counter + 1) * 0x1.0p-32;
    const double r = sqrt(-2.0 * log(u1));
    return (float)(r * cos(2.0 * 3.14159265358979323846 * u2));
}

uint64_t qto_fnv1a64(const char* s) {
    uint64_t h = 0xCBF29CE484222325ull;
    for (; *s; ++s) {
        h ^= (uint8_t)*s;
        h *= 0x100000001B3ull;
    }
    return h;
}

static uint32_t f2u(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    return u;
}
static float u2f(uint32_t u) {
    float x;
    memcpy(&x, &u, 4);
    return x;
}

float qto_bf16_round(float x) {
    if (isnan(x)) return x;
    uint32_t b = f2u(x);
    b += 0x7FFFu + ((b >> 16) & 1u);
    return u2f(b & 0xFFFF0000u);
}

float qto_sr_bf16(float x, uint64_t seed, uint64_t stream, uint64_t counter) {
    if (isnan(x)) return x;
    uint32_t b = f2u(x);
    if ((b & 0xFFFFu) == 0) return x;
    b += qto_rng_uniform(seed, stream, counter) & 0xFFFFu;
    return u2f(b & 0xFFFF0000u);
}

/* ------------------------------------------------------------------------- */
/* tensorops: src/tensorops.cpp                                               */
/* ------------------------------------------------------------------------- */
static float rnd(float v, int r) { return r ? qto_bf16_round(v) : v; }

/* matmul_tn (ScaledQuant), src/tensorops.cpp:41-59 */
void qto_matmul_fp8(const uint8_t* a, int64_t M, int64_t K, int akind, float ascale, const uint8_t* b, int64_t N,
                    int bkind, float bscale, int round_bf16, float* out) {
    const float* da = tab(akind)->decode;
    const float* db = tab(bkind)->decode;
    const float denom = ascale * bscale;
    for (int64_t m = 0; m < M; ++m)
        for (int64_t n = 0; n < N; ++n) {
            float acc = 0.0f;
            for (int64_t k = 0; k < K; ++k) acc += da[a[m * K + k]] * db[b[n * K + k]];
            out[m * N + n] = rnd(acc / denom, round_bf16);
        }
}

/* matmul_tn (Tensor), src/tensorops.cpp:24-39 */
void qto_matmul_f32(const float* a, int64_t M, int64_t K, const float* b, int64_t N, int round_bf16, float* out) {
    for (int64_t m = 0; m < M; ++m)
        for (int64_t n = 0; n < N; ++n) {
            float acc = 0.0f;
            for (int64_t k = 0; k < K; ++k) acc += a[m * K + k] * b[n * K + k];
            out[m * N + n] = rnd(acc, round_bf16);
        }
}

/* rmsnorm_residual_fused, src/tensorops.cpp:61-86 (Bf16 rounding) */
void qto_rmsnorm_fwd(const float* x, const float* res, const float* gamma, int64_t rows, int64_t d, float eps,
                     float* nr_out, float* normed, float* absmax) {
    float am = 0.0f;
    for (int64_t r = 0; r < rows; ++r) {
        float* nrp = nr_out + r * d;
        for (int64_t i = 0; i < d; ++i) nrp[i] = x ? qto_bf16_round(x[r * d + i] + res[r * d + i]) : res[r * d + i];
        float ssq = 0.0f;
        for (int64_t i = 0; i < d; ++i) ssq += nrp[i] * nrp[i];
        const float inv = 1.0f / sqrtf(ssq / (float)d + eps);
        for (int64_t i = 0; i < d; ++i) {
            const float v = qto_bf16_round((nrp[i] * inv) * gamma[i]);
            normed[r * d + i] = v;
            const float a = fabsf(v);
            if (a > am || isnan(a)) am = a;
        }
    }
    *absmax = am;
}

/* rmsnorm_residual_backward, src/tensorops.cpp:88-112 */
void qto_rmsnorm_bwd(const float* nr, const float* gamma, int64_t rows, int64_t d, float eps, const float* dy,
                     const float* d_extra, float* d_in, float* d_gamma) {
    for (int64_t i = 0; i < d; ++i) d_gamma[i] = 0.0f;
    for (int64_t r = 0; r < rows; ++r) {
        const float* n = nr + r * d;
        const float* y = dy + r * d;
        float ssq = 0.0f;
        for (int64_t i = 0; i < d; ++i) ssq += n[i] * n[i];
        const float inv = 1.0f / sqrtf(ssq / (float)d + eps);
        float dot = 0.0f;
        for (int64_t i = 0; i < d; ++i) dot += y[i] * gamma[i] * n[i];
        const float inv3_over_d = inv * inv * inv / (float)d;
        for (int64_t i = 0; i < d; ++i) {
            float v = y[i] * gamma[i] * inv - n[i] * inv3_over_d * dot;
            if (d_extra) v += d_extra[r * d + i];
            d_in[r * d + i] = qto_bf16_round(v);
            d_gamma[i] += y[i] * n[i] * inv;
        }
    }
}

static float silu(float x) { return x / (1.0f + expf(-x)); }

/* swiglu_fused, src/tensorops.cpp:114-132 */
void qto_swiglu_fwd(const float* gu, int64_t rows, int64_t two_h, float* h, float* absmax) {
    const int64_t hh = two_h / 2;
    float am = 0.0f;
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t i = 0; i < hh; ++i) {
            const float v = qto_bf16_round(silu(gu[r * two_h + i]) * gu[r * two_h + hh + i]);
            h[r * hh + i] = v;
            const float a = fabsf(v);
            if (a > am || isnan(a)) am = a;
        }
    *absmax = am;
}

/* swiglu_backward, src/tensorops.cpp:134-153 */
void qto_swiglu_bwd(const float* gu, int64_t rows, int64_t two_h, const float* dh, float* dgu) {
    const int64_t hh = two_h / 2;
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t i = 0; i < hh; ++i) {
            const float g = gu[r * two_h + i], u = gu[r * two_h + hh + i], go = dh[r * hh + i];
            const float sig = 1.0f / (1.0f + expf(-g));
            const float dsilu = sig * (1.0f + g * (1.0f - sig));
            dgu[r * two_h + i] = qto_bf16_round(go * u * dsilu);
            dgu[r * two_h + hh + i] = qto_bf16_round(go * (g * sig));
        }
}

/* attn_row_forward, src/tensorops.cpp:191-218 */
static void attn_row(const float* qr, const float* kb, const float* vb, int64_t row, int64_t D, float inv_sqrt_d,
                     float* probs, float* out_row) {
    float mx = -INFINITY;
    for (int64_t j = 0; j <= row; ++j) {
        float s = 0.0f;
        for (int64_t i = 0; i < D; ++i) s += qr[i] * kb[j * D + i];
        probs[j] = s * inv_sqrt_d;
        mx = mx < probs[j] ? probs[j] : mx;
    }
    float denom = 0.0f;
    for (int64_t j = 0; j <= row; ++j) {
        probs[j] = expf(probs[j] - mx);
        denom += probs[j];
    }
    const float inv_denom = 1.0f / denom;
    for (int64_t j = 0; j <= row; ++j) probs[j] *= inv_denom;
    for (int64_t i = 0; i < D; ++i) out_row[i] = 0.0f;
    for (int64_t j = 0; j <= row; ++j)
        for (int64_t i = 0; i < D; ++i) out_row[i] += probs[j] * vb[j * D + i];
}

/* sdpa_chunked, src/tensorops.cpp:227-255 (results are chunk-invariant) */
void qto_sdpa_fwd(const float* q, const float* k, const float* v, int64_t H, int64_t Hkv, int64_t T, int64_t D,
                  float* out) {
    const int64_t group = H / Hkv;
    const float inv_sqrt_d = 1.0f / sqrtf((float)D);
    float* probs = (float*)malloc(sizeof(float) * (size_t)T);
    float* orow = (float*)malloc(sizeof(float) * (size_t)D);
    for (int64_t h = 0; h < H; ++h) {
        const int64_t kvh = h / group;
        for (int64_t t = 0; t < T; ++t) {
            attn_row(q + (h * T + t) * D, k + kvh * T * D, v + kvh * T * D, t, D, inv_sqrt_d, probs, orow);
            for (int64_t i = 0; i < D; ++i) out[(h * T + t) * D + i] = qto_bf16_round(orow[i]);
        }
    }
    free(probs);
    free(orow);
}

/* sdpa_chunked_backward, src/tensorops.cpp:257-303 */
void qto_sdpa_bwd(const float* q, const float* k, const float* v, const float* go, int64_t H, int64_t Hkv, int64_t T,
                  int64_t D, float* dq, float* dk, float* dv) {
    const int64_t group = H / Hkv;
    const float inv_sqrt_d = 1.0f / sqrtf((float)D);
    memset(dq, 0, sizeof(float) * (size_t)(H * T * D));
    memset(dk, 0, sizeof(float) * (size_t)(Hkv * T * D));
    memset(dv, 0, sizeof(float) * (size_t)(Hkv * T * D));
    float* probs = (float*)malloc(sizeof(float) * (size_t)T);
    float* orow = (float*)malloc(sizeof(float) * (size_t)D);
    for (int64_t h = 0; h < H; ++h) {
        const int64_t kvh = h / group;
        const float* kb = k + kvh * T * D;
        const float* vb = v + kvh * T * D;
        float* dkb = dk + kvh * T * D;
        float* dvb = dv + kvh * T * D;
        for (int64_t t = 0; t < T; ++t) {
            const float* qr = q + (h * T + t) * D;
            const float* g = go + (h * T + t) * D;
            attn_row(qr, kb, vb, t, D, inv_sqrt_d, probs, orow);
            float pdp = 0.0f;
            for (int64_t i = 0; i < D; ++i) pdp += g[i] * orow[i];
            float* dqr = dq + (h * T + t) * D;
            for (int64_t j = 0; j <= t; ++j) {
                float dpj = 0.0f;
                for (int64_t i = 0; i < D; ++i) dpj += g[i] * vb[j * D + i];
                const float ds = probs[j] * (dpj - pdp) * inv_sqrt_d;
                for (int64_t i = 0; i < D; ++i) {
                    dqr[i] += ds * kb[j * D + i];
                    dkb[j * D + i] += ds * qr[i];
                    dvb[j * D + i] += probs[j] * g[i];
                }
            }
        }
    }
    for (int64_t i = 0; i < H * T * D; ++i) dq[i] = qto_bf16_round(dq[i]);
    for (int64_t i = 0; i < Hkv * T * D; ++i) {
        dk[i] = qto_bf16_round(dk[i]);
        dv[i] = qto_bf16_round(dv[i]);
    }
    free(probs);
    free(orow);
}

/* embedding_backward_sorted, src/tensorops.cpp:317-342 (stable order by id,
 * ascending positions within an id) */
int qto_embedding_backward(const int32_t* ids, int64_t n, const float* grad_out, int64_t d, int64_t vocab,
                           float* out) {
    for (int64_t p = 0; p < n; ++p)
        if (ids[p] < 0 || ids[p] >= vocab) return -2;
    memset(out, 0, sizeof(float) * (size_t)(vocab * d));
    /* counting sort by id keeps positions ascending inside each id (stable) */
    int64_t* cnt = (int64_t*)calloc((size_t)vocab + 1, sizeof(int64_t));
    int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    for (int64_t p = 0; p < n; ++p) cnt[ids[p] + 1]++;
    for (int64_t v = 0; v < vocab; ++v) cnt[v + 1] += cnt[v];
    for (int64_t p = 0; p < n; ++p) pos[cnt[ids[p]]++] = p;
    for (int64_t s = 0; s < n; ++s) {
        const int64_t p = pos[s];
        float* dst = out + (int64_t)ids[p] * d;
        for (int64_t i = 0; i < d; ++i) dst[i] += grad_out[p * d + i];
    }
    free(cnt);
    free(pos);
    return 0;
}

/* fused_cross_entropy_chunked, src/tensorops.cpp:344-410 */
int qto_cross_entropy(const float* hidden, int64_t N, int64_t d, const float* lm_w, int64_t V, const int32_t* targets,
                      int with_grads, float* loss, float* d_hidden, float* d_lm_w) {
    for (int64_t t = 0; t < N; ++t)
        if (targets[t] < 0 || targets[t] >= V) return -2;
    float* lrow = (float*)malloc(sizeof(float) * (size_t)V);
    const float inv_n = 1.0f / (float)N;
    if (with_grads) memset(d_lm_w, 0, sizeof(float) * (size_t)(V * d));
    float loss_sum = 0.0f;
    for (int64_t t = 0; t < N; ++t) {
        const float* h = hidden + t * d;
        for (int64_t vv = 0; vv < V; ++vv) {
            float acc = 0.0f;
            for (int64_t i = 0; i < d; ++i) acc += h[i] * lm_w[vv * d + i];
            lrow[vv] = acc;
        }
        float mx = lrow[0];
        for (int64_t vv = 1; vv < V; ++vv) mx = mx < lrow[vv] ? lrow[vv] : mx;
        float denom = 0.0f;
        for (int64_t vv = 0; vv < V; ++vv) denom += expf(lrow[vv] - mx);
        const float lse = mx + logf(denom);
        loss_sum += lse - lrow[targets[t]];
        if (!with_grads) continue;
        const float inv_denom = 1.0f / denom;
        for (int64_t vv = 0; vv < V; ++vv) {
            float p = expf(lrow[vv] - mx) * inv_denom;
            if (vv == targets[t]) p -= 1.0f;
            lrow[vv] = p * inv_n;
        }
        for (int64_t i = 0; i < d; ++i) {
            float acc = 0.0f;
            for (int64_t vv = 0; vv < V; ++vv) acc += lrow[vv] * lm_w[vv * d + i];
            d_hidden[t * d + i] = qto_bf16_round(acc);
        }
        for (int64_t vv = 0; vv < V; ++vv) {
            const float dl = lrow[vv];
            if (dl == 0.0f) continue;
            for (int64_t i = 0; i < d; ++i) d_lm_w[vv * d + i] += dl * h[i];
        }
    }
    *loss = loss_sum * inv_n;
    free(lrow);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* optimizer: src/optim.cpp:37-110; accumulation: src/model.cpp:448-464       */
/* ------------------------------------------------------------------------- */
static uint64_t stream_of(const char* prefix, const char* name, const char* suffix) {
    char buf[512];
    size_t n = 0;
    for (const char* p = prefix; *p && n < sizeof(buf) - 1; ++p) buf[n++] = *p;
    for (const char* p = name; *p && n < sizeof(buf) - 1; ++p) buf[n++] = *p;
    for (const char* p = suffix; *p && n < sizeof(buf) - 1; ++p) buf[n++] = *p;
    buf[n] = 0;
    return qto_fnv1a64(buf);
}

/* update_range + make_ctx (src/optim.cpp:37-70), step is the 1-based step
 * being applied; returns -1 on a non-finite scaled gradient */
int qto_adamw_range(const char* name, float* p, float* m, float* v, const float* g, int64_t numel, int64_t lo,
                    int64_t hi, float lr, float b1, float b2, float eps, float wd, int bf16_moments, int bf16_params,
                    uint64_t seed, int64_t step, float grad_scale) {
    const uint64_t sm = stream_of("adamw/", name, "/m");
    const uint64_t sv = stream_of("adamw/", name, "/v");
    const uint64_t sw = stream_of("adamw/", name, "/w");
    const float bc1 = 1.0f - powf(b1, (float)step);
    const float bc2 = 1.0f - powf(b2, (float)step);
    const uint64_t base = (uint64_t)(step - 1) * (uint64_t)numel;
    for (int64_t i = lo; i < hi; ++i) {
        const float gi = g[i] * grad_scale;
        if (!isfinite(gi)) return -1;
        const float m_new = b1 * m[i] + (1.0f - b1) * gi;
        const float v_new = b2 * v[i] + (1.0f - b2) * gi * gi;
        const float mhat = m_new / bc1;
        const float vhat = v_new / bc2;
        const float upd = mhat / (sqrtf(vhat) + eps) + wd * p[i];
        const float p_new = p[i] - lr * upd;
        const uint64_t ctr = base + (uint64_t)i;
        m[i] = bf16_moments ? qto_sr_bf16(m_new, seed, sm, ctr) : m_new;
        v[i] = bf16_moments ? qto_sr_bf16(v_new, seed, sv, ctr) : v_new;
        p[i] = bf16_params ? qto_sr_bf16(p_new, seed, sw, ctr) : p_new;
    }
    return 0;
}

/* grad_norm_block_partials, src/optim.cpp:87-99 (256-element f64 blocks) */
double qto_grad_norm_partials(const float* g, int64_t lo, int64_t hi) {
    double total = 0.0;
    for (int64_t b = lo; b < hi; b += 256) {
        const int64_t end = b + 256 < hi ? b + 256 : hi;
        double partial = 0.0;
        for (int64_t i = b; i < end; ++i) {
            const double x = g[i];
            partial += x * x;
        }
        total += partial;
    }
    return total;
}

/* GradAccumulator::accumulate, src/model.cpp:448-464 */
void qto_grad_accumulate(const char* name, float* buf, const float* g, int64_t n, int f32_mode, uint64_t seed,
                         uint64_t micro_step) {
    const uint64_t stream = stream_of("gradaccum/", name, "");
    const uint64_t base = micro_step * (uint64_t)n;
    for (int64_t i = 0; i < n; ++i) {
        const float s = buf[i] + g[i];
        buf[i] = f32_mode ? s : qto_sr_bf16(s, seed, stream, base + (uint64_t)i);
    }
}

/* normal_init, src/model.cpp:56-65 */
void qto_init_normal(float* t, int64_t n, float std, uint64_t seed, const char* name) {
    const uint64_t stream = stream_of("init/", name, "");
    for (int64_t i = 0; i < n; ++i) t[i] = qto_bf16_round(std * qto_rng_normal(seed, stream, (uint64_t)i));
}

/* shard_layout, src/comms.cpp:69-73 */
void qto_shard_layout(int64_t numel, int workers, int64_t* padded, int64_t* per_worker) {
    const int64_t unit = 256 * (int64_t)workers;
    *padded = (numel + unit - 1) / unit * unit;
    *per_worker = *padded / workers;
}
