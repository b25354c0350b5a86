/*
 * odyssey_oracle.c -- CPU restatement of the reference's W4A8 FastGEMM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * library: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product path (libodyssey_b200.so and
 * the paper_2311_09550_b200 package) never links or calls it.
 *
 * Parity pin: every function below is checked against (a) golden vectors
 * produced by the reference itself (oracle/gen_golden.cpp compiled against
 * /root/reference/proj/src, fixtures committed under tests/golden/), and
 * (b) the known-answer tests the reference's own suite holds
 * (proj/tests/test_gemm.cpp:55-127, test_quantizer.cpp:9-119,
 * pipeline.cpp:149-232).  See tests/test_oracle_golden.py.
 *
 * Numeric contract (identical to the reference, which is plain libstdc++):
 *   - scale:  S = max(|gamma*max(w)|, |beta*min(w)|) / qmax, S<=0 -> 2^-24
 *   - codes:  clamp(roundf(x / S), lo, hi)   (IEEE division, half-away round)
 *   - fast GEMM: acc = sum a*(16*w) in int32, acc >>= 4, out = (float)acc*(sa*sw)
 * Build with -ffp-contract=off and without -ffast-math (see oracle/Makefile).
 */
#include <math.h>
#include <pthread.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_EINVAL 1

/* proj/src/core/tensor.hpp:14 -- kMinScale */
static const float kMinScale = 0x1.0p-24f;
/* proj/src/core/gemm.cpp:14 -- 127*127*K must stay below 2^31 */
static const size_t kMaxK = (size_t)1 << 17;

/* ------------------------------------------------------------------ RNG */
/* proj/src/core/rng.hpp:10-52 -- splitmix64 + Box-Muller */
typedef struct oracle_rng {
    uint64_t state;
    double spare;
    int have_spare;
} oracle_rng;

void oracle_rng_init(oracle_rng* r, uint64_t seed) {
    r->state = seed;
    r->spare = 0.0;
    r->have_spare = 0;
}

uint64_t oracle_rng_next_u64(oracle_rng* r) {
    uint64_t z = (r->state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

double oracle_rng_uniform(oracle_rng* r) {
    return (double)(oracle_rng_next_u64(r) >> 11) * 0x1.0p-53;
}

int64_t oracle_rng_uniform_int(oracle_rng* r, int64_t lo, int64_t hi) {
    uint64_t span = (uint64_t)(hi - lo) + 1;
    return lo + (int64_t)(oracle_rng_next_u64(r) % span);
}

double oracle_rng_gaussian(oracle_rng* r) {
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    double u1 = oracle_rng_uniform(r);
    double u2 = oracle_rng_uniform(r);
    while (u1 <= 1e-300) u1 = oracle_rng_uniform(r);
    double rad = sqrt(-2.0 * log(u1));
    double theta = 2.0 * 3.14159265358979323846 * u2;
    r->spare = rad * sin(theta);
    r->have_spare = 1;
    return rad * cos(theta);
}

/* v = (float)(gaussian() * stddev) for each element, in order
 * (proj/src/core/bench.cpp:80-83; stddev 1.0 reproduces the activation fill). */
void oracle_rng_fill_gaussian(oracle_rng* r, float* out, size_t n, double stddev) {
    for (size_t i = 0; i < n; ++i) out[i] = (float)(oracle_rng_gaussian(r) * stddev);
}

/* ------------------------------------------------------------ quantizer */
/* proj/src/core/quantize.cpp:12-18 -- round half away from zero, clamp */
static int32_t clamp_code(float x, int32_t lo, int32_t hi) {
    float r = roundf(x);
    if (r < (float)lo) return lo;
    if (r > (float)hi) return hi;
    return (int32_t)r;
}

static float fmax_ref(float a, float b) { return (a < b) ? b : a; } /* std::max */
static float fmin_ref(float a, float b) { return (b < a) ? b : a; } /* std::min */

/* proj/src/core/quantize.cpp:22-35 */
int oracle_compute_scale_symmetric(const float* w, size_t n, int bits, float gamma, float beta,
                                   float* out) {
    if (n == 0) return ORACLE_EINVAL;
    if (!(gamma > 0.0f && gamma <= 1.0f && beta > 0.0f && beta <= 1.0f)) return ORACLE_EINVAL;
    float wmax = w[0], wmin = w[0];
    for (size_t i = 0; i < n; ++i) {
        wmax = fmax_ref(wmax, w[i]);
        wmin = fmin_ref(wmin, w[i]);
    }
    float qmax = (float)((1 << (bits - 1)) - 1);
    float s = fmax_ref(fabsf(gamma * wmax), fabsf(beta * wmin)) / qmax;
    *out = s > 0.0f ? s : kMinScale;
    return ORACLE_OK;
}

/* proj/src/core/quantize.cpp:37-47 -- code = clamp(round(w / S)) (division, not reciprocal) */
int oracle_quantize_symmetric(const float* w, size_t n, int bits, float gamma, float beta,
                              int8_t* codes, float* scale) {
    float s;
    int rc = oracle_compute_scale_symmetric(w, n, bits, gamma, beta, &s);
    if (rc) return rc;
    const int32_t lo = -(1 << (bits - 1));
    const int32_t hi = (1 << (bits - 1)) - 1;
    for (size_t i = 0; i < n; ++i) codes[i] = (int8_t)clamp_code(w[i] / s, lo, hi);
    *scale = s;
    return ORACLE_OK;
}

/* proj/src/core/quantize.cpp:113-132 -- dynamic per-token symmetric INT8 */
int oracle_quantize_activations_per_token(const float* a, size_t m, size_t k, int8_t* codes,
                                          float* scales) {
    if (m == 0 || k == 0) return ORACLE_EINVAL;
    for (size_t r = 0; r < m; ++r) {
        int rc = oracle_quantize_symmetric(a + r * k, k, 8, 1.0f, 1.0f, codes + r * k, &scales[r]);
        if (rc) return rc;
    }
    return ORACLE_OK;
}

/* proj/src/core/quantize.cpp:75-111 restricted to the hot path's per-channel
 * granularity; gamma/beta may be NULL (1.0 everywhere, tensor.hpp:86-87). */
int oracle_quantize_weights_per_channel(const float* w, size_t n, size_t k, int bits,
                                        const float* gamma, const float* beta, int8_t* codes,
                                        float* scales) {
    if (n == 0 || k == 0) return ORACLE_EINVAL;
    if (bits != 4 && bits != 8) return ORACLE_EINVAL;
    for (size_t r = 0; r < n; ++r) {
        float g = gamma ? gamma[r] : 1.0f;
        float b = beta ? beta[r] : 1.0f;
        int rc = oracle_quantize_symmetric(w + r * k, k, bits, g, b, codes + r * k, &scales[r]);
        if (rc) return rc;
    }
    return ORACLE_OK;
}

/* --------------------------------------------------------- int4 packing */
/* proj/src/core/tensor.cpp:30-60 -- element 2k low nibble, 2k+1 high nibble;
 * odd tail leaves the last high nibble zero.  bytes must hold (count+1)/2. */
int oracle_pack_int4(const int8_t* codes, size_t count, uint8_t* bytes) {
    memset(bytes, 0, (count + 1) / 2);
    for (size_t i = 0; i < count; ++i) {
        if (codes[i] < -8 || codes[i] > 7) return ORACLE_EINVAL;
        uint8_t nib = (uint8_t)codes[i] & 0x0F;
        if (i % 2 == 0)
            bytes[i / 2] = (uint8_t)((bytes[i / 2] & 0xF0) | nib);
        else
            bytes[i / 2] = (uint8_t)((bytes[i / 2] & 0x0F) | (nib << 4));
    }
    return ORACLE_OK;
}

/* proj/src/core/tensor.cpp:42-47 -- sign-extended get */
int8_t oracle_int4_get(const uint8_t* bytes, size_t i) {
    uint8_t byte = bytes[i / 2];
    uint8_t nib = (i % 2 == 0) ? (byte & 0x0F) : (byte >> 4);
    return (int8_t)(nib >= 8 ? (int)nib - 16 : (int)nib);
}

/* proj/src/core/gemm.cpp:49-54 -- SINT4 -> S8 lane equal to value*16 */
int8_t oracle_unpack_sint4_as_high_nibble(const uint8_t* bytes, size_t i) {
    uint8_t byte = bytes[i / 2];
    uint8_t shifted = (i % 2 == 0) ? (uint8_t)(byte << 4) : (uint8_t)(byte & 0xF0);
    return (int8_t)shifted;
}

/* ----------------------------------------------------------- fast GEMM */
typedef struct gemm_job {
    const int8_t* a;      /* M x K activation codes */
    const float* sa;      /* M per-token scales (NULL for accumulator mode) */
    const int8_t* lanes;  /* N x K high-nibble lanes */
    const float* sw;      /* N per-channel scales */
    size_t n, k;
    size_t r0, r1;
    int32_t* acc;         /* accumulator mode output (M x N), pre-shift */
    float* out;           /* epilogue mode output (M x N) */
} gemm_job;

static void* gemm_rows(void* p) {
    gemm_job* j = (gemm_job*)p;
    for (size_t i = j->r0; i < j->r1; ++i) {
        const int8_t* ai = j->a + i * j->k;
        for (size_t c = 0; c < j->n; ++c) {
            const int8_t* wj = j->lanes + c * j->k;
            int32_t s = 0;
            for (size_t kk = 0; kk < j->k; ++kk) s += (int32_t)ai[kk] * (int32_t)wj[kk];
            if (j->acc) {
                j->acc[i * j->n + c] = s; /* gemm.cpp:244 (before the shift) */
            } else {
                s >>= 4;                  /* gemm.cpp:269 -- exact */
                j->out[i * j->n + c] = (float)s * (j->sa[i] * j->sw[c]); /* gemm.cpp:273 */
            }
        }
    }
    return NULL;
}

/* Row-chunk fan-out over M, one fresh thread per chunk, mirroring
 * parallel_for_rows (proj/src/core/parallel.cpp:36-54). */
static void run_rows(gemm_job* base, size_t m, int threads) {
    size_t workers = threads > 0 ? (size_t)threads : 1;
    if (workers > m) workers = m;
    if (workers <= 1) {
        base->r0 = 0;
        base->r1 = m;
        gemm_rows(base);
        return;
    }
    size_t chunk = (m + workers - 1) / workers;
    pthread_t* tids = (pthread_t*)calloc(workers, sizeof(pthread_t));
    gemm_job* jobs = (gemm_job*)calloc(workers, sizeof(gemm_job));
    size_t launched = 0;
    for (size_t w = 0; w < workers; ++w) {
        size_t b = w * chunk, e = b + chunk < m ? b + chunk : m;
        if (b >= e) break;
        jobs[w] = *base;
        jobs[w].r0 = b;
        jobs[w].r1 = e;
        pthread_create(&tids[w], NULL, gemm_rows, &jobs[w]);
        ++launched;
    }
    for (size_t w = 0; w < launched; ++w) pthread_join(tids[w], NULL);
    free(tids);
    free(jobs);
}

/* proj/src/core/gemm.cpp:219-225 -- serial widening pre-pass */
static int8_t* unpack_lanes(const uint8_t* packed, size_t count) {
    int8_t* lanes = (int8_t*)malloc(count ? count : 1);
    for (size_t i = 0; i < count; ++i) lanes[i] = oracle_unpack_sint4_as_high_nibble(packed, i);
    return lanes;
}

/* proj/src/core/gemm.cpp:229-249 -- int32 accumulators of sum a*(16w), before >>4.
 * w_packed is the flat PackedInt4Buffer over N x K (tensor.hpp:43-64). */
int oracle_gemm_w4a8_fast_accumulators(const int8_t* a_codes, const uint8_t* w_packed, size_t m,
                                       size_t n, size_t k, int threads, int32_t* acc) {
    if (m == 0 || n == 0 || k == 0 || k > kMaxK) return ORACLE_EINVAL;
    int8_t* lanes = unpack_lanes(w_packed, n * k);
    gemm_job j = {a_codes, NULL, lanes, NULL, n, k, 0, 0, acc, NULL};
    run_rows(&j, m, threads);
    free(lanes);
    return ORACLE_OK;
}

/* proj/src/core/gemm.cpp:251-279 -- the FastGEMM engine with its epilogue */
int oracle_gemm_w4a8_fast(const int8_t* a_codes, const float* sa, const uint8_t* w_packed,
                          const float* sw, size_t m, size_t n, size_t k, int threads, float* out) {
    if (m == 0 || n == 0 || k == 0 || k > kMaxK) return ORACLE_EINVAL;
    int8_t* lanes = unpack_lanes(w_packed, n * k);
    gemm_job j = {a_codes, sa, lanes, sw, n, k, 0, 0, NULL, out};
    run_rows(&j, m, threads);
    free(lanes);
    return ORACLE_OK;
}

/* proj/src/core/quantize.cpp:134-146 -- symmetric per-row dequantize, q*S */
void oracle_dequantize_rows(const int8_t* codes, const float* scales, size_t rows, size_t cols,
                            float* out) {
    for (size_t r = 0; r < rows; ++r)
        for (size_t c = 0; c < cols; ++c) out[r * cols + c] = (float)codes[r * cols + c] * scales[r];
}

/* proj/src/core/tensor.cpp:176-196 -- fixed-order f32 matmul against b^T */
void oracle_matmul_f32(const float* a, const float* bt, size_t m, size_t n, size_t k, float* out) {
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j) {
            float acc = 0.0f;
            for (size_t kk = 0; kk < k; ++kk) acc += a[i * k + kk] * bt[j * k + kk];
            out[i * n + j] = acc;
        }
}

/* proj/src/core/bench.cpp:14-22 -- FNV-1a 64 checksum */
uint64_t oracle_fnv1a(const void* data, size_t bytes) {
    const uint8_t* p = (const uint8_t*)data;
    uint64_t h = 0xcbf29ce484222325ULL;
    for (size_t i = 0; i < bytes; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

/* quantize.cpp:37-47 with the scale supplied by the caller: the row-parallel TP
 * restatement (scale of the full row applied to a K-shard). */
void oracle_quantize_with_scale(const float* x, size_t n, int bits, float scale, int8_t* codes) {
    const int32_t lo = -(1 << (bits - 1));
    const int32_t hi = (1 << (bits - 1)) - 1;
    for (size_t i = 0; i < n; ++i) codes[i] = (int8_t)clamp_code(x[i] / scale, lo, hi);
}

/* ---------------------------------------------- comparison engines */
/* proj/src/core/quantize.cpp:75-111 with PerGroup granularity: one symmetric scale per
 * (row, group of g columns); scales laid out [row][group] (tensor.cpp:117-125). */
int oracle_quantize_weights_per_group(const float* w, size_t n, size_t k, size_t g, int bits, int8_t* codes,
                                      float* scales) {
    if (g == 0 || k % g) return ORACLE_EINVAL;
    const size_t groups = k / g;
    for (size_t r = 0; r < n; ++r)
        for (size_t gi = 0; gi < groups; ++gi) {
            int rc = oracle_quantize_symmetric(w + r * k + gi * g, g, bits, 1.0f, 1.0f, codes + r * k + gi * g,
                                               &scales[r * groups + gi]);
            if (rc) return rc;
        }
    return ORACLE_OK;
}

/* proj/src/core/gemm.cpp:281-311 -- W8A8: acc = sum a*w (int32), out = float(acc)*(sa*sw) */
void oracle_gemm_w8a8(const int8_t* a, const float* sa, const int8_t* w, const float* sw, size_t m, size_t n,
                      size_t k, float* out) {
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j) {
            int32_t acc = 0;
            for (size_t kk = 0; kk < k; ++kk) acc += (int32_t)a[i * k + kk] * (int32_t)w[j * k + kk];
            out[i * n + j] = (float)acc * (sa[i] * sw[j]);
        }
}

/* proj/src/core/gemm.cpp:123-161 -- fine-grained: per group an int32 sub-sum, then
 * acc += float(sub) * (sa * s_group) in f32, groups in order */
void oracle_gemm_finegrained(const int8_t* a, const float* sa, const int8_t* w, const float* ws, size_t g,
                             size_t m, size_t n, size_t k, float* out) {
    const size_t groups = k / g;
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j) {
            float acc = 0.0f;
            for (size_t gi = 0; gi < groups; ++gi) {
                int32_t sub = 0;
                for (size_t kk = 0; kk < g; ++kk)
                    sub += (int32_t)a[i * k + gi * g + kk] * (int32_t)w[j * k + gi * g + kk];
                acc += (float)sub * (sa[i] * ws[j * groups + gi]);
            }
            out[i * n + j] = acc;
        }
}

/* proj/src/core/gemm.cpp:163-202 + 56-75 -- asymmetric (offset) path: nibble u = q + 8,
 * widened and 8 subtracted, acc = sum a*(u - 8), out = float(acc)*(sa*sw) */
void oracle_gemm_asymmetric(const int8_t* a, const float* sa, const int8_t* w, const float* sw, size_t m,
                            size_t n, size_t k, float* out) {
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j) {
            int32_t acc = 0;
            for (size_t kk = 0; kk < k; ++kk) {
                const uint8_t u = (uint8_t)(w[j * k + kk] + 8); /* pack_uint4_offset */
                acc += (int32_t)a[i * k + kk] * ((int32_t)u - 8);
            }
            out[i * n + j] = (float)acc * (sa[i] * sw[j]);
        }
}

/* proj/src/core/gemm.cpp:105-121 -- W4A16: f32 activations against dequantized weights,
 * acc += a * (float(code) * scale), sequential over k (scales [row][group], g = group) */
void oracle_gemm_w4a16(const float* a, const int8_t* w, const float* ws, size_t g, size_t m, size_t n, size_t k,
                       float* out) {
    const size_t groups = k / g;
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j) {
            float acc = 0.0f;
            for (size_t kk = 0; kk < k; ++kk) {
                const float wf = (float)w[j * k + kk] * ws[j * groups + kk / g];
                acc += a[i * k + kk] * wf;
            }
            out[i * n + j] = acc;
        }
}

/* ------------------------------------------------------------ LWC (clip.cpp) */
/* proj/src/core/clip.cpp:11-24 -- candidate grid */
size_t oracle_clip_candidates(float gmin, float step, float* out, size_t cap) {
    size_t n = 0;
    for (int i = 0; n + 1 < cap; ++i) {
        float v = gmin + (float)i * step;
        if (v >= 1.0f - 1e-6f) break;
        out[n++] = v;
    }
    out[n++] = 1.0f;
    return n;
}

/* proj/src/core/clip.cpp:40-51 */
static double mse_for_scale(const float* w, size_t k, int bits, float scale) {
    const float lo = (float)(-(1 << (bits - 1)));
    const float hi = (float)((1 << (bits - 1)) - 1);
    double acc = 0.0;
    for (size_t i = 0; i < k; ++i) {
        float c = roundf(w[i] / scale);
        c = fmin_ref(fmax_ref(c, lo), hi);
        double e = (double)w[i] - (double)c * (double)scale;
        acc += e * e;
    }
    return acc / (double)k;
}

/* proj/src/core/clip.cpp:55-103 -- per row: the (gamma, beta) pair minimising the MSE,
 * ties to larger gamma+beta, then larger gamma */
int oracle_optimize_clipping(const float* w, size_t n, size_t k, int bits, float gmin, float step, float* gamma,
                             float* beta, float* mse_before, float* mse_after) {
    if (n * k == 0 || !(gmin > 0.0f && gmin <= 1.0f) || !(step > 0.0f)) return ORACLE_EINVAL;
    float cand[4096];
    const size_t nc = oracle_clip_candidates(gmin, step, cand, 4096);
    const float qmax = (float)((1 << (bits - 1)) - 1);
    for (size_t r = 0; r < n; ++r) {
        const float* ch = w + r * k;
        float wmax = ch[0], wmin = ch[0];
        for (size_t i = 0; i < k; ++i) {
            wmax = fmax_ref(wmax, ch[i]);
            wmin = fmin_ref(wmin, ch[i]);
        }
        double best = 0.0, ident = 0.0;
        float bg = 1.0f, bb = 1.0f;
        int first = 1;
        for (size_t gi = 0; gi < nc; ++gi)
            for (size_t bi = 0; bi < nc; ++bi) {
                const float g = cand[gi], b = cand[bi];
                float s = fmax_ref(fabsf(g * wmax), fabsf(b * wmin)) / qmax;
                if (!(s > 0.0f)) s = kMinScale;
                const double mse = mse_for_scale(ch, k, bits, s);
                if (g == 1.0f && b == 1.0f) ident = mse;
                const int better = first || mse < best ||
                                   (mse == best && (g + b > bg + bb || (g + b == bg + bb && g > bg)));
                if (better) {
                    best = mse;
                    bg = g;
                    bb = b;
                    first = 0;
                }
            }
        gamma[r] = bg;
        beta[r] = bb;
        mse_before[r] = (float)ident;
        mse_after[r] = (float)best;
    }
    return ORACLE_OK;
}
