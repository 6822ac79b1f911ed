/*
 * bermuda_oracle.c -- CPU restatement of the reference nested-MC path walker.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * engine in paper_0805_1827_b200/.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it; the product never does.
 *
 * It restates, in plain C compiled with -ffp-contract=off (as the reference
 * builds its Cython module, pkg/setup.py:41), the reference algorithm of
 *   pkg/src/bermuda/_kernels/_core.pyx   (Philox, AS241, path walker, solves)
 *   pkg/src/bermuda/rng.py               (SplitMix64 key derivation)
 *   pkg/src/bermuda/boundary_cmc.py      (training-point sampler)
 * and extends it, with the same conventions, to what BASELINE.json asks for but
 * the reference cannot express (geometric / arithmetic basket puts, log-space
 * boundary surfaces, bisection solves, forward point sampling).  Each function
 * names the reference lines it follows.  Pinned against the built reference in
 * tests/test_oracle_pin.py and tests/golden/.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_API __attribute__((visibility("default")))

/* ---------------------------------------------------------------- RNG ---- */

/* SplitMix64 finaliser (rng.py:67-76). */
static uint64_t orc_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* (seed, phase, item, date) -> (key64, stream64)   (rng.py:79-89). */
ORC_API void orc_derive_words(uint64_t seed, uint64_t phase, uint64_t item, uint64_t date,
                              uint64_t *key64, uint64_t *stream64) {
    const uint64_t golden = 0x9E3779B97F4A7C15ULL;
    uint64_t fields[3] = {phase, item, date};
    uint64_t h = orc_mix64(seed + golden);
    for (int i = 0; i < 3; ++i) h = orc_mix64(h ^ (fields[i] + golden));
    *key64 = h;
    *stream64 = orc_mix64(h + 0xD6E8FEB86659FD93ULL);
}

/* Philox4x32-10 on counter (call lo, call hi, stream lo, stream hi) with key
 * (key lo, key hi); words packed as (x0<<32|x1, x2<<32|x3)  (_core.pyx:23-52,
 * rng.py:105-128). */
static void orc_philox(uint64_t key, uint64_t stream, uint64_t call, uint64_t *w0, uint64_t *w1) {
    uint32_t x[4] = {(uint32_t)call, (uint32_t)(call >> 32), (uint32_t)stream, (uint32_t)(stream >> 32)};
    uint32_t k[2] = {(uint32_t)key, (uint32_t)(key >> 32)};
    for (int round = 0; round < 10; ++round) {
        uint64_t a = (uint64_t)0xD2511F53u * x[0];
        uint64_t b = (uint64_t)0xCD9E8D57u * x[2];
        uint32_t y0 = (uint32_t)(b >> 32) ^ x[1] ^ k[0];
        uint32_t y2 = (uint32_t)(a >> 32) ^ x[3] ^ k[1];
        x[1] = (uint32_t)b;
        x[3] = (uint32_t)a;
        x[0] = y0;
        x[2] = y2;
        k[0] += 0x9E3779B9u;
        k[1] += 0xBB67AE85u;
    }
    *w0 = ((uint64_t)x[0] << 32) | x[1];
    *w1 = ((uint64_t)x[2] << 32) | x[3];
}

/* 53-bit open-interval uniform (_core.pyx:55-56, rng.py:145-148). */
static double orc_uniform(uint64_t bits) {
    return ((double)(bits >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}

static double orc_horner(const double *c, int n, double x) {
    /* c[0] is the highest-order coefficient; acc = acc*x + c[i] (rng.py:172-176) */
    double acc = c[0];
    for (int i = 1; i < n; ++i) acc = acc * x + c[i];
    return acc;
}

/* Wichura AS241 / PPND16, highest order first (rng.py:151-211). */
static const double AS_A[8] = {2.5090809287301226727e3, 3.3430575583588128105e4, 6.7265770927008700853e4,
                               4.5921953931549871457e4, 1.3731693765509461125e4, 1.9715909503065514427e3,
                               1.3314166789178437745e2, 3.3871328727963666080};
static const double AS_B[8] = {5.2264952788528545610e3, 2.8729085735721942674e4, 3.9307895800092710610e4,
                               2.1213794301586595867e4, 5.3941960214247511077e3, 6.8718700749205790830e2,
                               4.2313330701600911252e1, 1.0};
static const double AS_C[8] = {7.74545014278341407640e-4, 2.27238449892691845833e-2, 2.41780725177450611770e-1,
                               1.27045825245236838258, 3.64784832476320460504, 5.76949722146069140550,
                               4.63033784615654529590, 1.42343711074968357734};
static const double AS_D[8] = {1.05075007164441684324e-9, 5.47593808499534494600e-4, 1.51986665636164571966e-2,
                               1.48103976427480074590e-1, 6.89767334985100004550e-1, 1.67638483018380384940,
                               2.05319162663775882187, 1.0};
static const double AS_E[8] = {2.01033439929228813265e-7, 2.71155556874348757815e-5, 1.24266094738807843860e-3,
                               2.65321895265761230930e-2, 2.96560571828504891230e-1, 1.78482653991729133580,
                               5.46378491116411436990, 6.65790464350110377720};
static const double AS_F[8] = {2.04426310338993978564e-15, 1.42151175831644588870e-7, 1.84631831751005468180e-5,
                               7.86869131145613259100e-4, 1.48753612908506148525e-2, 1.36929880922735805310e-1,
                               5.99832206555887937690e-1, 1.0};

static double orc_ndtri(double u) {
    double q = u - 0.5;
    if (fabs(q) <= 0.425) {
        double r = 0.180625 - q * q;
        return q * orc_horner(AS_A, 8, r) / orc_horner(AS_B, 8, r);
    }
    double r = sqrt(-log(q < 0.0 ? u : 1.0 - u));
    double z;
    if (r <= 5.0) {
        r = r - 1.6;
        z = orc_horner(AS_C, 8, r) / orc_horner(AS_D, 8, r);
    } else {
        r = r - 5.0;
        z = orc_horner(AS_E, 8, r) / orc_horner(AS_F, 8, r);
    }
    return q < 0.0 ? -z : z;
}

ORC_API void orc_raw_fill(uint64_t key, uint64_t stream, uint64_t start, int64_t count, uint64_t *out) {
    for (int64_t i = 0; i < count; ++i) {
        uint64_t idx = start + (uint64_t)i, w0, w1;
        orc_philox(key, stream, idx >> 1, &w0, &w1);
        out[i] = (idx & 1) ? w1 : w0;
    }
}

ORC_API void orc_normals_fill(uint64_t key, uint64_t stream, uint64_t start, int64_t count, double *out) {
    for (int64_t i = 0; i < count; ++i) {
        uint64_t idx = start + (uint64_t)i, w0, w1;
        orc_philox(key, stream, idx >> 1, &w0, &w1);
        out[i] = orc_ndtri(orc_uniform((idx & 1) ? w1 : w0));
    }
}

/* ------------------------------------------------------------ context ---- */

enum { PAY_MAXCALL = 0, PAY_PUT = 1, PAY_CALL = 2, PAY_GEOPUT = 3, PAY_BASKETPUT = 4 };
enum { RULE_EUROPEAN = 0, RULE_IMMEDIATE = 1, RULE_IZ = 2, RULE_CMC = 3 };

/* Flat market + rule description: the reference MarketPack / RulePack
 * (packs.py:44-71, 100-193) plus iz_space (0 = price-space argmax surfaces,
 * the reference's; 1 = log-space surface of the last asset, for d>1 puts). */
typedef struct {
    int d, n_dates, payoff_kind;
    double strike;
    const double *step_mu, *step_vol, *chol, *disc_steps;
    int rule_kind, call_like, imm_date, nbasis, iz_space;
    const double *iz_coeffs, *iz_lo, *iz_hi;
    const int32_t *cmc_starts, *cmc_counts, *cmc_feat;
    const double *cmc_thr, *cmc_pol, *cmc_alpha, *cmc_intercept;
    /* supplied-normals mode: draw idx i reads normals[i - normals_base] */
    const double *normals;
    uint64_t normals_base, normals_count;
} orc_ctx;

typedef struct {
    uint64_t key, stream, call;
    int valid;
    double u0, u1;
} orc_cache;

static double orc_draw(const orc_ctx *c, uint64_t key, uint64_t stream, uint64_t idx, orc_cache *cache) {
    if (c->normals) {
        uint64_t off = idx - c->normals_base;
        return off < c->normals_count ? c->normals[off] : NAN;
    }
    uint64_t call = idx >> 1;
    if (!cache->valid || cache->call != call || cache->key != key || cache->stream != stream) {
        uint64_t w0, w1;
        orc_philox(key, stream, call, &w0, &w1);
        cache->key = key;
        cache->stream = stream;
        cache->call = call;
        cache->valid = 1;
        cache->u0 = orc_uniform(w0);
        cache->u1 = orc_uniform(w1);
    }
    return orc_ndtri((idx & 1) ? cache->u1 : cache->u0);
}

/* Derived classifier feature at index d (d>1): max for the max-call
 * (boundary_cmc.py:38-52, _core.pyx:275-282), arithmetic mean for the basket
 * put, geometric mean for the geometric put. */
static double orc_mean_log(const orc_ctx *c, const double *v) {
    double s = 0.0;
    for (int i = 0; i < c->d; ++i) s += log(v[i]);
    return s / c->d;
}

static double orc_aggregate(const orc_ctx *c, const double *v) {
    double a;
    switch (c->payoff_kind) {
    case PAY_GEOPUT:
        return exp(orc_mean_log(c, v));
    case PAY_BASKETPUT:
        a = 0.0;
        for (int i = 0; i < c->d; ++i) a += v[i];
        return a / c->d;
    default:
        a = v[0];
        for (int i = 1; i < c->d; ++i)
            if (v[i] > a) a = v[i];
        return a;
    }
}

/* Exercise value (_core.pyx:211-224 plus the two basket puts). */
static double orc_payoff(const orc_ctx *c, const double *v) {
    double p;
    switch (c->payoff_kind) {
    case PAY_MAXCALL: p = orc_aggregate(c, v) - c->strike; break;
    case PAY_PUT: p = c->strike - v[0]; break;
    case PAY_CALL: p = v[0] - c->strike; break;
    default: p = c->strike - orc_aggregate(c, v); break;
    }
    return p > 0.0 ? p : 0.0;
}

/* Quadratic surface value sum_b coeff[b]*basis_b(w) in the reference basis
 * order [1, w_a, w_a*w_b (a<=b)] (packs.py:74-93, _core.pyx:247-265). */
static double orc_quad(const double *row, const double *w, int k) {
    double b = row[0];
    for (int a = 0; a < k; ++a) b += row[1 + a] * w[a];
    int pos = 1 + k;
    for (int a = 0; a < k; ++a)
        for (int bb = a; bb < k; ++bb) b += row[pos++] * w[a] * w[bb];
    return b;
}

/* Boundary-surface decision at date m (_core.pyx:227-268); iz_space 1 is the
 * log-space surface of asset d-1 over the other log prices. */
static int orc_iz_stop(const orc_ctx *c, int m, const double *v) {
    double w[64];
    int d = c->d, k = d - 1;
    if (d == 1) {
        double b = c->iz_coeffs[m * c->nbasis];
        if (c->call_like) return v[0] >= (b < c->strike ? c->strike : b);
        return v[0] <= (b > c->strike ? c->strike : b);
    }
    if (c->iz_space == 1) {
        for (int j = 0; j < k; ++j) {
            double z = log(v[j]);
            w[j] = z < c->iz_lo[j] ? c->iz_lo[j] : (z > c->iz_hi[j] ? c->iz_hi[j] : z);
        }
        const double *row = c->iz_coeffs + ((size_t)m * d + (d - 1)) * c->nbasis;
        return log(v[d - 1]) <= orc_quad(row, w, k);
    }
    int istar = 0;
    for (int i = 1; i < d; ++i)
        if (v[i] > v[istar]) istar = i;
    int cc = 0;
    for (int j = 0; j < d; ++j) {
        if (j == istar) continue;
        double z = v[j];
        w[cc] = z < c->iz_lo[cc] ? c->iz_lo[cc] : (z > c->iz_hi[cc] ? c->iz_hi[cc] : z);
        ++cc;
    }
    double b = orc_quad(c->iz_coeffs + ((size_t)m * d + istar) * c->nbasis, w, k);
    if (b < c->strike) b = c->strike;
    return v[istar] >= b;
}

/* Stump-score decision (_core.pyx:271-287). */
static int orc_cmc_stop(const orc_ctx *c, int m, const double *v) {
    double s = c->cmc_intercept[m];
    double agg = c->d > 1 ? orc_aggregate(c, v) : v[0];
    int t0 = c->cmc_starts[m], t1 = t0 + c->cmc_counts[m];
    for (int t = t0; t < t1; ++t) {
        int f = c->cmc_feat[t];
        double x = f < c->d ? v[f] : agg;
        if (x > c->cmc_thr[t]) s += c->cmc_alpha[t] * c->cmc_pol[t];
        else s -= c->cmc_alpha[t] * c->cmc_pol[t];
    }
    return s > 0.0;
}

/* One stopped path from date m_start (_core.pyx:290-323).  draws of step k,
 * asset a sit at base + k*d + a. */
static double orc_path(const orc_ctx *c, const double *start, int m_start, uint64_t key, uint64_t stream,
                       uint64_t base, orc_cache *cache, int *stop_date) {
    double v[64], z[64];
    int d = c->d, n_steps = c->n_dates - m_start;
    memcpy(v, start, sizeof(double) * d);
    *stop_date = 0;
    for (int k = 0; k < n_steps; ++k) {
        int m = m_start + k + 1;
        for (int a = 0; a < d; ++a) z[a] = orc_draw(c, key, stream, base + (uint64_t)(k * d + a), cache);
        for (int i = 0; i < d; ++i) {
            double y = 0.0;
            for (int a = 0; a < d; ++a) y += c->chol[i * d + a] * z[a];
            v[i] = v[i] * exp(c->step_mu[i] + c->step_vol[i] * y);
        }
        double pay = orc_payoff(c, v);
        if (pay <= 0.0) continue;
        int stop;
        if (c->rule_kind == RULE_EUROPEAN) stop = m == c->n_dates;
        else if (c->rule_kind == RULE_IMMEDIATE) stop = m == c->imm_date;
        else if (m == c->n_dates) stop = 1;
        else if (c->rule_kind == RULE_IZ) stop = orc_iz_stop(c, m, v);
        else stop = orc_cmc_stop(c, m, v);
        if (stop) {
            *stop_date = m;
            return pay * c->disc_steps[m - m_start];
        }
    }
    return 0.0;
}

ORC_API int orc_payoff_value(const orc_ctx *c, const double *v, double *out) {
    *out = orc_payoff(c, v);
    return 0;
}

ORC_API int orc_decision(const orc_ctx *c, int m, const double *v) {
    if (orc_payoff(c, v) <= 0.0) return 0;
    if (c->rule_kind == RULE_EUROPEAN) return m == c->n_dates;
    if (c->rule_kind == RULE_IMMEDIATE) return m == c->imm_date;
    if (m == c->n_dates) return 1;
    return c->rule_kind == RULE_IZ ? orc_iz_stop(c, m, v) : orc_cmc_stop(c, m, v);
}

/* Per-path discounted values + stop dates (the per-path view of
 * stopped_sums: path p's draws start at base + p*per_path). */
ORC_API int orc_path_values(const orc_ctx *c, const double *start, int m_start, int64_t n_paths, uint64_t key,
                            uint64_t stream, uint64_t draw_base, double *out, int32_t *stop_dates) {
    if (c->n_dates - m_start <= 0) return -1;
    uint64_t per_path = (uint64_t)(c->n_dates - m_start) * c->d;
    orc_cache cache = {0};
    for (int64_t p = 0; p < n_paths; ++p) {
        int sd;
        out[p] = orc_path(c, start, m_start, key, stream, draw_base + (uint64_t)p * per_path, &cache, &sd);
        if (stop_dates) stop_dates[p] = sd;
    }
    return 0;
}

/* Sequential sum and sum of squares (_core.pyx:402-430). */
ORC_API int orc_stopped_sums(const orc_ctx *c, const double *start, int m_start, int64_t n_paths, uint64_t key,
                             uint64_t stream, uint64_t draw_base, double *sum, double *sumsq) {
    if (c->n_dates - m_start <= 0) return -1;
    uint64_t per_path = (uint64_t)(c->n_dates - m_start) * c->d;
    orc_cache cache = {0};
    double s = 0.0, ss = 0.0;
    for (int64_t p = 0; p < n_paths; ++p) {
        int sd;
        double val = orc_path(c, start, m_start, key, stream, draw_base + (uint64_t)p * per_path, &cache, &sd);
        s += val;
        ss += val * val;
    }
    *sum = s;
    *sumsq = ss;
    return 0;
}

/* --------------------------------------------------------- I&Z solves ---- */

/* Probe state for the payoff-driving scalar u (_core.pyx:476-483 for
 * iz_space 0, where u is the probed asset's price and seeds above u are
 * pulled to u - 0.01K; iz_space 1 sets the last asset so that the
 * geometric mean of the state equals u). */
static void orc_probe_state(const orc_ctx *c, const double *seed, int asset, double u, double *start) {
    int d = c->d;
    if (c->iz_space == 1) {
        double sl = 0.0;
        for (int j = 0; j < d - 1; ++j) {
            start[j] = seed[j];
            sl += log(seed[j]);
        }
        start[d - 1] = exp(d * log(u) - sl);
        return;
    }
    int j = 0;
    for (int i = 0; i < d; ++i) {
        if (i == asset) start[i] = u;
        else {
            start[i] = seed[j] <= u ? seed[j] : u - 0.01 * c->strike;
            ++j;
        }
    }
}

static double orc_probe_level(const orc_ctx *c, const double *seed, int asset, double u) {
    double start[64];
    orc_probe_state(c, seed, asset, u, start);
    return c->iz_space == 1 ? start[c->d - 1] : u;
}

static double orc_mean_paths(const orc_ctx *c, const double *start, int m, int n_inner, uint64_t key,
                             uint64_t stream, uint64_t base) {
    double s, ss;
    orc_stopped_sums(c, start, m, n_inner, key, stream, base, &s, &ss);
    return s / n_inner;
}

/* Fixed-point solve u <- K +/- C(u) with armed stop and trailing average
 * (_core.pyx:433-512).  Returns the level of the probed asset. */
ORC_API int orc_iz_solve(const orc_ctx *c, const double *seed, int asset, int m, int n_inner, double eps,
                         int max_iter, int avg_window, uint64_t key, uint64_t stream, double *level,
                         int32_t *iterations, int32_t *converged) {
    if (c->n_dates - m <= 0) return -1;
    double start[64];
    double *hist = (double *)malloc(sizeof(double) * (max_iter + 1));
    if (!hist) return -2;
    uint64_t slab = (uint64_t)n_inner * (uint64_t)(c->n_dates - m) * c->d;
    double x = c->strike;
    int armed = 0, conv = 0, it = 0;
    hist[0] = x;
    for (int k = 0; k < max_iter; ++k) {
        orc_probe_state(c, seed, asset, x, start);
        double cont = orc_mean_paths(c, start, m, n_inner, key, stream, (uint64_t)k * slab);
        double x_new = c->call_like ? c->strike + cont : c->strike - cont;
        double step = x_new - x;
        it = k + 1;
        if (!armed && (c->call_like ? step <= 0.0 : step >= 0.0)) armed = 1;
        x = x_new;
        hist[it] = x;
        if (armed && fabs(step) < eps) {
            conv = 1;
            break;
        }
    }
    int n_avg = avg_window < it + 1 ? avg_window : it + 1;
    double acc = 0.0;
    for (int i = it + 1 - n_avg; i <= it; ++i) acc += hist[i];
    free(hist);
    *level = orc_probe_level(c, seed, asset, acc / n_avg);
    *iterations = it;
    *converged = conv;
    return 0;
}

/* Bisection on the payoff-driving scalar over [lo, hi] to width tol, with
 * common random numbers (draw_base 0 for every evaluation).  Exercise is
 * optimal where payoff - C > 0: above the boundary for calls, below it for
 * puts.  BASELINE.json configs 1-2 (no reference counterpart). */
ORC_API int orc_iz_bisect(const orc_ctx *c, const double *seed, int asset, int m, int n_inner, double lo,
                          double hi, double tol, int max_iter, uint64_t key, uint64_t stream, double *level,
                          int32_t *iterations, int32_t *converged) {
    if (c->n_dates - m <= 0) return -1;
    double start[64];
    int it = 0;
    while (hi - lo > tol && it < max_iter) {
        double mid = 0.5 * (lo + hi);
        orc_probe_state(c, seed, asset, mid, start);
        double gain = orc_payoff(c, start) - orc_mean_paths(c, start, m, n_inner, key, stream, 0);
        int exercise = gain > 0.0;
        if (c->call_like == exercise) hi = mid;
        else lo = mid;
        ++it;
    }
    *level = orc_probe_level(c, seed, asset, 0.5 * (lo + hi));
    *iterations = it;
    *converged = hi - lo <= tol;
    return 0;
}

/* ------------------------------------------------------------- CMC ------ */

/* beta_i = payoff(x_i) - mean continuation (_core.pyx:515-550). */
ORC_API int orc_cmc_labels(const orc_ctx *c, const double *points, int64_t n, int m, int n_label,
                           const uint64_t *keys, const uint64_t *streams, uint64_t draw_base, double *out) {
    if (c->n_dates - m <= 0) return -1;
    for (int64_t i = 0; i < n; ++i) {
        const double *x = points + i * c->d;
        double s, ss;
        orc_stopped_sums(c, x, m, n_label, keys[i], streams[i], draw_base, &s, &ss);
        out[i] = orc_payoff(c, x) - s / n_label;
    }
    return 0;
}

/* Training point at date m.  mode 0 is the reference sampler
 * (boundary_cmc.py:164-177 with market.py:180-220): terminal draw from S0
 * over [0, T] with draws 0..d-1, then a Brownian bridge to t_m with draws
 * d..2d-1.  mode 1 steps forward from S0 over dates 1..m with the walker's
 * step (draws (k*d + a)).  sig_sqrt_T[i] = sigma_i*sqrt(T), bridge_sd[i] =
 * sigma_i*sd, log_s0 = log(s0), drift_T = log_drift*T: the host computes
 * these scalars exactly as the reference does.  lam = t_m / T. */
ORC_API int orc_sample_points(const orc_ctx *c, int mode, int m, int64_t n, const uint64_t *keys,
                              const uint64_t *streams, const double *s0, const double *drift_T,
                              const double *sig_sqrt_T, const double *log_s0, const double *bridge_sd, double lam,
                              double *out) {
    int d = c->d;
    for (int64_t i = 0; i < n; ++i) {
        double z[128], term[64], y;
        double *x = out + i * d;
        orc_cache cache = {0};
        if (mode == 1) {
            memcpy(x, s0, sizeof(double) * d);
            for (int k = 0; k < m; ++k) {
                for (int a = 0; a < d; ++a) z[a] = orc_draw(c, keys[i], streams[i], (uint64_t)(k * d + a), &cache);
                for (int r = 0; r < d; ++r) {
                    y = 0.0;
                    for (int a = 0; a < d; ++a) y += c->chol[r * d + a] * z[a];
                    x[r] = x[r] * exp(c->step_mu[r] + c->step_vol[r] * y);
                }
            }
            continue;
        }
        for (int a = 0; a < 2 * d; ++a) z[a] = orc_draw(c, keys[i], streams[i], (uint64_t)a, &cache);
        for (int r = 0; r < d; ++r) {
            y = 0.0;
            for (int a = 0; a < d; ++a) y += z[a] * c->chol[r * d + a];
            term[r] = s0[r] * exp(drift_T[r] + sig_sqrt_T[r] * y);
        }
        if (m == c->n_dates) {
            memcpy(x, term, sizeof(double) * d);
            continue;
        }
        for (int r = 0; r < d; ++r) {
            y = 0.0;
            for (int a = 0; a < d; ++a) y += z[d + a] * c->chol[r * d + a];
            x[r] = exp((1.0 - lam) * log_s0[r] + lam * log(term[r]) + bridge_sd[r] * y);
        }
    }
    return 0;
}

/* ----------------------------------------------- batched (threads) ----- */
/* The restated CPU pricer (oracle/restated.py) for the configs the reference
 * cannot express: independent items spread over the host cores (POSIX
 * threads, a shared atomic item counter), one stream per item as in the
 * engine.  ORC_THREADS overrides the thread count (default: online cores). */
#include <pthread.h>
#include <stdatomic.h>
#include <unistd.h>

typedef struct {
    atomic_long next;
    int64_t n;
    void (*fn)(void *arg, int64_t i);
    void *arg;
} orc_pool;

static void *orc_worker(void *p) {
    orc_pool *pool = (orc_pool *)p;
    for (;;) {
        int64_t i = atomic_fetch_add(&pool->next, 1);
        if (i >= pool->n) break;
        pool->fn(pool->arg, i);
    }
    return NULL;
}

ORC_API int orc_threads(void) {
    const char *e = getenv("ORC_THREADS");
    long t = e ? atol(e) : sysconf(_SC_NPROCESSORS_ONLN);
    return t < 1 ? 1 : (t > 512 ? 512 : (int)t);
}

static void orc_parallel_for(int64_t n, void (*fn)(void *, int64_t), void *arg) {
    orc_pool pool;
    atomic_init(&pool.next, 0);
    pool.n = n;
    pool.fn = fn;
    pool.arg = arg;
    int nt = orc_threads();
    if (nt > n) nt = (int)n;
    pthread_t th[512];
    int started = 0;
    for (int t = 1; t < nt; ++t)
        if (pthread_create(&th[started], NULL, orc_worker, &pool) == 0) ++started;
    orc_worker(&pool);
    for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
}

typedef struct {
    const orc_ctx *c;
    const double *points;
    int m, n_label;
    const uint64_t *keys, *streams;
    uint64_t draw_base;
    double *out;
} orc_labels_job;

static void orc_labels_item(void *p, int64_t i) {
    const orc_labels_job *j = (const orc_labels_job *)p;
    orc_cmc_labels(j->c, j->points + i * j->c->d, 1, j->m, j->n_label, j->keys + i, j->streams + i, j->draw_base,
                   j->out + i);
}

/* orc_cmc_labels over the host cores. */
ORC_API int orc_cmc_labels_mt(const orc_ctx *c, const double *points, int64_t n, int m, int n_label,
                              const uint64_t *keys, const uint64_t *streams, uint64_t draw_base, double *out) {
    if (c->n_dates - m <= 0) return -1;
    orc_labels_job j = {c, points, m, n_label, keys, streams, draw_base, out};
    orc_parallel_for(n, orc_labels_item, &j);
    return 0;
}

typedef struct {
    const orc_ctx *c;
    const double *seeds;
    int seed_stride;
    const int32_t *assets;
    int m, n_inner, max_iter;
    double lo, hi, tol;
    uint64_t seed;
    int64_t item_lo;
    double *level;
    int32_t *iterations, *converged;
} orc_bisect_job;

static void orc_bisect_item(void *p, int64_t i) {
    const orc_bisect_job *j = (const orc_bisect_job *)p;
    uint64_t key, stream;
    orc_derive_words(j->seed, 1, (uint64_t)(j->item_lo + i), (uint64_t)j->m, &key, &stream);
    double zero = 0.0;
    orc_iz_bisect(j->c, j->seed_stride ? j->seeds + i * j->seed_stride : &zero, j->assets[i], j->m, j->n_inner, j->lo,
                  j->hi, j->tol, j->max_iter, key, stream, j->level + i, j->iterations + i, j->converged + i);
}

/* n bisection solves (orc_iz_bisect) on streams derive(seed, IZ_CALC, item_lo + j, m), over the host cores. */
ORC_API int orc_iz_bisect_batch(const orc_ctx *c, const double *seeds, int seed_stride, const int32_t *assets,
                                int64_t n, int m, int n_inner, double lo, double hi, double tol, int max_iter,
                                uint64_t seed, int64_t item_lo, double *level, int32_t *iterations,
                                int32_t *converged) {
    if (c->n_dates - m <= 0) return -1;
    orc_bisect_job j = {c, seeds, seed_stride, assets, m, n_inner, max_iter, lo, hi, tol, seed, item_lo, level,
                        iterations, converged};
    orc_parallel_for(n, orc_bisect_item, &j);
    return 0;
}

typedef struct {
    const orc_ctx *c;
    const double *s0;
    int64_t n_paths, block_lo;
    uint64_t seed;
    double *out;
} orc_price_job;

static void orc_price_item(void *p, int64_t i) {
    const orc_price_job *j = (const orc_price_job *)p;
    const int64_t b = j->block_lo + i;
    int64_t cnt = j->n_paths - b * 4096;
    if (cnt > 4096) cnt = 4096;
    uint64_t key, stream;
    orc_derive_words(j->seed, 3, (uint64_t)b, 0, &key, &stream);
    double s, q;
    orc_stopped_sums(j->c, j->s0, 0, cnt, key, stream, 0, &s, &q);
    j->out[3 * i] = (double)cnt;
    j->out[3 * i + 1] = s;
    j->out[3 * i + 2] = q;
}

/* Per-block (count, sum, sumsq) of 4096-path pricing blocks [block_lo, block_hi)
 * (pricer.py:154-164) on streams derive(seed, PRICING, b, 0), over the host cores. */
ORC_API int orc_price_blocks(const orc_ctx *c, const double *s0, int64_t n_paths, uint64_t seed, int64_t block_lo,
                             int64_t block_hi, double *out) {
    orc_price_job j = {c, s0, n_paths, block_lo, seed, out};
    orc_parallel_for(block_hi - block_lo, orc_price_item, &j);
    return 0;
}
