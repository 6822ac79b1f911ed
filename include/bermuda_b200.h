/*
 * bermuda_b200.h -- C ABI of the B200 nested-Monte-Carlo engine
 * (libbermuda_b200.so, built from paper_0805_1827_b200/csrc/).
 *
 * Drop-in boundary for the reference package `bermuda` (arXiv 0805.1827):
 * every entry point replaces one function of the reference's duck-typed
 * kernel-backend module (pkg/src/bermuda/_kernels/core_backend.py:12-58,
 * numpy_backend.py:19-190) or one phase body of its builders, and is cited
 * below.  Plain C types only: no torch, no numpy.
 *
 * Buffers.  Every array argument may be HOST memory (pageable or pinned) or
 * DEVICE memory of the context's GPU; the library inspects each pointer.
 * Host inputs are staged to HBM and host outputs copied back before the call
 * returns.  When every output of a call is device memory the call is
 * stream-ordered and returns without synchronising (see brm_ctx_set_stream).
 *
 * Errors.  Functions return BRM_OK (0) or a status; brm_last_error() gives
 * the message (thread-local).  The Python shim maps BRM_EINVAL to ValueError
 * (the reference raises ValueError for a start date with no remaining
 * exercise dates, _core.pyx:406-407, 445-446, 524-525) and BRM_ENOMEM to
 * MemoryError (_core.pyx:418-421).
 *
 * Precision modes (per context).  BRM_MODE_PARITY reproduces the reference
 * pipeline: Philox4x32-10 words, 53-bit uniforms and AS241 normals in fp64
 * with the reference draw indexing (_core.pyx:4-7) and no FMA contraction,
 * so draws are the reference's draws and per-path values agree to the last
 * ulp of exp().  BRM_MODE_FAST steps paths in fp32 with Box-Muller normals
 * from the same Philox counter space and accumulates in fp64 (BASELINE.json
 * configs 3-4); it agrees with the reference statistically only.
 */
#ifndef BERMUDA_B200_H
#define BERMUDA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define BRM_ABI_VERSION 3

enum brm_status {
    BRM_OK = 0,
    BRM_EINVAL = 1,   /* invalid argument            -> ValueError   */
    BRM_ENOMEM = 2,   /* allocation failure          -> MemoryError  */
    BRM_ECUDA = 3,    /* CUDA runtime / launch error -> RuntimeError */
    BRM_ENODEV = 4    /* no usable sm_100 device     -> RuntimeError */
};

enum brm_mode { BRM_MODE_PARITY = 0, BRM_MODE_FAST = 1 };

/* Payoff codes: 0-2 are the reference's (packs.py:33-35); 3-4 are the
 * BASELINE.json configs 2 and 4 the reference cannot express. */
enum brm_payoff {
    BRM_PAY_MAXCALL = 0, BRM_PAY_PUT = 1, BRM_PAY_CALL = 2,
    BRM_PAY_GEOPUT = 3, BRM_PAY_BASKETPUT = 4
};

/* Rule kinds (packs.py:28-31). */
enum brm_rule_kind { BRM_RULE_EUROPEAN = 0, BRM_RULE_IMMEDIATE = 1, BRM_RULE_IZ = 2, BRM_RULE_CMC = 3 };

/* Stream phases (rng.py:55-61). */
enum brm_phase { BRM_PHASE_GLP = 0, BRM_PHASE_IZ_CALC = 1, BRM_PHASE_CMC_CALC = 2, BRM_PHASE_PRICING = 3 };

/* Market pack (packs.py:44-71).  Arrays are host or device. */
typedef struct brm_market_desc {
    int32_t d, n_dates, payoff_kind;
    double strike;
    const double *step_mu;     /* [d]          log drift per exercise step  */
    const double *step_vol;    /* [d]          sigma*sqrt(dt)                */
    const double *chol;        /* [d*d]        correlation factor, row-major */
    const double *disc_steps;  /* [n_dates+1]  exp(-r*k*dt)                  */
    const double *s0;          /* [d]                                        */
} brm_market_desc;

/* Rule pack (packs.py:100-193).  iz_space 0 is the reference's price-space
 * surfaces of the argmax asset (_core.pyx:227-268); 1 is a log-space surface
 * of the last asset over the other log prices (geometric put, config 2). */
typedef struct brm_rule_desc {
    int32_t kind, call_like, imm_date;
    int32_t nbasis, iz_space;
    const double *iz_coeffs;   /* [(n_dates+1)*d*nbasis] */
    const double *iz_lo, *iz_hi; /* [d-1] clamp box (log box when iz_space 1) */
    int32_t n_stumps;
    const int32_t *cmc_starts, *cmc_counts; /* [n_dates+1] */
    const int32_t *cmc_feat;   /* [n_stumps]; index d = derived feature */
    const double *cmc_thr, *cmc_pol, *cmc_alpha; /* [n_stumps] */
    const double *cmc_intercept; /* [n_dates+1] */
} brm_rule_desc;

typedef struct brm_ctx brm_ctx;

int brm_abi_version(void);
const char *brm_last_error(void);
int brm_device_count(int32_t *count);

/* Context = device-resident copy of one (MarketPack, RulePack) pair; replaces
 * the reference's cached _CtxHolder (core_backend.py:23-33, _core.pyx:334-378). */
int brm_ctx_create(const brm_market_desc *market, const brm_rule_desc *rule, int32_t device, int32_t mode,
                   brm_ctx **out);
int brm_ctx_destroy(brm_ctx *ctx);
/* Device-resident backward induction (the date loop of build_cmc_rule,
 * boundary_cmc.py:248-278, without a host round trip per date): a CMC
 * context whose dates start empty (intercept -1, never exercise) with room
 * for `capacity` stumps per date (<= 1024).  brm_ctx_set_ensemble writes
 * date `date`'s ensemble -- arrays sized [capacity], *count stumps used,
 * *intercept -- into the image on the context's stream (inputs may be
 * device pointers, e.g. the outputs of brm_fit_ensemble with
 * BRM_FIT_DEVICE_RESULT), building the date's step tables on the device.
 * The image equals the one brm_ctx_create builds for the same ensembles
 * (RulePack.from_stumps, packs.py:149-182) up to the layout. */
int brm_ctx_create_cmc(const brm_market_desc *market, int32_t call_like, int32_t capacity, int32_t device,
                       int32_t mode, brm_ctx **out);
int brm_ctx_set_ensemble(brm_ctx *ctx, int32_t date, const int32_t *feat, const double *thr, const double *pol,
                         const double *alpha, const int32_t *count, const double *intercept);
/* Launch on a caller-owned cudaStream_t (e.g. torch's current stream); NULL restores the context's own. */
int brm_ctx_set_stream(brm_ctx *ctx, void *cuda_stream);
/* Fixed-input mode: draw index i of every stream reads normals[i - base]
 * instead of the generator (north star "identical host-supplied normal
 * draws").  normals == NULL returns to the generator. */
int brm_ctx_supply_normals(brm_ctx *ctx, const double *normals, uint64_t base, uint64_t count);

/* ---- RNG (rng.py:79-216; _core.pyx:149-181) ---------------------------- */
int brm_derive_words(uint64_t seed, uint32_t phase, uint64_t item, uint64_t date, uint64_t *key64,
                     uint64_t *stream64);
int brm_raw_uint64(int32_t device, uint64_t key64, uint64_t stream64, uint64_t start, int64_t count,
                   uint64_t *out);
int brm_normals(int32_t device, uint64_t key64, uint64_t stream64, uint64_t start, int64_t count,
                double *out);

/* Self-test of the walker's branch-free fp64 exp / divide / log / sqrt against
 * CUDA's exp / __ddiv_rn / log / __dsqrt_rn (kind 0 exp_nb(a), 1 exp(a),
 * 2 div_nb(a, b), 3 a / b, 4 log_nb(a), 5 log(a), 6 sqrt_nb(a), 7 sqrt(a)),
 * and of AdaBoost's parallel cumsum against the sequential one (kind 8:
 * out = np.cumsum order of a[0..n) by one thread, 10: by the parity
 * AdaBoost's block-parallel exact scan; a >= 0). */
int brm_selftest_math(int32_t device, int32_t kind, const double *a, const double *b, int64_t n, double *out);

/* ---- Path walker ------------------------------------------------------- */
/* stopped_sums (core_backend.py:36-41, _core.pyx:402-430). */
int brm_stopped_sums(brm_ctx *ctx, const double *start_values, int32_t m_start, int64_t n_paths,
                     uint64_t key64, uint64_t stream64, uint64_t draw_base, double *sum, double *sumsq);
/* Per-path discounted values and stop dates (0 = never exercised) of the
 * same paths stopped_sums folds: path p starts at draw_base + p*per_path. */
int brm_path_values(brm_ctx *ctx, const double *start_values, int32_t m_start, int64_t n_paths,
                    uint64_t key64, uint64_t stream64, uint64_t draw_base, double *values,
                    int32_t *stop_dates);
/* Exercise decision of the context's rule for n states at date m
 * (pricer.py:104-133 iz_exercise_rule / cmc_exercise_rule). */
int brm_decisions(brm_ctx *ctx, const double *states, int64_t n, int32_t m, int32_t *out);

/* Final pricing: blocks [block_lo, block_hi) of PATH_BLOCK=4096 paths, block
 * b on StreamKey(seed, PRICING, b) from s0 at date 0; out_stats[b-block_lo] =
 * (count, sum, sumsq)  (pricer.py:154-164). */
int brm_price_blocks(brm_ctx *ctx, int64_t n_paths, uint64_t seed, int64_t block_lo, int64_t block_hi,
                     double *out_stats);

/* cmc_labels (core_backend.py:52-58, _core.pyx:515-550): beta_i =
 * payoff(x_i) - mean of n_label stopped paths from x_i at date m on stream
 * (keys[i], streams[i]) from draw_base.  keys == NULL derives them on the
 * device as StreamKey(seed, CMC_CALC, item_lo + i, m) (boundary_cmc.py:220). */
int brm_cmc_labels(brm_ctx *ctx, const double *points, int64_t n, int32_t m, int32_t n_label,
                   const uint64_t *keys, const uint64_t *streams, uint64_t seed, int64_t item_lo,
                   uint64_t draw_base, double *out_beta);

/* Training points at date m for items [item_lo, item_lo+n) on
 * StreamKey(seed, CMC_CALC, item, m).  mode 0 = the reference sampler
 * (terminal draw + Brownian bridge, boundary_cmc.py:164-177, labels then
 * start at draw 2d); mode 1 = forward from S0 over dates 1..m (labels start
 * at draw m*d).  bridge holds 4*d+1 host-computed scalars:
 * [drift_T(d), sig_sqrt_T(d), log_s0(d), bridge_sd(d), lam]. */
int brm_sample_points(brm_ctx *ctx, int32_t mode, int32_t m, uint64_t seed, int64_t item_lo, int64_t n,
                      const double *bridge, double *out_points);

/* ---- I&Z probes (_core.pyx:433-512; BASELINE bisection) ----------------- */
/* n probes; seeds [n*(d-1)] (row-major), assets [n]; keys NULL derives
 * StreamKey(seed, IZ_CALC, item_lo + i, m) (boundary_iz.py:288).
 * solver 0: fixed point u <- K +/- C(u) from K, fresh draws per iteration,
 *           armed |step| < eps stop, mean of the last avg_window iterates.
 * solver 1: bisection of payoff - C on [lo, hi] to width tol with common
 *           random numbers.  Levels are prices of the probed asset. */
int brm_iz_solve(brm_ctx *ctx, int32_t solver, const double *seeds, const int32_t *assets, int64_t n,
                 int32_t m, int32_t n_inner, double eps, int32_t max_iter, int32_t avg_window, double lo,
                 double hi, double tol, const uint64_t *keys, const uint64_t *streams, uint64_t seed,
                 int64_t item_lo, double *out_level, int32_t *out_iterations, int32_t *out_converged);

/* ---- CMC date step: sampler + features + labels (boundary_cmc.py:210-227) */
/* Items [item_lo, item_lo+n) of date m: sample the training point (sampler
 * 0 = reference bridge, 1 = forward; bridge as in brm_sample_points), write
 * its classifier features out_features[i*F + f] with F = d+1 for d>1 (the
 * d prices plus the payoff aggregate: max for the max-call as the reference's
 * classifier_features, boundary_cmc.py:38-52; arithmetic / geometric mean for
 * the basket / geometric puts) and F = 1 for d = 1, and its label
 * out_beta[i] = payoff - continuation with n_label paths under the
 * context's (later-dates) rule, continuing the point's stream after the
 * sampler draws. */
int brm_cmc_calc(brm_ctx *ctx, int32_t sampler, int32_t m, uint64_t seed, int64_t item_lo, int64_t n,
                 int32_t n_label, const double *bridge, double *out_features, double *out_beta);

/* ---- AdaBoost stumps (boosting.py:126-206) ------------------------------ */
/* xs [n*F] row-major features, betas [n] (y = +1 iff beta > 0), weights [n]
 * initial weights or NULL for 1/n.  BRM_MODE_PARITY replays numpy's
 * summation orders (sequential cumsum, pairwise sum) and the reference tie
 * rules.  flags BRM_FIT_SINGLE_STUMP: one fit_stump search (boosting.py:
 * 126-171) with the given weights, no boosting rules.  Outputs sized
 * [rounds]; *out_count stumps picked; out_err the weighted error of each;
 * *out_intercept the ensemble intercept.  stream: cudaStream_t or NULL.
 * flags BRM_FIT_DEVICE_RESULT: every output (count and intercept included)
 * is a device pointer, the stump arrays are written in full ([rounds],
 * entries past *out_count unspecified) and the call returns without
 * synchronising: results are ordered on `stream`.  out_n_pos (may be NULL;
 * host or device) receives the number of positive labels, the report's
 * positive_fraction * n (boundary_cmc.py:275).
 * Parity mode runs the split search's cumsums as a block-parallel exact
 * scan (integer adds inside a binade, one fp64 add per binade crossing), one
 * CTA per feature and one grid barrier per round; the column sort is an own
 * bitonic + merge-path kernel. */
#define BRM_FIT_SINGLE_STUMP 1
#define BRM_FIT_DEVICE_RESULT 2
int brm_fit_ensemble(int32_t device, int32_t mode, int32_t flags, void *stream, const double *xs,
                     const double *betas, const double *weights, int64_t n, int32_t F, int32_t rounds,
                     int32_t *out_feat, double *out_thr, double *out_pol, double *out_alpha, double *out_err,
                     int32_t *out_count, double *out_intercept, int32_t *out_n_pos);

/* Column sort of a DEVICE feature matrix ahead of its fit, ordered on `stream`
 * (any stream): a later brm_fit_ensemble on the same xs / n / F waits for it
 * and skips its own transpose and sort -- same sorted columns, same stumps.
 * brm_ctx_set_presort(ctx, 1) makes brm_cmc_calc do this for the points it
 * samples, on a high-priority side stream beside the label walk (the sort
 * needs only the features, boundary_cmc.py:264-271).  An unused sort is
 * dropped by the next presort of that matrix (at most 4 are kept). */
int brm_fit_presort(int32_t device, void *stream, const double *xs, int64_t n, int32_t F);
int brm_ctx_set_presort(brm_ctx *ctx, int32_t on);

/* ---- Device-resident I&Z date step (boundary_iz.py:328-357) ------------- */
/* Fit date m's boundary surface(s) on the device and write them into the
 * context's rule image, ordered on the context's stream (no host round trip:
 * the next, earlier date's brm_iz_solve on the same context uses them).
 * design [J*nb] row-major quadratic basis of k_coords coordinates (host or
 * device); levels [n_fits*J] (host or device; their logs for a log-space
 * surface); n_fits = d for price surfaces (fit g is asset g's surface), 1 for
 * the log-space surface (written to every row).  Rank-deficient designs fall
 * back to the cross-term-free basis as brm_lstsq.  out_coeffs [n_fits*nb] and
 * out_rank [n_fits] are optional (NULL), host or device. */
int brm_iz_fit(brm_ctx *ctx, int32_t m, const double *design, int32_t J, int32_t nb, int32_t k_coords,
               const double *levels, int32_t n_fits, int32_t log_space, double *out_coeffs, int32_t *out_rank);

/* ---- Quadratic boundary regression (boundary_iz.py:250-276) ------------- */
/* Least squares over the design [n*nb] (row-major), fp64 Householder QR with
 * column pivoting on the device; rank-deficient designs fall back to the
 * cross-term-free basis over k coordinates (zeros in dropped columns) and set
 * *out_rank_deficient. */
int brm_lstsq(int32_t device, void *stream, const double *design, const double *levels, int64_t n, int32_t nb,
              int32_t k_coords, double *out_coeffs, int32_t *out_rank_deficient);

/* ---- Launch accounting (bench.py) -------------------------------------- */
/* Kernel families: 0 walker (pricing / labels / stopped_sums), 1 probe
 * clusters, 2 AdaBoost, 3 sampler, 4 unit fold, 5 lstsq, 6 RNG fills,
 * 7 decisions, 8 auxiliary.  Launches are always counted; with profiling
 * enabled every launch is bracketed by CUDA events on its stream.
 * path_steps counts path-steps executed by walker / probe kernels. */
enum brm_prof_kind { BRM_PROF_WALK = 0, BRM_PROF_IZ = 1, BRM_PROF_BOOST = 2, BRM_PROF_SAMPLE = 3,
                     BRM_PROF_FINISH = 4, BRM_PROF_LSTSQ = 5, BRM_PROF_RNG = 6, BRM_PROF_DEC = 7,
                     BRM_PROF_AUX = 8, BRM_PROF_KINDS = 9 };
int brm_profile_enable(int32_t on);
int brm_profile_reset(void);
int brm_profile_read(int32_t kind, double *ms, uint64_t *launches, uint64_t *path_steps);
/* Host<->device bytes staged by the library since the last brm_profile_reset. */
int brm_transfer_read(uint64_t *h2d_bytes, uint64_t *d2h_bytes);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* BERMUDA_B200_H */
