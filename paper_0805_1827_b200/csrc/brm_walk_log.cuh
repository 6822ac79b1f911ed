// brm_walk_log.cuh -- the log-price walker instances, parity draws in fp64:
//   LOG_MAXCALL_CMC  max-call payoff, CMC rule, independent assets (C3 / C5;
//                    walk_units<.., WALK_CMC_LOG>)
//   LOG_GEOPUT_IZ    geometric-average put, I&Z log-space surface, independent
//                    assets (the probe clusters of C2; iz_probes<.., 2>)
//
// The reference's _path_value (_core.pyx:290-323) steps prices,
// v_i <- v_i * exp(mu_i + vol_i z_i), and needs d exponentials per step.  For
// this payoff and rule nothing on the path needs the prices themselves:
//   * the max-call payoff is max_i v_i - K, and max_i v_i = exp(max_i x_i)
//     for x_i = log v_i, so "payoff > 0" is x_max > log K and the payoff value
//     is needed once per path, at the stop date;
//   * a stump asks v_f > t, which is x_f > log t (the derived feature
//     max_i v_i likewise), so the rule's step functions are searched over
//     log-thresholds (build_log_tables, brm_model.cuh).
// The state therefore is the log-price, x_i <- x_i + (mu_i + vol_i z_i): two
// fp64 operations per asset-step where the price step costs ~20, and one
// exponential per path.  Draws are the reference's (Philox + AS241, the same
// draw indices), so the log-prices differ from the logs of the reference's
// prices only by rounding (a few 1e-16 relative in the price; the K-scaled
// 1e-12 parity tolerance of DESIGN.md section 4 holds with three orders of
// margin), and a decision can differ only for a state within that rounding of
// a threshold -- the same caveat the price stepper already carries, because
// CUDA's exp and glibc's differ in the last bit.
//
// Exactness guards: "in the money" within 1e-13 of log K and stump scores
// inside the rounding bound bound[m] are decided in price space from
// exp(x) (rare branches), so the decision is the price-space decision of the
// state exp(x) whenever the cheap test cannot be trusted.
//
// A stopped path leaves (x_max, stop date) in its shared-memory slot; the
// payoff (exp(x_max) - K) disc is formed afterwards by all lanes of the CTA
// (finish_log_values) instead of by the two or three lanes of a warp that
// stop in a given step.
//
// The geometric put needs even less: its payoff K - exp(mean_i x_i) and its
// log-space boundary surface (x_d against a quadratic in the other x_j) are
// functions of the log-prices, so the price stepper's d exponentials and d
// logarithms per step become one exponential per stopped path.
#pragma once
#include "brm_walk.cuh"

namespace brm {

// Stump score of the state exp(x) in stump order (the reference's sequential
// sum, _core.pyx:271-287); reached only when the table sum is inside bound[m]
// or the search trees did not fit in shared memory.
template <int D>
__device__ __forceinline__ bool cmc_stop_exact_log(const Model<double> &M, int m, const double *x, double xmax) {
  double v_of[D + 1];
#pragma unroll
  for (int i = 0; i < D; ++i) v_of[i] = exp_nb(x[i]);
  v_of[D] = exp_nb(xmax);
  double s = M.icept[m];
  const int t0 = M.starts[m], t1 = t0 + M.counts[m];
  for (int t = t0; t < t1; ++t) {
    const double v = v_of[M.feat[t]];
    s = v > M.thr[t] ? r_add(s, M.ap[t]) : r_sub(s, M.ap[t]);
  }
  return s > 0.0;
}

__device__ __forceinline__ double lds_f64(unsigned addr) {
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

// One level of a search tree: a <- 2 a + k + 8 [t < x] (k = 8 - tree base),
// the comparison as a predicated add (three instructions with the load).
__device__ __forceinline__ unsigned tree_step(unsigned a, unsigned k, double t, double x) {
  unsigned na = 2u * a + k;
  asm("{ .reg .pred p; setp.lt.f64 p, %1, %2; @p add.u32 %0, %0, 8; }" : "+r"(na) : "d"(t), "d"(x));
  return na;
}

// Stump score through the per-feature search trees (build_log_tables): D + 1
// branch-free searches in lock-step, then a pairwise sum.  The sum is in a
// different order than the reference's, so it decides only outside the
// rounding bound bound[m] (see cmc_stop, brm_model.cuh).
template <int D>
__device__ __forceinline__ bool cmc_stop_log(const Model<double> &M, int m, const double *x, double xmax) {
  if (M.lt_base == 0) return cmc_stop_exact_log<D>(M, m, x, xmax);  // uniform
  constexpr int FN = D + 1;
  // a[f]: byte address of the current node; a <- 2a + (8 - base) + 8 [node < x]
  unsigned a[FN], kf[FN];
  const unsigned date = M.lt_base + (unsigned)(m - 1) * (unsigned)M.lt_date;
#pragma unroll
  for (int f = 0; f < FN; ++f) {
    a[f] = date + (unsigned)f * (unsigned)M.lt_s1;
    kf[f] = 8u - a[f];
  }
  const int dmin = min(M.lt_d1, M.lt_d2);
#pragma unroll 1
  for (int l = 0; l < dmin; ++l) {
    double t[FN];
#pragma unroll
    for (int f = 0; f < FN; ++f) t[f] = lds_f64(a[f]);
#pragma unroll
    for (int f = 0; f < FN; ++f) a[f] = tree_step(a[f], kf[f], t[f], f < D ? x[f < D ? f : 0] : xmax);
  }
#pragma unroll 1
  for (int l = dmin; l < M.lt_d1; ++l) {  // deeper asset trees
    double t[D];
#pragma unroll
    for (int f = 0; f < D; ++f) t[f] = lds_f64(a[f]);
#pragma unroll
    for (int f = 0; f < D; ++f) a[f] = tree_step(a[f], kf[f], t[f], x[f]);
  }
#pragma unroll 1
  for (int l = dmin; l < M.lt_d2; ++l)  // deeper derived-feature tree
    a[D] = tree_step(a[D], kf[D], lds_f64(a[D]), xmax);
  double val[FN];
#pragma unroll
  for (int f = 0; f < FN; ++f) val[f] = lds_f64(a[f]);
#pragma unroll
  for (int w = 1; w < FN; w <<= 1)
#pragma unroll
    for (int f = 0; f + w < FN; f += 2 * w) val[f] = r_add(val[f], val[f + w]);
  const double s = r_add(M.icept[m], val[0]);
  const double B = M.bound[m];
  if (s > B) return true;
  if (s < -B) return false;
  return cmc_stop_exact_log<D>(M, m, x, xmax);
}

// Parity draws of one step, consumed group by group: after a group's normals
// are final (central branch per lane, tail draws through the warp queue, as
// step_draws_compact) the log-prices of the group's assets step at once, so
// only one group of normals is live.  Queue slots come from one ballot per
// draw (the rank of the lane among the lanes whose draw is a tail draw).
// inc (optional): the step's increments mu_i + vol_i z_i, for the draw cache
// of the bisection probes (iz_probes, brm_kernels.cuh).
template <int D, bool EVEN>
__device__ __forceinline__ void step_log_prices(const Model<double> &M, const PhiloxKey &K, uint64_t idx0, double *x,
                                                bool active, double *wbuf, unsigned short *widx, unsigned lt_mask,
                                                double *inc = nullptr) {
  constexpr int NC = EVEN ? D / 2 : D / 2 + 1;
  constexpr int G = TailGroup<D>::G;
  static_assert(D % G == 0, "the log-price walker steps whole draw groups");
  const uint64_t c0 = idx0 >> 1;
  const bool odd = EVEN ? false : (idx0 & 1);
  const int ncalls = EVEN ? NC : (int)(((idx0 + D - 1) >> 1) - c0) + 1;
  double z[D];
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    if (j < ncalls) {
      const Philox4 p = philox(K, c0 + j);
      const double u0 = uniform_x2(philox_word(p, 0)), u1 = uniform_x2(philox_word(p, 1));
      if (2 * j < D) z[2 * j] = odd ? u1 : u0;
      if (2 * j + 1 < D && !odd) z[2 * j + 1] = u1;
      if (j > 0 && 2 * j - 1 < D && odd) z[2 * j - 1] = u0;
    }
  }
  const unsigned lane = threadIdx.x & 31;
#pragma unroll
  for (int g0 = 0; g0 < D; g0 += G) {
    bool tail[G];
    int total = 0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const double q = fma(z[g0 + g], 0x1p-54, -0.5);
      const bool central = fabs(q) <= 0.425;
      tail[g] = !central && active;
      const double c = as241_central(q);
      if (central) z[g0 + g] = c;
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const unsigned mask = __ballot_sync(0xffffffffu, tail[g]);
      if (tail[g]) {
        const int slot = lane * G + g;
        wbuf[slot] = z[g0 + g];
        widx[total + __popc(mask & lt_mask)] = (unsigned short)slot;
      }
      total += __popc(mask);
    }
    if (total != 0) {
      __syncwarp();
      for (int j = lane; j < total; j += 32) {
        const int slot = widx[j];
        const double u = __dmul_rn(wbuf[slot], 0x1p-54);  // exact
        wbuf[slot] = as241_tail(u, __dsub_rn(u, 0.5));
      }
      __syncwarp();
#pragma unroll
      for (int g = 0; g < G; ++g)
        if (tail[g]) z[g0 + g] = wbuf[lane * G + g];
      __syncwarp();
    }
#pragma unroll
    for (int a = g0; a < g0 + G; ++a) {
      const double dx = fma(M.vol[a], z[a], M.mu[a]);
      if (inc) inc[a] = dx;
      x[a] = r_add(x[a], dx);
    }
  }
}

enum { LOG_MAXCALL_CMC = 0, LOG_GEOPUT_IZ = 1 };

// Log-space boundary decision of the geometric put (iz_stop's iz_space == 1
// branch, brm_model.cuh, on the state's own log-prices).
template <int D>
__device__ __forceinline__ double iz_surface_log(const Model<double> &M, int m, const double *x) {
  constexpr int k = D - 1;
  double w[k];
#pragma unroll
  for (int j = 0; j < k; ++j) w[j] = x[j] < M.izlo[j] ? M.izlo[j] : (x[j] > M.izhi[j] ? M.izhi[j] : x[j]);
  const double *row = M.izc + ((size_t)m * D + (D - 1)) * M.nbasis;
  return quad_surface<D>(row, w, k);
}

template <int D>
__device__ __forceinline__ bool iz_stop_log(const Model<double> &M, int m, const double *x) {
  return x[D - 1] <= iz_surface_log<D>(M, m, x);
}

// Decision of a path at date m in state x: true when it stops; xstop is then
// x_max (LOG_MAXCALL_CMC; the payoff is formed by finish_log_values) or the
// discounted payoff itself (LOG_GEOPUT_IZ).
template <int D, int KIND>
__device__ __forceinline__ bool log_state_stops(const Model<double> &M, double log_strike, int m, int m_start,
                                                const double *x, double &xstop) {
  if constexpr (KIND == LOG_GEOPUT_IZ) {
    // geometric mean in log space: the same sequential sum and divide as geo_payoff (brm_walk.cuh)
    double sx = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) sx = r_add(sx, x[i]);
    const double g = __ddiv_rn(sx, (double)D);
    const double dk = r_sub(log_strike, g);
    bool itm = dk > 0.0;
    if (fabs(dk) <= 1e-13) itm = r_sub(M.strike, exp_nb(g)) > 0.0;  // decide at the money in price space
    const bool stop = itm && (m == M.n_dates || iz_stop_log<D>(M, m, x));
    if (stop) xstop = r_mul(r_sub(M.strike, exp_nb(g)), M.disc[m - m_start]);
    return stop;
  } else {
    double xmax = x[0];
#pragma unroll
    for (int i = 1; i < D; ++i)
      if (x[i] > xmax) xmax = x[i];
    const double dk = r_sub(xmax, log_strike);
    bool itm = dk > 0.0;
    if (fabs(dk) <= 1e-13) itm = r_sub(exp_nb(xmax), M.strike) > 0.0;  // decide at the money in price space
    const bool stop = itm && (m == M.n_dates || cmc_stop_log<D>(M, m, x, xmax));
    if (stop) xstop = xmax;
    return stop;
  }
}

// Walk paths [p0, p1) of one unit from the shared start log-prices x_start
// (lane refill as walk_paths, brm_walk.cuh).
// RECORD (bisection probes of the geometric put, first pass): every path is
// stepped to expiry and leaves, per step, what the later passes need -- they
// differ from this one only in the start of the probed (last) asset:
//   rec[(k * rec_paths + p) * 3 + 0]  the last asset's increment mu + vol z
//   rec[... + 1]  the other assets' log-price sum, ((0 + x_0) + x_1) + ...
//                 (the leading part of geo_payoff's sequential sum)
//   rec[... + 2]  the boundary surface over the other assets' log-prices
//                 (+inf at expiry: any in-the-money path stops)
// (a plane per step, paths contiguous: a warp's replay loads are coalesced).
// The value is that of the path's first stop.  replay_geoput_log replays.
// LOG_MAXCALL_CMC: slot p - p0 of vals receives the stopped path's x_max and
// stopm its stop date (0: expired worthless); finish_log_values turns them
// into discounted payoffs.  LOG_GEOPUT_IZ: vals receives the discounted payoff
// itself (stopm unused; the probe clusters fold vals as they are).
template <int D, int KIND = LOG_MAXCALL_CMC, bool RECORD = false>
__device__ void walk_paths_log(const Model<double> &M, const double *x_start, double log_strike, int m_start,
                               int n_steps, uint64_t key, uint64_t stream, uint64_t base0, int p0, int p1,
                               double *vals, unsigned char *stopm, int *s_next, unsigned long long *step_count,
                               const TailQueue &tq, double *rec = nullptr, int rec_paths = 0) {
  static_assert(D > 1, "the log-price walkers are d > 1 instances");
  const uint64_t stride = (uint64_t)n_steps * (uint64_t)D;
  const unsigned lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const PhiloxKey K = philox_key(key, stream);
  double x[D];

  unsigned nsteps = 0;
  int p = p0 + threadIdx.x;
  bool have = p < p1;
  int k = 0;
  uint64_t base = base0 + (uint64_t)(have ? p : 0) * stride;
#pragma unroll
  for (int i = 0; i < D; ++i) x[i] = x_start[i];
  [[maybe_unused]] bool stopped = false;  // RECORD: the path's first stop is kept while it steps on
  [[maybe_unused]] double xkeep = 0.0;
  [[maybe_unused]] int mkeep = 0;

  while (__any_sync(0xffffffffu, have)) {
    bool done = false;
    double xstop = 0.0;
    int stop_m = 0;
    // the whole warp draws (the tail pass is warp-cooperative); lanes without
    // a path step a dummy state at a valid index and discard it
    [[maybe_unused]] double inc[D];
    step_log_prices<D, D % 2 == 0>(M, K, base + (uint64_t)k * (uint64_t)D, x, have, tq.buf, tq.idx, lt_mask,
                                   RECORD ? inc : nullptr);
    if (have) {
      ++nsteps;
      const int m = m_start + k + 1;
      if constexpr (RECORD) {
        static_assert(!RECORD || KIND == LOG_GEOPUT_IZ, "the draw cache is the geometric put's");
        double *dst = rec + ((size_t)k * rec_paths + p) * 3;
        double sa = 0.0;
#pragma unroll
        for (int i = 0; i < D - 1; ++i) sa = r_add(sa, x[i]);
        dst[0] = inc[D - 1];
        dst[1] = sa;
        dst[2] = m == M.n_dates ? __longlong_as_double(0x7ff0000000000000LL) : iz_surface_log<D>(M, m, x);
        if (!stopped && log_state_stops<D, KIND>(M, log_strike, m, m_start, x, xkeep)) {
          stopped = true;
          mkeep = m;
        }
        if (k + 1 == n_steps) {
          done = true;
          xstop = xkeep;
          stop_m = mkeep;
        } else {
          ++k;
        }
      } else if (log_state_stops<D, KIND>(M, log_strike, m, m_start, x, xstop)) {
        stop_m = m;
        done = true;
      } else if (k + 1 == n_steps) {
        done = true;
      } else {
        ++k;
      }
    }
    if (done) {
      vals[p - p0] = xstop;
      if constexpr (KIND == LOG_MAXCALL_CMC) stopm[p - p0] = (unsigned char)stop_m;
    }
    const unsigned need = __ballot_sync(0xffffffffu, done);
    if (need) {
      const int leader = __ffs(need) - 1;
      int got = 0;
      if ((int)lane == leader) got = atomicAdd(s_next, __popc(need));
      got = __shfl_sync(0xffffffffu, got, leader);
      if (done) {
        p = got + __popc(need & lt_mask);
        have = p < p1;
        k = 0;
        base = base0 + (uint64_t)(have ? p : 0) * stride;
#pragma unroll
        for (int i = 0; i < D; ++i) x[i] = x_start[i];
        if constexpr (RECORD) {
          stopped = false;
          xkeep = 0.0;
          mkeep = 0;
        }
      }
    }
  }
  if (step_count) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) nsteps += __shfl_down_sync(0xffffffffu, nsteps, off);
    if (lane == 0 && nsteps) atomicAdd(step_count, (unsigned long long)nsteps);
  }
}

// Bisection probes, passes after the first (common random numbers: every pass
// walks the same paths from another start state): path p's log-prices are
// x_start + the recorded increments, added in step order exactly as
// walk_paths_log adds them, so a replayed pass returns the bits a re-simulated
// pass would -- without drawing a single normal.  Paths are assigned to
// threads statically (a replayed path-step is ~80 instructions and a
// coalesced read of D doubles); vals as walk_paths_log.
// Bisection probes of the geometric put, passes after the first (common random
// numbers: every pass walks the same paths, from start states that differ in
// the probed asset only).  A thread replays its paths (static assignment) for
// n_cand candidate levels at once -- the midpoints of the next bisection
// levels -- from one read of the record: per step and candidate
//   xl += inc;  s = sa + xl;  g = s / D;  stop iff g < log K and xl <= b,
// the operations, in the order, of walk_paths_log's LOG_GEOPUT_IZ step, so a
// candidate's values are the bits a re-simulated pass would produce, without
// drawing a normal or evaluating a surface.  xl0[t]: the probed asset's start
// log-price of candidate t; vals[t * stride + (p - p0)] receives the values.
template <int D, int T>
__device__ __forceinline__ void replay_geoput_log(const Model<double> &M, double log_strike, int m_start, int n_steps,
                                                  const double *rec, int rec_paths, int p0, int p1, const double *xl0,
                                                  int n_cand, double *vals, int stride) {
  const size_t plane = (size_t)rec_paths * 3;
  for (int p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
    double xl[T], val[T];
    unsigned live = n_cand >= 32 ? 0xffffffffu : (1u << n_cand) - 1u;
#pragma unroll
    for (int t = 0; t < T; ++t) {
      xl[t] = xl0[t < n_cand ? t : 0];
      val[t] = 0.0;
    }
    const double *src = rec + (size_t)p * 3;
    double inc = __ldcg(src), sa = __ldcg(src + 1), b = __ldcg(src + 2);
    for (int k = 0; k < n_steps && live; ++k) {
      const double cinc = inc, csa = sa, cb = b;
      if (k + 1 < n_steps) {  // the next step's record is in flight while this one is decided
        inc = __ldcg(src + (size_t)(k + 1) * plane);
        sa = __ldcg(src + (size_t)(k + 1) * plane + 1);
        b = __ldcg(src + (size_t)(k + 1) * plane + 2);
      }
      // the T candidates are independent chains: straight-line code for the decisions (their
      // divides interleave), one branch for the rare at-the-money guard, one for the stops
      double g[T];
      unsigned stops = 0, near = 0;
#pragma unroll
      for (int t = 0; t < T; ++t) {
        xl[t] = r_add(xl[t], cinc);
        // (div_nb: __ddiv_rn's bits for normal operands -- a sum of log-prices over D; a sum
        // next to zero takes the guard's library path)
        const double sx = r_add(csa, xl[t]);
        g[t] = div_nb(sx, (double)D);
        const double dk = r_sub(log_strike, g[t]);
        near |= ((fabs(dk) <= 1e-13 || !(fabs(sx) >= 0x1p-1000)) ? 1u : 0u) << t;
        stops |= ((dk > 0.0 && xl[t] <= cb) ? 1u : 0u) << t;
      }
      near &= live;
      if (near) {
#pragma unroll
        for (int t = 0; t < T; ++t) {
          if ((near >> t) & 1u) {
            g[t] = __ddiv_rn(r_add(csa, xl[t]), (double)D);
            const double dk = r_sub(log_strike, g[t]);
            bool itm = dk > 0.0;
            if (fabs(dk) <= 1e-13) itm = r_sub(M.strike, exp_nb(g[t])) > 0.0;  // decide at the money in price space
            stops = (stops & ~(1u << t)) | ((itm && xl[t] <= cb) ? 1u << t : 0u);
          }
        }
      }
      stops &= live;
      if (stops) {
        const double disc = M.disc[k + 1];
#pragma unroll
        for (int t = 0; t < T; ++t)
          if ((stops >> t) & 1u) val[t] = r_mul(r_sub(M.strike, exp_nb(g[t])), disc);
        live &= ~stops;
      }
    }
#pragma unroll
    for (int t = 0; t < T; ++t)
      if (t < n_cand) vals[(size_t)t * stride + (p - p0)] = val[t];
  }
}

// (x_max, stop date) of every path of the chunk -> discounted payoff
// (exp(x_max) - K) disc[m - m_start] in place, and the optional per-path
// outputs.  All threads; the caller synchronises before and after.
__device__ __forceinline__ void finish_log_values(const Model<double> &M, int m_start, int p0, int n, double *vals,
                                                  const unsigned char *stopm, double *path_out, int32_t *stop_out) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int m = stopm[i];
    const double v = m ? r_mul(r_sub(exp_nb(vals[i]), M.strike), M.disc[m - m_start]) : 0.0;
    vals[i] = v;
    if (path_out) path_out[p0 + i] = v;
    if (stop_out) stop_out[p0 + i] = m;
  }
}

}  // namespace brm
