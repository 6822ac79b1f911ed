// brm_walk.cuh -- the lane-refilling path walker shared by every kernel.
//
// A CTA walks the paths [p0, p1) of one work unit (a pricing block, a CMC
// training point, one I&Z probe iteration).  Each lane walks one path at a
// time; when its path stops (or expires) the lane writes the discounted value
// into shared memory at the path's slot and takes the next unclaimed path
// from a CTA-wide counter (one atomic per warp per refill), so lanes never
// idle behind a long path of a warp-mate.  Because values land at their path
// slot, the chunk's (sum, sum of squares) is then folded in a fixed order and
// is bit-identical run to run whatever the lane schedule was.
#pragma once
#include "brm_model.cuh"

namespace brm {

struct NormalSrc {
  const double *ptr;  // supplied normals (fixed-input mode) or nullptr
  uint64_t base, count;
};

// This warp's slice of the CTA's AS241 tail queue (parity mode).
struct TailQueue {
  double *buf;
  unsigned short *idx;
};

__device__ __forceinline__ double supplied_normal(const NormalSrc &s, uint64_t idx) {
  const uint64_t off = idx - s.base;
  return off < s.count ? s.ptr[off] : __longlong_as_double(0x7ff8000000000000LL);
}

// Fast mode: steps are call-aligned, dp = d rounded up to a multiple of 4.
__host__ __device__ __forceinline__ int fast_dp(int d) { return (d + 3) & ~3; }

template <bool FAST>
using RealT = typename std::conditional<FAST, float, double>::type;

// Draws of step k of a path: parity indices base + k*d + a (reference
// _core.pyx:4-7); fast positions pos + k*dp + a.
template <int D, bool FAST, bool EVEN = false>
__device__ __forceinline__ void path_step_draws(int d, const PhiloxKey &K, uint64_t base, int k,
                                                const NormalSrc &ns, RealT<FAST> *z, bool active,
                                                const TailQueue &tq) {
  if (ns.ptr) {
    const uint64_t idx0 = base + (uint64_t)k * (uint64_t)d;
#pragma unroll
    for (int a = 0; a < dim_of<D>(d); ++a) z[a] = (RealT<FAST>)supplied_normal(ns, idx0 + a);
    return;
  }
  if constexpr (FAST) {
    step_draws_fast<D>(K, base + (uint64_t)k * (uint64_t)fast_dp(d), z, d);
  } else if constexpr (D > 0) {
    step_draws_compact<D, EVEN>(K, base + (uint64_t)k * (uint64_t)d, z, active, tq.buf, tq.idx);
  } else {
    step_draws<D>(K, base + (uint64_t)k * (uint64_t)d, z, d);
  }
}

// Stride (in draw indices / positions) between consecutive paths of a unit.
template <bool FAST>
__host__ __device__ __forceinline__ uint64_t path_stride(int d, int n_steps, bool supplied) {
  if (FAST && !supplied) return (uint64_t)n_steps * (uint64_t)fast_dp(d);
  return (uint64_t)n_steps * (uint64_t)d;
}

// First draw index / position of a unit that starts at parity draw_base.
// Fast mode starts at the first Philox call not touched by parity draws
// [0, draw_base), so sampler draws and path draws never share a counter.
template <bool FAST>
__host__ __device__ __forceinline__ uint64_t unit_base(uint64_t draw_base, bool supplied) {
  if (FAST && !supplied) return 4 * ((draw_base + 1) / 2);  // first call past the parity draws, call-aligned
  return draw_base;
}

// Walk paths [p0, p1) of one unit from the shared start state.  *s_next must
// hold p0 + blockDim.x (set by the caller, followed by __syncthreads()).
// Geometric put in fp64 (GEO kernels): the step's log prices, formed once
// with the straight-line log (CUDA's log bits for the positive normal prices
// a walk produces), feed both the geometric mean -- the same sequential sum,
// divide and exp as aggregate() -- and a log-space I&Z surface.
template <int D>
__device__ __forceinline__ double geo_payoff(const Model<double> &M, const double *v, double &agg, double *lv) {
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    lv[i] = (v[i] >= 0x1p-1022 && v[i] < 0x1p1023) ? log_nb(v[i]) : log(v[i]);
    s = __dadd_rn(s, lv[i]);
  }
  agg = exp_nb(__ddiv_rn(s, (double)D));
  const double p = __dsub_rn(M.strike, agg);
  return p > 0.0 ? p : 0.0;
}

// Specialised steps (each instance launched only for its payoff / rule; code
// a kernel never runs still costs registers and instruction cache):
// WALK_GEO: the geometric put (geo_payoff); WALK_CMC: a CMC rule (the
// labels and pricing of C3-C5); WALK_CMC_UNIT: the max-call payoff under a
// CMC rule with independent assets (unit diagonal factor: C3, C5);
// WALK_CMC_LOWER: fast mode, CMC rule, lower-triangular factor (C4);
// WALK_CMC_LOG: WALK_CMC_UNIT's case in parity mode with the state kept as
// log-prices (brm_walk_log.cuh).
// WALK_CMC_COLCONST: WALK_CMC_LOWER's case with a column-constant factor
// (fast_step_colconst, brm_model.cuh): equicorrelated assets (C4).
enum { WALK_GENERIC = 0, WALK_GEO = 1, WALK_CMC = 2, WALK_CMC_UNIT = 3, WALK_CMC_LOWER = 4, WALK_CMC_LOG = 5,
       WALK_CMC_COLCONST = 6 };

template <int D, bool FAST, int SPEC = WALK_GENERIC>
__device__ void walk_paths(const Model<RealT<FAST>> &M, const RealT<FAST> *s_start, int m_start, int n_steps,
                           uint64_t key, uint64_t stream, uint64_t base0, int p0, int p1, const NormalSrc &ns,
                           double *vals, int *s_next, double *path_out, int32_t *stop_out,
                           unsigned long long *step_count, const TailQueue &tq,
                           [[maybe_unused]] const float4 *cc_rows = nullptr) {
  using R = RealT<FAST>;
  const int d = dim_of<D>(M.d);
  const uint64_t stride = path_stride<FAST>(d, n_steps, ns.ptr != nullptr);
  const unsigned lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  constexpr int NV = D > 0 ? D : kMaxD;
  const PhiloxKey K = philox_key(key, stream);
  R v[NV], z[NV];

  unsigned nsteps = 0;
  int p = p0 + threadIdx.x;
  bool have = p < p1;
  int k = 0;
  uint64_t base = base0 + (uint64_t)(have ? p : 0) * stride;
#pragma unroll
  for (int i = 0; i < dim_of<D>(d); ++i) v[i] = s_start[i];

  while (__any_sync(0xffffffffu, have)) {
    bool done = false;
    double val = 0.0;
    int stop_m = 0;
    // draws are generated by the whole warp (the tail pass is warp-cooperative);
    // lanes without a path draw at a valid dummy index and discard the result
    constexpr bool kFused = FAST && D > 0;
    // full (non-triangular) factor: generic step
    const bool fused = SPEC == WALK_CMC_COLCONST || (kFused && !ns.ptr && M.chol_lower != 0);
    // the CMC instances are launched only with even draw bases (host check)
    constexpr bool kCmc = SPEC == WALK_CMC || SPEC == WALK_CMC_UNIT || SPEC == WALK_CMC_LOWER ||
                          SPEC == WALK_CMC_COLCONST;
    if (!fused) path_step_draws<D, FAST, kCmc && D % 2 == 0>(d, K, base, k, ns, z, have, tq);
    if (have) {
      ++nsteps;
      if constexpr (SPEC == WALK_CMC_COLCONST && FAST && D > 0) {
        fast_step_colconst<(D > 0 ? D : 1)>(cc_rows, v, K, base + (uint64_t)k * (uint64_t)fast_dp(D));
      } else if constexpr (SPEC == WALK_CMC_LOWER && FAST && D > 0) {
        fast_step_fused<(D > 0 ? D : 1), true>(M, v, K, base + (uint64_t)k * (uint64_t)fast_dp(D));
      } else if constexpr (SPEC == WALK_CMC_UNIT && FAST && D > 1) {
        fast_step_unit<(D > 1 ? D : 2)>(reinterpret_cast<const float2 *>(cc_rows), v, K,
                                        base + (uint64_t)k * (uint64_t)fast_dp(D));
      } else if constexpr (SPEC == WALK_CMC_UNIT && FAST && D > 0) {
        fast_step_diag<(D > 0 ? D : 1)>(M, v, K, base + (uint64_t)k * (uint64_t)fast_dp(D));
      } else if constexpr (SPEC == WALK_CMC_UNIT && !FAST) {
        // y_i = 0 + 1.0 * z_i == z_i exactly (gbm_step's unit-diagonal branch)
#pragma unroll
        for (int i = 0; i < dim_of<D>(d); ++i) v[i] = r_mul(v[i], r_exp(r_add(M.mu[i], r_mul(M.vol[i], z[i]))));
      } else if constexpr (kFused) {
        if (!fused) gbm_step<D>(M, v, z);
        else fast_step_fused<(D > 0 ? D : 1)>(M, v, K, base + (uint64_t)k * (uint64_t)fast_dp(D));
      } else {
        gbm_step<D>(M, v, z);
      }
      const int m = m_start + k + 1;
      R agg;
      bool stop;
      R pay;
      if constexpr (SPEC == WALK_CMC_UNIT && D > 1) {
        // max-call payoff under the CMC rule (aggregate's max: strict >, first
        // maximum; written out for fp32, where it schedules better)
        if constexpr (FAST) {
          agg = v[0];
#pragma unroll
          for (int i = 1; i < D; ++i)
            if (v[i] > agg) agg = v[i];
        } else {
          agg = aggregate<D>(M, v);
        }
        pay = r_sub(agg, M.strike);
        pay = pay > (R)0 ? pay : (R)0;
        stop = pay > (R)0 && (m == M.n_dates || cmc_stop<D>(M, m, v, agg));
      } else if constexpr (kCmc && D > 1) {
        // rule_stop's CMC branch only (no I&Z surface code in the kernel)
        pay = payoff_agg<D>(M, v, agg);
        stop = pay > (R)0 && (m == M.n_dates || cmc_stop<D>(M, m, v, agg));
      } else if constexpr (SPEC == WALK_GEO && !FAST && D > 1) {
        R lv[D > 1 ? D : 1];
        pay = geo_payoff<D>(M, v, agg, lv);
        stop = pay > (R)0 && (m == M.n_dates || (M.rule == RULE_IZ ? iz_stop<D>(M, m, v, lv)
                                                                  : rule_stop<D>(M, m, v, agg)));
      } else {
        pay = payoff_agg<D>(M, v, agg);
        stop = pay > (R)0 && rule_stop<D>(M, m, v, agg);
      }
      if (stop) {
        val = (double)pay * M.disc[m - m_start];
        stop_m = m;
        done = true;
      } else if (k + 1 == n_steps) {
        done = true;
      } else {
        ++k;
      }
    }
    if (done) {
      vals[p - p0] = val;
      if (path_out) path_out[p] = val;
      if (stop_out) stop_out[p] = stop_m;
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
        for (int i = 0; i < dim_of<D>(d); ++i) v[i] = s_start[i];
      }
    }
  }
  if (step_count) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) nsteps += __shfl_down_sync(0xffffffffu, nsteps, off);
    if (lane == 0 && nsteps) atomicAdd(step_count, (unsigned long long)nsteps);
  }
}

// Fixed-order fold of vals[0..n) into (sum, sumsq); result valid in thread 0.
// Thread t folds a contiguous run, then a shuffle tree and a warp-order pass.
__device__ inline void fold_values(const double *vals, int n, double *s_red, double &sum, double &sumsq) {
  const int nt = blockDim.x;
  const int per = (n + nt - 1) / nt;
  const int lo = threadIdx.x * per;
  const int hi = min(lo + per, n);
  double s = 0.0, q = 0.0;
  for (int i = lo; i < hi; ++i) {
    const double x = vals[i];
    s = __dadd_rn(s, x);
    q = __dadd_rn(q, __dmul_rn(x, x));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, off));
    q = __dadd_rn(q, __shfl_down_sync(0xffffffffu, q, off));
  }
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_red[2 * warp] = s;
    s_red[2 * warp + 1] = q;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    s = 0.0;
    q = 0.0;
    for (int w = 0; w < (nt + 31) / 32; ++w) {
      s = __dadd_rn(s, s_red[2 * w]);
      q = __dadd_rn(q, s_red[2 * w + 1]);
    }
    sum = s;
    sumsq = q;
  }
}

}  // namespace brm
