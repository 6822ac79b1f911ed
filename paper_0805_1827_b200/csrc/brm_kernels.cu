// brm_kernels.cu -- non-template kernels and the dimension dispatch.
#include "brm_kernels.cuh"

namespace brm {

// Fold each unit's chunk partials in chunk order.  mode 0: out[u] = (sum,
// sumsq); mode 1: pricing stats out[u] = (count, sum, sumsq); mode 2: CMC
// label out[u] = payoff(point_u) - sum / n_label (fp64, _core.pyx:548).
__global__ void finish_units(FinishParams P) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= P.n_units) return;
  double s = 0.0, q = 0.0;
  for (int c = 0; c < P.chunks_per_unit; ++c) {
    s = __dadd_rn(s, P.partials[2 * ((size_t)u * P.chunks_per_unit + c)]);
    q = __dadd_rn(q, P.partials[2 * ((size_t)u * P.chunks_per_unit + c) + 1]);
  }
  if (P.mode == 0) {
    P.out[2 * (size_t)u] = s;
    P.out[2 * (size_t)u + 1] = q;
  } else if (P.mode == 1) {
    const int64_t cnt64 = P.total_paths - (int64_t)u * P.per_unit;
    P.out[3 * (size_t)u] = (double)(cnt64 < P.per_unit ? cnt64 : P.per_unit);
    P.out[3 * (size_t)u + 1] = s;
    P.out[3 * (size_t)u + 2] = q;
  } else {
    Model<double> M{};
    M.d = P.d;
    M.payoff = P.payoff;
    M.strike = P.strike;
    const double *x = P.points + (size_t)u * P.points_stride;
    P.out[u] = __dsub_rn(payoff<0>(M, x), __ddiv_rn(s, (double)P.per_unit));
  }
}

// --------------------------------------------------------- training points ----
// mode 0: terminal GBM draw over [0, T] (draws 0..d-1) then the Brownian
// bridge to t_m (draws d..2d-1) exactly as boundary_cmc.py:164-177 with
// market.py:180-220 (z @ L^T summed over a in order); mode 1: forward steps
// over dates 1..m with the walker's step and parity draws k*d + a.
// Derived classifier feature x[d] (boundary_cmc.py:38-52 for the max-call).
__device__ inline void write_aggregate(const SampleParams &P, double *x) {
  if (P.out_stride <= P.d) return;
  Model<double> M{};
  M.d = P.d;
  M.payoff = P.payoff;
  x[P.d] = aggregate<0>(M, x);
}

__global__ void sample_points(SampleParams P) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  const int d = P.d;
  uint64_t key, stream;
  derive_words(P.seed, 2 /* CMC_CALC */, (uint64_t)(P.item_lo + i), (uint64_t)P.m, key, stream);
  double *x = P.out + i * P.out_stride;
  const double *L = P.chol;
  if (P.mode == 1) {
    double v[kMaxD], z[kMaxD];
    for (int a = 0; a < d; ++a) v[a] = P.s0[a];
    for (int k = 0; k < P.m; ++k) {
      for (int a = 0; a < d; ++a) z[a] = normal_at(key, stream, (uint64_t)k * d + a);
      for (int r = 0; r < d; ++r) {
        double y = 0.0;
        for (int a = 0; a < d; ++a)
          if (L[r * d + a] != 0.0) y = __dadd_rn(y, __dmul_rn(L[r * d + a], z[a]));
        v[r] = __dmul_rn(v[r], exp(__dadd_rn(P.step_mu[r], __dmul_rn(P.step_vol[r], y))));
      }
    }
    for (int a = 0; a < d; ++a) x[a] = v[a];
    write_aggregate(P, x);
    return;
  }
  const double *drift_T = P.bridge, *sig_sqrt_T = P.bridge + d, *log_s0 = P.bridge + 2 * d;
  const double *bsd = P.bridge + 3 * d;
  const double lam = P.bridge[4 * d];
  double term[kMaxD];
  for (int r = 0; r < d; ++r) {
    double y = 0.0;
    for (int a = 0; a < d; ++a)
      if (L[r * d + a] != 0.0) y = __dadd_rn(y, __dmul_rn(normal_at(key, stream, (uint64_t)a), L[r * d + a]));
    term[r] = __dmul_rn(P.s0[r], exp(__dadd_rn(drift_T[r], __dmul_rn(sig_sqrt_T[r], y))));
  }
  if (P.m == P.n_dates) {
    for (int r = 0; r < d; ++r) x[r] = term[r];
    write_aggregate(P, x);
    return;
  }
  const double one_m_lam = __dsub_rn(1.0, lam);
  for (int r = 0; r < d; ++r) {
    double y = 0.0;
    for (int a = 0; a < d; ++a)
      if (L[r * d + a] != 0.0) y = __dadd_rn(y, __dmul_rn(normal_at(key, stream, (uint64_t)(d + a)), L[r * d + a]));
    const double lm = __dadd_rn(__dadd_rn(__dmul_rn(one_m_lam, log_s0[r]), __dmul_rn(lam, log(term[r]))),
                                __dmul_rn(bsd[r], y));
    x[r] = exp(lm);
  }
  write_aggregate(P, x);
}

// ------------------------------------------------------------------ RNG ----
__global__ void fill_raw(uint64_t key, uint64_t stream, uint64_t start, int64_t count, uint64_t *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t idx = start + (uint64_t)i;
    out[i] = philox_word(philox(key, stream, idx >> 1), (int)(idx & 1));
  }
}

__global__ void fill_normals(uint64_t key, uint64_t stream, uint64_t start, int64_t count, double *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = normal_at(key, stream, start + (uint64_t)i);
}

// Math self-test: the branch-free exp / divide / log / sqrt against the library functions.
__global__ void math_selftest(int kind, const double *a, const double *b, int64_t n, double *out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  switch (kind) {
    case 0: out[i] = exp_nb(a[i]); break;
    case 1: out[i] = exp(a[i]); break;
    case 2: out[i] = div_nb(a[i], b[i]); break;
    case 3: out[i] = __ddiv_rn(a[i], b[i]); break;
    case 4: out[i] = log_nb(a[i]); break;
    case 5: out[i] = log(a[i]); break;
    case 6: out[i] = sqrt_nb(a[i]); break;
    default: out[i] = __dsqrt_rn(a[i]); break;
  }
}

// ---------------------------------------------------------- dispatch tables ----
KernelTriple kernels_d0(bool fast);
KernelTriple kernels_d1(bool fast);
KernelTriple kernels_d2(bool fast);
KernelTriple kernels_d3(bool fast);
KernelTriple kernels_d5(bool fast);
KernelTriple kernels_d10(bool fast);
KernelTriple kernels_d40(bool fast);

KernelTriple kernels_for(int d, bool fast) {
  switch (d) {
    case 1: return kernels_d1(fast);
    case 2: return kernels_d2(fast);
    case 3: return kernels_d3(fast);
    case 5: return kernels_d5(fast);
    case 10: return kernels_d10(fast);
    case 40: return kernels_d40(fast);
    default: return kernels_d0(fast);
  }
}

// ---- device-side ensemble upload (slotted CMC images) --------------------
// Double-double accumulation for the step-table values: the host build sums
// in long double; either is far inside the rounding bound that guards the
// table decision (cmc_stop), so decisions stay exact.
struct DD {
  double hi, lo;
};
__device__ __forceinline__ DD dd_add(DD a, DD b) {
  const double s = __dadd_rn(a.hi, b.hi), bb = __dsub_rn(s, a.hi);
  double e = __dadd_rn(__dsub_rn(a.hi, __dsub_rn(s, bb)), __dsub_rn(b.hi, bb));
  const double t = __dadd_rn(a.lo, b.lo), bt = __dsub_rn(t, a.lo);
  const double f = __dadd_rn(__dsub_rn(a.lo, __dsub_rn(t, bt)), __dsub_rn(b.lo, bt));
  e = __dadd_rn(e, t);
  double hi = __dadd_rn(s, e);
  e = __dsub_rn(e, __dsub_rn(hi, s));
  e = __dadd_rn(e, f);
  const double h2 = __dadd_rn(hi, e);
  return DD{h2, __dsub_rn(e, __dsub_rn(h2, hi))};
}

// Writes date m's ensemble (count and intercept read on the device) into its
// slot: stumps, the per-feature sorted thresholds padded with +inf to a power
// of two minus one, the step-table values and the rounding bound -- the same
// image brm_ctx_create builds on the host (brm_capi.cu).
__global__ void __launch_bounds__(256) set_ensemble(unsigned char *blob, ModelHdr h, int m, int R, SlotDims slot,
                                                    const int32_t *feat, const double *thr, const double *pol,
                                                    const double *alpha, const int32_t *count,
                                                    const double *intercept) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *s_thr = reinterpret_cast<double *>(smem_raw);
  double *s_ap = s_thr + R;
  double *s_hi = s_ap + R;               // [8][R] per-warp rank sums (double-double)
  double *s_lo = s_hi + 8 * R;
  int *s_feat = reinterpret_cast<int *>(s_lo + 8 * R);
  int *s_rank = s_feat + R;              // rank r among the feature's distinct thresholds (-1-r: repeat)
  int *s_first = s_rank + R;
  __shared__ int s_u[kMaxD + 1], s_toff[kMaxD + 1], s_voff[kMaxD + 1], s_p[kMaxD + 1];
  double *gd = reinterpret_cast<double *>(blob);
  int32_t *gi = reinterpret_cast<int32_t *>(blob + 8 * (size_t)h.n_dbl);
  const int F = h.nfeat;
  const int c = max(0, min(*count, R));
  const double ic = *intercept;
  for (int t = threadIdx.x; t < c; t += blockDim.x) {
    s_thr[t] = thr[t];
    s_ap[t] = __dmul_rn(alpha[t], pol[t]);  // the product the reference forms per vote
    s_feat[t] = feat[t];
  }
  for (int f = threadIdx.x; f < F; f += blockDim.x) s_u[f] = 0;
  __syncthreads();
  // distinct thresholds per feature (first occurrence in stump order) and
  // their ranks (c <= R stumps: O(c^2) compares)
  for (int t = threadIdx.x; t < c; t += blockDim.x) {
    const int f = s_feat[t];
    const double x = s_thr[t];
    bool first = true;
    for (int q = 0; q < t && first; ++q) first = !(s_feat[q] == f && s_thr[q] == x);
    s_first[t] = first;
    if (first) atomicAdd(&s_u[f], 1);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < c; t += blockDim.x) {
    const int f = s_feat[t];
    const double x = s_thr[t];
    int r = 0;
    for (int q = 0; q < c; ++q) r += s_first[q] && s_feat[q] == f && s_thr[q] < x;
    s_rank[t] = s_first[t] ? r : -1 - r;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int to = m * slot.ts, vo = m * slot.vs;
    for (int f = 0; f < F; ++f) {
      int P = 1;
      while (P < s_u[f] + 1) P <<= 1;
      s_p[f] = P;
      s_toff[f] = to;
      s_voff[f] = vo;
      gi[h.o_toff + m * F + f] = to;
      gi[h.o_tcnt + m * F + f] = P;
      gi[h.o_voff + m * F + f] = vo;
      to += P - 1;
      vo += s_u[f] + 1;
    }
    gi[h.o_counts + m] = c;
    gd[h.o_icept + m] = ic;
    double absum = fabs(ic);
    for (int t = 0; t < c; ++t) absum = __dadd_rn(absum, fabs(s_ap[t]));
    gd[h.o_bound + m] = __dadd_rn(__dmul_rn(4.0 * (double)(c + F + 4), ldexp(absum, -53)), 1e-300);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < c; t += blockDim.x) {
    gd[h.o_thr + m * R + t] = s_thr[t];
    gd[h.o_ap + m * R + t] = s_ap[t];
    gi[h.o_feat + m * R + t] = s_feat[t];
    if (s_rank[t] >= 0) gd[h.o_tt + s_toff[s_feat[t]] + s_rank[t]] = s_thr[t];
  }
  for (int f = 0; f < F; ++f)
    for (int k = s_u[f] + threadIdx.x; k < s_p[f] - 1; k += blockDim.x)
      gd[h.o_tt + s_toff[f] + k] = __longlong_as_double(0x7ff0000000000000LL);
  // table values: T[0] = -sum(ap), T[k+1] = T[k] + 2 * (votes of rank k), one warp per feature
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double *whi = s_hi + warp * R, *wlo = s_lo + warp * R;
  for (int f = warp; f < F; f += blockDim.x >> 5) {
    const int u = s_u[f];
    for (int k = lane; k < u; k += 32) {
      DD acc{0.0, 0.0};
      for (int t = 0; t < c; ++t) {
        const int rk = s_rank[t] >= 0 ? s_rank[t] : -1 - s_rank[t];
        if (s_feat[t] == f && rk == k) acc = dd_add(acc, DD{s_ap[t], 0.0});
      }
      whi[k] = acc.hi;
      wlo[k] = acc.lo;
    }
    __syncwarp();
    if (lane == 0) {
      DD acc{0.0, 0.0};
      for (int t = 0; t < c; ++t)
        if (s_feat[t] == f) acc = dd_add(acc, DD{-s_ap[t], 0.0});
      double *tv = gd + h.o_tv + s_voff[f];
      tv[0] = __dadd_rn(acc.hi, acc.lo);
      for (int k = 0; k < u; ++k) {
        acc = dd_add(acc, DD{2.0 * whi[k], 2.0 * wlo[k]});
        tv[k + 1] = __dadd_rn(acc.hi, acc.lo);
      }
    }
    __syncwarp();
  }
}

size_t set_ensemble_smem(int capacity) { return (size_t)capacity * (2 * 8 + 16 * 8 + 3 * 4); }
void *set_ensemble_kernel() { return (void *)&set_ensemble; }

void *finish_kernel() { return (void *)&finish_units; }
void *sample_kernel() { return (void *)&sample_points; }
void *fill_raw_kernel() { return (void *)&fill_raw; }
void *fill_normals_kernel() { return (void *)&fill_normals; }
void *math_selftest_kernel() { return (void *)&math_selftest; }

}  // namespace brm
