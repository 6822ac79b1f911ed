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

// Math self-test: the branch-free exp / divide against the library functions.
__global__ void math_selftest(int kind, const double *a, const double *b, int64_t n, double *out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  switch (kind) {
    case 0: out[i] = exp_nb(a[i]); break;
    case 1: out[i] = exp(a[i]); break;
    case 2: out[i] = div_nb(a[i], b[i]); break;
    default: out[i] = __ddiv_rn(a[i], b[i]); break;
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

void *finish_kernel() { return (void *)&finish_units; }
void *sample_kernel() { return (void *)&sample_points; }
void *fill_raw_kernel() { return (void *)&fill_raw; }
void *fill_normals_kernel() { return (void *)&fill_normals; }
void *math_selftest_kernel() { return (void *)&math_selftest; }

}  // namespace brm
