// Micro-benchmark + exactness check: sequential fp64 prefix sum of nonnegative
// values vs the integer binade-scan warp emulation (candidate for brm_boost.cu).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <random>

__device__ void seq_chain(const double *in, double *out, int n, double &acc) {
  for (int k = 0; k < n; ++k) {
    acc = __dadd_rn(acc, in[k]);
    out[k] = acc;
  }
}

// Exact emulation: inside the binade of s, RN(s + x) = s + ulp*rint(x/ulp)
// (no tie), computed on integer mantissas.
__device__ void int_chain(const double *__restrict__ in, double *__restrict__ out, int cnt, double &acc,
                          int *passes) {
  constexpr int IT = 16, BLK = 32 * IT;
  const int lane = threadIdx.x & 31;
  double s = acc;
  int k = 0;
  while (k < cnt) {
    const unsigned long long sb = __double_as_longlong(s);
    const int E = (int)(sb >> 52) & 0x7ff;
    if (E == 0) {  // zero / subnormal prefix: sequential
      s = __dadd_rn(s, in[k]);
      if (lane == 0) out[k] = s;
      ++k;
      continue;
    }
    if (lane == 0 && passes) ++*passes;
    const long long ms = (long long)((sb & 0xFFFFFFFFFFFFFull) | 0x10000000000000ull);  // s / ulp
    const long long L = (1ll << 53) - ms;                                                  // room in the binade
    long long pre[IT];
    int bad = IT;
    long long run = 0;
#pragma unroll
    for (int t = 0; t < IT; ++t) {
      const int j = k + IT * lane + t;
      long long q = 0;
      if (j < cnt) {
        const unsigned long long xb = __double_as_longlong(in[j]);
        const int Ex = (int)(xb >> 52) & 0x7ff;
        const long long mx = (long long)(xb & 0xFFFFFFFFFFFFFull) | (Ex ? 0x10000000000000ll : 0);
        const int sh = E - (Ex ? Ex : 1);
        if (sh < 0) {
          bad = min(bad, t);  // x >= 2^(e+1): leaves the binade
        } else if (sh == 0) {
          q = mx;
        } else if (sh <= 53) {
          const long long half = 1ll << (sh - 1), rem = mx & ((half << 1) - 1);
          q = (mx >> sh) + (rem > half ? 1 : 0);
          if (rem == half) bad = min(bad, t);  // tie: depends on the parity of s
        }
      }
      run += q;
      pre[t] = run;
    }
    long long incl = run;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const long long o = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += o;
    }
    const long long excl = incl - run;
    int first = 1 << 30;
#pragma unroll
    for (int t = IT - 1; t >= 0; --t) {
      const int j = k + IT * lane + t;
      if (j < cnt && (t == bad || excl + pre[t] >= L)) first = IT * lane + t;
    }
    first = (int)__reduce_min_sync(0xffffffffu, (unsigned)first);
    const unsigned long long ebits = sb & 0xFFF0000000000000ull;
#pragma unroll
    for (int t = 0; t < IT; ++t) {
      const int idx = IT * lane + t, j = k + idx;
      if (j < cnt && idx < first)
        out[j] = __longlong_as_double((long long)(ebits | (unsigned long long)((ms + excl + pre[t]) & 0xFFFFFFFFFFFFFll)));
    }
    if (first == (1 << 30)) {
      const long long tot = __shfl_sync(0xffffffffu, incl, 31);
      s = __longlong_as_double((long long)(ebits | (unsigned long long)((ms + tot) & 0xFFFFFFFFFFFFFll)));
      k += min(BLK, cnt - k);
    } else {
      const int prev = first - 1;
      long long qp = 0;
      if (prev >= 0) {
        long long mine = excl;
#pragma unroll
        for (int t = 0; t < IT; ++t)
          if (t == prev % IT) mine = excl + pre[t];
        qp = __shfl_sync(0xffffffffu, mine, prev / IT);
      }
      const double sp = __longlong_as_double((long long)(ebits | (unsigned long long)((ms + qp) & 0xFFFFFFFFFFFFFll)));
      s = __dadd_rn(sp, in[k + first]);
      if (lane == 0) out[k + first] = s;
      k += first + 1;
    }
  }
  acc = s;
}

// the kernel's serial_chain (loads batched 8 ahead)
__device__ __forceinline__ void batched_chain(const double *__restrict__ in, double *__restrict__ out, int cnt,
                                             double &acc) {
  constexpr int B = 8;
  int k = 0;
  double cur[B];
  if (cnt >= B) {
#pragma unroll
    for (int j = 0; j < B; ++j) cur[j] = in[j];
  }
  for (; k + B <= cnt; k += B) {
    double nxt[B];
    const bool more = k + 2 * B <= cnt;
#pragma unroll
    for (int j = 0; j < B; ++j) nxt[j] = more ? in[k + B + j] : 0.0;
#pragma unroll
    for (int j = 0; j < B; ++j) {
      acc = __dadd_rn(acc, cur[j]);
      out[k + j] = acc;
    }
#pragma unroll
    for (int j = 0; j < B; ++j) cur[j] = nxt[j];
  }
  for (; k < cnt; ++k) {
    acc = __dadd_rn(acc, in[k]);
    out[k] = acc;
  }
}

// both read from / write to shared memory, as in the AdaBoost kernel (tiles of 4096)
constexpr int T = 4096;
template <int U>
__device__ __forceinline__ void unrolled_chain(const double *__restrict__ in, double *__restrict__ out, int cnt,
                                               double &acc) {
#pragma unroll U
  for (int k = 0; k < cnt; ++k) {
    acc = __dadd_rn(acc, in[k]);
    out[k] = acc;
  }
}

// ping-pong: chunk A summed while chunk B loads, then the reverse (no moves)
template <int C>
__device__ __forceinline__ void pingpong_chain(const double *__restrict__ in, double *__restrict__ out, int cnt,
                                               double &acc) {
  int k = 0;
  double a[C], b[C];
  if (cnt >= 2 * C) {
#pragma unroll
    for (int j = 0; j < C; ++j) a[j] = in[j];
  }
  for (; k + 2 * C <= cnt; k += 2 * C) {
#pragma unroll
    for (int j = 0; j < C; ++j) b[j] = in[k + C + j];
#pragma unroll
    for (int j = 0; j < C; ++j) {
      acc = __dadd_rn(acc, a[j]);
      out[k + j] = acc;
    }
    const bool more = k + 4 * C <= cnt;
#pragma unroll
    for (int j = 0; j < C; ++j) a[j] = more ? in[k + 2 * C + j] : 0.0;
#pragma unroll
    for (int j = 0; j < C; ++j) {
      acc = __dadd_rn(acc, b[j]);
      out[k + C + j] = acc;
    }
  }
  for (; k < cnt; ++k) {
    acc = __dadd_rn(acc, in[k]);
    out[k] = acc;
  }
}

template <int V>
__global__ void run_var(const double *in, double *out, int n, long long *cyc) {
  extern __shared__ double sm[];
  double *si = sm, *so = sm + T;
  double acc = 0.0;
  long long tot = 0;
  for (int t0 = 0; t0 < n; t0 += T) {
    const int tn = min(T, n - t0);
    for (int j = threadIdx.x; j < tn; j += blockDim.x) si[j] = in[t0 + j];
    __syncthreads();
    long long a = clock64();
    if (threadIdx.x == blockDim.x - 32) {
      if (V == 0) unrolled_chain<8>(si, so, tn, acc);
      if (V == 1) unrolled_chain<16>(si, so, tn, acc);
      if (V == 2) unrolled_chain<32>(si, so, tn, acc);
      if (V == 3) pingpong_chain<8>(si, so, tn, acc);
      if (V == 4) pingpong_chain<16>(si, so, tn, acc);
    }
    tot += clock64() - a;
    __syncthreads();
    for (int j = threadIdx.x; j < tn; j += blockDim.x) out[t0 + j] = so[j];
    __syncthreads();
  }
  if (threadIdx.x == blockDim.x - 32) *cyc = tot;
}

__global__ void run_seq(const double *in, double *out, int n, long long *cyc) {
  extern __shared__ double sm[];
  double *si = sm, *so = sm + T;
  double acc = 0.0;
  long long tot = 0;
  for (int t0 = 0; t0 < n; t0 += T) {
    const int tn = min(T, n - t0);
    for (int j = threadIdx.x; j < tn; j += blockDim.x) si[j] = in[t0 + j];
    __syncthreads();
    long long a = clock64();
    if (threadIdx.x == 0) seq_chain(si, so, tn, acc);
    tot += clock64() - a;
    __syncthreads();
    for (int j = threadIdx.x; j < tn; j += blockDim.x) out[t0 + j] = so[j];
    __syncthreads();
  }
  if (threadIdx.x == 0) *cyc = tot;
}

template <int WARPS>
__global__ void run_batched(const double *in, double *out, int n, long long *cyc) {
  extern __shared__ double sm[];
  double *si = sm, *so = sm + T;
  double acc = 0.0;
  long long tot = 0;
  for (int t0 = 0; t0 < n; t0 += T) {
    const int tn = min(T, n - t0);
    for (int j = threadIdx.x; j < tn; j += blockDim.x) si[j] = in[t0 + j];
    __syncthreads();
    long long a = clock64();
    if (threadIdx.x == blockDim.x - 32) batched_chain(si, so, tn, acc);
    tot += clock64() - a;
    __syncthreads();
    for (int j = threadIdx.x; j < tn; j += blockDim.x) out[t0 + j] = so[j];
    __syncthreads();
  }
  if (threadIdx.x == blockDim.x - 32) *cyc = tot;
}

__global__ void run_warp(const double *in, double *out, int n, long long *cyc, int *passes) {
  extern __shared__ double sm[];
  double *si = sm, *so = sm + T;
  double acc = 0.0;
  long long tot = 0;
  for (int t0 = 0; t0 < n; t0 += T) {
    const int tn = min(T, n - t0);
    for (int j = threadIdx.x; j < tn; j += blockDim.x) si[j] = in[t0 + j];
    __syncthreads();
    long long a = clock64();
    int_chain(si, so, tn, acc, passes);
    tot += clock64() - a;
    __syncthreads();
    for (int j = threadIdx.x; j < tn; j += blockDim.x) out[t0 + j] = so[j];
    __syncthreads();
  }
  if (threadIdx.x == 0) *cyc = tot;
}

static double r1ref(const std::vector<double> &h, int i) {  // sequential prefix, cached
  static std::vector<double> c;
  static const double *key = nullptr;
  if (key != h.data() || c.size() != h.size()) {
    key = h.data();
    c.resize(h.size());
    double s = 0.0;
    for (size_t j = 0; j < h.size(); ++j) c[j] = (s += h[j]);
  }
  return c[i];
}

int main() {
  std::mt19937_64 rng(1);
  const int n = 10000;
  int bad_total = 0;
  for (int trial = 0; trial < 6; ++trial) {
    std::vector<double> h(n);
    std::lognormal_distribution<double> ln(0.0, trial < 3 ? 0.2 : 2.0);
    double tot = 0;
    for (auto &x : h) tot += (x = ln(rng));
    for (auto &x : h) x /= tot;           // normalised AdaBoost-like weights
    if (trial == 5)
      for (int i = 0; i < n; ++i) h[i] = 1.0 / n;  // uniform first round
    double *din, *o1, *o2;
    long long *cyc;
    int *passes;
    cudaMalloc(&din, 8 * n); cudaMalloc(&o1, 8 * n); cudaMalloc(&o2, 8 * n); cudaMalloc(&cyc, 16);
    cudaMalloc(&passes, 4); cudaMemset(passes, 0, 4);
    cudaMemcpy(din, h.data(), 8 * n, cudaMemcpyHostToDevice);
    long long c1, c2;
    int np;
    cudaFuncSetAttribute(run_seq, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * T * 8);
    cudaFuncSetAttribute(run_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * T * 8);
    run_seq<<<1, 32, 2 * T * 8>>>(din, o1, n, cyc);
    cudaMemcpy(&c1, cyc, 8, cudaMemcpyDeviceToHost);
    {
      long long cb1, cb8;
      cudaFuncSetAttribute(run_batched<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * T * 8);
      cudaFuncSetAttribute(run_batched<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * T * 8);
      run_batched<1><<<1, 32, 2 * T * 8>>>(din, o2, n, cyc + 1);
      cudaMemcpy(&cb1, cyc + 1, 8, cudaMemcpyDeviceToHost);
      run_batched<8><<<1, 256, 2 * T * 8>>>(din, o2, n, cyc + 1);
      cudaMemcpy(&cb8, cyc + 1, 8, cudaMemcpyDeviceToHost);
      printf("  batched chain: 1 warp %.1f cyc/elem, 8 warps (chain on warp 7) %.1f cyc/elem\n", (double)cb1 / n,
             (double)cb8 / n);
    }
    {
      const char *names[] = {"unroll8", "unroll16", "unroll32", "pingpong8", "pingpong16"};
      void (*ks[])(const double *, double *, int, long long *) = {run_var<0>, run_var<1>, run_var<2>, run_var<3>,
                                                                  run_var<4>};
      for (int v = 0; v < 5; ++v) {
        long long cv;
        cudaFuncSetAttribute(ks[v], cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * T * 8);
        ks[v]<<<1, 256, 2 * T * 8>>>(din, o2, n, cyc + 1);
        cudaMemcpy(&cv, cyc + 1, 8, cudaMemcpyDeviceToHost);
        std::vector<double> rv(n);
        cudaMemcpy(rv.data(), o2, 8 * n, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int i = 0; i < n; ++i) bad += rv[i] != r1ref(h, i);
        printf("  %s: %.1f cyc/elem (mismatches %d)\n", names[v], (double)cv / n, bad);
      }
    }
    run_warp<<<1, 32, 2 * T * 8>>>(din, o2, n, cyc + 1, passes);
    cudaMemcpy(&c2, cyc + 1, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&np, passes, 4, cudaMemcpyDeviceToHost);
    std::vector<double> r1(n), r2(n);
    cudaMemcpy(r1.data(), o1, 8 * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(r2.data(), o2, 8 * n, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < n; ++i) bad += r1[i] != r2[i];
    bad_total += bad;
    printf("trial %d: seq %.1f cyc/elem, warp %.1f cyc/elem (%d passes), mismatches %d\n", trial, (double)c1 / n,
           (double)c2 / n, np, bad);
  }
  return bad_total ? 1 : 0;
}
