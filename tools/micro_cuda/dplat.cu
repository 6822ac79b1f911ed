// Dependent-chain latency of fp64 DADD / DMUL / DFMA and of a separately rounded Horner step (registers only).
#include <cstdio>
template <int K>
__global__ void chain(double *out, double a, double b, long long *cyc, int n) {
  double x = a, y = b;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (K == 0) x = __dadd_rn(x, y);
      if (K == 1) x = __dmul_rn(x, y);
      if (K == 2) x = fma(x, y, a);
      if (K == 3) x = __dadd_rn(__dmul_rn(x, y), a);
      if (K == 4) x = __fadd_rn((float)x, (float)y);
    }
  }
  long long t1 = clock64();
  out[0] = x;
  cyc[0] = t1 - t0;
}
int main() {
  double *out; long long *cyc, h;
  cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  const int n = 4096;
  const char *names[] = {"DADD", "DMUL", "DFMA", "DMUL+DADD (Horner step)", "FADD"};
#define RUN(K) chain<K><<<1, 1>>>(out, 1.0000001, 0.9999999, cyc, n); chain<K><<<1, 1>>>(out, 1.0000001, 0.9999999, cyc, n); \
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("%s: %.2f cycles per dependent op\n", names[K], (double)h / (32.0 * n));
  RUN(0) RUN(1) RUN(2) RUN(3) RUN(4)
  return 0;
}
