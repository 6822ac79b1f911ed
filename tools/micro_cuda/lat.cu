// Dependent-chain latency of fp64 add on this GPU (one thread, clock64).
#include <cstdio>
__global__ void chain(double *out, const double *in, long long *cyc, int n) {
  double acc = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, in[i & 1023]);
  long long t1 = clock64();
  out[0] = acc;
  cyc[0] = t1 - t0;
}
__global__ void chain_smem(double *out, const double *in, long long *cyc, int n) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = in[i];
  __syncthreads();
  if (threadIdx.x) return;
  double acc = 0.0, a2 = 0.0;
  long long t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, s[i & 1023]);
  long long t1 = clock64();
  out[0] = acc;
  cyc[0] = t1 - t0;
}
int main() {
  double *in, *out; long long *cyc, h;
  cudaMalloc(&in, 8192); cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  cudaMemset(in, 0, 8192);
  const int n = 1 << 20;
  chain<<<1, 1>>>(out, in, cyc, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  chain<<<1, 1>>>(out, in, cyc, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("global-operand DADD chain: %.2f cycles/add\n", (double)h / n);
  chain_smem<<<1, 256>>>(out, in, cyc, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("smem-operand DADD chain: %.2f cycles/add\n", (double)h / n);
  return 0;
}
