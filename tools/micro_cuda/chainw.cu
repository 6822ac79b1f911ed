// Micro-benchmark of warp_chain (brm_chain.cuh) vs a sequential chain, from shared memory.
#define BRM_CHAIN_STATS 1
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../../paper_0805_1827_b200/csrc/brm_chain.cuh"
using namespace brm;
__global__ void k_seq(const double *g, double *o, int n, long long *cyc) {
  extern __shared__ double sm[];
  double *in = sm, *out = sm + n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) in[i] = g[i];
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    double s = 0;
    for (int k = 0; k < n; ++k) { s = __dadd_rn(s, in[k]); out[k] = s; }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[0] = clock64() - t0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) o[i] = out[i];
}
__global__ void k_warp(const double *g, double *o, int n, long long *cyc) {
  extern __shared__ double sm[];
  double *in = sm, *out = sm + chain_padded_len(n);
  for (int i = threadIdx.x; i < n; i += blockDim.x) in[chain_pos<true>(i)] = g[i];
  __syncthreads();
  long long t0 = clock64();
  double acc = 0.0;
  if (threadIdx.x < 32) warp_chain<true, CHAIN_T>(in, out, n, acc);
  __syncthreads();
  if (threadIdx.x == 0) cyc[0] = clock64() - t0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) o[i] = out[chain_pos<true>(i)];
}
int main() {
  const int n = 10000;
  std::vector<double> h(n);
  srand(1);
  for (int i = 0; i < n; ++i) h[i] = (rand() / (double)RAND_MAX) / (n / 2);
  double *g, *o1, *o2; long long *cyc, c1, c2;
  cudaMalloc(&g, 8 * n); cudaMalloc(&o1, 8 * n); cudaMalloc(&o2, 8 * n); cudaMalloc(&cyc, 8);
  cudaMemcpy(g, h.data(), 8 * n, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_seq, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * (n + n / 16 + 2));
  cudaFuncSetAttribute(k_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * (n + n / 16 + 2));
  for (int r = 0; r < 3; ++r) {
    k_seq<<<1, 256, 16 * (n + n / 16 + 2)>>>(g, o1, n, cyc); cudaMemcpy(&c1, cyc, 8, cudaMemcpyDeviceToHost);
    k_warp<<<1, 256, 16 * (n + n / 16 + 2)>>>(g, o2, n, cyc); cudaMemcpy(&c2, cyc, 8, cudaMemcpyDeviceToHost);
  }
  long long st[6];
  cudaMemcpyFromSymbol(st, g_chain_stats, sizeof st);
  printf("3 runs: tiles %lld events %lld seq-elems %lld seq-cycles %lld tile-cycles %lld\n", st[0], st[1], st[2], st[3], st[4]);
  std::vector<double> a(n), b(n);
  cudaMemcpy(a.data(), o1, 8 * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), o2, 8 * n, cudaMemcpyDeviceToHost);
  int diff = 0;
  for (int i = 0; i < n; ++i) diff += a[i] != b[i];
  printf("n=%d sequential %.2f cyc/elem, warp %.2f cyc/elem, mismatches %d (%s)\n", n, (double)c1 / n, (double)c2 / n, diff,
         cudaGetErrorString(cudaGetLastError()));
}
