// Does an fp64 instruction hold the sub-partition's issue port for both cycles
// of its 16-lane pass?  Each warp runs NF independent fp64 FMA chains and NI
// independent integer chains per loop trip (inline PTX, so neither compiler
// folds them); W warps per SM sub-partition.  If integer work issued in the
// shadow of the fp64 pipe, time(NF, NI) would be max(2*NF, NI) cycles per trip
// per warp; if the port is held, 2*NF + NI.
#include <cstdio>
template <int NF, int NI>
__global__ void mix(double *out, int *iout, double a, int s, long long *cyc, int n) {
  double x[8];
  int v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { x[j] = a + j + threadIdx.x; v[j] = s + j + threadIdx.x; }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j < NF) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(x[j]) : "d"(a));
        if (j < NI) asm volatile("mad.lo.s32 %0, %0, %1, %1;" : "+r"(v[j]) : "r"(s));
      }
    }
  }
  long long t1 = clock64();
  double acc = 0; int iacc = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) { acc += x[j]; iacc += v[j]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  iout[blockIdx.x * blockDim.x + threadIdx.x] = iacc;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <int NF, int NI>
void run(int warps_per_smsp, double *out, int *iout, long long *cyc) {
  const int n = 2048, threads = warps_per_smsp * 4 * 32;
  long long h;
  for (int rep = 0; rep < 2; ++rep) mix<NF, NI><<<148, threads>>>(out, iout, 1.0000001, 3, cyc, n);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double per_trip = (double)h / (4.0 * n);  // cycles per (NF fp64 + NI int) of one warp
  printf("W=%d NF=%d NI=%d: %.2f cycles per trip per warp -> %.2f per sub-partition trip-set (W warps); "
         "2*NF*W=%d, NI*W=%d, sum=%d\n", warps_per_smsp, NF, NI, per_trip, per_trip, 2 * NF * warps_per_smsp,
         NI * warps_per_smsp, (2 * NF + NI) * warps_per_smsp);
}
int main() {
  double *out; int *iout; long long *cyc;
  cudaMalloc(&out, 8 * 148 * 1024); cudaMalloc(&iout, 4 * 148 * 1024); cudaMalloc(&cyc, 8);
  for (int w : {1, 2, 4, 8}) {
    if (w == 1) { run<8, 0>(1, out, iout, cyc); run<0, 8>(1, out, iout, cyc); run<8, 8>(1, out, iout, cyc); run<4, 8>(1, out, iout, cyc); run<8, 4>(1, out, iout, cyc); }
    if (w == 2) { run<8, 0>(2, out, iout, cyc); run<0, 8>(2, out, iout, cyc); run<8, 8>(2, out, iout, cyc); run<4, 8>(2, out, iout, cyc); run<8, 4>(2, out, iout, cyc); }
    if (w == 4) { run<8, 0>(4, out, iout, cyc); run<0, 8>(4, out, iout, cyc); run<8, 8>(4, out, iout, cyc); run<4, 8>(4, out, iout, cyc); run<8, 4>(4, out, iout, cyc); }
    if (w == 8) { run<8, 0>(8, out, iout, cyc); run<0, 8>(8, out, iout, cyc); run<8, 8>(8, out, iout, cyc); run<4, 8>(8, out, iout, cyc); run<8, 4>(8, out, iout, cyc); }
  }
  return 0;
}
