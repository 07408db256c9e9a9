// Class-task microbenchmark: the round-1 DIF form (radix-3 combine with twiddles + FFT16) vs the Good-Thomas form
// (no twiddles + tangent FFT16) of the pruned length-48 inverse transform, with Y-like inputs (one row per lane,
// ld = 1) and Z-like inputs (ld = 41 pencils), W warps per SM, r = warp % 3.  Prints cycles per task per warp.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1701_01608_b200/csrc/fft_dev.cuh"
using namespace fks;
constexpr int K = 31;

__device__ __forceinline__ void x_dif(const double2* base, int ld, int r, double2 (&u)[16]) {
  u[0] = base[15 * ld];
  if (r == 0) {
#pragma unroll
    for (int m = 1; m < 16; m++) u[m] = fftd::cadd(base[(m + 15) * ld], base[(m - 1) * ld]);
  } else {
    const double sg = (r == 1) ? -0.86602540378443864676 : 0.86602540378443864676;
#pragma unroll
    for (int m = 1; m < 16; m++) {
      const double2 a = base[(m + 15) * ld], v = base[(m - 1) * ld];
      double2 acc;
      acc.x = fma(-0.5, v.x, a.x);
      acc.x = fma(-sg, v.y, acc.x);
      acc.y = fma(-0.5, v.y, a.y);
      acc.y = fma(sg, v.x, acc.y);
      u[m] = fftd::cmul_s<1>(fftd::c_tw48[r * m], acc);
    }
  }
  fftd::fft16<1>(u);
}
__device__ __forceinline__ void x_gt(const double2* base, int ld, int r, double2 (&u)[16]) {
  u[0] = base[15 * ld];
  if (r == 0) {
#pragma unroll
    for (int m = 1; m < 16; m++) u[fftd::pfa_n2(m)] = fftd::cadd(base[(m + 15) * ld], base[(m - 1) * ld]);
  } else {
    const double sg = (r == 1) ? 0.86602540378443864676 : -0.86602540378443864676;
#pragma unroll
    for (int m = 1; m < 16; m++) u[fftd::pfa_n2(m)] = fftd::pfa_combine(m, base[(m + 15) * ld], base[(m - 1) * ld], -0.5, sg);
  }
  fftd::fft16i(u);
}

template <int GT, int LD>
__global__ void tasks(double* out, int iters, long long* cyc) {
  extern __shared__ double2 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int IN = (LD == 1) ? 32 * K : K * 41;
  double2* in = sm + warp * (IN + 16 * 32 + 2);
  double2* o = in + IN;
  for (int i = lane; i < IN; i += 32) in[i] = make_double2(i * 1e-3, 1.0 - i * 1e-3);
  __syncwarp();
  const int r = warp % 3;
  const double2* base = (LD == 1) ? in + lane * K : in + lane;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    double2 u[16];
    if (GT) x_gt(base, LD, r, u); else x_dif(base, LD, r, u);
#pragma unroll
    for (int q = 0; q < 16; q++) o[q * 32 + lane] = u[fftd::qslot(q)];
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
  if (o[lane].x == 12345.0) out[0] = 1;
}

template <int GT, int LD>
void run(int warps, long long* dcyc, double* dout) {
  const int iters = 2000;
  constexpr int IN = (LD == 1) ? 32 * K : K * 41;
  size_t sh = (size_t)warps * (IN + 16 * 32 + 2) * 16;
  cudaFuncSetAttribute(tasks<GT, LD>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (sh > 227 * 1024) { printf("skip W=%d\n", warps); return; }
  tasks<GT, LD><<<148, 32 * warps, sh>>>(dout, iters, dcyc);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  tasks<GT, LD><<<148, 32 * warps, sh>>>(dout, iters, dcyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[148 * 32]; cudaMemcpy(h, dcyc, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0; for (int w = 0; w < warps; w++) s += h[w];
  printf("{\"form\": \"%s\", \"ld\": %d, \"warps_per_sm\": %d, \"cycles_per_task_per_warp\": %.0f, \"ms\": %.3f, "
         "\"tasks_per_us_per_sm\": %.2f}\n", GT ? "good-thomas" : "dif", LD, warps, s / warps / iters, ms,
         (double)warps * iters / (ms * 1e3));
}

int main() {
  fftd::fill_twiddles();
  long long* dcyc; double* dout;
  cudaMalloc(&dcyc, 148 * 32 * sizeof(long long)); cudaMalloc(&dout, 8);
  for (int w : {4, 8, 12}) {
    run<0, 1>(w, dcyc, dout); run<1, 1>(w, dcyc, dout);
    run<0, 41>(w, dcyc, dout); run<1, 41>(w, dcyc, dout);
  }
  return 0;
}
