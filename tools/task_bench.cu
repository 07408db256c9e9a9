// Throughput of the bare class task of the term-loop kernel (31 smem loads -> radix-3 combine -> FFT16 ->
// 16 smem stores), no synchronisation: FP64 lane-instructions per clock per SM vs warps per SM.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1701_01608_b200/csrc/fft_dev.cuh"
using namespace fks;
constexpr int K = 31;

__device__ __forceinline__ void xform48(const double2* base, int ld, int r, double2 (&u)[16]) {
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

struct InK {
  const double2* b;
  __device__ __forceinline__ bool nz(int i) const { return i <= 15 || i >= 33; }
  __device__ __forceinline__ double2 operator()(int i) const { return b[i <= 15 ? i + 15 : i - 33]; }
};
template <int R>
__device__ __forceinline__ void xform48t(const double2* base, double2 (&u)[16]) {
  fftd::dif_class<3, 1, R>(InK{base}, u);
}

template <int MODE>  // 0: smem out, runtime r; 1: register out, runtime r; 2: smem out, template r; 3: smem out, dual
__global__ void tasks(double* out, int iters) {
  extern __shared__ double2 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* in = sm + warp * (K * 32 + 16 * 32 + 2);
  double2* o = in + K * 32 + 2;
  for (int i = lane; i < K * 32 + 2; i += 32) in[i] = make_double2(i * 1e-3, 1.0 - i * 1e-3);
  __syncwarp();
  double2 acc = make_double2(0, 0);
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    const int r = it % 3;
    const double2* b = in + lane * K + (it & 1) * 16 * 0 + ((it >> 1) & 1);  // varies: defeats hoisting
    double2 u[16];
    if (MODE == 2) {
      if (r == 0) xform48t<0>(b, u); else if (r == 1) xform48t<1>(b, u); else xform48t<2>(b, u);
    } else if (MODE == 3) {
      double2 v[16];
      const double2* b2 = in + ((lane + 7) & 31) * K + ((it >> 1) & 1);
      xform48(b, 1, r, u);
      xform48(b2, 1, r, v);
#pragma unroll
      for (int q = 0; q < 16; q++) o[q * 32 + lane] = fftd::cadd(u[q], v[q]);
      continue;
    } else {
      xform48(b, 1, r, u);
    }
    if (MODE != 1) {
#pragma unroll
      for (int q = 0; q < 16; q++) o[q * 32 + lane] = u[q];
    } else {
#pragma unroll
      for (int q = 0; q < 16; q++) acc = fftd::cadd(acc, u[q]);
    }
  }
  long long t1 = clock64();
  if (acc.x == 1234.5) out[0] = acc.y;
  if (lane == 0) ((long long*)out)[1 + blockIdx.x * 16 + warp] = t1 - t0;  // every warp: take the slowest
}

int main() {
  double* out;
  cudaMalloc(&out, 8192 * sizeof(double));
  fftd::fill_twiddles();
  const char* names[] = {"smem_out_runtime_r", "reg_out_runtime_r", "smem_out_template_r", "smem_out_dual"};
  for (int mode = 0; mode < 4; mode++) {
    for (int w : {4, 8, 12, 16}) {
      const int smem = w * (K * 32 + 16 * 32 + 2) * 16;
      auto kern = mode == 0 ? tasks<0> : mode == 1 ? tasks<1> : mode == 2 ? tasks<2> : tasks<3>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      const int iters = 600;
      kern<<<148, w * 32, smem>>>(out, 30);
      cudaDeviceSynchronize();
      kern<<<148, w * 32, smem>>>(out, iters);
      cudaError_t e = cudaDeviceSynchronize();
      static long long cyc[148 * 16];
      cudaMemcpy(cyc, out + 1, sizeof(cyc), cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < 148; i++)
        for (int ww = 0; ww < w; ww++) mx = cyc[i * 16 + ww] > mx ? cyc[i * 16 + ww] : mx;
      const double tasks_per_iter = mode == 3 ? 2.0 : 1.0;
      printf("{\"mode\": \"%s\", \"warps\": %d, \"err\": %d, \"clk_per_iter\": %.0f, \"sm_clk_per_task\": %.1f}\n",
             names[mode], w, (int)e, mx / iters, mx / iters / (w * tasks_per_iter));
    }
  }
  return 0;
}
