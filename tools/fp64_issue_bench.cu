// FP64 issue/latency microbenchmark: one CTA per SM with W warps, each thread running ILP independent DFMA
// (or DADD) chains.  Reports FP64 lane-ops per clock per SM (peak 64) -> how many warps x ILP saturate the pipe.
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP, int OP>  // OP 0 DFMA, 1 DADD, 2 DMUL
__global__ void chains(double* out, int iters, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; i++) x[i] = threadIdx.x * 1e-3 + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) x[i] = OP == 1 ? x[i] + a : (OP == 2 ? x[i] * a : fma(x[i], a, b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; i++) s += x[i];
  if (s == 1234.5678) out[0] = s;
  if (threadIdx.x == 0) ((long long*)out)[1 + blockIdx.x] = t1 - t0;
}

template <int ILP, int OP>
void run(int warps, int sms, double* out) {
  const int iters = 4096;
  chains<ILP, OP><<<sms, warps * 32>>>(out, 64, 1.0000001, 1e-9);
  cudaDeviceSynchronize();
  chains<ILP, OP><<<sms, warps * 32>>>(out, iters, 1.0000001, 1e-9);
  cudaDeviceSynchronize();
  long long cyc[256];
  cudaMemcpy(cyc, out + 1, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < sms; i++) mx = cyc[i] > mx ? cyc[i] : mx;
  const double ops = (double)iters * ILP * warps * 32;
  printf("{\"op\": \"%s\", \"warps_per_sm\": %d, \"ilp\": %d, \"lane_ops_per_clk_sm\": %.2f, \"clk_per_dependent_op\": %.2f}\n",
         OP == 1 ? "dadd" : (OP == 2 ? "dmul" : "dfma"), warps, ILP, ops / mx, (double)mx / iters);
}

int main() {
  double* out;
  cudaMalloc(&out, 4096 * sizeof(double));
  int sms = 148;
  for (int w : {8, 16, 32}) {
    run<8, 0>(w, sms, out);
    run<8, 1>(w, sms, out);
    run<8, 2>(w, sms, out);
    run<4, 1>(w, sms, out);
  }
  return 0;
}
