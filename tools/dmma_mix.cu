// Do DMMA (mma.sync f64, tensor cores) and DFMA share one pipe on B200?  One CTA per SM; warps of the first half
// run DFMA chains, warps of the second half DMMA chains (mode 0: all DFMA, 1: all DMMA, 2: half / half).  Each
// warp does a fixed amount of work, so if the two kinds run on separate units the mixed kernel takes about the
// time of the slower half alone; if they share the FP64 pipe, about the sum.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_mix tools/dmma_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512, 1) mix(int mode, int iters, double* out) {
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const bool dm = mode == 1 || (mode == 2 && warp >= nw / 2);
  double s = 0;
  if (!dm) {
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; i++) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; it++) {
#pragma unroll
      for (int i = 0; i < 16; i++) x[i] = fma(x[i], 1.0000001, 1e-9);
    }
#pragma unroll
    for (int i = 0; i < 16; i++) s += x[i];
  } else {
    double a = threadIdx.x * 1e-3, b = 1.0001, c[8][2];
#pragma unroll
    for (int i = 0; i < 8; i++) { c[i][0] = 0; c[i][1] = 0; }
    for (int it = 0; it < iters / 4; it++) {  // one m8n8k4 = 256 FMA per warp = 8 per lane: 8 chains x iters/4
#pragma unroll
      for (int i = 0; i < 8; i++)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  }
  if (s == 1234.5678) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {8, 16}) {
    for (int mode = 0; mode < 3; mode++) {
      mix<<<sms, 32 * warps>>>(mode, 100, out);
      cudaEventRecord(e0);
      mix<<<sms, 32 * warps>>>(mode, iters, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      // per warp: DFMA 16 x iters x 32 lanes FMA;  DMMA 8 x iters/4 x 256 FMA = same FMA count per warp
      const double fma_per_warp = 16.0 * iters * 32;
      const double tf = 2.0 * fma_per_warp * warps * sms / (ms * 1e-3) / 1e12;
      printf("{\"warps\": %d, \"mode\": \"%s\", \"ms\": %.3f, \"tflops_all_warps\": %.2f}\n", warps,
             mode == 0 ? "dfma" : mode == 1 ? "dmma" : "half_dfma_half_dmma", ms, tf);
    }
  }
  return 0;
}
