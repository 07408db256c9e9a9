// Box-facts microbenchmarks for the FKS collision kernel design.
// Measures: FP64 DFMA peak, DMMA (mma.sync f64) rate, max active clusters per cluster size,
// DSMEM store bandwidth, L2 read bandwidth, SMEM LDS.128 bandwidth.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; i++) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += x[i];
  if (s == 1234.5678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0001;
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; i++) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; i++) s += c[i][0] + c[i][1];
  if (s == 1234.5678) out[0] = s;
}

// Each CTA of the cluster writes `bytes_per_cta` bytes into the next CTA's smem, `reps` times.
__global__ void dsmem_kernel(int reps, int words, double* out) {
  extern __shared__ double4 sm4[];
  cg::cluster_group cl = cg::this_cluster();
  unsigned r = cl.block_rank();
  unsigned n = cl.num_blocks();
  double4* dst = cl.map_shared_rank(sm4, (r + 1) % n);
  cl.sync();
  double4 v = make_double4(r, 1, 2, 3);
  for (int k = 0; k < reps; k++) {
    for (int i = threadIdx.x; i < words; i += blockDim.x) { dst[i] = v; v.x += 1.0; }
  }
  cl.sync();
  if (threadIdx.x == 0 && sm4[0].x == -1.0) out[0] = 1;
}

// Same, but remote 8-byte stores.
__global__ void dsmem8_kernel(int reps, int words, double* out) {
  extern __shared__ double sm8[];
  cg::cluster_group cl = cg::this_cluster();
  unsigned r = cl.block_rank();
  unsigned n = cl.num_blocks();
  double* dst = cl.map_shared_rank(sm8, (r + 1) % n);
  cl.sync();
  double v = r;
  for (int k = 0; k < reps; k++) {
    for (int i = threadIdx.x; i < words; i += blockDim.x) { dst[i] = v; v += 1.0; }
  }
  cl.sync();
  if (threadIdx.x == 0 && sm8[0] == -1.0) out[0] = 1;
}

__global__ void l2_read_kernel(const double4* __restrict__ buf, size_t n4, int reps, double* out) {
  double acc = 0;
  for (int k = 0; k < reps; k++) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
      double2 v = __ldcg((const double2*)&buf[i]); double2 w = __ldcg(((const double2*)&buf[i]) + 1);
      acc += v.x + w.y;
    }
  }
  if (acc == 1234.5678) out[0] = acc;
}

__global__ void smem_kernel(int reps, double* out) {
  extern __shared__ double2 s2[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s2[i] = make_double2(i, i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  int idx = threadIdx.x;
  for (int k = 0; k < reps; k++) {
#pragma unroll 8
    for (int j = 0; j < 32; j++) {
      double2 v = s2[(idx + j * 256) & 8191];
      acc.x += v.x; acc.y += v.y;
    }
  }
  if (acc.x == 1234.5678) out[0] = acc.x + acc.y;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_per_block_optin\": %zu, \"smem_per_sm\": %zu, \"regs_per_sm\": %d, \"clock_khz\": %d, \"cc\": \"%d.%d\"}\n",
         p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin, p.sharedMemPerMultiprocessor,
         p.regsPerMultiprocessor, clk, p.major, p.minor);
  double* out; CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // FP64 DFMA peak
  {
    int blocks = p.multiProcessorCount * 8, threads = 256, iters = 20000;
    dfma_kernel<<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * iters * (double)blocks * threads;
    printf("{\"test\": \"dfma\", \"tflops\": %.3f, \"ms\": %.3f}\n", flops / ms / 1e9, ms);
  }
  // DMMA
  {
    int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4000;
    dmma_kernel<<<blocks, threads>>>(out, 10);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 4 * (double)iters * blocks * (threads / 32);
    printf("{\"test\": \"dmma_m8n8k4\", \"tflops\": %.3f, \"ms\": %.3f}\n", flops / ms / 1e9, ms);
  }
  // Max active clusters
  {
    int sizes[] = {1, 2, 3, 4, 6, 8, 12, 16};
    size_t smems[] = {64 * 1024, 100 * 1024, 150 * 1024, 200 * 1024, 227 * 1024};
    CK(cudaFuncSetAttribute(dsmem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    CK(cudaFuncSetAttribute(dsmem_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (size_t sm : smems) {
      for (int cs : sizes) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs * 64); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = sm;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        int ncl = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, dsmem_kernel, &cfg);
        if (e != cudaSuccess) { cudaGetLastError(); ncl = -1; }
        printf("{\"test\": \"max_active_clusters\", \"cluster\": %d, \"smem_kb\": %zu, \"clusters\": %d, \"ctas\": %d}\n",
               cs, sm / 1024, ncl, ncl * cs);
      }
    }
  }
  // DSMEM bandwidth
  {
    CK(cudaFuncSetAttribute(dsmem8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    CK(cudaFuncSetAttribute(dsmem8_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    int sizes[] = {2, 4, 8, 16};
    for (int which = 0; which < 2; which++)
    for (int cs : sizes) {
      size_t sm = 128 * 1024; int words = which == 0 ? (int)(sm / 32) : (int)(sm / 8); int reps = 200;
      cudaLaunchConfig_t cfg = {};
      int ncl = 0;
      cfg.gridDim = dim3(cs * 256); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = sm;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      if (which == 0) cudaOccupancyMaxActiveClusters(&ncl, dsmem_kernel, &cfg);
      else cudaOccupancyMaxActiveClusters(&ncl, dsmem8_kernel, &cfg);
      cfg.gridDim = dim3(cs * ncl);
      void* args[] = {&reps, &words, &out};
      cudaError_t e;
      if (which == 0) e = cudaLaunchKernelExC(&cfg, (void*)dsmem_kernel, args);
      else e = cudaLaunchKernelExC(&cfg, (void*)dsmem8_kernel, args);
      if (e != cudaSuccess) { printf("launch err %s\n", cudaGetErrorString(e)); continue; } CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      if (which == 0) e = cudaLaunchKernelExC(&cfg, (void*)dsmem_kernel, args);
      else e = cudaLaunchKernelExC(&cfg, (void*)dsmem8_kernel, args);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      double bytes = (double)sm * reps * cs * ncl;
      printf("{\"test\": \"dsmem_store%s\", \"cluster\": %d, \"ctas\": %d, \"GBps_total\": %.1f, \"B_per_clk_per_sm_at_1.9GHz\": %.2f}\n",
             which == 0 ? "32B" : "8B", cs, cs * ncl, bytes / ms / 1e6, bytes / ms / 1e6 / (cs * ncl) / 1.9);
    }
  }
  // L2 read bandwidth (64 MB working set)
  {
    size_t bytes = 64ull << 20; double4* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 0, bytes));
    size_t n4 = bytes / 32; int reps = 20;
    int blocks = p.multiProcessorCount * 4;
    l2_read_kernel<<<blocks, 512>>>(buf, n4, 2, out); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    l2_read_kernel<<<blocks, 512>>>(buf, n4, reps, out);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"test\": \"l2_read_64MB\", \"GBps\": %.1f}\n", (double)bytes * reps / ms / 1e6);
    cudaFree(buf);
    bytes = 4ull << 30; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 0, bytes)); n4 = bytes / 32; reps = 2;
    l2_read_kernel<<<blocks, 512>>>(buf, n4, 1, out); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    l2_read_kernel<<<blocks, 512>>>(buf, n4, reps, out);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"test\": \"hbm_read_4GB\", \"GBps\": %.1f}\n", (double)bytes * reps / ms / 1e6);
    cudaFree(buf);
  }
  // SMEM LDS.128
  {
    CK(cudaFuncSetAttribute(smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024));
    int blocks = p.multiProcessorCount * 4, reps = 2000;
    smem_kernel<<<blocks, 256, 128 * 1024>>>(10, out); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    smem_kernel<<<blocks, 256, 128 * 1024>>>(reps, out);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double bytes = 16.0 * 32 * reps * 256.0 * blocks;
    printf("{\"test\": \"smem_lds128\", \"GBps_total\": %.1f, \"B_per_clk_per_sm_at_1.9GHz\": %.2f}\n",
           bytes / ms / 1e6, bytes / ms / 1e6 / p.multiProcessorCount / 1.9);
  }
  return 0;
}
