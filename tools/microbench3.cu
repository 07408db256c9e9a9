// Microbenchmarks for the hot-kernel design (B200, sm_100a): per-SM throughput of
//   (1) tcgen05.ld 32x32b.x32 (TMEM -> registers) and tcgen05.st,
//   (2) LDS.128 from shared memory,
//   (3) DFMA alone, and DFMA warps sharing the SM with TMEM-load or LDS.128 warps.
// One CTA per SM, W warps; every warp loops `iters` times.  Prints one JSON line per test.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench3 tools/microbench3.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void tld32(uint32_t addr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tst32(uint32_t addr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      ::"r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
        "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
        "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// mode bits: 1 = TMEM-load warps, 2 = LDS.128 warps, 4 = DFMA warps, 8 = TMEM-store warps.
// Warps are assigned round-robin over the enabled roles (role = warp % nroles).
__global__ void __launch_bounds__(512, 1) mix_kernel(int mode, int iters, double* out, unsigned long long* clk) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t tbase_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&tbase_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  double2* sm2 = reinterpret_cast<double2*>(smem);
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm2[i] = make_double2(i * 1e-3, i * 2e-3);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tbase_sh + ((uint32_t)(32 * (warp & 3)) << 16);
  int roles[4], nr = 0;
  for (int b = 0; b < 4; b++) if (mode & (1 << b)) roles[nr++] = b;
  const int role = roles[warp % nr];
  unsigned long long t0 = clock64();
  double acc = 0.0;
  if (role == 0) {  // TMEM loads: 4 KB per instruction per warp
    uint32_t x = 0;
    for (int it = 0; it < iters; it++) {
      uint32_t v[32];
      tld32(tb + (uint32_t)(32 * ((it + warp) & 7)), v);
#pragma unroll
      for (int k = 0; k < 32; k++) x ^= v[k];
    }
    acc = (double)x;
  } else if (role == 1) {  // LDS.128: 512 B per instruction per warp
    double2 a = make_double2(0, 0);
    const double2* p = sm2 + lane;
    for (int it = 0; it < iters; it++) {
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const double2 v = p[((it * 8 + k) & 63) * 32];
        a.x += v.x;
        a.y -= v.y;
      }
    }
    acc = a.x + a.y;
  } else if (role == 2) {  // DFMA, 8 independent chains
    double c[8];
#pragma unroll
    for (int k = 0; k < 8; k++) c[k] = lane + k;
    for (int it = 0; it < iters; it++) {
#pragma unroll
      for (int r = 0; r < 8; r++)
#pragma unroll
        for (int k = 0; k < 8; k++) c[k] = fma(c[k], 0.999999, 1e-9);
    }
#pragma unroll
    for (int k = 0; k < 8; k++) acc += c[k];
  } else {  // TMEM stores
    uint32_t v[32];
#pragma unroll
    for (int k = 0; k < 32; k++) v[k] = k + lane;
    for (int it = 0; it < iters; it++) {
      v[0] += 1;
      tst32(tb + (uint32_t)(32 * ((it + warp) & 7)), v);
    }
    acc = v[0];
  }
  unsigned long long t1 = clock64();
  if (lane == 0) clk[blockIdx.x * 16 + warp] = t1 - t0;
  if (acc == 12345.678) out[threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase_sh));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  unsigned long long* clk;
  cudaMalloc(&out, 4096 * sizeof(double));
  cudaMalloc(&clk, sms * 16 * sizeof(unsigned long long));
  const int smem = 64 * 1024;
  cudaFuncSetAttribute(mix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[16] = {};
  struct T { int mode, warps; } tests[] = {{1, 4}, {1, 8}, {1, 16}, {2, 4}, {2, 8}, {2, 16}, {4, 8}, {4, 16},
                                          {8, 4}, {8, 16}, {5, 16}, {6, 16}, {3, 16}, {7, 12}};
  (void)names;
  for (auto t : tests) {
    const int iters = 20000;
    mix_kernel<<<sms, 32 * t.warps, smem>>>(t.mode, 100, out, clk);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mix_kernel<<<sms, 32 * t.warps, smem>>>(t.mode, iters, out, clk);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[16 * 4];
    cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
    // per-role cycles (max over the role's warps in CTA 0) and bytes / lane-ops per SM per cycle
    int roles[4], nr = 0;
    for (int b = 0; b < 4; b++) if (t.mode & (1 << b)) roles[nr++] = b;
    printf("{\"mode\": %d, \"warps\": %d, \"ms\": %.3f, \"err\": %d", t.mode, t.warps, ms, (int)err);
    for (int r = 0; r < nr; r++) {
      unsigned long long mx = 0;
      int nw = 0;
      for (int w = 0; w < t.warps; w++)
        if (w % nr == r) { if (h[w] > mx) mx = h[w]; nw++; }
      const int role = roles[r];
      double per = 0;
      const char* nm = "";
      if (role == 0) { per = (double)nw * iters * 4096.0 / mx; nm = "tmem_ld_B_per_clk"; }
      if (role == 1) { per = (double)nw * iters * 8 * 512.0 / mx; nm = "lds128_B_per_clk"; }
      if (role == 2) { per = (double)nw * iters * 64 * 32.0 / mx; nm = "dfma_lanes_per_clk"; }
      if (role == 3) { per = (double)nw * iters * 4096.0 / mx; nm = "tmem_st_B_per_clk"; }
      printf(", \"%s\": %.2f, \"%s_warps\": %d", nm, per, nm, nw);
    }
    printf("}\n");
  }
  return 0;
}
