// Microbenchmarks for the hot-kernel redesign: DSMEM (16 B stores / loads / bulk copies) inside a 6-CTA
// cluster with an all-to-all pattern, and TMEM (tcgen05.ld/st 32x32b.x16) throughput per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench2 microbench2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int CL = 6;
constexpr int SM_BYTES = 190464;

__device__ __forceinline__ unsigned crank() { unsigned r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, unsigned r) { uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }

// each thread stores 16 B words round-robin to all 6 CTAs (including itself)
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(384, 1) dsm_st16(int reps, double* out, int mode) {
  extern __shared__ __align__(16) unsigned char sm[];
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  uint32_t rb[CL];
  for (int d = 0; d < CL; d++) rb[d] = mapa(base, d);
  csync();
  const int words = SM_BYTES / 16;
  double v = threadIdx.x;
  for (int k = 0; k < reps; k++) {
    for (int i = threadIdx.x; i < words; i += blockDim.x) {
      const int d = (i + k) % CL;
      if (mode == 0) {
        asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(rb[d] + i * 16), "d"(v), "d"(v + 1.0) : "memory");
      } else if (mode == 1) {
        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(rb[d] + i * 16), "d"(v) : "memory");
        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(rb[d] + i * 16 + 8), "d"(v + 1.0) : "memory");
      } else {
        // same destination for the whole warp-row: d fixed per (k) to test all-to-one burst
        asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(rb[k % CL] + i * 16), "d"(v), "d"(v + 1.0) : "memory");
      }
      v += 1.0;
    }
  }
  csync();
  if (threadIdx.x == 0 && v == -1.0) out[0] = v;
}

__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(384, 1) dsm_ld16(int reps, double* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  for (int i = threadIdx.x; i < SM_BYTES / 8; i += blockDim.x) reinterpret_cast<double*>(sm)[i] = i;
  uint32_t rb[CL];
  for (int d = 0; d < CL; d++) rb[d] = mapa(base, d);
  csync();
  const int words = SM_BYTES / 16;
  double acc = 0.0;
  for (int k = 0; k < reps; k++) {
    for (int i = threadIdx.x; i < words; i += blockDim.x) {
      const int d = (i + k) % CL;
      double a, b;
      asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "r"(rb[d] + i * 16));
      acc += a + b;
    }
  }
  csync();
  if (threadIdx.x == 0 && acc == -1.0) out[0] = acc;
}

// bulk copies: warp 0 lane 0 issues cp.async.bulk shared::cluster <- shared::cta, chunk bytes each, to all others
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(128, 1) dsm_bulk(int reps, int chunk, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t bar_a = (uint32_t)__cvta_generic_to_shared(&bar);
  const unsigned me = crank();
  const int half = SM_BYTES / 2;  // send from first half into the receivers' second half
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  csync();
  int nchunks = half / chunk;
  uint32_t phase = 0;
  for (int k = 0; k < reps; k++) {
    // expect (CL-1) * nchunks * chunk bytes arriving into my barrier
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_a), "r"((CL - 1) * nchunks * chunk) : "memory");
    }
    csync();  // all barriers armed
    if (threadIdx.x == 0) {
      for (int d = 1; d < CL; d++) {
        const unsigned dst = (me + d) % CL;
        const uint32_t rbar = mapa(bar_a, dst);
        for (int c = 0; c < nchunks; c++) {
          // each sender writes a disjoint slice of the receiver's second half
          const uint32_t src = base + c * chunk;
          const int slots = half / chunk;
          const uint32_t dsta = mapa(base + half + (((d - 1) * nchunks + c) % slots) * chunk, dst);
          asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(dsta), "r"(src), "r"(chunk), "r"(rbar) : "memory");
        }
      }
    }
    // wait for my incoming bytes
    if (threadIdx.x == 0) {
      uint32_t done = 0;
      long long guard = 0;
      while (!done && ++guard < 20000000LL) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(bar_a), "r"(phase) : "memory");
      }
    }
    phase ^= 1;
    csync();
  }
  if (threadIdx.x == 0 && reps < 0) out[0] = 1;
}

// TMEM throughput: each warp loads/stores its lane slice, x16 (16 x 32-bit per thread)
__global__ void __launch_bounds__(384, 1) tmem_bw(int reps, int mode, double* out) {
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t ta = tb + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(128 * (warp >> 2));
  uint32_t v[16];
  for (int i = 0; i < 16; i++) v[i] = threadIdx.x + i;
  uint32_t acc = 0;
  for (int k = 0; k < reps; k++) {
    for (int c = 0; c < 128; c += 16) {
      if (mode == 0) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(ta + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        acc += v[0] ^ v[15];
      } else {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                     ::"r"(ta + c), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                       "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
        v[0] += 1;
      }
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
  if (acc == 12345u) out[0] = acc;
}

int main() {
  double* out; CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  int nsm = 148;
  CK(cudaFuncSetAttribute(dsm_st16, cudaFuncAttributeMaxDynamicSharedMemorySize, SM_BYTES));
  CK(cudaFuncSetAttribute(dsm_ld16, cudaFuncAttributeMaxDynamicSharedMemorySize, SM_BYTES));
  CK(cudaFuncSetAttribute(dsm_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, SM_BYTES));
  const int ncl = 22, reps = 100;
  const double clk = 1.9e9;
  double bytes = (double)SM_BYTES * reps * 5.0 / 6.0;  // remote part per CTA
  for (int mode = 0; mode < 4; mode++) {
    if (mode == 2) continue;  // st.async needs an mbarrier operand; not used
    dsm_st16<<<ncl * CL, 384, SM_BYTES>>>(2, out, mode); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dsm_st16<<<ncl * CL, 384, SM_BYTES>>>(reps, out, mode); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"test\": \"dsmem_st_all2all_c6\", \"mode\": %d, \"remote_B_per_clk_per_sm\": %.2f, \"ms\": %.3f}\n", mode, bytes / (ms * 1e-3) / clk, ms);
  }
  dsm_ld16<<<ncl * CL, 384, SM_BYTES>>>(2, out); CK(cudaDeviceSynchronize());
  cudaEventRecord(e0); dsm_ld16<<<ncl * CL, 384, SM_BYTES>>>(reps, out); cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"test\": \"dsmem_ld16_all2all_c6\", \"remote_B_per_clk_per_sm\": %.2f, \"ms\": %.3f}\n", bytes / (ms * 1e-3) / clk, ms);
  for (int chunk : {1024}) {
    dsm_bulk<<<ncl * CL, 128, SM_BYTES>>>(2, chunk, out); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dsm_bulk<<<ncl * CL, 128, SM_BYTES>>>(reps, chunk, out); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    int nch = (SM_BYTES / 2) / chunk;
    double b = (double)(CL - 1) * nch * chunk * reps;
    printf("{\"test\": \"dsmem_bulk_c6\", \"chunk\": %d, \"recv_B_per_clk_per_sm\": %.2f, \"ms\": %.3f}\n", chunk, b / (ms * 1e-3) / clk, ms);
  }
  for (int mode = 0; mode < 2; mode++) {
    tmem_bw<<<nsm, 384>>>(2, mode, out); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); tmem_bw<<<nsm, 384>>>(2000, mode, out); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double b = 2000.0 * 8 * 16 * 4 * 384;  // per SM
    printf("{\"test\": \"tmem_%s_x16\", \"B_per_clk_per_sm\": %.2f, \"ms\": %.3f}\n", mode == 0 ? "ld" : "st", b / (ms * 1e-3) / clk, ms);
  }
  return 0;
}
