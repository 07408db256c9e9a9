// Macroscopic moments (ToConservative / ToPrimitive) and the BGK operator, fused with the FKS transport gather
// (SURVEY §8(f) NEXT-1 and NEXT-3).
//
//   U_j = sum_k phi(v_k) f_{j,k} dv^3,  phi = (1, v, |v|^2/2)
//   (rho, u, T):  u = (rho u)/rho,  (3/2) rho T = E - rho |u|^2 / 2
//   E_{j,k} = rho (2 pi T)^{-3/2} exp(-|v_k - u|^2 / 2T)   (0 if rho <= 0 or T <= 0, reading A26)
//   Q_BGK = nu (E - f)
//   BGK step: f_out = f* + nu dt (E[f*] - f*),  f* = transported f_in                      (Eq. disc_relax)
//
// HBM-bound: one thread-block cluster per spatial cell stages the whole cell in shared memory (C CTAs x 64 KB,
// asynchronous copies all in flight; 3 CTAs per SM overlap one cell's loads with another's stores), so f is read
// once and f_out written once (16 B per cell-velocity point for the step, the algorithmic minimum).  The
// Maxwellian is separable: 3N exponentials per cell instead of N^3.  The moments are reduced in a fixed order (per thread, warp
// butterfly, warps in order, cluster ranks in order over distributed shared memory), so every CTA of the cluster
// computes bit-identical (rho, u, T).
#include <cooperative_groups.h>

#include "fks_internal.cuh"

namespace fks {
namespace cg = cooperative_groups;

namespace macro {

constexpr int NT = 256;  // threads per CTA
enum Mode { MOMENTS = 0, BGK_Q = 1, BGK_STEP = 2 };

struct Args {
  const double* fin;
  double* out;        // BGK_Q: Q;  BGK_STEP: f_out;  MOMENTS: unused
  double* U;          // optional [n_cells][5] conservative moments of the (transported) input
  double* W;          // optional [n_cells][5] primitive (rho, u_x, u_y, u_z, T)
  long long n_cells;
  int N;
  int C;              // CTAs per cell (cluster size)
  int chunk;          // velocity points per CTA (C * chunk >= N^3), staged in shared memory
  int vec16;          // 1: contiguous 16-byte staging of the whole chunk (no shift, fin 16-B aligned)
  int in16, out16;    // fin / out 16-byte aligned (element pairs move as one 16-byte access)
  double L, h;        // box half-width, node spacing 2L/N
  double coef;        // BGK_Q: nu;  BGK_STEP: nu * dt
  Shift sh;           // BGK_STEP: transport shifts (identity when all zero)
};

// (kx, ky, kz) of flat index q, advanced by a fixed stride with carries (no division in the loops)
struct Idx {
  int x, y, z;
  __device__ __forceinline__ void init(int q, int N) { z = q % N; y = (q / N) % N; x = q / (N * N); }
  __device__ __forceinline__ void step(int a, int b, int c, int N) {  // + (a N^2 + b N + c), 0 <= b, c < N
    z += c;
    const int cz = z >= N;
    z -= cz ? N : 0;
    y += b + cz;
    const int cy = y >= N;
    y -= cy ? N : 0;
    x += a + cy;
  }
};

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

// v_k = -L + k h rounded exactly like the oracle's velocity_nodes (no FMA contraction)
__device__ __forceinline__ double node(int k, const Args& A) { return __dadd_rn(-A.L, __dmul_rn((double)k, A.h)); }

// NC = N when instantiated for one velocity size (index arithmetic by constants), 0 = runtime N
template <int MODE, int NC>
__global__ void __launch_bounds__(NT) macro_kernel(const Args A) {
  extern __shared__ __align__(16) double sf[];  // this CTA's velocity points [q0, q1) of the cell
  __shared__ double s_red[NT / 32][5];
  __shared__ double s_part[16][5];  // partial sums of every CTA of the cluster (pushed by their owners)
  __shared__ int sx[kMaxN], sy[kMaxN], sz[kMaxN];
  __shared__ double gx[kMaxN], gy[kMaxN], gz[kMaxN];  // separable Maxwellian factors
  __shared__ double vn[kMaxN], wn[kMaxN];             // node v_k and v_k^2 / 2
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const long long cell = (long long)blockIdx.x / A.C;
  const int N = NC ? NC : A.N, tid = threadIdx.x;
  const long long nv = (long long)N * N * N;
  const int q0 = rank * A.chunk;
  const int q1 = (int)min((long long)q0 + A.chunk, nv);  // this CTA's velocity points are [q0, q1)
  const int nh = max(q1 - q0, 0);
  // Distributed shared memory may only be accessed once every CTA of the cluster is running: arrive here, wait
  // just before the DSMEM push below (the wait hides behind the staging copies).
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");

  // ---- stage the cell's points in shared memory (asynchronous copies, all in flight at once) ----
  if (MODE == BGK_STEP) {  // source cell of every (axis, velocity index): (j - delta) mod grid
    const int jz = (int)(cell % A.sh.nz), jy = (int)((cell / A.sh.nz) % A.sh.ny);
    const int jx = (int)(cell / ((long long)A.sh.nz * A.sh.ny));
    if (tid < N) {
      int a = (jx - A.sh.delta[0][tid]) % A.sh.nx; if (a < 0) a += A.sh.nx;
      int b = (jy - A.sh.delta[1][tid]) % A.sh.ny; if (b < 0) b += A.sh.ny;
      int c = (jz - A.sh.delta[2][tid]) % A.sh.nz; if (c < 0) c += A.sh.nz;
      sx[tid] = a; sy[tid] = b; sz[tid] = c;
    }
    __syncthreads();
  }
  if (tid < N) {
    const double v = node(tid, A);
    vn[tid] = v;
    wn[tid] = 0.5 * v * v;
  }
  // every thread handles element pairs (kz, kz + 1) of one velocity row (N even): 16-byte copies and stores
  const int pa = (2 * NT) / (N * N), pb = ((2 * NT) / N) % N, pc = (2 * NT) % N;  // stride 2 NT in base N
  if (A.vec16) {
    const double* src = A.fin + cell * nv + q0;
    for (int j = 2 * tid; j < nh; j += 2 * NT) cp_async16(sf + j, src + j);
  } else {
    Idx k;
    k.init(q0 + 2 * tid, N);
    for (int j = 2 * tid; j < nh; j += 2 * NT) {
      long long s0 = cell, s1 = cell;
      if (MODE == BGK_STEP) {
        const long long row = (long long)sx[k.x] * A.sh.ny + sy[k.y];
        s0 = row * A.sh.nz + sz[k.z];
        s1 = row * A.sh.nz + sz[k.z + 1];
      }
      const double* g = A.fin + s0 * nv + q0 + j;
      if (s0 == s1 && A.in16) {
        cp_async16(sf + j, g);  // both from one source cell (the common case): one 16-byte copy
      } else {
        cp_async8(sf + j, g);
        cp_async8(sf + j + 1, A.fin + s1 * nv + q0 + j + 1);
      }
      k.step(pa, pb, pc, N);
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();

  // ---- moments: per-thread partial sums, fixed-order reduction (thread, warp butterfly, warps, ranks) ----
  double m[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  {
    Idx k;
    k.init(q0 + 2 * tid, N);
    for (int j = 2 * tid; j < nh; j += 2 * NT) {
      const double2 f = *reinterpret_cast<const double2*>(sf + j);
      const double vx = vn[k.x], vy = vn[k.y], wxy = wn[k.x] + wn[k.y];
      m[0] += f.x;
      m[0] += f.y;
      m[1] = fma(f.x + f.y, vx, m[1]);
      m[2] = fma(f.x + f.y, vy, m[2]);
      m[3] = fma(f.x, vn[k.z], m[3]);
      m[3] = fma(f.y, vn[k.z + 1], m[3]);
      m[4] = fma(f.x, wxy + wn[k.z], m[4]);
      m[4] = fma(f.y, wxy + wn[k.z + 1], m[4]);
      k.step(pa, pb, pc, N);
    }
  }
#pragma unroll
  for (int a = 0; a < 5; a++) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m[a] += __shfl_xor_sync(0xffffffffu, m[a], o);
  }
  if ((tid & 31) == 0) {
#pragma unroll
    for (int a = 0; a < 5; a++) s_red[tid >> 5][a] = m[a];
  }
  __syncthreads();
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // every peer CTA has started
  if (tid < 5 * A.C) {  // push this CTA's partial sum of component a into CTA r's s_part[rank][a]
    const int a = tid % 5, r = tid / 5;
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NT / 32; w++) s += s_red[w][a];
    cluster.map_shared_rank(&s_part[0][0], r)[rank * 5 + a] = s;
  }
  cluster.sync();  // all pushes landed; afterwards nobody touches another CTA's shared memory
  double U[5];
#pragma unroll
  for (int a = 0; a < 5; a++) U[a] = 0.0;
#pragma unroll 1
  for (int r = 0; r < A.C; r++) {
#pragma unroll
    for (int a = 0; a < 5; a++) U[a] += s_part[r][a];
  }
  const double h3 = A.h * A.h * A.h;
#pragma unroll
  for (int a = 0; a < 5; a++) U[a] *= h3;

  const double rho = U[0];
  const double ux = U[1] / rho, uy = U[2] / rho, uz = U[3] / rho;
  const double T = (U[4] - 0.5 * rho * (ux * ux + uy * uy + uz * uz)) / (1.5 * rho);
  if (rank == 0 && tid == 0) {
    if (A.U) {
#pragma unroll
      for (int a = 0; a < 5; a++) A.U[cell * 5 + a] = U[a];
    }
    if (A.W) {
      double* w = A.W + cell * 5;
      w[0] = rho; w[1] = ux; w[2] = uy; w[3] = uz; w[4] = T;
    }
  }
  if (MODE == MOMENTS) return;

  // ---- local Maxwellian E = rho (2 pi T)^{-3/2} e^{-|v-u|^2/2T}, separable: cM gx[kx] gy[ky] gz[kz] ----
  const bool have_M = (rho > 0.0) && (T > 0.0);
  const double two_pi_T = 2.0 * 3.14159265358979323846 * T;
  const double cM = have_M ? rho / (two_pi_T * sqrt(two_pi_T)) : 0.0;
  if (tid < N) {
    const double inv2T = have_M ? 1.0 / (2.0 * T) : 0.0;
    const double v = node(tid, A);
    gx[tid] = have_M ? exp(-(v - ux) * (v - ux) * inv2T) : 0.0;
    gy[tid] = have_M ? exp(-(v - uy) * (v - uy) * inv2T) : 0.0;
    gz[tid] = have_M ? exp(-(v - uz) * (v - uz) * inv2T) : 0.0;
  }
  __syncthreads();
  double* out = A.out + cell * nv + q0;
  Idx k;
  k.init(q0 + 2 * tid, N);
  for (int j = 2 * tid; j < nh; j += 2 * NT) {
    const double2 f = *reinterpret_cast<const double2*>(sf + j);
    const double cxy = cM * gx[k.x] * gy[k.y];
    const double d0 = A.coef * (cxy * gz[k.z] - f.x), d1 = A.coef * (cxy * gz[k.z + 1] - f.y);
    const double2 r = MODE == BGK_Q ? make_double2(d0, d1) : make_double2(f.x + d0, f.y + d1);
    if (A.out16) {
      __stcs(reinterpret_cast<double2*>(out + j), r);
    } else {
      __stcs(out + j, r.x);
      __stcs(out + j + 1, r.y);
    }
    k.step(pa, pb, pc, N);
  }
}

template <int MODE, int NC>
static cudaError_t launch(const Args& A, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(macro_kernel<MODE, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (A.C > 8) {
    e = cudaFuncSetAttribute(macro_kernel<MODE, NC>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(A.n_cells * A.C), 1, 1);
  cfg.blockDim = dim3(NT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = A.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, macro_kernel<MODE, NC>, A);
}

}  // namespace macro

// Launch one macro kernel over n_cells cells (MODE: 0 moments, 1 BGK operator, 2 BGK step with transport).
// U = dv^3 sum_p mpart[cell][p] (p in order), W = (rho, u, T) exactly as macro_kernel derives them
__global__ void moments_finish_kernel(const double* __restrict__ mpart, int parts, long long n, double h3, double* U,
                                      double* W) {
  const long long cell = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (cell >= n) return;
  double u[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int p = 0; p < parts; p++) {
#pragma unroll
    for (int a = 0; a < 5; a++) u[a] += mpart[(cell * parts + p) * 5 + a];
  }
#pragma unroll
  for (int a = 0; a < 5; a++) u[a] *= h3;
  if (U) {
#pragma unroll
    for (int a = 0; a < 5; a++) U[cell * 5 + a] = u[a];
  }
  if (W) {
    const double rho = u[0];
    const double ux = u[1] / rho, uy = u[2] / rho, uz = u[3] / rho;
    const double T = (u[4] - 0.5 * rho * (ux * ux + uy * uy + uz * uz)) / (1.5 * rho);
    double* w = W + cell * 5;
    w[0] = rho; w[1] = ux; w[2] = uy; w[3] = uz; w[4] = T;
  }
}

void launch_moments_finish(Ctx& c, const double* mpart, int parts, long long n_cells, double* U, double* W,
                           cudaStream_t st) {
  if (n_cells <= 0) return;
  const double h = 2.0 * c.p.L / c.N;
  moments_finish_kernel<<<(unsigned)((n_cells + 127) / 128), 128, 0, st>>>(mpart, parts, n_cells, h * h * h, U, W);
  c.launches++;
}

fks_status launch_macro(Ctx& c, int mode, const double* fin, double* out, double* U, double* W, long long n_cells,
                        double coef, const Shift* sh, cudaStream_t st) {
  if (n_cells <= 0) return FKS_OK;
  macro::Args A{};
  A.fin = fin; A.out = out; A.U = U; A.W = W;
  A.n_cells = n_cells;
  A.N = c.N;
  A.L = c.p.L;
  A.h = 2.0 * c.p.L / c.N;
  A.coef = coef;
  if (sh) A.sh = *sh;
  const long long nv = (long long)c.N * c.N * c.N;
  // 8192 points (64 KB) per CTA -> 3 CTAs per SM; 16384 (128 KB) when a cell would need more than 8 CTAs
#ifndef MACRO_CHUNK
#define MACRO_CHUNK 8192
#endif
  long long chunk = MACRO_CHUNK;
  long long C = (nv + chunk - 1) / chunk;
  if (C > 8) { chunk = 16384; C = (nv + chunk - 1) / chunk; }
  if (C > 16) { set_error("moments/BGK: N^3 too large for one 16-CTA cluster"); return FKS_ERR_UNSUPPORTED; }
  chunk = (nv + C - 1) / C;
  chunk += chunk & 1;  // even, so 16-byte staging stays aligned per CTA
  A.C = (int)C;
  A.chunk = (int)chunk;
  bool ident = true;
  if (sh) {
    for (int a = 0; a < 3; a++)
      for (int k = 0; k < c.N; k++) ident = ident && sh->delta[a][k] == 0;
  }
  A.in16 = ((uintptr_t)fin & 15) == 0;
  A.out16 = ((uintptr_t)out & 15) == 0;
  A.vec16 = (mode != 2 || ident) && A.in16;
  if (n_cells * C > 0x7fffffffLL) { set_error("moments/BGK: too many cells for one launch"); return FKS_ERR_INVALID; }
  const size_t smem = (size_t)chunk * sizeof(double);
  cudaError_t e;
  if (c.N == 32) {  // the paper's velocity grid: constant index arithmetic
    e = mode == 0 ? macro::launch<macro::MOMENTS, 32>(A, smem, st)
      : mode == 1 ? macro::launch<macro::BGK_Q, 32>(A, smem, st) : macro::launch<macro::BGK_STEP, 32>(A, smem, st);
  } else {
    e = mode == 0 ? macro::launch<macro::MOMENTS, 0>(A, smem, st)
      : mode == 1 ? macro::launch<macro::BGK_Q, 0>(A, smem, st) : macro::launch<macro::BGK_STEP, 0>(A, smem, st);
  }
  c.launches++;
  if (e != cudaSuccess) return cuda_status(e, "moments/BGK launch");
  return cuda_status(cudaPeekAtLastError(), "moments/BGK launch");
}

}  // namespace fks
