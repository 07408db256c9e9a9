// Fast path for N = 32 (P = 48): the term loop (rows a3-a5 of DESIGN.md §2) as ONE fused sm_100a kernel.
//
// One thread-block cluster of 6 CTAs per cell (measured: clusters of 6 occupy 132 of 148 SMs with ~190 KB
// of shared memory per CTA, clusters of 8 only 120).  CTA c owns the 8 padded z-planes pz in [8c, 8c+8) and
// 1/6 of the (lx, ly) pencils.  Per separated term t (T+1 = 33 or 65 times per cell):
//
//   Z phase  thread <- pencil (lx,ly): Z(l) = (a_t + i b_t)(l) f^(l) for the 31 lz (coalesced loads of the
//            pencil-interleaved f^ and table), then the pruned 48-point inverse transform along z; the 48
//            outputs W1(lx,ly,pz) go straight into the owner CTA's shared memory through DSMEM.
//   Y phase  thread <- (plane, lx): 31 -> 48 along y, in place: every thread first pulls its W1 column into
//            registers, then the region is overwritten with Y(lx,py,pz).
//   X phase  thread <- (plane, py): 31 -> 48 along x, then G(p) += Re z_t(p) * Im z_t(p)  (= A_t * B_t with the
//            balanced tables), G resident in TENSOR MEMORY (TMEM, 147 KB per CTA) for the whole term loop.
//
// Every pruned transform is z(p) = sum_{l=-15..15} Z(l) e^{2 pi i l p/48}, computed as a radix-3 DIF combine of
// the 31 inputs (outputs p = 3q + r, r = 0,1,2) followed by three 16-point radix-4x4 FFTs held in registers.
// Forward and back transforms still use the generic per-axis kernels (DESIGN.md §7 "next").
#include <cooperative_groups.h>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include "fks_internal.cuh"

namespace fks {
namespace f32 {

constexpr int N = 32, K = 31, P = 48;
constexpr int CL = 6;                 // CTAs per cell (cluster size)
constexpr int PL = P / CL;            // z-planes per CTA = 8
constexpr int NT = 384;               // threads per CTA: one per (plane, py) in the X phase
constexpr int NPEN = K * K;           // 961 pencils
constexpr int R_ELEMS = PL * P * K;   // complex elements of the shared region (Y layout) = 11904
constexpr int R_BYTES = R_ELEMS * 16; // 190464 B  (>= the W1 layout PL*K*K*16 = 123008 B)
constexpr int Y_THREADS = PL * K;     // 248

__constant__ double2 c_w48[48];       // e^{+2 pi i m/48}

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

__device__ __forceinline__ uint32_t mapa(uint32_t laddr, unsigned rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(laddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster(uint32_t addr, double2 v) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(v.x), "d"(v.y) : "memory");
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 w, double2 a) {
  return make_double2(fma(w.x, a.x, -w.y * a.y), fma(w.x, a.y, w.y * a.x));
}

// radix-3 DIF combine for output class r: u(m) = w48^{mr} (Z(m) + w3^{-r} Z(m-16)); x[i] = Z(i - 15)
template <int r>
__device__ __forceinline__ void combine(const double2 (&x)[K], double2 (&u)[16]) {
  u[0] = x[15];
#pragma unroll
  for (int m = 1; m < 16; m++) {
    const double2 a = x[m + 15], b = x[m - 1];
    if (r == 0) {
      u[m] = cadd(a, b);
    } else {
      const double ci = (r == 1) ? -0.86602540378443864676 : 0.86602540378443864676;
      double sr = fma(-0.5, b.x, a.x);
      sr = fma(-ci, b.y, sr);
      double si = fma(-0.5, b.y, a.y);
      si = fma(ci, b.x, si);
      u[m] = cmul(c_w48[(m * r) % 48], make_double2(sr, si));
    }
  }
}

__device__ __forceinline__ void bfly4_inv(double2& x0, double2& x1, double2& x2, double2& x3) {
  const double2 a = cadd(x0, x2), b = csub(x0, x2), c = cadd(x1, x3), d = csub(x1, x3);
  x0 = cadd(a, c);
  x2 = csub(a, c);
  x1 = make_double2(b.x - d.y, b.y + d.x);  // b + i d
  x3 = make_double2(b.x + d.y, b.y - d.x);  // b - i d
}

// twiddle by w16^k (k = m2*q1 in 0..9)
__device__ __forceinline__ double2 tw16(double2 v, int k) {
  const double h = 0.70710678118654752440;
  switch (k) {
    case 0: return v;
    case 2: return make_double2(h * (v.x - v.y), h * (v.x + v.y));
    case 4: return make_double2(-v.y, v.x);
    case 6: return make_double2(-h * (v.x + v.y), h * (v.x - v.y));
    default: return cmul(c_w48[3 * k], v);
  }
}

// in-place inverse 16-point DFT (positive exponent): on exit z(q) is at u[4*(q%4) + q/4]
__device__ __forceinline__ void fft16_inv(double2 (&u)[16]) {
#pragma unroll
  for (int m2 = 0; m2 < 4; m2++) bfly4_inv(u[m2], u[m2 + 4], u[m2 + 8], u[m2 + 12]);
#pragma unroll
  for (int m2 = 1; m2 < 4; m2++)
#pragma unroll
    for (int q1 = 1; q1 < 4; q1++) u[m2 + 4 * q1] = tw16(u[m2 + 4 * q1], m2 * q1);
#pragma unroll
  for (int q1 = 0; q1 < 4; q1++) bfly4_inv(u[4 * q1], u[4 * q1 + 1], u[4 * q1 + 2], u[4 * q1 + 3]);
}

// outputs z(3q + r), q = 0..15, of the pruned 48-point inverse transform of x
template <int r>
__device__ __forceinline__ void pruned48(const double2 (&x)[K], double2 (&u)[16]) {
  combine<r>(x, u);
  fft16_inv(u);
}
__device__ __forceinline__ int qslot(int q) { return 4 * (q & 3) + (q >> 2); }

// ---- TMEM helpers (tcgen05) --------------------------------------------------------------------------
__device__ __forceinline__ void tmem_ld32(uint32_t addr, uint32_t (&v)[32]) {
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
__device__ __forceinline__ void tmem_st32(uint32_t addr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      ::"r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
        "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
        "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t addr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
      ::"r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

struct HotArgs {
  const double2* fhatT;  // [cell][iz][pp], pp = ix*31 + iy
  const double2* tabT;   // [t][iz][pp]
  double* G;             // [cell][px][py][pz]
  int T1;                // T + 1 terms
};

template <int r>
__device__ __forceinline__ void x_accumulate(const double2 (&x)[K], uint32_t taddr, bool first) {
  double2 u[16];
  pruned48<r>(x, u);
#pragma unroll
  for (int h = 0; h < 2; h++) {  // two halves of 8 doubles (16 TMEM columns) to bound register pressure
    uint32_t g[16];
    const uint32_t a = taddr + r * 32 + h * 16;
    if (!first) tmem_ld16(a, g);
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const int q = 8 * h + j;
      const double2 z = u[qslot(q)];
      double acc = first ? z.x * z.y : fma(z.x, z.y, __hiloint2double((int)g[2 * j + 1], (int)g[2 * j]));
      g[2 * j] = (uint32_t)__double2loint(acc);
      g[2 * j + 1] = (uint32_t)__double2hiint(acc);
    }
    tmem_st16(a, g);
  }
}

template <int r>
__device__ __forceinline__ void z_scatter(const double2 (&x)[K], const uint32_t (&rbase)[CL], int lx, int ly) {
  double2 u[16];
  pruned48<r>(x, u);
#pragma unroll
  for (int q = 0; q < 16; q++) {
    const int pz = 3 * q + r, d = pz / PL, s = pz % PL;
    st_cluster(rbase[d] + (uint32_t)(((s * K + lx) * K + ly) * 16), u[qslot(q)]);
  }
}

template <int r>
__device__ __forceinline__ void y_store(const double2 (&x)[K], double2* R, int s, int lx) {
  double2 u[16];
  pruned48<r>(x, u);
#pragma unroll
  for (int q = 0; q < 16; q++) {
    const int py = 3 * q + r;
    R[(s * P + py) * K + lx] = u[qslot(q)];
  }
}

__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(NT, 1) hot_kernel(HotArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  double2* R = reinterpret_cast<double2*>(smem);
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5;
  const unsigned crank = cluster_rank();
  const long long cell = blockIdx.x / CL;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                 ::"r"((uint32_t)__cvta_generic_to_shared(&tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tmem_base_sh;
  // thread's TMEM row: lane 32*(warp%4) + lane, 96 columns (48 doubles) at column 96*(warp/4)
  const uint32_t taddr = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(96 * (warp >> 2));

  const int p0 = (int)(crank * NPEN) / CL, p1 = (int)((crank + 1) * NPEN) / CL;
  const int npc = p1 - p0;
  const uint32_t lbase = (uint32_t)__cvta_generic_to_shared(R);
  uint32_t rbase[CL];
#pragma unroll
  for (int d = 0; d < CL; d++) rbase[d] = mapa(lbase, d);

  // all CTAs of the cluster are running before any DSMEM traffic
  cluster_arrive();
  cluster_wait();
  cluster_arrive();  // "R free" for term 0

  const long long fstride = (long long)K * NPEN;
  for (int t = 0; t < A.T1; t++) {
    // ---------------- Z phase ----------------
    double2 x[K];
    const bool zact = tid < npc;
    const int pp = p0 + tid, lx = pp / K, ly = pp - (pp / K) * K;
    if (zact) {
      const double2* fh = A.fhatT + cell * fstride + pp;
      const double2* tb = A.tabT + (long long)t * fstride + pp;
#pragma unroll
      for (int i = 0; i < K; i++) {
        const double2 f = __ldg(fh + i * NPEN), ab = __ldg(tb + i * NPEN);
        x[i] = make_double2(fma(ab.x, f.x, -ab.y * f.y), fma(ab.x, f.y, ab.y * f.x));
      }
    }
    cluster_wait();  // every CTA finished reading its region for the previous term
    if (zact) {
      z_scatter<0>(x, rbase, lx, ly);
      z_scatter<1>(x, rbase, lx, ly);
      z_scatter<2>(x, rbase, lx, ly);
    }
    cluster_arrive();
    cluster_wait();  // all W1 planes delivered

    // ---------------- Y phase (in place) ----------------
    const bool yact = tid < Y_THREADS;
    const int ys = tid / K, ylx = tid - (tid / K) * K;
    if (yact) {
#pragma unroll
      for (int i = 0; i < K; i++) x[i] = R[(ys * K + ylx) * K + i];
    }
    __syncthreads();
    if (yact) {
      y_store<0>(x, R, ys, ylx);
      y_store<1>(x, R, ys, ylx);
      y_store<2>(x, R, ys, ylx);
    }
    __syncthreads();

    // ---------------- X phase ----------------
    const int xs = tid / P, xpy = tid - (tid / P) * P;
#pragma unroll
    for (int i = 0; i < K; i++) x[i] = R[(xs * P + xpy) * K + i];
    cluster_arrive();  // done reading the region: the next term may write into it
    const bool first = (t == 0);
    x_accumulate<0>(x, taddr, first);
    x_accumulate<1>(x, taddr, first);
    x_accumulate<2>(x, taddr, first);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  cluster_wait();

  // ---------------- write G[cell][px][py][pz] ----------------
  {
    const int xs = tid / P, xpy = tid - (tid / P) * P;
    const int pz = (int)crank * PL + xs;
    double* Gc = A.G + cell * (long long)(P * P * P);
#pragma unroll
    for (int r = 0; r < 3; r++) {
      uint32_t g[32];
      tmem_ld32(taddr + r * 32, g);
#pragma unroll
      for (int q = 0; q < 16; q++) {
        const int px = 3 * q + r;
        Gc[(px * P + xpy) * P + pz] = __hiloint2double((int)g[2 * q + 1], (int)g[2 * q]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

// f^ [cell][ix][iy][iz] -> [cell][iz][ix*31+iy]
__global__ void transpose_hat_kernel(const double2* __restrict__ in, double2* __restrict__ out, long long n) {
  const long long total = n * K * NPEN;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long cell = i / (K * NPEN);
    const int rem = (int)(i - cell * K * NPEN), iz = rem / NPEN, pp = rem - iz * NPEN;
    out[i] = in[cell * K * NPEN + (long long)pp * K + iz];
  }
}

}  // namespace f32

bool fast_available(const Ctx& c) { return c.N == 32 && c.P == 48; }

size_t xform32_ws_bytes_per_cell();
void xform32_forward(Ctx& c, const double* fin, double2* fhT, double2* scratch, long long n, cudaStream_t st);
void xform32_back(Ctx& c, const double* G, double2* scratch_a, double2* scratch_b, const double* fin, double* out,
                  long long n, bool euler, double s, cudaStream_t st);

size_t fast_ws_bytes_per_cell(const Ctx&) { return xform32_ws_bytes_per_cell(); }

fks_status fast_prepare(Ctx& c) {
  using namespace f32;
  double2 w[48];
  for (int m = 0; m < 48; m++) {
    const long double a = 2.0L * 3.14159265358979323846264338327950288L * m / 48.0L;
    w[m] = make_double2((double)cosl(a), (double)sinl(a));
  }
  cudaError_t e = cudaMemcpyToSymbol(c_w48, w, sizeof(w));
  if (e != cudaSuccess) return cuda_status(e, "fast constants");
  size_t n = (size_t)(c.T + 1) * K * NPEN;
  e = cudaMalloc(&c.d_abT, n * sizeof(double2));
  if (e != cudaSuccess) { cudaGetLastError(); return cuda_status(e, "fast table allocation"); }
  // reuse the transpose kernel over the T+1 tables: each "cell" is one term
  transpose_hat_kernel<<<(unsigned)std::min<size_t>((n + 255) / 256, 4096), 256>>>(c.d_ab, c.d_abT, c.T + 1);
  c.launches++;
  e = cudaFuncSetAttribute(hot_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, R_BYTES);
  if (e != cudaSuccess) return cuda_status(e, "fast kernel attributes");
  c.fast_cluster = CL;
  return cuda_status(cudaDeviceSynchronize(), "fast prepare");
}

fks_status fast_collision(Ctx& c, const double* fin, double* out, long long n, bool euler, double s,
                          cudaStream_t st) {
  using namespace f32;
  // workspace: f^T [n][K^3] complex | scratch [n][P*K*16] complex | G [n][P^3] fp64
  double2* fhT = reinterpret_cast<double2*>(c.d_ws);
  double2* scratch = fhT + n * K * NPEN;
  double* G = reinterpret_cast<double*>(scratch + n * (long long)P * K * 16);
  c.prof.begin(1, st);
  xform32_forward(c, fin, fhT, scratch, n, st);
  c.prof.end(1, st);

  c.prof.begin(2, st);
  HotArgs A{fhT, c.d_abT, G, c.T + 1};
  hot_kernel<<<(unsigned)(n * CL), NT, R_BYTES, st>>>(A);
  c.launches++;
  c.prof.end(2, st);
  fks_status rc = cuda_status(cudaPeekAtLastError(), "fast hot kernel launch");
  if (rc) return rc;

  c.prof.begin(3, st);
  xform32_back(c, G, scratch, fhT, fin, out, n, euler, s, st);
  c.prof.end(3, st);
  return cuda_status(cudaPeekAtLastError(), "fast collision");
}

}  // namespace fks
