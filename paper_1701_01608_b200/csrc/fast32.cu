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
#include <cstdlib>
#include <string>
#include "fks_internal.cuh"

namespace fks {
namespace f32 {

constexpr int N = 32, K = 31, P = 48;
constexpr int CL = 6;                 // CTAs per cell (cluster size)
constexpr int PL = P / CL;            // z-planes per CTA = 8
constexpr int NT = 384;               // threads per CTA: one per (plane, py) in the X phase
constexpr int NPEN = K * K;           // 961 pencils
constexpr int R_ELEMS = PL * P * K;   // complex elements of the shared region (Y layout) = 11904
constexpr int R_BYTES = R_ELEMS * 16; // 190464 B: Y planes of this CTA in shared memory
constexpr int Y_THREADS = PL * K;     // 248

__constant__ double2 c_w48[48];       // e^{+2 pi i m/48}

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 w, double2 a) {
  return make_double2(fma(w.x, a.x, -w.y * a.y), fma(w.x, a.y, w.y * a.x));
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

__device__ __forceinline__ int qslot(int q) { return 4 * (q & 3) + (q >> 2); }

// ---- TMEM helpers (tcgen05) --------------------------------------------------------------------------
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

// ---- mbarrier + TMA bulk copies (global -> this CTA's shared memory) ----------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  uint32_t done = 0;
  long long spins = 0;
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(a), "r"(parity) : "memory");
    if (++spins > (1LL << 28)) asm volatile("trap;");  // never hang the GPU on a byte-count bug
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
                 "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}

struct HotArgs {
  const double2* fhatT;  // [cell][LHN]: lower-half pencils in per-CTA blocks (xform32.cu lh_offset)
  const double2* tabT;   // [t][LHN]
  double* G;             // [cell][px][py][pz]
  double2* W1;           // [cluster][2][pz][pp]: double-buffered, L2-resident exchange of the z-pass output
  long long n_cells;
  int T1;                // T + 1 terms
  long long* dbg;        // optional phase timestamps (tools/phase_timing.py); nullptr in production
};

constexpr int W1_BUF = P * NPEN;  // complex elements per buffer (738 KB)
constexpr int LHN = K * (NPEN / 2 + 1);  // lower-half block layout: 14911 complex per cell / per term

// Pack / unpack one complex double as 4 x 32-bit TMEM words.
__device__ __forceinline__ void pack4(uint32_t* w, double2 v) {
  w[0] = (uint32_t)__double2loint(v.x); w[1] = (uint32_t)__double2hiint(v.x);
  w[2] = (uint32_t)__double2loint(v.y); w[3] = (uint32_t)__double2hiint(v.y);
}
__device__ __forceinline__ double2 unpack4(const uint32_t* w) {
  return make_double2(__hiloint2double((int)w[1], (int)w[0]), __hiloint2double((int)w[3], (int)w[2]));
}

// u(m) for one output class r from a = Z(m) (m = 1..15) and b = Z(m-16)
template <int r>
__device__ __forceinline__ double2 comb1(int m, double2 a, double2 b) {
  if (r == 0) return cadd(a, b);
  const double ci = (r == 1) ? -0.86602540378443864676 : 0.86602540378443864676;
  double sr = fma(-0.5, b.x, a.x);
  sr = fma(-ci, b.y, sr);
  double si = fma(-0.5, b.y, a.y);
  si = fma(ci, b.x, si);
  return cmul(c_w48[(m * r) % 48], make_double2(sr, si));
}

// Parked-input variant: xa[j] = Z(j) for j = 0..15 in registers; Z(m-16), m = 1..15, parked in TMEM at tP
// (4 chunks of 4 complex = 16 columns each).
template <int r>
__device__ __forceinline__ void combine_parked(const double2 (&xa)[16], uint32_t tP, double2 (&u)[16]) {
  u[0] = xa[0];
#pragma unroll
  for (int c = 0; c < 4; c++) {
    uint32_t w[16];
    tmem_ld16(tP + 16 * c, w);
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const int m = 4 * c + k + 1;
      if (m <= 15) u[m] = comb1<r>(m, xa[m], unpack4(w + 4 * k));
    }
  }
}

// Shared-memory variant: row[i] = Z(i - 15), i = 0..30
template <int r>
__device__ __forceinline__ void combine_smem(const double2* row, double2 (&u)[16]) {
  u[0] = row[15];
#pragma unroll
  for (int m = 1; m < 16; m++) u[m] = comb1<r>(m, row[m + 15], row[m - 1]);
}

// Park b = Z(i - 15), i = 0..14, given by `get(i)`; keep xa[j] = Z(j) = input i = j + 15.
template <typename Get>
__device__ __forceinline__ void load_and_park(Get get, uint32_t tP, double2 (&xa)[16]) {
#pragma unroll
  for (int c = 0; c < 4; c++) {
    uint32_t w[16];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const int i = 4 * c + k;
      if (i < 15) pack4(w + 4 * k, get(i));
      else { w[4 * k] = w[4 * k + 1] = w[4 * k + 2] = w[4 * k + 3] = 0u; }
    }
    tmem_st16(tP + 16 * c, w);
  }
#pragma unroll
  for (int j = 0; j < 16; j++) xa[j] = get(15 + j);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// one output class r of the z-pass of one pencil: inputs Z(i - 15) at Zs[i * ld], outputs to W1b[pz][pp]
template <int r>
__device__ __forceinline__ void z_task(const double2* Zs, int ld, double2* W1b, int pp, bool act) {
  double2 u[16];
  u[0] = Zs[15 * ld];
#pragma unroll
  for (int m = 1; m < 16; m++) u[m] = comb1<r>(m, Zs[(m + 15) * ld], Zs[(m - 1) * ld]);
  fft16_inv(u);
  if (act) {
#pragma unroll
    for (int q = 0; q < 16; q++) W1b[(3 * q + r) * NPEN + pp] = u[qslot(q)];
  }
}

template <int r>
__device__ __forceinline__ void z_out(const double2 (&xa)[16], uint32_t tP, double2* W1b, int pp, bool act) {
  double2 u[16];
  combine_parked<r>(xa, tP, u);
  fft16_inv(u);
  if (act) {
#pragma unroll
    for (int q = 0; q < 16; q++) W1b[(3 * q + r) * NPEN + pp] = u[qslot(q)];
  }
}

template <int r>
__device__ __forceinline__ void y_out(const double2 (&xa)[16], uint32_t tP, double2* Ysh, int s, int lx, bool act) {
  double2 u[16];
  combine_parked<r>(xa, tP, u);
  fft16_inv(u);
  if (act) {
#pragma unroll
    for (int q = 0; q < 16; q++) Ysh[(s * P + 3 * q + r) * K + lx] = u[qslot(q)];
  }
}

template <int r>
__device__ __forceinline__ void x_acc(const double2* row, uint32_t tG, bool first) {
  double2 u[16];
  combine_smem<r>(row, u);
  fft16_inv(u);
#pragma unroll
  for (int h = 0; h < 2; h++) {  // two halves of 8 doubles (16 TMEM columns)
    uint32_t g[16];
    const uint32_t a = tG + r * 32 + h * 16;
    if (!first) tmem_ld16(a, g);
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const double2 z = u[qslot(8 * h + j)];
      const double acc = first ? z.x * z.y : fma(z.x, z.y, __hiloint2double((int)g[2 * j + 1], (int)g[2 * j]));
      g[2 * j] = (uint32_t)__double2loint(acc);
      g[2 * j + 1] = (uint32_t)__double2hiint(acc);
    }
    tmem_st16(a, g);
  }
}

// Persistent kernel: one 6-CTA cluster per resident cell slot, looping over cells.
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(NT, 1) hot_kernel(HotArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  double2* Ysh = reinterpret_cast<double2*>(smem);  // [PL][P][K]
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5;
  const unsigned crank = cluster_rank();
  const long long cid = blockIdx.x / CL, ncl = gridDim.x / CL;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                 ::"r"((uint32_t)__cvta_generic_to_shared(&tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tmem_base_sh;
  // TMEM row of this thread: lane 32*(warp%4) + lane; per warp slot (warp/4): G in 96 columns, parking in 64
  const uint32_t trow = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
  const uint32_t tG = trow + (uint32_t)(96 * (warp >> 2));
  const uint32_t tP = trow + 288u + (uint32_t)(64 * (warp >> 2));

  // Hermitian pairing: CTA c stages the lower-half pencils pp in [h0, h1) (pp <= 480) and also transforms their
  // mirrors 960 - pp = (-lx, -ly): Z(-lx,-ly,lz) = (a+ib)(lx,ly,-lz) conj(f^(lx,ly,-lz)) (a, b even; f real)
  constexpr int NLOW = NPEN / 2 + 1;  // 481 pencils with pp <= 480 (pp = 480 is its own mirror)
  const int h0 = (int)(crank * NLOW) / CL, h1 = (int)((crank + 1) * NLOW) / CL;
  const int nh = h1 - h0;                       // staged pencils (80 or 81)
  const int nmir = (h1 == NLOW) ? nh - 1 : nh;  // mirrors (the centre pencil has none)
  double2* W1c = A.W1 + cid * 2LL * W1_BUF;
  const long long fstride = (long long)K * NPEN;

  __shared__ __align__(8) uint64_t bar;
  if (tid == 0) mbar_init(&bar);
  __syncthreads();
  uint32_t parity = 0;
  double2* stage = Ysh;  // the Y region doubles as the staging area of each phase's inputs
  long long* dbg = (A.dbg && tid == 0) ? A.dbg + (long long)blockIdx.x * 64 : nullptr;
  for (long long cell = cid; cell < A.n_cells; cell += ncl) {
    for (int t = 0; t < A.T1; t++) {
      const bool rec = dbg && cell == cid && t >= 2 && t < 6;
      if (rec) dbg[(t - 2) * 8 + 0] = clock64();
      double2* W1b = W1c + (t & 1) * (long long)W1_BUF;
      // ---------------- Z phase ----------------
      // stage f^[cell][lz][p0..p1) and table[t][lz][p0..p1) (31 contiguous runs each) into shared memory
      __syncthreads();  // previous X phase done with the region
      if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t blk = (uint32_t)(K * nh) * 16u;  // this CTA's contiguous block (lower-half layout)
        mbar_expect(&bar, 2u * blk);
        bulk_g2s(stage, A.fhatT + cell * (long long)LHN + K * h0, blk, &bar);
        bulk_g2s(stage + K * nh, A.tabT + (long long)t * LHN + K * h0, blk, &bar);
      }
      mbar_wait(&bar, parity);
      parity ^= 1;
      if (rec) dbg[(t - 2) * 8 + 6] = clock64();
      // Z of the staged pencils (over the f^ stage) and of their mirrors (over the table stage): the element
      // pair {i, 30 - i} of pencil j is handled by one thread, so the in-place writes never race.
      for (int e = tid; e < 16 * nh; e += NT) {
        const int i = e / nh, j = e - (e / nh) * nh, i2 = 30 - i;
        const double2 f1 = stage[i * nh + j], a1 = stage[(K + i) * nh + j];
        const double2 f2 = stage[i2 * nh + j], a2 = stage[(K + i2) * nh + j];
        stage[i * nh + j] = make_double2(fma(a1.x, f1.x, -a1.y * f1.y), fma(a1.x, f1.y, a1.y * f1.x));
        stage[i2 * nh + j] = make_double2(fma(a2.x, f2.x, -a2.y * f2.y), fma(a2.x, f2.y, a2.y * f2.x));
        // mirror at lz index i uses (a+ib) and conj(f^) at index 30 - i
        stage[(K + i) * nh + j] = make_double2(fma(a2.x, f2.x, a2.y * f2.y), fma(-a2.x, f2.y, a2.y * f2.x));
        stage[(K + i2) * nh + j] = make_double2(fma(a1.x, f1.x, a1.y * f1.y), fma(-a1.x, f1.y, a1.y * f1.x));
      }
      __syncthreads();
      if (rec) dbg[(t - 2) * 8 + 7] = clock64();
      // (pencil, r) tasks, warp-uniform r: slot k = r*192 + j; j < nh: staged pencil, nh <= j < nh + nmir: mirror
      for (int k = tid; k < 3 * 192; k += NT) {
        const int r = k / 192, j = k - r * 192;
        const bool act = j < nh + nmir;
        const bool mir = j >= nh;
        const int jj = act ? (mir ? j - nh : j) : 0;
        const double2* Zs = stage + (mir ? K * nh : 0) + jj;
        const int pp = mir ? (NPEN - 1) - (h0 + jj) : h0 + jj;
        if (r == 0) z_task<0>(Zs, nh, W1b, pp, act);
        else if (r == 1) z_task<1>(Zs, nh, W1b, pp, act);
        else z_task<2>(Zs, nh, W1b, pp, act);
      }
      if (rec) dbg[(t - 2) * 8 + 1] = clock64();
      cluster_arrive();
      cluster_wait();  // the z-pass output of every CTA is in W1b (release/acquire at cluster scope)
      if (rec) dbg[(t - 2) * 8 + 2] = clock64();

      // ---------------- Y phase ----------------
      // stage this CTA's 8 planes W1b[8c + s][0..961) into the region, then transform in place
      if (tid == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect(&bar, (uint32_t)(PL * NPEN * 16));
        for (int sp = 0; sp < PL; sp++)
          bulk_g2s(stage + sp * NPEN, W1b + (long long)(crank * PL + sp) * NPEN, NPEN * 16, &bar);
      }
      mbar_wait(&bar, parity);
      parity ^= 1;
      {
        const bool act = tid < Y_THREADS;
        const int ys = act ? tid / K : 0, ylx = act ? tid - (tid / K) * K : 0;
        const double2* src = stage + ys * NPEN + ylx * K;
        double2 xa[16];
        if (warp < 8) load_and_park([&](int i) { return src[i]; }, tP, xa);
        __syncthreads();  // every input is in registers / TMEM: the region may now receive Y
        if (warp < 8) {
          y_out<0>(xa, tP, Ysh, ys, ylx, act);
          y_out<1>(xa, tP, Ysh, ys, ylx, act);
          y_out<2>(xa, tP, Ysh, ys, ylx, act);
        }
      }
      if (rec) dbg[(t - 2) * 8 + 3] = clock64();
      __syncthreads();
      if (rec) dbg[(t - 2) * 8 + 4] = clock64();

      // ---------------- X phase (all warps) ----------------
      {
        const int xs = tid / P, xpy = tid - (tid / P) * P;
        const double2* row = Ysh + (xs * P + xpy) * K;
        const bool first = (t == 0);
        x_acc<0>(row, tG, first);
        x_acc<1>(row, tG, first);
        x_acc<2>(row, tG, first);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      if (rec) dbg[(t - 2) * 8 + 5] = clock64();
    }
    // ---------------- write G[cell][px][py][pz] ----------------
    {
      const int xs = tid / P, xpy = tid - (tid / P) * P;
      const int pz = (int)crank * PL + xs;
      double* Gc = A.G + cell * (long long)(P * P * P);
#pragma unroll
      for (int r = 0; r < 3; r++) {
#pragma unroll
        for (int h = 0; h < 2; h++) {
          uint32_t g[16];
          tmem_ld16(tG + r * 32 + h * 16, g);
#pragma unroll
          for (int j = 0; j < 8; j++) {
            const int px = 3 * (8 * h + j) + r;
            Gc[(px * P + xpy) * P + pz] = __hiloint2double((int)g[2 * j + 1], (int)g[2 * j]);
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}


// ======================================================================================================
// v3: teams of 12 CTAs per cell, TWO CTAs per SM (cooperative persistent grid, global-memory team barrier).
// Each CTA owns 4 z-planes and ~1/12 of the pencils; per SM the two resident CTAs belong to different cells,
// so one CTA's L2 staging / barrier wait overlaps the other's FP64 work.
// ======================================================================================================
namespace t12 {
constexpr int TM = 12;                      // CTAs per cell (team)
constexpr int PL = P / TM;                  // 4 planes per CTA
constexpr int NT = 192;                     // threads per CTA: one per (plane, py) in the X phase
constexpr int R_BYTES = PL * P * K * 16;    // 95232 B
constexpr int Y_THREADS = PL * K;           // 124
constexpr int ZSLOT = 96;                   // task slots per output class (>= 41 staged + 41 mirrored pencils)

struct Args {
  const double2* fhatT;  // [cell][LHN], 12 blocks
  const double2* tabT;   // [t][LHN], 12 blocks
  double* G;             // [cell][px][py][pz]
  double2* W1;           // [team][2][pz][pp]
  unsigned* ctr;         // [team * 32]: monotonic team-barrier counters (zeroed before launch)
  long long n_cells;
  int T1;
  long long* dbg;
  long long phase_shift;  // start delay of warp group 1, in clock cycles
};

__device__ __forceinline__ void team_barrier(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    unsigned v;
    long long spins = 0;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if (++spins > (1LL << 30)) asm volatile("trap;");
    } while (v < target);
  }
  __syncthreads();
}

// Group-local barrier of the 6 warps of warp group g (named barrier 1 + g; barrier 0 is __syncthreads).
__device__ __forceinline__ void gsync(int g) { asm volatile("bar.sync %0, 192;" ::"r"(1 + g) : "memory"); }

__device__ __forceinline__ void team_barrier_g(unsigned* ctr, unsigned target, int g, int ltid) {
  gsync(g);
  if (ltid == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    unsigned v;
    long long spins = 0;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if (++spins > (1LL << 30)) asm volatile("trap;");
    } while (v < target);
  }
  gsync(g);
}

// One CTA of 384 threads = two independent "virtual CTAs" (warp groups of 6 warps), each the k-th member of a
// different team; they share the SM's TMEM (256 columns each) and shared memory (95 KB each).
__global__ void __launch_bounds__(2 * NT, 1) hot_kernel_t12(Args A) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t tmem_base_sh;
  __shared__ __align__(8) uint64_t bars[2];
  const int tid = threadIdx.x, warp = tid >> 5;
  const int g = warp / 6, ltid = tid - g * NT, lwarp = warp - 6 * g;
  double2* Ysh = reinterpret_cast<double2*>(smem + g * R_BYTES);  // [PL][P][K]; also the staging area
  double2* stage = Ysh;
  uint64_t* bar = &bars[g];
  const int v = g * gridDim.x + blockIdx.x;  // virtual CTA id: the two groups of a CTA belong to different teams
  const int team = v / TM, k = v - (v / TM) * TM, nteams = (2 * gridDim.x) / TM;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                 ::"r"((uint32_t)__cvta_generic_to_shared(&tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (ltid == 0) mbar_init(bar);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tmem_base_sh;
  const uint32_t trow = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(256 * g);
  const uint32_t tG = trow + (uint32_t)(96 * (lwarp >> 2));  // local warps 0-3: cols 0-95, 4-5: 96-191
  const uint32_t tP = trow + 192u;                           // parking (Y phase: local warps 0-3 only)

  constexpr int NLOW = NPEN / 2 + 1;
  const int h0 = (k * NLOW) / TM, h1 = ((k + 1) * NLOW) / TM;
  const int nh = h1 - h0;
  const int nmir = (h1 == NLOW) ? nh - 1 : nh;
  double2* W1c = A.W1 + (long long)team * 2LL * W1_BUF;
  unsigned* ctr = A.ctr + team * 32;
  unsigned target = 0;
  uint32_t parity = 0;
  long long* dbg = (A.dbg && ltid == 0) ? A.dbg + (long long)v * 64 : nullptr;
  // Start the second warp group about half a term later so that the memory-bound Z/Y phases of one group
  // overlap the compute-bound X phase of the other (A.phase_shift cycles; 0 disables).
  if (g == 1 && A.phase_shift > 0) {
    const long long t0 = clock64();
    while (clock64() - t0 < A.phase_shift) __nanosleep(1000);
  }

  for (long long cell = team; cell < A.n_cells; cell += nteams) {
    for (int t = 0; t < A.T1; t++) {
      const bool rec = dbg && cell == team && t >= 2 && t < 6;
      if (rec) dbg[(t - 2) * 8 + 0] = clock64();
      double2* W1b = W1c + (t & 1) * (long long)W1_BUF;
      // ---------------- Z phase ----------------
      gsync(g);
      if (ltid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t blk = (uint32_t)(K * nh) * 16u;
        mbar_expect(bar, 2u * blk);
        bulk_g2s(stage, A.fhatT + cell * (long long)LHN + K * h0, blk, bar);
        bulk_g2s(stage + K * nh, A.tabT + (long long)t * LHN + K * h0, blk, bar);
      }
      mbar_wait(bar, parity);
      parity ^= 1;
      if (rec) dbg[(t - 2) * 8 + 6] = clock64();
      for (int e = ltid; e < 16 * nh; e += NT) {
        const int i = e / nh, j = e - (e / nh) * nh, i2 = 30 - i;
        const double2 f1 = stage[i * nh + j], a1 = stage[(K + i) * nh + j];
        const double2 f2 = stage[i2 * nh + j], a2 = stage[(K + i2) * nh + j];
        stage[i * nh + j] = make_double2(fma(a1.x, f1.x, -a1.y * f1.y), fma(a1.x, f1.y, a1.y * f1.x));
        stage[i2 * nh + j] = make_double2(fma(a2.x, f2.x, -a2.y * f2.y), fma(a2.x, f2.y, a2.y * f2.x));
        stage[(K + i) * nh + j] = make_double2(fma(a2.x, f2.x, a2.y * f2.y), fma(-a2.x, f2.y, a2.y * f2.x));
        stage[(K + i2) * nh + j] = make_double2(fma(a1.x, f1.x, a1.y * f1.y), fma(-a1.x, f1.y, a1.y * f1.x));
      }
      gsync(g);
      if (rec) dbg[(t - 2) * 8 + 7] = clock64();
      for (int kk = ltid; kk < 3 * ZSLOT; kk += NT) {
        const int r = kk / ZSLOT, j = kk - r * ZSLOT;
        const bool act = j < nh + nmir;
        const bool mir = j >= nh;
        const int jj = act ? (mir ? j - nh : j) : 0;
        const double2* Zs = stage + (mir ? K * nh : 0) + jj;
        const int pp = mir ? (NPEN - 1) - (h0 + jj) : h0 + jj;
        if (r == 0) z_task<0>(Zs, nh, W1b, pp, act);
        else if (r == 1) z_task<1>(Zs, nh, W1b, pp, act);
        else z_task<2>(Zs, nh, W1b, pp, act);
      }
      if (rec) dbg[(t - 2) * 8 + 1] = clock64();
      target += TM;
      team_barrier_g(ctr, target, g, ltid);  // every member of the team has stored its z-pass output
      if (rec) dbg[(t - 2) * 8 + 2] = clock64();

      // ---------------- Y phase ----------------
      if (ltid == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect(bar, (uint32_t)(PL * NPEN * 16));
        for (int sp = 0; sp < PL; sp++)
          bulk_g2s(stage + sp * NPEN, W1b + (long long)(k * PL + sp) * NPEN, NPEN * 16, bar);
      }
      mbar_wait(bar, parity);
      parity ^= 1;
      {
        const bool act = ltid < Y_THREADS;
        const int ys = act ? ltid / K : 0, ylx = act ? ltid - (ltid / K) * K : 0;
        const double2* src = stage + ys * NPEN + ylx * K;
        double2 xa[16];
        if (lwarp < 4) load_and_park([&](int i) { return src[i]; }, tP, xa);
        gsync(g);
        if (lwarp < 4) {
          y_out<0>(xa, tP, Ysh, ys, ylx, act);
          y_out<1>(xa, tP, Ysh, ys, ylx, act);
          y_out<2>(xa, tP, Ysh, ys, ylx, act);
        }
      }
      if (rec) dbg[(t - 2) * 8 + 3] = clock64();
      gsync(g);
      if (rec) dbg[(t - 2) * 8 + 4] = clock64();
      // ---------------- X phase ----------------
      {
        const int xs = ltid / P, xpy = ltid - (ltid / P) * P;
        const double2* row = Ysh + (xs * P + xpy) * K;
        const bool first = (t == 0);
        x_acc<0>(row, tG, first);
        x_acc<1>(row, tG, first);
        x_acc<2>(row, tG, first);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      if (rec) dbg[(t - 2) * 8 + 5] = clock64();
    }
    {
      const int xs = ltid / P, xpy = ltid - (ltid / P) * P;
      const int pz = k * PL + xs;
      double* Gc = A.G + cell * (long long)(P * P * P);
#pragma unroll
      for (int r = 0; r < 3; r++) {
#pragma unroll
        for (int h = 0; h < 2; h++) {
          uint32_t gg[16];
          tmem_ld16(tG + r * 32 + h * 16, gg);
#pragma unroll
          for (int j = 0; j < 8; j++) {
            const int px = 3 * (8 * h + j) + r;
            Gc[(px * P + xpy) * P + pz] = __hiloint2double((int)gg[2 * j + 1], (int)gg[2 * j]);
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}
}  // namespace t12

}  // namespace f32

bool fast_available(const Ctx& c) { return c.N == 32 && c.P == 48; }

size_t xform32_ws_bytes_per_cell();
cudaError_t xform32_prepare();
void xform32_tables_lh(const double2* ab, double2* abL, int T1, int nb);
void xform32_forward(Ctx& c, const double* fin, double2* fhT, double2* scratch, long long n, int nb, cudaStream_t st);
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
  if (e == cudaSuccess) e = xform32_prepare();
  if (e != cudaSuccess) return cuda_status(e, "fast constants");
  e = cudaFuncSetAttribute(hot_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, R_BYTES);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(t12::hot_kernel_t12, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * t12::R_BYTES);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(t12::hot_kernel_t12, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return cuda_status(e, "fast kernel attributes");
  // variant: two CTAs per SM (teams of 12, default) unless FKS_HOT=c6 or the occupancy does not allow it
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, t12::hot_kernel_t12, 2 * t12::NT, 2 * t12::R_BYTES);
  if (e != cudaSuccess) { cudaGetLastError(); per_sm = 0; }
  if (std::getenv("FKS_DEBUG")) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, t12::hot_kernel_t12);
    fprintf(stderr, "[fks] t12 occupancy per SM = %d (err %d), regs %d, static smem %zu, dyn %d, maxthreads %d\n",
            per_sm, (int)e, fa.numRegs, fa.sharedSizeBytes, t12::R_BYTES, fa.maxThreadsPerBlock);

  }
  const char* hv = std::getenv("FKS_HOT");
  const bool want_c6 = hv && std::string(hv) == "c6";
  c.fast_variant = (!want_c6 && per_sm >= 1) ? t12::TM : CL;
  size_t w1_elems;
  if (c.fast_variant == t12::TM) {
    c.fast_nteams = (2 * c.num_sms) / t12::TM;  // two virtual CTAs (warp groups) per SM
    w1_elems = (size_t)c.fast_nteams * 2 * W1_BUF;
    e = cudaMalloc(&c.d_ctr, (size_t)c.fast_nteams * 32 * sizeof(unsigned));
    if (e != cudaSuccess) { cudaGetLastError(); return cuda_status(e, "team counters"); }
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL * 64);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = R_BYTES;
    int ncl = 0;
    e = cudaOccupancyMaxActiveClusters(&ncl, hot_kernel, &cfg);
    if (e != cudaSuccess || ncl <= 0) { cudaGetLastError(); ncl = 22; }
    c.fast_ncl = ncl;
    w1_elems = (size_t)ncl * 2 * W1_BUF;
  }
  size_t n = (size_t)(c.T + 1) * LHN;
  e = cudaMalloc(&c.d_abT, n * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc(&c.d_w1, w1_elems * sizeof(double2));
  if (e != cudaSuccess) { cudaGetLastError(); return cuda_status(e, "fast path allocation"); }
  xform32_tables_lh(c.d_ab, c.d_abT, c.T + 1, c.fast_variant);
  c.launches++;
  c.fast_cluster = c.fast_variant;
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
  xform32_forward(c, fin, fhT, scratch, n, c.fast_variant, st);
  c.prof.end(1, st);

  c.prof.begin(2, st);
  if (c.fast_variant == t12::TM) {
    const char* ps = std::getenv("FKS_PHASE_SHIFT");
    t12::Args A{fhT, c.d_abT, G, c.d_w1, c.d_ctr, n, c.T + 1, c.dbg, ps ? std::atoll(ps) : 15000LL};
    // teams are formed from the 2 * grid virtual CTAs; keep an even team count so both warp groups have work
    long long nt = std::min<long long>(c.fast_nteams, n);
    if (nt % 2) nt += (nt < c.fast_nteams) ? 1 : -1;
    if (nt < 2) nt = 2;
    cudaMemsetAsync(c.d_ctr, 0, (size_t)c.fast_nteams * 32 * sizeof(unsigned), st);
    void* args[] = {&A};
    cudaError_t e = cudaLaunchCooperativeKernel((void*)t12::hot_kernel_t12, dim3((unsigned)(nt * t12::TM / 2)),
                                                dim3(2 * t12::NT), args, 2 * t12::R_BYTES, st);
    if (e != cudaSuccess) { c.prof.end(2, st); return cuda_status(e, "cooperative hot kernel launch"); }
  } else {
    HotArgs A{fhT, c.d_abT, G, c.d_w1, n, c.T + 1, c.dbg};
    const long long ncl = std::min<long long>(c.fast_ncl, n);
    hot_kernel<<<(unsigned)(ncl * CL), NT, R_BYTES, st>>>(A);
  }
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
