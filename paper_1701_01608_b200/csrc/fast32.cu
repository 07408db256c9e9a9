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
#include "fft_dev.cuh"

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
// Waiting warps are suspended by the hardware (try_wait with a suspend-time hint) instead of spinning: spinning
// waiters cost ~14 % of the issue slots of the working warps sharing their sub-partition (ncu, hot kernel v4).
// Waiting warps back off exponentially (test_wait + nanosleep 32 ns .. 1 us): spinning waiters issued ~35 % of
// all instructions of the 16-warp term-loop kernel (ncu) and took issue slots from the working warps.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  uint32_t done = 0;
  unsigned ns = 32;
  long long spins = 0;
  while (true) {
    asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(a), "r"(parity) : "memory");
    if (done) break;
    __nanosleep(ns);
    if (ns < 1024) ns <<= 1;
    if (++spins > (1LL << 24)) asm volatile("trap;");  // never hang the GPU on a byte-count bug
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
  double* G;             // [cell][px][pz][py]
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
            Gc[(px * P + pz) * P + xpy] = __hiloint2double((int)g[2 * j + 1], (int)g[2 * j]);
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
  double* G;             // [cell][px][pz][py]
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
            Gc[(px * P + pz) * P + xpy] = __hiloint2double((int)gg[2 * j + 1], (int)gg[2 * j]);
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

// ======================================================================================================
// v4: decoupled warp roles.  Teams of 12 CTAs per cell, ONE CTA per SM (4 z-planes and ~1/12 of the pencils
// each).  Inside a CTA:
//   * 2 Z warps produce the z-pass output W1 of term tg into a triple-buffered, L2-resident team buffer and
//     publish it with a monotonic team counter (zdone); they run up to NB terms ahead of the consumers.
//   * 6 YX warps form 2 groups of 3 ("pairs" of z-planes).  A group loads its two W1 planes with one TMA bulk
//     copy per plane (prefetched during the previous term), acknowledges consumption (ydone), and runs a fixed
//     5-round schedule synchronised only by a 96-thread named barrier:
//        R1  Y_0(p0)  Y_0(p1)  Y_1(p0)        Y_c: y-pass of output class c (py = 3q + c), 31 lanes
//        R2  X(0,0)   X(0,1)   X(0,2)          X(c, rx): x-pass class rx of the 32 rows of class c
//        R3  Y_1(p1)  Y_2(p0)  Y_2(p1)         (input planes free -> prefetch W1 of the next term)
//        R4  X(1,*)   R5  X(2,*)               G += Re z * Im z in TMEM
//     Warp (group g, role rx) always handles px class rx, so its G accumulators (16 doubles per lane and row
//     class) stay in its TMEM lane quarter for the whole cell.
// ======================================================================================================
namespace v4 {
constexpr int TM = 12;                        // CTAs (members) per team = per cell
constexpr int PLN = P / TM;                   // 4 z-planes per member
constexpr int NB = 4;                         // W1 team buffers (Z warps run ahead by < NB terms)
// V4_G6 = 1: 16 warps (2 YX groups of 6 + 4 Z warps, <= 128 registers)
// V4_G4 = 1: 12 warps (2 YX groups of 4 + 4 Z warps, <= 168 registers); both 0: 8 warps (groups of 3 + 2 Z warps)
#ifndef V4_G6
#define V4_G6 1
#endif
#if V4_G6
#undef V4_G4
#define V4_G4 1
#endif
#ifndef V4_G4
#define V4_G4 1
#endif
// V4_XP = 1 (with G6): X warps park their rows in TMEM and run all three px classes from there
#ifndef V4_XP
#define V4_XP 1
#endif
#if V4_G6
constexpr int GW = 6;                         // warps per YX group
#ifndef V4_NZW
#define V4_NZW 4
#endif
#elif V4_G4
constexpr int GW = 4;                         // warps per YX group
#ifndef V4_NZW
#define V4_NZW 4
#endif
#else
constexpr int GW = 3;
#ifndef V4_NZW
#define V4_NZW 2
#endif
#endif
constexpr int NYX = 2 * GW, NZW = V4_NZW;     // YX warps (2 groups of GW), Z warps
constexpr int NTHR = 32 * (NYX + NZW);        // 288
constexpr int NZT = 32 * NZW;                 // Z threads
constexpr int MAXH = 41;                      // max staged pencils per member (481 / 12 rounded up)
constexpr int ZSLOT = 96;                     // Z task slots per output class (>= 41 + 41)
constexpr int YB = 16 * K;                    // complex elements of one Y class buffer [16 rows][31]
constexpr int W1IN_B = NPEN * 16;             // 15376 B: one W1 plane
constexpr int YBUF_B = YB * 16;               // 7936 B
#if V4_G4
constexpr int NYSLOT = 3;                     // Y class slots per plane (one per class: Y(c) never waits for X(c'))
#else
constexpr int NYSLOT = 2;                     // slot 0: class 0 then 2, slot 1: class 1
#endif
constexpr int PLANE_B = W1IN_B + NYSLOT * YBUF_B;  // per owned plane
constexpr int ZBLK_B = K * MAXH * 16;         // 20336 B
constexpr int OFF_Z = PLN * PLANE_B;          // 124992
constexpr int SMEM_B = OFF_Z + 3 * ZBLK_B;    // Z: products (2) + the cell's f^ block (tables are read from L2)
constexpr int CTR_STRIDE = 256;               // counter words per team (one 128-B line per counter)
// Synchronisation (exact because buffer b = tg % NB is refilled only after all consumers of its previous
// generation acknowledged it):  W1(tg) is complete when zcnt[b] == TM (tg / NB + 1);  buffer b may be
// overwritten with W1(tg) when ycnt[b] == 2 TM (tg / NB)  (2 YX groups per member).

struct Args {
  const double2* fhatT;  // [cell][LHN], 12 blocks
  const double2* tabT;   // [t][LHN], 12 blocks
  double* G;             // [cell][px][pz][py]
  double2* W1;           // [team][NB][P][NPEN]
  unsigned* ctr;         // [team][CTR_STRIDE]: per W1 buffer b: zcnt at 32 b, ycnt at 32 (NB + b) (zeroed)
  long long n_cells;
  int T1;
  int nteams;
  long long* dbg;        // optional per-phase clock64 stamps (tools/phase_timing.py); nullptr in production
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void poll_ge(const unsigned* p, unsigned target) {
  long long spins = 0;
  while (ld_acquire(p) < target) {
    __nanosleep(128);
    if (++spins > (1LL << 25)) asm volatile("trap;");  // never hang the GPU on a counting bug
  }
}
// publication of W1 by one thread after a named barrier: release semantics are cumulative over the stores the
// barrier made visible to it (a separate fence.sc cost ~1.3 K cycles per term)
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int vload(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ void nbar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

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

// Inputs of a pruned length-48 inverse transform: modes l = -15..15 stored at base[(l + 15) * ld]; transform
// index i = l mod 48 (16..32 absent).
struct InK {
  const double2* base; int ld;
  __device__ __forceinline__ bool nz(int i) const { return i <= 15 || i >= 33; }
  __device__ __forceinline__ double2 operator()(int i) const { return base[(i <= 15 ? i + 15 : i - 33) * ld]; }
};

// Pruned inverse transform of one output class r (runtime, warp-uniform): z(3q + r) = sum_{l=-15..15} Z(l)
// e^{2 pi i l (3q + r)/48}, inputs Z(l) at base[(l + 15) * ld].  Radix-3 combine (only l mod 48 in 0..15 and
// 33..47 are present) + FFT16; z(3q + r) ends in u[qslot(q)].  ONE instance per warp role keeps the kernel's hot
// code inside the instruction cache (templated per-class copies thrashed it: ncu no_instruction stalls).
__device__ __forceinline__ void xform48(const double2* base, int ld, int r, double2 (&u)[16]) {
  u[0] = base[15 * ld];
  if (r == 0) {
#pragma unroll
    for (int m = 1; m < 16; m++) u[m] = fftd::cadd(base[(m + 15) * ld], base[(m - 1) * ld]);
  } else {
    // w3^{2r} = (-1/2, -+ sin(2pi/3)) for r = 1, 2;  twiddle w48^{r m}
    const double sg = (r == 1) ? -0.86602540378443864676 : 0.86602540378443864676;
    const double2* tw = fftd::c_tw48;
#pragma unroll
    for (int m = 1; m < 16; m++) {
      const double2 a = base[(m + 15) * ld], v = base[(m - 1) * ld];
      double2 acc;
      acc.x = fma(-0.5, v.x, a.x);
      acc.x = fma(-sg, v.y, acc.x);
      acc.y = fma(-0.5, v.y, a.y);
      acc.y = fma(sg, v.x, acc.y);
      u[m] = fftd::cmul_s<1>(tw[r * m], acc);
    }
  }
  fftd::fft16<1>(u);
}

// Two independent class-r transforms interleaved (ILP 2) for the fused R4+R5 X round.
__device__ __forceinline__ void xform48x2(const double2* b1, const double2* b2, int r, double2 (&u)[16],
                                          double2 (&v)[16]) {
  u[0] = b1[15];
  v[0] = b2[15];
  if (r == 0) {
#pragma unroll
    for (int m = 1; m < 16; m++) {
      u[m] = fftd::cadd(b1[m + 15], b1[m - 1]);
      v[m] = fftd::cadd(b2[m + 15], b2[m - 1]);
    }
  } else {
    const double sg = (r == 1) ? -0.86602540378443864676 : 0.86602540378443864676;
#pragma unroll
    for (int m = 1; m < 16; m++) {
      const double2 w = fftd::c_tw48[r * m];
      const double2 a1 = b1[m + 15], c1 = b1[m - 1], a2 = b2[m + 15], c2 = b2[m - 1];
      double2 s1, s2;
      s1.x = fma(-0.5, c1.x, a1.x); s2.x = fma(-0.5, c2.x, a2.x);
      s1.x = fma(-sg, c1.y, s1.x);  s2.x = fma(-sg, c2.y, s2.x);
      s1.y = fma(-0.5, c1.y, a1.y); s2.y = fma(-0.5, c2.y, a2.y);
      s1.y = fma(sg, c1.x, s1.y);   s2.y = fma(sg, c2.x, s2.y);
      u[m] = fftd::cmul_s<1>(w, s1);
      v[m] = fftd::cmul_s<1>(w, s2);
    }
  }
  fftd::fft16<1>(u);
  fftd::fft16<1>(v);
}

// Two class-r transforms of inputs with stride ld, interleaved (Z dual tasks).
__device__ __forceinline__ void xform48x2s(const double2* b1, const double2* b2, int ld, int r, double2 (&u)[16],
                                           double2 (&v)[16]) {
  u[0] = b1[15 * ld];
  v[0] = b2[15 * ld];
  if (r == 0) {
#pragma unroll
    for (int m = 1; m < 16; m++) {
      u[m] = fftd::cadd(b1[(m + 15) * ld], b1[(m - 1) * ld]);
      v[m] = fftd::cadd(b2[(m + 15) * ld], b2[(m - 1) * ld]);
    }
  } else {
    const double sg = (r == 1) ? -0.86602540378443864676 : 0.86602540378443864676;
#pragma unroll
    for (int m = 1; m < 16; m++) {
      const double2 w = fftd::c_tw48[r * m];
      const double2 a1 = b1[(m + 15) * ld], c1 = b1[(m - 1) * ld], a2 = b2[(m + 15) * ld], c2 = b2[(m - 1) * ld];
      double2 s1, s2;
      s1.x = fma(-0.5, c1.x, a1.x); s2.x = fma(-0.5, c2.x, a2.x);
      s1.x = fma(-sg, c1.y, s1.x);  s2.x = fma(-sg, c2.y, s2.x);
      s1.y = fma(-0.5, c1.y, a1.y); s2.y = fma(-0.5, c2.y, a2.y);
      s1.y = fma(sg, c1.x, s1.y);   s2.y = fma(sg, c2.x, s2.y);
      u[m] = fftd::cmul_s<1>(w, s1);
      v[m] = fftd::cmul_s<1>(w, s2);
    }
  }
  fftd::fft16<1>(u);
  fftd::fft16<1>(v);
}

__device__ __forceinline__ void tmem_ld16_async(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void g_accumulate(uint32_t tcol, const double2 (&u)[16]) {
  uint32_t gw[32];
  tmem_ld32(tcol, gw);
#pragma unroll
  for (int q = 0; q < 16; q++) {
    const double2 z = u[fftd::qslot(q)];
    const double acc = fma(z.x, z.y, __hiloint2double((int)gw[2 * q + 1], (int)gw[2 * q]));
    gw[2 * q] = (uint32_t)__double2loint(acc);
    gw[2 * q + 1] = (uint32_t)__double2hiint(acc);
  }
  tmem_st32(tcol, gw);
}

__global__ void __launch_bounds__(NTHR, 1) hot_kernel_v4(Args A) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t tmem_base_sh;
  __shared__ __align__(8) uint64_t bar_w1[2];
  __shared__ __align__(8) uint64_t bar_tab, bar_fh;
  // YX groups (V4_G4): per-group completion counters instead of round barriers
  __shared__ int s_yc[2][3], s_xc[2][3], s_yall[2], s_w1iss[2];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int team = blockIdx.x / TM, k = blockIdx.x - (blockIdx.x / TM) * TM;
  constexpr int NLOW = NPEN / 2 + 1;
  const int h0 = (k * NLOW) / TM, h1 = ((k + 1) * NLOW) / TM;
  const int nh = h1 - h0;
  const int nmir = (h1 == NLOW) ? nh - 1 : nh;
  double2* W1t = A.W1 + (long long)team * NB * W1_BUF;
  unsigned* zcnt = A.ctr + (long long)team * CTR_STRIDE;  // + 32 b
  unsigned* ycnt = zcnt + 32 * NB;                         // + 32 b
  const long long ncell_team = (team < A.n_cells) ? (A.n_cells - 1 - team) / A.nteams + 1 : 0;
  const long long total_tg = ncell_team * A.T1;

  if (warp == 0) {
#if V4_G6 && V4_XP
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                 ::"r"((uint32_t)__cvta_generic_to_shared(&tmem_base_sh)));
#else
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;"
                 ::"r"((uint32_t)__cvta_generic_to_shared(&tmem_base_sh)));
#endif
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&bar_w1[0]);
    mbar_init(&bar_w1[1]);
    mbar_init(&bar_tab);
    mbar_init(&bar_fh);
    for (int i = 0; i < 6; i++) { (&s_yc[0][0])[i] = 0; (&s_xc[0][0])[i] = 0; }
    s_yall[0] = s_yall[1] = 0;
    s_w1iss[0] = s_w1iss[1] = 0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tmem_base_sh;

  if (warp < NYX) {
#if V4_G6 && V4_XP
    // --------------------------------- YX warps, X rows parked in TMEM -------------------------------------
    // 6 X warps (one per group and row class c; warps 0..5 -> (g,c) = (0,0) (0,1) (0,2) (1,2) (1,0) (1,1), lane
    // quarters 0,1,2,3,0,1) and 6 Y warps (6..11 -> (g, c) = (w-6)/3, (w-6)%3).  Per term t:
    //   Y(g,c): wait W1(t) and slot c free (X(g,c) parked term t-1); class c of the y-pass of both planes
    //           -> slot c; count yc[g][c] = t+1; the last Y warp of the group done with W1(t) prefetches W1(t+1).
    //   X(g,c): wait yc[g][c] = t+1; load its 32 rows of class c once, park them in TMEM (124 columns), free the
    //           slot (xc[g][c] = t+1), then the three px classes from TMEM with G += Re z Im z (3 x 32 columns).
    const bool isx = warp < 6;
    const int g = isx ? ((warp >= 3) ? 1 : 0) : (warp - 6) / 3;
    const int c = isx ? (warp < 3 ? warp : (warp == 3 ? 2 : warp - 4)) : (warp - 6) % 3;
    double2* pb0 = reinterpret_cast<double2*>(smem + (2 * g) * PLANE_B);
    double2* pb1 = reinterpret_cast<double2*>(smem + (2 * g + 1) * PLANE_B);
    double2* in0 = pb0;
    double2* in1 = pb1;
    auto ybuf = [&](int pl, int slot) { return (pl ? pb1 : pb0) + NPEN + slot * YB; };
    const int pz0 = PLN * k + 2 * g;
    const uint32_t tX = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(warp >= 4 && warp < 6 ? 224 : 0);
    const uint32_t tPark = tX + 96u;
    const int xp = lane >> 4, xq = lane & 15;
    int* yc = s_yc[g];
    int* xc = s_xc[g];
    auto wait_ge = [&](const int* ptr, int target) {
      if (lane == 0) {
        long long spins = 0;
        unsigned ns = 32;
        while (vload(ptr) < target) {
          __nanosleep(ns);
          if (ns < 512) ns <<= 1;
          if (++spins > (1LL << 26)) asm volatile("trap;");
        }
      }
      __syncwarp();
    };
    auto issue_w1 = [&](long long tgi) {
      const double2* src = W1t + (tgi % NB) * (long long)W1_BUF + (long long)pz0 * NPEN;
      asm volatile("fence.proxy.async.global;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect(&bar_w1[g], 2u * W1IN_B);
      bulk_g2s(in0, src, W1IN_B, &bar_w1[g]);
      bulk_g2s(in1, src + NPEN, W1IN_B, &bar_w1[g]);
    };
    auto try_issue_w1 = [&](long long tz, bool block) {  // lane 0: bulk-copy W1(tz) once per group
      if (tz >= total_tg) return;
      if (vload(&s_w1iss[g]) > (int)tz) return;
      if (vload(&s_yall[g]) < 3 * (int)tz) {
        if (!block) return;
        long long spins = 0;
        while (vload(&s_yall[g]) < 3 * (int)tz) { __nanosleep(64); if (++spins > (1LL << 26)) asm volatile("trap;"); }
      }
      unsigned* zc = zcnt + 32 * (tz % NB);
      const unsigned target = (unsigned)(TM * (tz / NB + 1));
      if (block) poll_ge(zc, target);
      else if (ld_acquire(zc) < target) return;
      if (atomicCAS(&s_w1iss[g], (int)tz, (int)tz + 1) == (int)tz) issue_w1(tz);
    };
    uint32_t par = 0;
    long long tg = 0;
#pragma unroll 1
    for (long long cell = team; cell < A.n_cells; cell += A.nteams) {
#pragma unroll 1
      for (int t = 0; t < A.T1; t++, tg++) {
        const int T = (int)tg;
        long long* st = (A.dbg && lane == 0 && warp == 6 && cell == team && t >= 2 && t < 6)
                            ? A.dbg + (long long)blockIdx.x * 128 + (t - 2) * 16 : nullptr;
        if (st) st[0] = clock64();
        if (!isx) {
          // ---------------- Y warp ----------------
          if (lane == 0 && c == 0) try_issue_w1(tg, true);
          mbar_wait(&bar_w1[g], par);
          if (c == 0 && lane == 0) {
            __threadfence();
            atomicAdd(ycnt + 32 * (tg % NB), 1u);  // this group has consumed W1(tg)
          }
          if (st) st[1] = clock64();
          wait_ge(&xc[c], T);  // slot c: X(g, c) of term t-1 has parked its rows
#pragma unroll 1
          for (int pl = 0; pl < 2; pl++) {
            double2 u[16];
            xform48((pl ? in1 : in0) + (lane < K ? lane : K - 1) * K, 1, c, u);
            if (lane < K) {
              double2* ydst = ybuf(pl, c) + lane;
#pragma unroll
              for (int q = 0; q < 16; q++) ydst[q * K] = u[fftd::qslot(q)];
            }
          }
          __syncwarp();
          if (lane == 0) {
            __threadfence_block();
            atomicAdd(&yc[c], 1);
            if (atomicAdd(&s_yall[g], 1) + 1 == 3 * (T + 1)) try_issue_w1(tg + 1, false);  // prefetch
          }
          if (st) st[2] = clock64();
        } else {
          // ---------------- X warp ----------------
          wait_ge(&yc[c], T + 1);
          if (t == 0) {  // first term of the cell: zero the three G blocks
            uint32_t zw[32];
#pragma unroll
            for (int i = 0; i < 32; i++) zw[i] = 0u;
#pragma unroll 1
            for (int rx = 0; rx < 3; rx++) tmem_st32(tX + 32u * rx, zw);
          }
          {  // park the row (31 complex = 124 words) in this lane's TMEM columns, 8 values per store
            const double2* row = ybuf(xp, c) + xq * K;
#pragma unroll
            for (int ch = 0; ch < 4; ch++) {
              uint32_t w[32];
#pragma unroll
              for (int k2 = 0; k2 < 8; k2++) {
                const int i = 8 * ch + k2;
                const double2 v = (i < K) ? row[i] : make_double2(0.0, 0.0);
                w[4 * k2] = (uint32_t)__double2loint(v.x);
                w[4 * k2 + 1] = (uint32_t)__double2hiint(v.x);
                w[4 * k2 + 2] = (uint32_t)__double2loint(v.y);
                w[4 * k2 + 3] = (uint32_t)__double2hiint(v.y);
              }
              tmem_st32(tPark + 32u * ch, w);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          }
          __syncwarp();
          if (lane == 0) {
            __threadfence_block();
            atomicAdd(&xc[c], 1);  // the Y slot may be refilled
          }
#pragma unroll 1
          for (int rx = 0; rx < 3; rx++) {
            double2 u[16];
            const double sg = (rx == 1) ? -0.86602540378443864676 : 0.86602540378443864676;
#pragma unroll
            for (int mm = 0; mm < 4; mm++) {  // x[4mm..4mm+3] (a) and x[16+4mm..19+4mm] (b) -> u[4mm+1..4mm+4]
              uint32_t wa[16], wb[16];
              tmem_ld16_async(tPark + 16u * mm, wa);
              tmem_ld16_async(tPark + 64u + 16u * mm, wb);
              tmem_wait_ld();
#pragma unroll
              for (int k2 = 0; k2 < 4; k2++) {
                const int m = 4 * mm + k2 + 1;
                const double2 va = make_double2(__hiloint2double((int)wa[4 * k2 + 1], (int)wa[4 * k2]),
                                                __hiloint2double((int)wa[4 * k2 + 3], (int)wa[4 * k2 + 2]));
                if (mm == 3 && k2 == 3) { u[0] = va; continue; }  // x[15]
                const double2 vb = make_double2(__hiloint2double((int)wb[4 * k2 + 1], (int)wb[4 * k2]),
                                                __hiloint2double((int)wb[4 * k2 + 3], (int)wb[4 * k2 + 2]));
                if (rx == 0) {
                  u[m] = fftd::cadd(vb, va);
                } else {
                  double2 acc;
                  acc.x = fma(-0.5, va.x, vb.x);
                  acc.x = fma(-sg, va.y, acc.x);
                  acc.y = fma(-0.5, va.y, vb.y);
                  acc.y = fma(sg, va.x, acc.y);
                  u[m] = fftd::cmul_s<1>(fftd::c_tw48[rx * m], acc);
                }
              }
            }
            fftd::fft16<1>(u);
            g_accumulate(tX + 32u * rx, u);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          if (t == A.T1 - 1) {  // G[cell][px = 3q' + rx][pz][py = 3 xq + c]
            double* Gc = A.G + cell * (long long)(P * P * P) + (long long)(pz0 + xp) * P;
#pragma unroll 1
            for (int rx = 0; rx < 3; rx++) {
              uint32_t gw[32];
              tmem_ld32(tX + 32u * rx, gw);
#pragma unroll
              for (int q = 0; q < 16; q++)
                Gc[(long long)(3 * q + rx) * P * P + 3 * xq + c] = __hiloint2double((int)gw[2 * q + 1], (int)gw[2 * q]);
            }
          }
        }
        par ^= 1;
      }
    }
#else
    // ---------------------------------------------- YX warps ----------------------------------------------
    const int g = warp / GW, wr = warp - GW * (warp / GW);
    double2* pb0 = reinterpret_cast<double2*>(smem + (2 * g) * PLANE_B);
    double2* pb1 = reinterpret_cast<double2*>(smem + (2 * g + 1) * PLANE_B);
    double2* in0 = pb0;                      // W1 plane 2g
    double2* in1 = pb1;                      // W1 plane 2g+1
    // Y class slots: slot 0 holds row class 0 then 2, slot 1 row class 1; plane 2g at pb0, 2g+1 at pb1
    auto ybuf = [&](int pl, int slot) { return (pl ? pb1 : pb0) + NPEN + slot * YB; };
    const int pz0 = PLN * k + 2 * g;
#if V4_G6
    const uint32_t tG = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));  // <= 2 blocks
#else
    const uint32_t tG = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(96 * g);
#endif
    const bool leader = (wr == 0 && lane == 0);
    auto issue_w1 = [&](long long tgi) {
      const double2* src = W1t + (tgi % NB) * (long long)W1_BUF + (long long)pz0 * NPEN;
      asm volatile("fence.proxy.async.global;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect(&bar_w1[g], 2u * W1IN_B);
      bulk_g2s(in0, src, W1IN_B, &bar_w1[g]);
      bulk_g2s(in1, src + NPEN, W1IN_B, &bar_w1[g]);
    };
    // X rows of this lane: plane (lane >> 4), row index q = lane & 15 (py = 3q + c)
    const int xp = lane >> 4, xq = lane & 15;
    uint32_t par = 0;
    bool issued = false;
    long long tg = 0;
#pragma unroll 1
    for (long long cell = team; cell < A.n_cells; cell += A.nteams) {
#pragma unroll 1
      for (int t = 0; t < A.T1; t++, tg++) {
        long long* st = (A.dbg && leader && g == 0 && cell == team && t >= 2 && t < 6)
                            ? A.dbg + (long long)blockIdx.x * 128 + (t - 2) * 16 : nullptr;
        if (st) st[0] = clock64();
#if V4_G4
        // Static per-warp task lists, synchronised by per-group completion counters (no round barriers):
        //   wr0: Y(0,p0) Y(2,p0) X(0,0) X(1,1)    wr1: Y(0,p1) Y(2,p1) X(0,1) X(2,0)
        //   wr2: Y(1,p0) X(0,2) X(2,1)            wr3: Y(1,p1) X(1,0) X(1,2) X(2,2)
        // One Y slot per class: Y(t, c, p) waits only for X(t-1, c, *) to have read slot c, X(t, c, rx) for both
        // planes of class c, so terms overlap.  X(c,rx) of a warp keeps its G block at TMEM column 32 * blk of the
        // warp's lane quarter (+96 per group).
        int* yc = s_yc[g];
        int* xc = s_xc[g];
        auto wait_ge = [&](const int* ptr, int target) {
          if (lane == 0) {
            long long spins = 0;
            unsigned ns = 32;
            while (vload(ptr) < target) {
              __nanosleep(ns);
              if (ns < 512) ns <<= 1;
              if (++spins > (1LL << 26)) asm volatile("trap;");
            }
          }
          __syncwarp();
        };
        auto try_issue_w1 = [&](long long tz, bool block) {  // lane 0 only: bulk-copy W1(tz) (once per group)
          if (tz >= total_tg) return;
          if (vload(&s_w1iss[g]) > (int)tz) return;
          if (vload(&s_yall[g]) < 6 * (int)tz) {  // input planes still read by Y(tz - 1)
            if (!block) return;
            long long spins = 0;
            while (vload(&s_yall[g]) < 6 * (int)tz) { __nanosleep(32); if (++spins > (1LL << 26)) asm volatile("trap;"); }
          }
          unsigned* zc = zcnt + 32 * (tz % NB);
          const unsigned target = (unsigned)(TM * (tz / NB + 1));
          if (block) poll_ge(zc, target);
          else if (ld_acquire(zc) < target) return;
          if (atomicCAS(&s_w1iss[g], (int)tz, (int)tz + 1) == (int)tz) issue_w1(tz);
        };
        if (lane == 0 && wr == 0) try_issue_w1(tg, true);
        if (st) st[1] = clock64();
        bool w1_seen = false;
#if V4_G6
        constexpr int NTASK = 3;
#else
        constexpr int NTASK = 4;
#endif
#pragma unroll 1
        for (int ti = 0; ti < NTASK; ti++) {
          int kind = 0, c = 0, rx = 0, pl = 0, blk = 0;  // kind 1 Y, 2 X
#if V4_G6
          // wr0: Y(0,p0) X(0,0) X(2,1)   wr1: Y(0,p1) X(0,1) X(2,2)   wr2: Y(1,p0) X(0,2)
          // wr3: Y(1,p1) X(1,0)          wr4: Y(2,p0) X(1,1)          wr5: Y(2,p1) X(1,2) X(2,0)
          if (ti == 0) { kind = 1; c = wr >> 1; pl = wr & 1; }
          else if (ti == 1) {
            kind = 2; blk = 0;
            c = wr < 3 ? 0 : 1;
            rx = wr < 3 ? wr : wr - 3;
          } else if (wr == 0 || wr == 1 || wr == 5) {
            kind = 2; blk = 1; c = 2;
            rx = wr == 0 ? 1 : (wr == 1 ? 2 : 0);
          }
#else
          if (wr == 0) {         // Y(0,p0) Y(2,p0) X(0,0) X(1,1)
            if (ti < 2) { kind = 1; c = 2 * ti; pl = 0; }
            else { kind = 2; c = ti - 2; rx = ti - 2; blk = ti - 2; }
          } else if (wr == 1) {  // Y(0,p1) Y(2,p1) X(0,1) X(2,0)
            if (ti < 2) { kind = 1; c = 2 * ti; pl = 1; }
            else if (ti == 2) { kind = 2; c = 0; rx = 1; blk = 0; }
            else { kind = 2; c = 2; rx = 0; blk = 1; }
          } else if (wr == 2) {  // Y(1,p0) X(0,2) X(2,1)
            if (ti == 0) { kind = 1; c = 1; pl = 0; }
            else if (ti == 1) { kind = 2; c = 0; rx = 2; blk = 0; }
            else if (ti == 2) { kind = 2; c = 2; rx = 1; blk = 1; }
          } else {               // Y(1,p1) X(1,0) X(1,2) X(2,2)
            if (ti == 0) { kind = 1; c = 1; pl = 1; }
            else { kind = 2; c = ti == 3 ? 2 : 1; rx = ti == 1 ? 0 : 2; blk = ti - 1; }
          }
#endif
          if (kind == 0) continue;
          const int T = (int)tg;
          if (kind == 1) {
            if (!w1_seen) {
              mbar_wait(&bar_w1[g], par);
              w1_seen = true;
              if (leader) {
                __threadfence();
                atomicAdd(ycnt + 32 * (tg % NB), 1u);  // this group has consumed W1(tg)
              }
            }
            wait_ge(&xc[c], 3 * T);  // slot c last read by X(t-1, c, *)
          } else {
            wait_ge(&yc[c], 2 * (T + 1));
            if (t == 0) {  // first term of the cell: zero this block
              uint32_t zw[32];
#pragma unroll
              for (int i = 0; i < 32; i++) zw[i] = 0u;
              tmem_st32(tG + 32u * blk, zw);
              asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            }
          }
          const double2* base;
          if (kind == 2) base = ybuf(xp, c) + xq * K;
          else base = (pl ? in1 : in0) + (lane < K ? lane : K - 1) * K;
          double2 u[16];
          xform48(base, 1, kind == 2 ? rx : c, u);
          if (kind == 2) {
            g_accumulate(tG + 32u * blk, u);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            if (t == A.T1 - 1) {  // last term of the cell: G[cell][px = 3q' + rx][pz][py = 3 xq + c]
              double* Gc = A.G + cell * (long long)(P * P * P) + (long long)(pz0 + xp) * P;
              uint32_t gw[32];
              tmem_ld32(tG + 32u * blk, gw);
#pragma unroll
              for (int q = 0; q < 16; q++)
                Gc[(long long)(3 * q + rx) * P * P + 3 * xq + c] = __hiloint2double((int)gw[2 * q + 1], (int)gw[2 * q]);
            }
            __syncwarp();
            if (lane == 0) {
              __threadfence_block();
              atomicAdd(&xc[c], 1);
            }
          } else {
            if (lane < K) {
              double2* ydst = ybuf(pl, c) + lane;
#pragma unroll
              for (int q = 0; q < 16; q++) ydst[q * K] = u[fftd::qslot(q)];
            }
            __syncwarp();
            if (lane == 0) {
              __threadfence_block();
              atomicAdd(&yc[c], 1);
              if (atomicAdd(&s_yall[g], 1) + 1 == 6 * (T + 1)) try_issue_w1(tg + 1, false);  // prefetch
            }
          }
        }
        par ^= 1;
        if (st) st[5] = clock64();
#else
        if (leader && !issued) {
          poll_ge(zcnt + 32 * (tg % NB), (unsigned)(TM * (tg / NB + 1)));
          issue_w1(tg);
        }
        mbar_wait(&bar_w1[g], par);
        par ^= 1;
        if (leader) {
          __threadfence();
          atomicAdd(ycnt + 32 * (tg % NB), 1u);  // this group has consumed W1(tg)
        }
        issued = false;
        if (st) st[1] = clock64();
        if (t == 0) {  // zero this warp's G accumulators (3 row classes x 16 doubles per lane)
          uint32_t zw[32];
#pragma unroll
          for (int i = 0; i < 32; i++) zw[i] = 0u;
#pragma unroll
          for (int c = 0; c < 3; c++) tmem_st32(tG + 32 * c, zw);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
#pragma unroll 1
        for (int rd = 0; rd < 4; rd++) {
          // task of this warp in round rd (see the schedule above; rd == 3 fuses R4 and R5)
          if (rd == 3) {
            double2 u[16], v[16];
            xform48x2(ybuf(xp, 1) + xq * K, ybuf(xp, 0) + xq * K, wr, u, v);
            g_accumulate(tG + 32u, u);
            g_accumulate(tG + 64u, v);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            nbar(1 + g, 32 * GW);
            if (st) st[5] = clock64();
            break;
          }
          const bool isx = (rd == 1);
          const double2* base;
          double2* ydst = nullptr;
          int r;
          uint32_t tcol = 0;
          if (isx) {
            base = ybuf(xp, 0) + xq * K;
            r = wr;
            tcol = tG;
          } else {
            // R1: (p0,c0) (p1,c0) (p0,c1);  R3: (p1,c1) (p0,c2) (p1,c2)
            const int code = (rd == 0) ? wr : 3 + wr;
            const int pl = (code == 1 || code == 3 || code == 5) ? 1 : 0;
            r = (code <= 1) ? 0 : (code <= 3 ? 1 : 2);
            const int slot = (r == 1) ? 1 : 0;
            base = (pl ? in1 : in0) + (lane < K ? lane : K - 1) * K;
            ydst = ybuf(pl, slot) + lane;
          }
          double2 u[16];
          xform48(base, 1, r, u);
          if (isx) {  // G(px = 3q + r, row) += Re z * Im z
            g_accumulate(tcol, u);
          } else if (lane < K) {
#pragma unroll
            for (int q = 0; q < 16; q++) ydst[q * K] = u[fftd::qslot(q)];
          }
          nbar(1 + g, 96);
          if (st) st[2 + rd] = clock64();
          if (rd == 2 && leader && tg + 1 < total_tg &&
              ld_acquire(zcnt + 32 * ((tg + 1) % NB)) >= (unsigned)(TM * ((tg + 1) / NB + 1))) {
            issue_w1(tg + 1);  // input planes are free: overlap the copy with R4/R5
            issued = true;
          }
        }
        if (t == A.T1 - 1) {  // G[cell][px = 3q' + wr][pz][py = 3 xq + c]
          double* Gc = A.G + cell * (long long)(P * P * P) + (long long)(pz0 + xp) * P;
#pragma unroll
          for (int c = 0; c < 3; c++) {
            uint32_t gw[32];
            tmem_ld32(tG + 32 * c, gw);
#pragma unroll
            for (int q = 0; q < 16; q++)
              Gc[(long long)(3 * q + wr) * P * P + 3 * xq + c] = __hiloint2double((int)gw[2 * q + 1], (int)gw[2 * q]);
          }
        }
#endif
      }
    }
#endif
  } else {
    // ---------------------------------------------- Z warps -----------------------------------------------
    const int zt = tid - 32 * NYX;  // 0..NZT-1
    double2* zp = reinterpret_cast<double2*>(smem + OFF_Z);
    double2* zm = reinterpret_cast<double2*>(smem + OFF_Z + ZBLK_B);
    double2* fh = reinterpret_cast<double2*>(smem + OFF_Z + 2 * ZBLK_B);  // the cell's f^ block (TMA, per cell)
    const uint32_t fblk = (uint32_t)(K * nh) * 16u;
    auto issue_fh = [&](long long cl) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect(&bar_fh, fblk);
      bulk_g2s(fh, A.fhatT + cl * (long long)LHN + K * h0, fblk, &bar_fh);
    };
    if (zt == 0 && ncell_team > 0) issue_fh(team);
    uint32_t par_fh = 0;
    long long tg = 0;
#pragma unroll 1
    for (long long cell = team; cell < A.n_cells; cell += A.nteams) {
      mbar_wait(&bar_fh, par_fh);
      par_fh ^= 1;
#pragma unroll 1
      for (int t = 0; t < A.T1; t++, tg++) {
        const double2* tb = A.tabT + (long long)t * LHN + K * h0;     // the member's table block (L2)
        long long* st = (A.dbg && zt == 0 && cell == team && t >= 2 && t < 6)
                            ? A.dbg + (long long)blockIdx.x * 128 + (t - 2) * 16 + 8 : nullptr;
        if (st) st[0] = clock64();
        if (st) st[1] = clock64();
        // products: Z = (a + ib) f^ for the staged pencils, and for their mirrors (-lx,-ly): (a + ib) conj(f^)
        // at the reversed lz (a, b even; f real)
        {  // element pairs {i, 30 - i} of pencil j, e = i * nh + j; i = e / nh by multiply-high (exact: e nh < 2^32).
           // Four iterations are loaded before any store (the product buffers never alias the staged inputs).
          const unsigned mdiv = 0xffffffffu / (unsigned)nh + 1u;
          const double2* __restrict__ fr = fh;  // f^ block in shared memory
          const double2* __restrict__ tr = tb;
          double2* __restrict__ pw = zp;
          double2* __restrict__ mw = zm;
          const int ne = 16 * nh;
          // every load of this thread (<= ZIT iterations) is issued before the first product: one L2 round trip
          constexpr int ZIT = (16 * MAXH + NZT - 1) / NZT;  // all table loads of this thread in one L2 round
#pragma unroll 1
          for (int zb = 0; zb * ZIT * NZT < ne; zb++) {
          const int zt0 = zt + zb * ZIT * NZT;
          double2 f1[ZIT], a1[ZIT], f2[ZIT], a2[ZIT];
          int o1[ZIT], o2[ZIT];
#pragma unroll
          for (int u = 0; u < ZIT; u++) {
            const int e = min(zt0 + u * NZT, ne - 1);
            const int i = (int)__umulhi((unsigned)e, mdiv), j = e - i * nh;
            o1[u] = i * nh + j;
            o2[u] = (30 - i) * nh + j;
            a1[u] = __ldg(tr + o1[u]);
            a2[u] = __ldg(tr + o2[u]);
          }
#pragma unroll
          for (int u = 0; u < ZIT; u++) {
            f1[u] = fr[o1[u]];  // shared memory
            f2[u] = fr[o2[u]];
            if (zt0 + u * NZT < ne) {
              pw[o1[u]] = make_double2(fma(a1[u].x, f1[u].x, -a1[u].y * f1[u].y), fma(a1[u].x, f1[u].y, a1[u].y * f1[u].x));
              pw[o2[u]] = make_double2(fma(a2[u].x, f2[u].x, -a2[u].y * f2[u].y), fma(a2[u].x, f2[u].y, a2[u].y * f2[u].x));
              mw[o1[u]] = make_double2(fma(a2[u].x, f2[u].x, a2[u].y * f2[u].y), fma(-a2[u].x, f2[u].y, a2[u].y * f2[u].x));
              mw[o2[u]] = make_double2(fma(a1[u].x, f1[u].x, a1[u].y * f1[u].y), fma(-a1[u].x, f1[u].y, a1[u].y * f1[u].x));
            }
          }
          }
        }
        nbar(3, NZT);  // products complete (after the cell's last term the f^ block is free)
        if (zt == 0 && t == A.T1 - 1 && cell + A.nteams < A.n_cells) issue_fh(cell + A.nteams);
        // publish W1(tg - 2) and W1(tg - 1) every second term: one store drain per pair (it costs ~1.4 K cycles
        // on the Z warps, which set the period; the consumers have slack)
        if (zt == 0 && tg >= 2 && (tg & 1) == 0) {
          __threadfence();
          atomicAdd(zcnt + 32 * ((tg - 2) % NB), 1u);
          atomicAdd(zcnt + 32 * ((tg - 1) % NB), 1u);
        }
        if (st) st[2] = clock64();
        if (zt == 0) {
          if (tg >= NB) poll_ge(ycnt + 32 * (tg % NB), (unsigned)(2 * TM * (tg / NB)));  // buffer free
        }
        nbar(3, NZT);
        if (st) st[3] = clock64();
        double2* W1b = W1t + (tg % NB) * (long long)W1_BUF;
#if V4_G4
        {  // 4 Z warps: single class tasks tau = r * na + j, 2 rounds of 128 threads cover 3 na <= 246
          const int na = nh + nmir;
#pragma unroll 1
          for (int kk = zt; kk < 2 * NZT; kk += NZT) {
            if (kk - lane >= 3 * na) break;  // no active lane in this warp (warp-uniform)
            const bool act = kk < 3 * na;
            const int kc = act ? kk : 0;
            const int r = kc / na, j = kc - r * na;
            const bool mir = j >= nh;
            const int jj = mir ? j - nh : j;
            double2 u[16];
            xform48((mir ? zm : zp) + jj, nh, r, u);
            if (act) {
              const int pp = mir ? (NPEN - 1) - (h0 + jj) : h0 + jj;
#pragma unroll
              for (int q = 0; q < 16; q++) W1b[(3 * q + r) * NPEN + pp] = u[fftd::qslot(q)];
            }
          }
        }
#else
        // dual class tasks: slot s -> class r = s / npair, pencils j1 = s % npair and j2 = j1 + npair (npair =
        // ceil(na / 2) <= 41, 3 npair <= 123 slots = 2 rounds of 64 threads); two interleaved transforms per thread
        const int na = nh + nmir, npair = (na + 1) / 2;
#pragma unroll 1
        for (int s0 = zt; s0 < 2 * NZT; s0 += NZT) {
          const bool act = s0 < 3 * npair;
          const int sc = act ? s0 : 0;
          const int r = sc / npair, j1 = sc - r * npair, j2 = j1 + npair;
          const bool act2 = act && j2 < na;
          const int j2c = act2 ? j2 : j1;
          const bool mir1 = j1 >= nh, mir2 = j2c >= nh;
          const int jj1 = mir1 ? j1 - nh : j1, jj2 = mir2 ? j2c - nh : j2c;
          double2 u[16], v[16];
          xform48x2s((mir1 ? zm : zp) + jj1, (mir2 ? zm : zp) + jj2, nh, r, u, v);
          if (act) {
            const int pp1 = mir1 ? (NPEN - 1) - (h0 + jj1) : h0 + jj1;
#pragma unroll
            for (int q = 0; q < 16; q++) W1b[(3 * q + r) * NPEN + pp1] = u[fftd::qslot(q)];
          }
          if (act2) {
            const int pp2 = mir2 ? (NPEN - 1) - (h0 + jj2) : h0 + jj2;
#pragma unroll
            for (int q = 0; q < 16; q++) W1b[(3 * q + r) * NPEN + pp2] = v[fftd::qslot(q)];
          }
        }
#endif
        nbar(3, NZT);
        if (st) st[4] = clock64();
      }
    }
    if (zt == 0 && tg > 0) {  // publish what is left (tg even: W1(tg-2), W1(tg-1); tg odd: W1(tg-1))
      __threadfence();
      if ((tg & 1) == 0 && tg >= 2) atomicAdd(zcnt + 32 * ((tg - 2) % NB), 1u);
      atomicAdd(zcnt + 32 * ((tg - 1) % NB), 1u);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
#if V4_G6 && V4_XP
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
#else
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
#endif
}
}  // namespace v4

// ======================================================================================================
// v5: "pencil tasks".  Same team structure as v4 (12 CTAs per cell, one CTA of 8 warps per SM, 4 z-planes and
// ~1/12 of the pencils per CTA, triple-buffered L2 exchange with per-buffer produce/consume counters), but
// every task loads its 31 inputs ONCE into registers and computes all three output classes from them (the
// class-task kernels re-read each input three times from shared memory, which cost as much smem bandwidth as
// the FP64 work).  Z products are formed on the fly (each product feeds exactly one pencil task), so there is
// no product pass.  Two rounds per term, separated by CTA barriers:
//     R1(t):  warps 0-3  Y(t) of plane w (31 lanes)          warp 4: Z(t+1) pencils [64, na)
//     R2(t):  warps 0-5  X(t) of rows 32w..32w+31 (192 rows)  warps 6-7: Z(t+2) pencils [0, 64)
// Z(t') is published (zcnt) after R1(t'-1); W1(t') is bulk-copied during R2(t'-1) and read by R1(t').
// ======================================================================================================
namespace v5 {
using v4::ld_acquire;
using v4::poll_ge;
using v4::tmem_ld32;
using v4::tmem_st32;
constexpr int TM = 12, PLN = 4, NB = 3, NW = 8, NTHR = 32 * NW;
constexpr int MAXH = 41;
constexpr int W1IN_B = NPEN * 16;                 // 15376
constexpr int YPL = P * K;                        // complex per plane of the Y region ([py][ix])
constexpr int ZBLK_B = K * MAXH * 16;             // 20336
constexpr int OFF_Y = PLN * W1IN_B;               // 61504
constexpr int OFF_FH = OFF_Y + PLN * YPL * 16;    // 156736
constexpr int OFF_TB = OFF_FH + ZBLK_B;           // 177072 (two buffers)
constexpr int SMEM_B = OFF_TB + 2 * ZBLK_B;       // 217744
constexpr int CTR_STRIDE = 256;
constexpr int ZA = 64;                            // Z pencils done in R2 (part A); the rest in R1 (part B)

struct Args {
  const double2* fhatT;  // [cell][LHN], 12 blocks
  const double2* tabT;   // [t][LHN], 12 blocks
  double* G;             // [cell][px][pz][py]
  double2* W1;           // [team][NB][P][NPEN]
  unsigned* ctr;         // [team][CTR_STRIDE]: zcnt[b] at 32 b, ycnt[b] at 32 (NB + b)
  long long n_cells;
  int T1;
  int nteams;
  long long* dbg;
};

// u = class r of the pruned inverse 48-point transform of x (modes l = -15..15 at x[l + 15]), r warp-uniform
__device__ __forceinline__ void xform48_regs(const double2 (&x)[K], int r, double2 (&u)[16]) {
  u[0] = x[15];
  if (r == 0) {
#pragma unroll
    for (int m = 1; m < 16; m++) u[m] = fftd::cadd(x[m + 15], x[m - 1]);
  } else {
    const double sg = (r == 1) ? -0.86602540378443864676 : 0.86602540378443864676;
    const double2* tw = fftd::c_tw48;
#pragma unroll
    for (int m = 1; m < 16; m++) {
      const double2 a = x[m + 15], v = x[m - 1];
      double2 acc;
      acc.x = fma(-0.5, v.x, a.x);
      acc.x = fma(-sg, v.y, acc.x);
      acc.y = fma(-0.5, v.y, a.y);
      acc.y = fma(sg, v.x, acc.y);
      u[m] = fftd::cmul_s<1>(tw[r * m], acc);
    }
  }
  fftd::fft16<1>(u);
}

struct ZTask {
  const double2* fh;   // staged f^ block [iz][j]
  const double2* tb;   // staged table block [iz][j]
  double2* W1b;        // W1 buffer of the term
  int nh, h0, tau;     // staged pencils, first pencil, task (tau < nh: staged pencil, else its mirror)
};
// One Z pencil task: products, three output classes, stores.  Not inlined: one copy serves every call site
// (prologue, R1, R2), which keeps the kernel's hot code small.
__device__ __noinline__ void z_pencil(const ZTask z) {
  const bool mir = z.tau >= z.nh;
  const int j = mir ? z.tau - z.nh : z.tau;
  double2 x[K];
#pragma unroll
  for (int i = 0; i < K; i++) {
    const int ii = mir ? (K - 1 - i) : i;  // mirror (-lx,-ly): (a + ib)(l') conj(f^(l')) at reversed lz
    const double2 f = z.fh[ii * z.nh + j], a = z.tb[ii * z.nh + j];
    x[i] = mir ? make_double2(fma(a.x, f.x, a.y * f.y), fma(-a.x, f.y, a.y * f.x))
               : make_double2(fma(a.x, f.x, -a.y * f.y), fma(a.x, f.y, a.y * f.x));
  }
  double2* W1b = z.W1b + (mir ? (NPEN - 1) - (z.h0 + j) : z.h0 + j);
#pragma unroll 1
  for (int r = 0; r < 3; r++) {
    double2 u[16];
    xform48_regs(x, r, u);
#pragma unroll
    for (int q = 0; q < 16; q++) W1b[(3 * q + r) * NPEN] = u[fftd::qslot(q)];
  }
}

enum { TK_NONE = 0, TK_Y = 1, TK_X = 2, TK_Z = 3 };

__global__ void __launch_bounds__(NTHR, 1) hot_kernel_v5(Args A) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t tmem_base_sh;
  __shared__ __align__(8) uint64_t bar_w1, bar_fh, bar_tab[2];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int team = blockIdx.x / TM, k = blockIdx.x - (blockIdx.x / TM) * TM;
  constexpr int NLOW = NPEN / 2 + 1;
  const int h0 = (k * NLOW) / TM, h1 = ((k + 1) * NLOW) / TM;
  const int nh = h1 - h0;
  const int nmir = (h1 == NLOW) ? nh - 1 : nh;
  const int na = nh + nmir;
  double2* W1t = A.W1 + (long long)team * NB * W1_BUF;
  unsigned* zcnt = A.ctr + (long long)team * CTR_STRIDE;
  unsigned* ycnt = zcnt + 32 * NB;
  const long long ncell_team = (team < A.n_cells) ? (A.n_cells - 1 - team) / A.nteams + 1 : 0;
  const long long TT = ncell_team * A.T1;  // terms of this team
  double2* w1in = reinterpret_cast<double2*>(smem);
  double2* ysh = reinterpret_cast<double2*>(smem + OFF_Y);
  double2* fh = reinterpret_cast<double2*>(smem + OFF_FH);
  double2* tbs = reinterpret_cast<double2*>(smem + OFF_TB);
  const uint32_t zblk = (uint32_t)(K * nh) * 16u;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;"
                 ::"r"((uint32_t)__cvta_generic_to_shared(&tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&bar_w1);
    mbar_init(&bar_fh);
    mbar_init(&bar_tab[0]);
    mbar_init(&bar_tab[1]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tmem_base_sh;
  if (TT == 0) goto done;
  {
    auto cell_of = [&](long long tz) { return team + (tz / A.T1) * (long long)A.nteams; };
    auto issue_tab = [&](long long tz) {  // table block of term tz into buffer tz % 2
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      uint64_t* b = &bar_tab[tz & 1];
      mbar_expect(b, zblk);
      bulk_g2s(tbs + (tz & 1) * (ZBLK_B / 16), A.tabT + (long long)(tz % A.T1) * LHN + K * h0, zblk, b);
    };
    auto issue_fh = [&](long long cell) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect(&bar_fh, zblk);
      bulk_g2s(fh, A.fhatT + cell * (long long)LHN + K * h0, zblk, &bar_fh);
    };
    auto w1_ready = [&](long long tz) {
      return ld_acquire(zcnt + 32 * (tz % NB)) >= (unsigned)(TM * (tz / NB + 1));
    };
    auto issue_w1 = [&](long long tz) {
      const double2* src = W1t + (tz % NB) * (long long)W1_BUF + (long long)(PLN * k) * NPEN;
      asm volatile("fence.proxy.async.global;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect(&bar_w1, PLN * W1IN_B);
      bulk_g2s(w1in, src, PLN * W1IN_B, &bar_w1);  // the member's 4 planes are contiguous
    };
    auto z_task = [&](long long tz, int tau) {
      z_pencil(ZTask{fh, tbs + (tz & 1) * (ZBLK_B / 16), W1t + (tz % NB) * (long long)W1_BUF, nh, h0, tau});
    };
    auto publish_z = [&](long long tz) {
      __threadfence();
      atomicAdd(zcnt + 32 * (tz % NB), 1u);
    };
    auto wait_buffer_free = [&](long long tz) {  // all members consumed W1(tz - NB)
      if (tz >= NB) poll_ge(ycnt + 32 * (tz % NB), (unsigned)(TM * (tz / NB)));
    };

    // ---------------- prologue: Z(0) complete, Z(1) part A ----------------
    uint32_t par_fh = 0;
    if (tid == 0) {
      issue_fh(cell_of(0));
      issue_tab(0);
      if (TT > 1) issue_tab(1);
    }
    if (warp >= 4) {
      mbar_wait(&bar_fh, par_fh);
      mbar_wait(&bar_tab[0], 0);
      const int tau = tid - 128;
      if (tau < na) z_task(0, tau);
    }
    __syncthreads();
    par_fh ^= 1;
    if (tid == 0) {
      publish_z(0);
      if (TT > 2) issue_tab(2);  // buffer 0 is free again
    }
    if (TT > 1 && warp >= 6) {
      const long long tz = 1;
      if (tz % A.T1 == 0) {  // new cell (T1 == 1 only)
        if (tid == 192) issue_fh(cell_of(tz));
        mbar_wait(&bar_fh, par_fh);
      }
      mbar_wait(&bar_tab[1], 0);
      const int tau = tid - 192;
      if (tau < ZA && tau < na) z_task(tz, tau);
    }
    if (TT > 1 && A.T1 == 1) par_fh ^= 1;
    __syncthreads();

    const bool leader = (tid == 0);
    bool w1_issued = false;
    uint32_t par_w1 = 0;
    const int xw = warp;                                  // X warps 0..5: rows 32 xw + lane
    const uint32_t tG = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(96 * (warp >> 2));
#pragma unroll 1
    for (long long tg = 0; tg < TT; tg++) {
      const int t = (int)(tg % A.T1);
      const long long cell = cell_of(tg);
      long long* st = (A.dbg && leader && tg >= 2 && tg < 6) ? A.dbg + (long long)blockIdx.x * 128 + (tg - 2) * 16 : nullptr;
      if (st) st[0] = clock64();
      // ---- W1(tg) in shared memory ----
      if (leader) {
        if (!w1_issued) {
          poll_ge(zcnt + 32 * (tg % NB), (unsigned)(TM * (tg / NB + 1)));
          issue_w1(tg);
        }
        w1_issued = false;
      }
      if (warp < 4) mbar_wait(&bar_w1, par_w1);
      par_w1 ^= 1;
      if (st) st[1] = clock64();
      if (leader) {
        __threadfence();
        atomicAdd(ycnt + 32 * (tg % NB), 1u);  // W1(tg) consumed by this member
      }
      // ---- R1: Y(tg) on warps 0-3, Z(tg+1) part B on warp 4 ----
      {
        int kind = TK_NONE;
        if (warp < 4 && lane < K) kind = TK_Y;
        else if (warp == 4 && tg + 1 < TT && ZA + lane < na) kind = TK_Z;
        if (kind == TK_Y) {
          const double2* src = w1in + warp * NPEN + lane * K;  // pencil lx = lane of plane w
          double2 x[K];
#pragma unroll
          for (int i = 0; i < K; i++) x[i] = src[i];
          double2* dst = ysh + warp * YPL + lane;             // Y[p][py][ix]
#pragma unroll 1
          for (int r = 0; r < 3; r++) {
            double2 u[16];
            xform48_regs(x, r, u);
#pragma unroll
            for (int q = 0; q < 16; q++) dst[(3 * q + r) * K] = u[fftd::qslot(q)];
          }
        } else if (kind == TK_Z) {
          z_task(tg + 1, ZA + lane);
        }
      }
      __syncthreads();
      if (st) st[2] = clock64();
      if (tid == 128 && tg + 1 < TT) publish_z(tg + 1);  // Z(tg+1) complete in this member
      if (tid == 192 && tg + 3 < TT) issue_tab(tg + 3);  // buffer (tg+1) % 2 is free
      // f^ of the next cell: last used by Z(tg+1) part B (this R1); first needed by Z(tg+2) part A (R2)
      const bool new_cell_z = (tg + 2 < TT) && ((tg + 2) % A.T1 == 0);
      if (new_cell_z && tid == 192) issue_fh(cell_of(tg + 2));
      if (leader && tg + 1 < TT && w1_ready(tg + 1)) {  // input planes are free: copy during R2
        issue_w1(tg + 1);
        w1_issued = true;
      }
      // ---- R2: X(tg) on warps 0-5, Z(tg+2) part A on warps 6-7 ----
      if (warp < 6) {
        if (t == 0) {  // zero this warp's G accumulators
          uint32_t zw[32];
#pragma unroll
          for (int i = 0; i < 32; i++) zw[i] = 0u;
#pragma unroll
          for (int c = 0; c < 3; c++) tmem_st32(tG + 32 * c, zw);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        const int rho = 32 * xw + lane, pl = rho / P, py = rho - (rho / P) * P;
        const double2* src = ysh + pl * YPL + py * K;
        double2 x[K];
#pragma unroll
        for (int i = 0; i < K; i++) x[i] = src[i];
#pragma unroll 1
        for (int r = 0; r < 3; r++) {
          double2 u[16];
          xform48_regs(x, r, u);
#pragma unroll
          for (int hh = 0; hh < 2; hh++) {
            uint32_t gw[16];
            tmem_ld16(tG + 32 * r + 16 * hh, gw);
#pragma unroll
            for (int q = 0; q < 8; q++) {
              const double2 z = u[fftd::qslot(8 * hh + q)];
              const double acc = fma(z.x, z.y, __hiloint2double((int)gw[2 * q + 1], (int)gw[2 * q]));
              gw[2 * q] = (uint32_t)__double2loint(acc);
              gw[2 * q + 1] = (uint32_t)__double2hiint(acc);
            }
            tmem_st16(tG + 32 * r + 16 * hh, gw);
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        if (t == A.T1 - 1) {  // G[cell][px = 3q + r][pz][py]
          double* Gc = A.G + cell * (long long)(P * P * P) + (long long)(PLN * k + pl) * P + py;
#pragma unroll 1
          for (int r = 0; r < 3; r++) {
            uint32_t gw[32];
            tmem_ld32(tG + 32 * r, gw);
#pragma unroll
            for (int q = 0; q < 16; q++)
              Gc[(long long)(3 * q + r) * P * P] = __hiloint2double((int)gw[2 * q + 1], (int)gw[2 * q]);
          }
        }
      } else if (tg + 2 < TT) {
        const long long tz = tg + 2;
        if (lane == 0) wait_buffer_free(tz);
        __syncwarp();
        if (tz % A.T1 == 0) {
          mbar_wait(&bar_fh, par_fh);
        }
        mbar_wait(&bar_tab[tz & 1], (uint32_t)((tz >> 1) & 1));
        const int tau = tid - 192;
        if (tau < na) z_task(tz, tau);
      }
      if (new_cell_z) par_fh ^= 1;
      __syncthreads();
      if (st) st[3] = clock64();
    }
  }
done:
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
}
}  // namespace v5

}  // namespace f32

bool fast_available(const Ctx& c) { return c.N == 32 && c.P == 48; }

size_t xform32_ws_bytes_per_cell();
cudaError_t xform32_prepare();
void xform32_tables_lh(const double2* ab, double2* abL, int T1, int nb);
void xform32_forward(Ctx& c, const double* fin, double2* fhT, double2* scratch, long long n, int nb, cudaStream_t st,
                     const GatherSrc* gs);
void xform32_back(Ctx& c, const double* G, double2* scratch_a, double2* scratch_b, const double* fin, double* out,
                  long long n, bool euler, double s, cudaStream_t st, const GatherSrc* gs);

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
  if (e == cudaSuccess) e = fftd::fill_twiddles();
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
  // variant: FKS_HOT = v4 (default: decoupled warp roles, one CTA per SM), t12 (two virtual CTAs per SM) or c6
  // (6-CTA clusters)
  const char* hv = std::getenv("FKS_HOT");
  const std::string want = hv ? std::string(hv) : std::string("v4");
  int v4_per_sm = 0;
  e = cudaFuncSetAttribute(v4::hot_kernel_v4, cudaFuncAttributeMaxDynamicSharedMemorySize, v4::SMEM_B);
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v4_per_sm, v4::hot_kernel_v4, v4::NTHR, v4::SMEM_B);
  if (e != cudaSuccess) { cudaGetLastError(); v4_per_sm = 0; }
  int v5_per_sm = 0;
  e = cudaFuncSetAttribute(v5::hot_kernel_v5, cudaFuncAttributeMaxDynamicSharedMemorySize, v5::SMEM_B);
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v5_per_sm, v5::hot_kernel_v5, v5::NTHR, v5::SMEM_B);
  if (e != cudaSuccess) { cudaGetLastError(); v5_per_sm = 0; }
  if (want == "v5" && v5_per_sm >= 1) c.fast_kernel = 5;
  else if (want == "v4" && v4_per_sm >= 1) c.fast_kernel = 4;
  else if (want != "c6" && per_sm >= 1) c.fast_kernel = 3;
  else c.fast_kernel = 2;
  c.fast_variant = (c.fast_kernel == 2) ? CL : t12::TM;
  size_t w1_elems;
  if (c.fast_kernel == 5) {
    c.fast_nteams = c.num_sms / v5::TM;
    w1_elems = (size_t)c.fast_nteams * v5::NB * W1_BUF;
    e = cudaMalloc(&c.d_ctr, (size_t)c.fast_nteams * v5::CTR_STRIDE * sizeof(unsigned));
    if (e != cudaSuccess) { cudaGetLastError(); return cuda_status(e, "team counters"); }
  } else if (c.fast_kernel == 4) {
    c.fast_nteams = c.num_sms / v4::TM;
    w1_elems = (size_t)c.fast_nteams * v4::NB * W1_BUF;
    e = cudaMalloc(&c.d_ctr, (size_t)c.fast_nteams * v4::CTR_STRIDE * sizeof(unsigned));
    if (e != cudaSuccess) { cudaGetLastError(); return cuda_status(e, "team counters"); }
  } else if (c.fast_kernel == 3) {
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
                          cudaStream_t st, const GatherSrc* gs) {
  using namespace f32;
  // workspace: f^T [n][K^3] complex | scratch [n][P*K*16] complex | G [n][P^3] fp64
  double2* fhT = reinterpret_cast<double2*>(c.d_ws);
  double2* scratch = fhT + n * K * NPEN;
  double* G = reinterpret_cast<double*>(scratch + n * (long long)P * K * 16);
  c.prof.begin(1, st);
  xform32_forward(c, fin, fhT, scratch, n, c.fast_variant, st, gs);
  c.prof.end(1, st);

  c.prof.begin(2, st);
  if (c.fast_kernel == 5) {
    const long long nt = std::min<long long>(c.fast_nteams, n);
    v5::Args A{fhT, c.d_abT, G, c.d_w1, c.d_ctr, n, c.T + 1, (int)nt, c.dbg};
    cudaMemsetAsync(c.d_ctr, 0, (size_t)c.fast_nteams * v5::CTR_STRIDE * sizeof(unsigned), st);
    void* args[] = {&A};
    cudaError_t e = cudaLaunchCooperativeKernel((void*)v5::hot_kernel_v5, dim3((unsigned)(nt * v5::TM)),
                                                dim3(v5::NTHR), args, v5::SMEM_B, st);
    if (e != cudaSuccess) { c.prof.end(2, st); return cuda_status(e, "cooperative hot kernel launch (v5)"); }
  } else if (c.fast_kernel == 4) {
    const long long nt = std::min<long long>(c.fast_nteams, n);
    v4::Args A{fhT, c.d_abT, G, c.d_w1, c.d_ctr, n, c.T + 1, (int)nt, c.dbg};
    cudaMemsetAsync(c.d_ctr, 0, (size_t)c.fast_nteams * v4::CTR_STRIDE * sizeof(unsigned), st);
    void* args[] = {&A};
    cudaError_t e = cudaLaunchCooperativeKernel((void*)v4::hot_kernel_v4, dim3((unsigned)(nt * v4::TM)),
                                                dim3(v4::NTHR), args, v4::SMEM_B, st);
    if (e != cudaSuccess) { c.prof.end(2, st); return cuda_status(e, "cooperative hot kernel launch (v4)"); }
  } else if (c.fast_kernel == 3) {
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
  xform32_back(c, G, scratch, fhT, fin, out, n, euler, s, st, gs);
  c.prof.end(3, st);
  return cuda_status(cudaPeekAtLastError(), "fast collision");
}

}  // namespace fks
