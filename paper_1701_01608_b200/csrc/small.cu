// Fast path for N = 16 (P = 24) and N = 24 (P = 36): the term loop (rows a3-a5 of DESIGN.md §2) as ONE persistent
// sm_100a kernel in which a CTA owns a whole (cell, z-class r, term chunk) unit — no inter-CTA exchange.
//
// Every pruned transform along one axis is z(p) = sum_{l=-h..h} Z(l) e^{2 pi i l p/P}, h = N/2 - 1, P = 3H, H = N/2
// (P:1589-1599 pruned to the retained modes K', A9, A10).  It is computed per output class r (p = 3q + r) as
//     y_r(n) = w_P^{n r} [ Z(n) + Z(n - H) w_3^{-r} ]   (n = 1..H-1;  y_r(0) = Z(0))
//     z(3q + r) = sum_n y_r(n) e^{2 pi i n q/H}          (an H-point inverse FFT held in registers, H = 8 or 12)
// so one "class task" produces H outputs.  Per term t and unit (cell, r):
//   Z tasks (one per lower-half pencil (lx, ly), together with its mirror (-lx, -ly)): the products
//     Z = (a_t + i b_t) f^ (mirror: (a_t + i b_t)(l) conj f^(l) at reversed lz, a_t, b_t even, f real) formed on
//     the fly from L2 (transposed, coalesced layouts), class r of the z-pass  ->  W1[lx][q][ly]   (shared memory)
//   Y tasks (lx, q) for each y-class r':  W1 along ly  ->  W2[q''][q][lx]                      (shared memory)
//   X tasks (q'', q, rx): W2 along lx  ->  z on the P-grid points (3q'+rx, 3q''+r', 3q+r);  G += Re z * Im z,
//     accumulated in TMEM over the unit's terms (the balanced tables make Re z = A_t, Im z = B_t).
// The unit's G block is written once; chunks of one cell are summed in a fixed order by small_reduce_kernel.
// Phases (one CTA barrier each, W2 double-buffered so that X of class r' overlaps Y of class r' + 1):
//   A: Z(t) + X2(t-1)    B: Y0(t)    C: X0(t) + Y1(t)    D: X1(t) + Y2(t)
// The per-warp task lists of every phase are a static schedule built on the host (small_schedule): X tasks are
// pinned to the TMEM lane quarter that holds their G block, the other tasks fill the least-loaded warps.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "fks_internal.cuh"

namespace fks {
namespace sm {

template <int N>
struct Geo {
  static constexpr int H = N / 2, P = 3 * H, K = N - 1, h = H - 1, KK = K * K, NLOW = (KK + 1) / 2;
  static constexpr int R = H / 4;                         // H = 4 R: FFT_H = radix-R x radix-4
  static constexpr int NZS = (NLOW + 31) / 32;            // Z slots (lower-half pencil + mirror per lane)
  static constexpr int NYL = K * H, NYS = (NYL + 31) / 32;       // Y lane tasks (q, lx) per class r'
  static constexpr int XSR = (H * H + 31) / 32, NXS = 3 * XSR;  // X slots per x-class rx, per y-class r'
  static constexpr int XQB = (NXS + 3) / 4;               // X TMEM column blocks per class r' and lane quarter
  static constexpr int TCOLS = (3 * XQB * 32 <= 128) ? 128 : (3 * XQB * 32 <= 256 ? 256 : 512);
  static constexpr int W1_E = KK * H;                     // W1[q][lx][ly]
  static constexpr int W2_E = H * H * K;                  // W2[q''][q][lx]
  static constexpr int SMEM = (W1_E + 2 * W2_E) * 16;
};

constexpr int kMaxWarps = 16, kMaxItems = 12;
enum { T_Z = 0, T_Y = 1, T_X = 2 };
// phases: 0 = A (Z + X of class 2), 1 = B (Y0), 2 = C (X0 + Y1), 3 = D (X1 + Y2)
struct Sched {
  unsigned char cnt[4][kMaxWarps];
  unsigned char item[4][kMaxWarps][kMaxItems];  // (type << 5) | slot
};
__constant__ Sched c_sched16, c_sched24;

struct Args {
  const double2* fhT;   // [cell][K][NLOW]: f^ of the lower-half pencils, lz-major (coalesced over pencils)
  const double2* tabT;  // [t][K][NLOW]: balanced (a_t k_t, b_t / k_t), same layout
  double* Gout;         // [cell][S][P^3] (S > 1) or [cell][P^3] (S = 1), layout [px][py][pz]
  long long n_cells;
  int T1, S;            // terms, term chunks per (cell, r)
  long long* dbg;       // optional clock64 stamps [cta][warp][step] of the first unit (FKS_PHASE_TIMING); nullptr
};

// ---- small complex helpers ---------------------------------------------------------------------------------
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 w, double2 v) {
  return make_double2(fma(w.x, v.x, -w.y * v.y), fma(w.x, v.y, w.y * v.x));
}
// 4-point inverse DFT in place (w4 = +i), natural order
__device__ __forceinline__ void bfly4(double2& x0, double2& x1, double2& x2, double2& x3) {
  const double2 a = cadd(x0, x2), b = csub(x0, x2), c = cadd(x1, x3), d = csub(x1, x3);
  x0 = cadd(a, c);
  x2 = csub(a, c);
  x1 = make_double2(b.x - d.y, b.y + d.x);
  x3 = make_double2(b.x + d.y, b.y - d.x);
}
// 3-point inverse DFT in place (w3 = e^{+2 pi i/3})
__device__ __forceinline__ void bfly3(double2& x0, double2& x1, double2& x2) {
  constexpr double s3 = 0.86602540378443864676;
  const double2 s = cadd(x1, x2), d = csub(x1, x2);
  const double2 m = make_double2(fma(-0.5, s.x, x0.x), fma(-0.5, s.y, x0.y));
  x0 = cadd(x0, s);
  x1 = make_double2(fma(-s3, d.y, m.x), fma(s3, d.x, m.y));  // the s3 products folded into FMAs: 12 instead of 14
  x2 = make_double2(fma(s3, d.y, m.x), fma(-s3, d.x, m.y));
}
// output slot of z(q) after fft_h: H = 4R, n = 4 n1 + n2, q = q1 + R q2 -> slot 4 q1 + q2
template <int R>
__device__ __forceinline__ constexpr int qslot(int q) { return 4 * (q % R) + q / R; }

// In-place H-point inverse DFT z(q) = sum_n u[n] e^{2 pi i n q/H}, H = 4R (R = 2: H = 8, R = 3: H = 12):
// H = 8: radix-2 over n1 (n = 4 n1 + n2), twiddle w_8^{q1 n2}, radix-4 over n2; H = 12: Good-Thomas 3 x 4 (below).
// z(q) ends in u[qslot<R>(q)].
template <int R>
__device__ __forceinline__ void fft_h(double2 (&u)[4 * R]) {
  constexpr double s2 = 0.70710678118654752440, s3 = 0.86602540378443864676;
  if (R == 2) {
#pragma unroll
    for (int n2 = 0; n2 < 4; n2++) {
      const double2 a = u[n2], b = u[4 + n2];
      u[n2] = cadd(a, b);
      u[4 + n2] = csub(a, b);
    }
    // w8^1 = s2 (1 + i), w8^2 = i, w8^3 = s2 (-1 + i)
    u[5] = make_double2(s2 * (u[5].x - u[5].y), s2 * (u[5].x + u[5].y));
    u[6] = make_double2(-u[6].y, u[6].x);
    u[7] = make_double2(-s2 * (u[7].x + u[7].y), s2 * (u[7].x - u[7].y));
#pragma unroll
    for (int q1 = 0; q1 < R; q1++) bfly4(u[4 * q1], u[4 * q1 + 1], u[4 * q1 + 2], u[4 * q1 + 3]);
  } else {
    // Good-Thomas (prime-factor) FFT12, 12 = 3 x 4 coprime: with n = (4 n1 + 3 n2) mod 12 and q = (4 k1 + 9 k2) mod 12,
    // w12^{nq} = w3^{n1 k1} w4^{n2 k2}, so the 3-point and 4-point stages need no twiddles between them (16 fewer
    // FP64 instructions than the Cooley-Tukey 3 x 4 form); the index maps are register renames after unrolling.
    double2 t[3][4];
#pragma unroll
    for (int n2 = 0; n2 < 4; n2++) {
      double2 a = u[(3 * n2) % 12], b = u[(4 + 3 * n2) % 12], c = u[(8 + 3 * n2) % 12];
      bfly3(a, b, c);
      t[0][n2] = a;
      t[1][n2] = b;
      t[2][n2] = c;
    }
#pragma unroll
    for (int k1 = 0; k1 < 3; k1++) bfly4(t[k1][0], t[k1][1], t[k1][2], t[k1][3]);
#pragma unroll
    for (int k1 = 0; k1 < 3; k1++)
#pragma unroll
      for (int k2 = 0; k2 < 4; k2++) u[qslot<R>((4 * k1 + 9 * k2) % 12)] = t[k1][k2];
  }
}

// twiddles w_P^m = e^{+2 pi i m/P} (P = 24, 36) in the constant bank: indexed by compile-time constants after
// unrolling, they become constant-bank operands of the DFMA / DMUL instructions (no load instructions)
__constant__ double2 c_tw24[24], c_tw36[36];
template <int P>
__device__ __forceinline__ double2 twc(int m) { return P == 24 ? c_tw24[m % 24] : c_tw36[m % 36]; }

// class-r combine (r a compile-time constant) of one pruned input vector x(l), l = -h..h stored at in(l + h):
// u[0] = x(0);  u[n] = w_P^{n r} (x(n) + x(n - H) w3^{-r}) for n >= 1,  w3^{-1} = (-1/2, -s3), w3^{-2} = (-1/2, s3)
template <int H, int r, class In>
__device__ __forceinline__ void combine(const In& in, double2 (&u)[H]) {
  constexpr double s3 = 0.86602540378443864676;
  constexpr double c3i = (r == 1) ? -s3 : s3;
  u[0] = in(H - 1);
#pragma unroll
  for (int n = 1; n < H; n++) {
    const double2 a = in(n + H - 1), v = in(n - 1);
    if (r == 0) {
      u[n] = cadd(a, v);
    } else {
      double2 acc;
      acc.x = fma(-0.5, v.x, a.x);
      acc.x = fma(-c3i, v.y, acc.x);
      acc.y = fma(-0.5, v.y, a.y);
      acc.y = fma(c3i, v.x, acc.y);
      u[n] = cmul(twc<3 * H>(r * n), acc);
    }
  }
}

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
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}


// ---- the three task kinds (one lane = one class task; the class is a compile-time constant) ----------------------
// Z: lower-half pencil jj (and its mirror) of class r: products from L2, z-pass, W1[q][lx][ly]
template <int N, int r>
__device__ __forceinline__ void z_task(double2* W1, const double2* fh, const double2* tabT, int slot, int lane, int t) {
  using G = Geo<N>;
  constexpr int H = G::H, K = G::K, R = G::R, NLOW = G::NLOW;
  const int j = 32 * slot + lane;
  const bool act = j < NLOW;
  const int jj = act ? j : NLOW - 1;
  const double2* tb = tabT + (long long)t * (K * NLOW) + jj;
  const double2* fp = fh + jj;
  // pencil (lx, ly) = lower-half pencil jj, mirror (-lx, -ly):  Zp(lz) = ab(l) f(l),  Zm(lz) = ab(l') conj f(l') with
  // l' = (lx, ly, -lz) (a_t, b_t even in l; f^ Hermitian).  Stored index i = lz + h.  The inputs are loaded in the
  // quadruples lz = +-n, +-(H - n) that complete u[n] and u[H - n] of both vectors (few live registers).
  constexpr double s3 = 0.86602540378443864676;
  constexpr double c3i = (r == 1) ? -s3 : s3;
  double2 up[H], um[H];
  auto prod = [&](int i, double2& zp, double2& zm) {
    const double2 a = __ldg(tb + (long long)i * NLOW), f = __ldg(fp + (long long)i * NLOW);
    const double by = a.y * f.y, bx = a.y * f.x;
    zp = make_double2(fma(a.x, f.x, -by), fma(a.x, f.y, bx));   // ab * f
    zm = make_double2(fma(a.x, f.x, by), fma(-a.x, f.y, bx));   // ab * conj f
  };
  auto comb = [&](double2 a, double2 v, int n) {  // w_P^{n r} (a + v w3^{-r})
    if (r == 0) return cadd(a, v);
    double2 acc;
    acc.x = fma(-0.5, v.x, a.x);
    acc.x = fma(-c3i, v.y, acc.x);
    acc.y = fma(-0.5, v.y, a.y);
    acc.y = fma(c3i, v.x, acc.y);
    return cmul(twc<3 * H>(r * n), acc);
  };
  prod(H - 1, up[0], um[0]);  // lz = 0
#pragma unroll
  for (int n = 1; n <= H / 2; n++) {
    // lz = n (idx n+h) -> A, -n (h-n) -> B, n-H (n-1) -> C, H-n (K-n) -> D
    double2 pA, mA, pB, mB, pC, mC, pD, mD;
    prod(n + H - 1, pA, mA);
    prod(n - 1, pC, mC);
    if (n < H / 2) {
      prod(H - 1 - n, pB, mB);
      prod(K - n, pD, mD);
    } else {
      pB = pC; mB = mC; pD = pA; mD = mA;
    }
    // pencil: x(n) = pA, x(n-H) = pC, x(H-n) = pD, x(-n) = pB;  mirror: x(n) = mB, x(n-H) = mD, x(H-n) = mC, x(-n) = mA
    up[n] = comb(pA, pC, n);
    um[n] = comb(mB, mD, n);
    if (n < H / 2) {
      up[H - n] = comb(pD, pB, H - n);
      um[H - n] = comb(mC, mA, H - n);
    }
  }
  const int ix = jj / K, iy = jj - ix * K;
  fft_h<R>(up);
  if (act) {
#pragma unroll
    for (int q = 0; q < H; q++) W1[(q * K + ix) * K + iy] = up[qslot<R>(q)];
  }
  fft_h<R>(um);
  if (act && j != NLOW - 1) {  // the centre pencil (0, 0) is its own mirror
#pragma unroll
    for (int q = 0; q < H; q++) W1[(q * K + (K - 1 - ix)) * K + (K - 1 - iy)] = um[qslot<R>(q)];
  }
}

// Y: lane task tau = q K + lx of y-class rp: W1[q][lx][.] along ly -> W2[q''][q][lx]
template <int N, int rp>
__device__ __forceinline__ void y_task(const double2* W1, double2* W2b, int slot, int lane) {
  using G = Geo<N>;
  constexpr int H = G::H, K = G::K, R = G::R;
  const int tau = 32 * slot + lane;
  const bool act = tau < G::NYL;
  const int tt = act ? tau : G::NYL - 1;
  const double2* in = W1 + tt * K;
  double2 u[H];
  combine<H, rp>([&](int i) { return in[i]; }, u);
  fft_h<R>(u);
  if (act) {
    const int q = tt / K, ix = tt - q * K;
    double2* out = W2b + q * K + ix;
#pragma unroll
    for (int q2 = 0; q2 < H; q2++) out[q2 * H * K] = u[qslot<R>(q2)];
  }
}

// X: slot of x-class rx (uniform per slot, lane task pen = q'' H + q): W2[q''][q][.] along lx -> G += Re z Im z
template <int N, int rx>
__device__ __forceinline__ void x_task(const double2* W2b, uint32_t col, int pen) {
  using G = Geo<N>;
  constexpr int H = G::H, K = G::K, R = G::R;
  const bool act = pen < H * H;
  const double2* in = W2b + (act ? pen : H * H - 1) * K;
  double2 u[H];
  combine<H, rx>([&](int i) { return in[i]; }, u);
  fft_h<R>(u);
  uint32_t gw[32];
  tmem_ld32(col, gw);
#pragma unroll
  for (int q = 0; q < H; q++) {
    const double2 z = u[qslot<R>(q)];
    const double g = __hiloint2double((int)gw[2 * q + 1], (int)gw[2 * q]);
    const double acc = act ? fma(z.x, z.y, g) : g;
    gw[2 * q] = (uint32_t)__double2loint(acc);
    gw[2 * q + 1] = (uint32_t)__double2hiint(acc);
  }
  tmem_st32(col, gw);  // (an asynchronous load issued before the transform measured 3 % slower on c1)
}

template <int N, int WARPS>
__global__ void __launch_bounds__(32 * WARPS, N == 16 ? 2 : 1) small_term_kernel(Args A) {
  using G = Geo<N>;
  constexpr int H = G::H, P = G::P, K = G::K, NLOW = G::NLOW;
  extern __shared__ __align__(16) unsigned char smem[];
  double2* W1 = reinterpret_cast<double2*>(smem);
  double2* W2 = W1 + G::W1_E;              // [2][H][H][K]
  __shared__ uint32_t tmem_base_sh;
  const Sched& sc = (N == 16) ? c_sched16 : c_sched24;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"((uint32_t)__cvta_generic_to_shared(&tmem_base_sh)), "r"(G::TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tq = tmem_base_sh + ((uint32_t)(32 * (warp & 3)) << 16);  // this warp's lane quarter
  // X block (r', s) lives in lane quarter s % 4, columns 32 (r' XQB + s / 4)
  auto xcol = [&](int rp, int s) { return tq + 32u * (uint32_t)(rp * G::XQB + (s >> 2)); };
  const long long units = A.n_cells * 3 * A.S;

#pragma unroll 1
  for (long long u = blockIdx.x; u < units; u += gridDim.x) {
    const long long cell = u / (3 * A.S);
    const int r = (int)((u / A.S) % 3), ch = (int)(u % A.S);
    const int t0 = (int)((long long)ch * A.T1 / A.S), t1 = (int)((long long)(ch + 1) * A.T1 / A.S);
    // zero this warp's G blocks (the X blocks it runs in phases A / C / D)
    {
      uint32_t zw[32];
#pragma unroll
      for (int i = 0; i < 32; i++) zw[i] = 0u;
#pragma unroll 1
      for (int ph = 0; ph < 4; ph++) {
        if (ph == 1) continue;
        const int rp = ph == 0 ? 2 : ph - 2;
#pragma unroll 1
        for (int i = 0; i < sc.cnt[ph][warp]; i++) {
          const int it = sc.item[ph][warp][i];
          if ((it >> 5) == T_X) tmem_st32(xcol(rp, it & 31), zw);
        }
      }
    }
    const double2* fh = A.fhT + cell * (long long)(K * NLOW);

#ifdef FKS_SMALL_PHASE_TIMING
    int dstep = 0;
#endif
    // phase runner: X items of class xr (-1: skip X), Z items of term zt (-1: skip Z), Y items of class yr
    auto run_phase = [&](int ph, int zt, int xr, int xb, int yr, int yb) {
#pragma unroll 1
      for (int i = 0; i < sc.cnt[ph][warp]; i++) {
        const int it = sc.item[ph][warp][i];
        const int ty = it >> 5, s = it & 31;
        if (ty == T_Z) {
          if (zt >= 0) {
            if (r == 0) z_task<N, 0>(W1, fh, A.tabT, s, lane, zt);
            else if (r == 1) z_task<N, 1>(W1, fh, A.tabT, s, lane, zt);
            else z_task<N, 2>(W1, fh, A.tabT, s, lane, zt);
          }
        } else if (ty == T_Y) {
          if (yr < 0) continue;
          double2* W2b = W2 + yb * G::W2_E;
          if (yr == 0) y_task<N, 0>(W1, W2b, s, lane);
          else if (yr == 1) y_task<N, 1>(W1, W2b, s, lane);
          else y_task<N, 2>(W1, W2b, s, lane);
        } else if (xr >= 0) {
          const double2* W2b = W2 + xb * G::W2_E;
          const int rx = s / G::XSR, pen = 32 * (s - rx * G::XSR) + lane;
          const uint32_t col = xcol(xr, s);
          if (rx == 0) x_task<N, 0>(W2b, col, pen);
          else if (rx == 1) x_task<N, 1>(W2b, col, pen);
          else x_task<N, 2>(W2b, col, pen);
        }
      }
#ifdef FKS_SMALL_PHASE_TIMING  // tools/phase_timing_small.py (a build variant: the stamps are not in the product)
      if (A.dbg && u == blockIdx.x && blockIdx.x < 32 && lane == 0 && dstep < 64) A.dbg[((long long)blockIdx.x * 16 + warp) * 128 + 2 * dstep] = clock64();
      __syncthreads();
      if (A.dbg && u == blockIdx.x && blockIdx.x < 32 && lane == 0 && dstep < 64) A.dbg[((long long)blockIdx.x * 16 + warp) * 128 + 2 * dstep + 1] = clock64();
      dstep++;
#else
      __syncthreads();
#endif
    };

    // phase sequence (ONE call site of run_phase keeps one copy of every task body in the kernel):
    //   per term t:  A: Z(t) + X2(t-1) [X2 reads the buffer Y2(t-1) wrote]   B: Y0(t) -> wb
    //                C: X0(t) from wb, Y1(t) -> wb^1    D: X1(t) from wb^1, Y2(t) -> wb    (then wb ^= 1)
    //   and a final drain phase A with X2(t1 - 1) only.  (Moving X2(t-1) into B, next to Y0(t), measured 4 %
    //   slower: phase A then holds only the long Z tasks.)
    int wb = 0;  // W2 buffer of the next Y0 pass
    const int nsteps = 4 * (t1 - t0) + 1;
#pragma unroll 1
    for (int k = 0; k < nsteps; k++) {
      const int ph = k & 3, t = t0 + (k >> 2);
      if (ph == 0) run_phase(0, t < t1 ? t : -1, t > t0 ? 2 : -1, wb ^ 1, -1, 0);
      else if (ph == 1) run_phase(1, -1, -1, 0, 0, wb);
      else if (ph == 2) run_phase(2, -1, 0, wb, 1, wb ^ 1);
      else { run_phase(3, -1, 1, wb ^ 1, 2, wb); wb ^= 1; }
    }

    // write the unit's G block: G[px = 3q' + rx][py = 3q'' + r'][pz = 3q + r]
    double* Gc = A.Gout + (A.S > 1 ? (cell * A.S + ch) : cell) * (long long)(P * P * P);
#pragma unroll 1
    for (int ph = 0; ph < 4; ph++) {
      if (ph == 1) continue;
      const int rp = ph == 0 ? 2 : ph - 2;
#pragma unroll 1
      for (int i = 0; i < sc.cnt[ph][warp]; i++) {
        const int it = sc.item[ph][warp][i];
        if ((it >> 5) != T_X) continue;
        const int s = it & 31;
        uint32_t gw[32];
        tmem_ld32(xcol(rp, s), gw);
        const int rx = s / G::XSR, pen = 32 * (s - rx * G::XSR) + lane;
        if (pen < H * H) {
          const int q2 = pen / H, q = pen - q2 * H;
          const int py = 3 * q2 + rp, pz = 3 * q + r;
#pragma unroll
          for (int qq = 0; qq < H; qq++)
            Gc[((long long)(3 * qq + rx) * P + py) * P + pz] = __hiloint2double((int)gw[2 * qq + 1], (int)gw[2 * qq]);
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_sh), "r"(G::TCOLS));
}

// f^ [cell][ix][iy][iz] (generic forward output)  ->  fhT[cell][iz][j], j < NLOW lower-half pencils
__global__ void fhat_lower_T_kernel(const double2* __restrict__ hat, double2* __restrict__ fhT, long long n, int K,
                                    int nlow) {
  const long long per = (long long)K * nlow;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * per; e += (long long)gridDim.x * blockDim.x) {
    const long long c = e / per;
    const int rem = (int)(e - c * per), iz = rem / nlow, j = rem - iz * nlow;
    fhT[e] = hat[(c * K * K + j) * K + iz];
  }
}

// sum of the S term-chunk partial G blocks of each cell, in chunk order (deterministic)
__global__ void small_reduce_kernel(const double* __restrict__ Gp, double* __restrict__ G, long long n, int S, long long P3) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * P3; e += (long long)gridDim.x * blockDim.x) {
    const long long c = e / P3, i = e - c * P3;
    const double* src = Gp + c * S * P3 + i;
    double s = src[0];
    for (int k = 1; k < S; k++) s += src[k * P3];
    G[e] = s;
  }
}

// ---- host: static per-phase schedule ---------------------------------------------------------------------------
template <int N>
static Sched make_schedule(int warps) {
  using G = Geo<N>;
  Sched s{};
  for (int ph = 0; ph < 4; ph++) {
    std::vector<int> load(warps, 0);
    auto put = [&](int w, int type, int slot, int dur) {
      s.item[ph][w][s.cnt[ph][w]++] = (unsigned char)((type << 5) | slot);
      load[w] += dur;
    };
    // X items first: pinned to the lane quarter of their TMEM block (slot % 4), least-loaded warp of it
    if (ph != 1) {
      for (int sl = 0; sl < G::NXS; sl++) {
        int best = -1;
        for (int w = sl % 4; w < warps; w += 4)
          if (best < 0 || load[w] < load[best]) best = w;
        put(best, T_X, sl, 1);
      }
    }
    // then the free items, longest first (Z: pencil + mirror = two class tasks)
    auto free_items = [&](int type, int n, int dur) {
      for (int sl = 0; sl < n; sl++) {
        int best = 0;
        for (int w = 1; w < warps; w++)
          if (load[w] < load[best]) best = w;
        put(best, type, sl, dur);
      }
    };
    if (ph == 0) free_items(T_Z, G::NZS, 2);
    else free_items(T_Y, G::NYS, 1);
  }
  return s;
}

#ifndef FKS_SMALL_WARPS24
#define FKS_SMALL_WARPS24 12
#endif
template <int N>
constexpr int warps_for() { return N == 16 ? 8 : FKS_SMALL_WARPS24; }

}  // namespace sm

bool small_available(const Ctx& c) { return (c.N == 16 || c.N == 24) && c.P == 3 * c.N / 2; }

// Test-only (fks.h): the host-built per-phase task schedule of the small-N kernel, no device needed.
extern "C" int fks_small_schedule(int N, int* warps, int* nzs, int* nys, int* nxs, unsigned char* cnt,
                                  unsigned char* items) {
  if (N != 16 && N != 24) return -1;
  const int W = N == 16 ? sm::warps_for<16>() : sm::warps_for<24>();
  const sm::Sched s = N == 16 ? sm::make_schedule<16>(W) : sm::make_schedule<24>(W);
  if (warps) *warps = W;
  if (nzs) *nzs = N == 16 ? sm::Geo<16>::NZS : sm::Geo<24>::NZS;
  if (nys) *nys = N == 16 ? sm::Geo<16>::NYS : sm::Geo<24>::NYS;
  if (nxs) *nxs = N == 16 ? sm::Geo<16>::NXS : sm::Geo<24>::NXS;
  for (int ph = 0; ph < 4; ph++)  // ABI layout cnt[4][16], items[4][16][12]
    for (int w = 0; w < 16; w++) {
      const bool in = w < sm::kMaxWarps;
      if (cnt) cnt[ph * 16 + w] = in ? s.cnt[ph][w] : 0;
      for (int i = 0; i < 12; i++)
        if (items) items[(ph * 16 + w) * 12 + i] = (in && i < sm::kMaxItems) ? s.item[ph][w][i] : 0;
    }
  return 0;
}

static int small_smax() { return 16; }

size_t small_ws_bytes_per_cell(const Ctx& c) {
  const size_t K = c.K, P = c.P, nlow = (K * K + 1) / 2;
  return generic_ws_bytes_per_cell(c) + 16 * K * nlow + 8 * (size_t)small_smax() * P * P * P;
}

template <int N>
static fks_status small_prepare_n(Ctx& c) {
  using G = sm::Geo<N>;
  constexpr int W = sm::warps_for<N>();
  sm::Sched s = sm::make_schedule<N>(W);
  cudaError_t e = cudaMemcpyToSymbol(N == 16 ? sm::c_sched16 : sm::c_sched24, &s, sizeof(s));
  {  // w_P^m, long double accuracy
    double2 tw[G::P];
    const long double pi = 3.14159265358979323846264338327950288L;
    for (int m = 0; m < G::P; m++) tw[m] = make_double2((double)cosl(2.0L * pi * m / G::P), (double)sinl(2.0L * pi * m / G::P));
    if (e == cudaSuccess) {
      if constexpr (N == 16) e = cudaMemcpyToSymbol(sm::c_tw24, tw, sizeof(tw));
      else e = cudaMemcpyToSymbol(sm::c_tw36, tw, sizeof(tw));
    }
  }
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(sm::small_term_kernel<N, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
  int per_sm = 0;
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sm::small_term_kernel<N, W>, 32 * W, G::SMEM);
  if (e != cudaSuccess) return cuda_status(e, "small-N kernel attributes");
  if (per_sm < 1) { set_error("small-N term kernel does not fit on one SM"); return FKS_ERR_UNSUPPORTED; }
  per_sm = std::min(per_sm, 512 / G::TCOLS);  // TMEM columns per SM
  c.small_ctas = per_sm * c.num_sms;
  // transposed lower-half tables [t][iz][j]
  const long long per = (long long)G::K * G::NLOW;
  e = cudaMalloc(&c.d_abT, (size_t)(c.T + 1) * per * sizeof(double2));
  if (e != cudaSuccess) { cudaGetLastError(); return cuda_status(e, "small-N table allocation"); }
  const long long tot = (long long)(c.T + 1) * per;
  sm::fhat_lower_T_kernel<<<(unsigned)std::min<long long>((tot + 255) / 256, 4096), 256>>>(c.d_ab, c.d_abT, c.T + 1,
                                                                                          G::K, G::NLOW);
  c.launches++;
  c.fast_variant = 3;  // CTAs per cell (one per z-class)
  c.fast_nteams = c.small_ctas;
  return cuda_status(cudaDeviceSynchronize(), "small-N prepare");
}

fks_status small_prepare(Ctx& c) { return c.N == 16 ? small_prepare_n<16>(c) : small_prepare_n<24>(c); }

// term chunks per (cell, r): a function of N and the term count only (at most small_smax()), so that the
// summation order of G — hence every bit of Q — does not depend on how a batch is split into calls or chunks
// Chunks of ~26 terms at N = 24 (c1: 10 chunks, 1920 units = 12.97 waves of the 148-CTA grid, so the last wave is
// full: 3.672 ms per c1 step vs 3.729 with 32-term chunks (11.7 waves), 3.722 with 20 and 3.818 with 16;
// profiles/r02_experiments.txt r2sc), ~3 terms at N = 16 (c0 has only 8 cells: parallelism over terms; c0 step
// 0.1275 ms with 8-term chunks (72 units), 0.1175 with 3 (144 units), 0.1245 with 2; r2c0).
static int small_chunks(const Ctx& c) {
  const int T1 = c.T + 1;
  static const int tpc_env = [] { const char* e = std::getenv("FKS_SMALL_TPC"); return e ? std::atoi(e) : 0; }();
  const int tpc = tpc_env > 0 ? tpc_env : (c.N == 24 ? 26 : 3);
  return std::max(1, std::min(small_smax(), (T1 + tpc - 1) / tpc));
}

template <int N>
static fks_status small_collision_n(Ctx& c, const double* fin, double* out, long long n, bool euler, double s,
                                    cudaStream_t st, const GatherSrc* gs) {
  using G = sm::Geo<N>;
  constexpr int W = sm::warps_for<N>();
  if (gs) {  // no fused gather on this path: materialise f* in `out`, then collide in place
    c.prof.begin(0, st);
    // the gather writes destination cell j at fout + j N^3: `out` holds cells [cell0, cell0 + n)
    const long long nv = (long long)N * N * N;
    fks_status rc = launch_transport_gather(c, gs->base, out - gs->cell0 * nv, gs->sh, st, gs->cell0, n);
    c.prof.end(0, st);
    if (rc) return rc;
    fin = out;
  }
  GenericWs w = generic_ws(c, n);
  const long long P3 = (long long)G::P * G::P * G::P;
  double2* fhT = reinterpret_cast<double2*>(reinterpret_cast<char*>(c.d_ws) + generic_ws_bytes_per_cell(c) * n);
  double* Gp = reinterpret_cast<double*>(fhT + n * G::K * G::NLOW);
  c.prof.begin(1, st);
  generic_forward(c, fin, n, st);
  const long long tot = n * G::K * G::NLOW;
  sm::fhat_lower_T_kernel<<<(unsigned)std::min<long long>((tot + 255) / 256, 8192), 256, 0, st>>>(w.hat, fhT, n, G::K,
                                                                                                 G::NLOW);
  c.launches++;
  c.prof.end(1, st);

  c.prof.begin(2, st);
  const int S = small_chunks(c);
  sm::Args A{fhT, c.d_abT, S > 1 ? Gp : w.G, n, c.T + 1, S, c.dbg};
  const long long units = 3 * n * S;
  const unsigned grid = (unsigned)std::min<long long>(units, c.small_ctas);
  sm::small_term_kernel<N, W><<<grid, 32 * W, G::SMEM, st>>>(A);
  c.launches++;
  if (S > 1) {
    sm::small_reduce_kernel<<<(unsigned)std::min<long long>((n * P3 + 255) / 256, 8192), 256, 0, st>>>(Gp, w.G, n, S, P3);
    c.launches++;
  }
  c.prof.end(2, st);
  fks_status rc = cuda_status(cudaPeekAtLastError(), "small-N term kernel launch");
  if (rc) return rc;
  c.prof.begin(3, st);
  generic_back(c, fin, out, n, euler, s, st);
  c.prof.end(3, st);
  return cuda_status(cudaPeekAtLastError(), "small-N collision");
}

fks_status small_collision(Ctx& c, const double* fin, double* out, long long n, bool euler, double s, cudaStream_t st,
                           const GatherSrc* gs) {
  return c.N == 16 ? small_collision_n<16>(c, fin, out, n, euler, s, st, gs)
                   : small_collision_n<24>(c, fin, out, n, euler, s, st, gs);
}

}  // namespace fks
