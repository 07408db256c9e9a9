// Register-resident FFT building blocks for the N = 32 / P = 48 kernels (sm_100a, fp64).
//
// Every transform of length n = 16R (R = 2: n = 32, R = 3: n = 48) is split by decimation in frequency into R
// output classes r:   X[R q + r] = sum_{m<16} w16^{S m q} * ( w_n^{S r m} * sum_{j<R} x[m + 16 j] w_R^{S j r} ),
// i.e. a radix-R combine of the (possibly pruned) inputs followed by one 16-point FFT (radix 4 x 4) held in
// registers.  S = -1 is the forward (e^{-i...}) and S = +1 the inverse direction; no normalisation.
// Twiddles come from per-translation-unit __constant__ tables indexed by compile-time constants (uniform LDC).
#pragma once
#include <cuda_runtime.h>

namespace fks {
namespace fftd {

static __constant__ double2 c_tw48[48];  // e^{+2 pi i m/48}
static __constant__ double2 c_tw32[32];  // e^{+2 pi i m/32}

// Fill this translation unit's twiddle tables (host; long double accuracy).
static inline cudaError_t fill_twiddles() {
  double2 w48[48], w32[32];
  const long double pi = 3.14159265358979323846264338327950288L;
  for (int m = 0; m < 48; m++) w48[m] = make_double2((double)cosl(2.0L * pi * m / 48), (double)sinl(2.0L * pi * m / 48));
  for (int m = 0; m < 32; m++) w32[m] = make_double2((double)cosl(2.0L * pi * m / 32), (double)sinl(2.0L * pi * m / 32));
  cudaError_t e = cudaMemcpyToSymbol(c_tw48, w48, sizeof(w48));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_tw32, w32, sizeof(w32));
  return e;
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// w * v (S = +1) or conj(w) * v (S = -1)
template <int S>
__device__ __forceinline__ double2 cmul_s(double2 w, double2 v) {
  if (S > 0) return make_double2(fma(w.x, v.x, -w.y * v.y), fma(w.x, v.y, w.y * v.x));
  return make_double2(fma(w.x, v.x, w.y * v.y), fma(w.x, v.y, -w.y * v.x));
}
// e^{S 2 pi i m / n} for n in {16, 32, 48} (m taken mod n)
template <int S, int n>
__device__ __forceinline__ double2 tw(int m) {
  m %= n;
  double2 w = (n == 32) ? c_tw32[m] : c_tw48[m * (48 / n)];
  return S > 0 ? w : make_double2(w.x, -w.y);
}

// radix-4 butterfly over m1 -> q1 with w4 = e^{S i pi/2} = S i
template <int S>
__device__ __forceinline__ void bfly4(double2& x0, double2& x1, double2& x2, double2& x3) {
  const double2 a = cadd(x0, x2), b = csub(x0, x2), c = cadd(x1, x3), d = csub(x1, x3);
  x0 = cadd(a, c);
  x2 = csub(a, c);
  if (S > 0) {
    x1 = make_double2(b.x - d.y, b.y + d.x);
    x3 = make_double2(b.x + d.y, b.y - d.x);
  } else {
    x1 = make_double2(b.x + d.y, b.y - d.x);
    x3 = make_double2(b.x - d.y, b.y + d.x);
  }
}

// v * e^{S 2 pi i k/16}, k in 0..9
template <int S>
__device__ __forceinline__ double2 tw16(double2 v, int k) {
  const double h = 0.70710678118654752440;
  switch (k) {
    case 0: return v;
    case 2: return S > 0 ? make_double2(h * (v.x - v.y), h * (v.x + v.y)) : make_double2(h * (v.x + v.y), h * (v.y - v.x));
    case 4: return S > 0 ? make_double2(-v.y, v.x) : make_double2(v.y, -v.x);
    case 6: return S > 0 ? make_double2(-h * (v.x + v.y), h * (v.x - v.y)) : make_double2(h * (v.y - v.x), -h * (v.x + v.y));
    default: return cmul_s<S>(c_tw48[3 * k], v);
  }
}

// In-place 16-point DFT z(q) = sum_m u[m] e^{S 2 pi i m q/16}; on exit z(q) is at u[qslot(q)].
__device__ __forceinline__ constexpr int qslot(int q) { return 4 * (q & 3) + (q >> 2); }
template <int S>
__device__ __forceinline__ void fft16(double2 (&u)[16]) {
#pragma unroll
  for (int m2 = 0; m2 < 4; m2++) bfly4<S>(u[m2], u[m2 + 4], u[m2 + 8], u[m2 + 12]);
#pragma unroll
  for (int m2 = 1; m2 < 4; m2++)
#pragma unroll
    for (int q1 = 1; q1 < 4; q1++) u[m2 + 4 * q1] = tw16<S>(u[m2 + 4 * q1], m2 * q1);
#pragma unroll
  for (int q1 = 0; q1 < 4; q1++) bfly4<S>(u[4 * q1], u[4 * q1 + 1], u[4 * q1 + 2], u[4 * q1 + 3]);
}

// Inverse (S = +1) 16-point DFT, same contract as fft16<1>, with the second stage's twiddles folded into its
// butterflies: w16^1 = C(1 + i t), w16^3 = C(t + i), w16^2 = h(1 + i), w16^6 = h(-1 + i), w16^9 = -C(1 + i t)
// (C = cos pi/8, t = tan pi/8, h = 1/sqrt 2), so each radix-4 butterfly of the second stage forms its rotated
// pair sums with DADD/DFMA and applies C or h inside the output FMAs: 144 FP64 instructions instead of 160.
__device__ __forceinline__ void fft16i(double2 (&u)[16]) {
  constexpr double h = 0.70710678118654752440, C = 0.92387953251128675613, t = 0.41421356237309504880;
#pragma unroll
  for (int m2 = 0; m2 < 4; m2++) bfly4<1>(u[m2], u[m2 + 4], u[m2 + 8], u[m2 + 12]);
  bfly4<1>(u[0], u[1], u[2], u[3]);
  {  // q1 = 1: twiddles 1, w, w^2, w^3
    const double2 x0 = u[4], x1 = u[5], x2 = u[6], x3 = u[7];
    const double ex = x2.x - x2.y, ey = x2.x + x2.y;
    const double ax = fma(h, ex, x0.x), ay = fma(h, ey, x0.y), bx = fma(-h, ex, x0.x), by = fma(-h, ey, x0.y);
    const double A = x1.x - x3.y, B = x1.x + x3.y, Cc = x1.y + x3.x, D = x1.y - x3.x;
    const double cx = fma(-t, D, A), cy = fma(t, B, Cc), dx = fma(-t, Cc, B), dy = fma(t, A, D);
    u[4] = make_double2(fma(C, cx, ax), fma(C, cy, ay));
    u[6] = make_double2(fma(-C, cx, ax), fma(-C, cy, ay));
    u[5] = make_double2(fma(-C, dy, bx), fma(C, dx, by));
    u[7] = make_double2(fma(C, dy, bx), fma(-C, dx, by));
  }
  {  // q1 = 2: twiddles 1, w^2, w^4 = i, w^6
    const double2 x0 = u[8], x1 = u[9], x2 = u[10], x3 = u[11];
    const double ax = x0.x - x2.y, ay = x0.y + x2.x, bx = x0.x + x2.y, by = x0.y - x2.x;
    const double px = x1.x - x3.x, py = x1.y - x3.y, sx = x1.x + x3.x, sy = x1.y + x3.y;
    const double cx = px - sy, cy = py + sx, dx = sx - py, dy = sy + px;
    u[8] = make_double2(fma(h, cx, ax), fma(h, cy, ay));
    u[10] = make_double2(fma(-h, cx, ax), fma(-h, cy, ay));
    u[9] = make_double2(fma(-h, dy, bx), fma(h, dx, by));
    u[11] = make_double2(fma(h, dy, bx), fma(-h, dx, by));
  }
  {  // q1 = 3: twiddles 1, w^3, w^6, w^9
    const double2 x0 = u[12], x1 = u[13], x2 = u[14], x3 = u[15];
    const double e1 = x2.x + x2.y, e2 = x2.x - x2.y;
    const double ax = fma(-h, e1, x0.x), ay = fma(h, e2, x0.y), bx = fma(h, e1, x0.x), by = fma(-h, e2, x0.y);
    const double A = x1.x - x3.y, B = x1.x + x3.y, Cc = x1.y + x3.x, D = x1.y - x3.x;
    const double cx = fma(t, B, -Cc), cy = fma(t, D, A), dx = fma(t, A, -D), dy = fma(t, Cc, B);
    u[12] = make_double2(fma(C, cx, ax), fma(C, cy, ay));
    u[14] = make_double2(fma(-C, cx, ax), fma(-C, cy, ay));
    u[13] = make_double2(fma(-C, dy, bx), fma(C, dx, by));
    u[15] = make_double2(fma(C, dy, bx), fma(-C, dx, by));
  }
}

// Good-Thomas (prime-factor) form of the pruned inverse length-48 transform, 48 = 3 x 16 coprime: with the input
// map n = (16 n1 + 3 n2) mod 48 and the output map k = (16 k1 + 33 k2) mod 48, e^{2 pi i n k/48} =
// w3^{n1 k1} w16^{n2 k2}: a 3-point DFT over n1 and a 16-point DFT over n2, no inter-stage twiddles.  For the
// retained modes l = -15..15 (transform index l mod 48; 16..32 absent) the group of n2 holds Z(m) and Z(m - 16),
// m = 3 n2 mod 16, and its class-r value is  w3^{-r j} (Z(m) + w3^{2r} Z(m - 16)),  j = 3 n2 div 16; the 16-point
// transform then leaves z(k) at slot k2 with k = 3 pfa_q(r, k2) + r.
__host__ __device__ __forceinline__ constexpr int pfa_q(int r, int k2) { return (5 * r + 11 * k2) & 15; }
__host__ __device__ __forceinline__ constexpr int pfa_n2(int m) { return (11 * m) & 15; }  // m = 3 n2 mod 16
// u[pfa_n2(m)] from a = Z(m), v = Z(m - 16), m = 1..15 (m is a constant after unrolling, so the branch folds), with
// w = w3^{2r} = (cr, -sg): r = 1, 2: cr = -1/2, sg = +-sin(2pi/3); r = 0: cr = 1, sg = 0 (every case reduces to a + v)
__device__ __forceinline__ double2 pfa_combine(int m, double2 a, double2 v, double cr, double sg) {
  const int j = (3 * pfa_n2(m)) >> 4;
  if (j == 0) {  // a + w v
    return make_double2(fma(sg, v.y, fma(cr, v.x, a.x)), fma(-sg, v.x, fma(cr, v.y, a.y)));
  } else if (j == 2) {  // conj(w) a + v
    return make_double2(fma(-sg, a.y, fma(cr, a.x, v.x)), fma(sg, a.x, fma(cr, a.y, v.y)));
  } else {  // w a + conj(w) v
    const double sx = a.x + v.x, sy = a.y + v.y, dx = a.x - v.x, dy = a.y - v.y;
    return make_double2(fma(cr, sx, sg * dy), fma(cr, sy, -sg * dx));
  }
}

// Radix-R combine of class r:  u[m] = w_n^{S r m} sum_j x[m + 16 j] w_R^{S j r},  n = 16 R.
// `in.nz(i)` (a compile-time constant after unrolling) marks structurally non-zero inputs; `in(i)` reads one.
template <int R, int S, int r, class In>
__device__ __forceinline__ void dif_combine(const In& in, double2 (&u)[16]) {
  constexpr double c3 = 0.86602540378443864676;  // sin(2 pi/3)
#pragma unroll
  for (int m = 0; m < 16; m++) {
    double2 acc = make_double2(0.0, 0.0);
    bool have = false;
#pragma unroll
    for (int j = 0; j < R; j++) {
      const int i = m + 16 * j;
      if (!in.nz(i)) continue;
      const double2 v = in(i);
      const int e = (j * r) % R;  // rotation by w_R^{S e}
      if (e == 0) {
        acc = have ? cadd(acc, v) : v;
      } else if (R == 2) {  // rotation by -1
        acc = have ? csub(acc, v) : make_double2(-v.x, -v.y);
      } else {  // R == 3: w3^{S e} = (-1/2, +-c3)
        const double sg = ((e == 1) == (S > 0)) ? c3 : -c3;
        if (have) {
          acc.x = fma(-0.5, v.x, acc.x);
          acc.x = fma(-sg, v.y, acc.x);
          acc.y = fma(-0.5, v.y, acc.y);
          acc.y = fma(sg, v.x, acc.y);
        } else {
          acc = make_double2(fma(-0.5, v.x, -sg * v.y), fma(-0.5, v.y, sg * v.x));
        }
      }
      have = true;
    }
    constexpr int n = 16 * R;
    u[m] = ((r * m) % n == 0) ? acc : cmul_s<S>(n == 32 ? c_tw32[(r * m) % n] : c_tw48[(r * m) % n], acc);
  }
}

// Full class-r transform: combine + FFT16; X[R q + r] ends up in u[qslot(q)].
template <int R, int S, int r, class In>
__device__ __forceinline__ void dif_class(const In& in, double2 (&u)[16]) {
  dif_combine<R, S, r>(in, u);
  fft16<S>(u);
}

}  // namespace fftd
}  // namespace fks
