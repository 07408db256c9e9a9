// Forward (a2) and back (a6-a7) transforms of the N = 32, P = 48 fast path.
//
// Both use the Hermitian symmetry of real data: only the half-spectrum lz >= 0 (resp. kz >= 0) is computed and
// the other half follows by conjugation.  Each kernel owns either a plane (two axes local in shared memory)
// or a set of columns (the third axis), so one cell's transform is 2 (forward) or 3 (back) kernels with the
// compact intermediates in the workspace.  The short transforms are register FFTs (fft_dev.cuh).
//
//   forward  Kf1 plane jx : f(jx,jy,jz)  --z (real, lz=0..15)--> --y (ly in K')-->  F2[cell][jx][ly][lz]
//            Kf2 column ly: F2(:,ly,lz)  --x (lx in K'), N^-3-->  f^T[cell][lz][lx*31+ly] and its conjugate at -l
//   back     Kb1 plane px : G[cell][px][pz/2][py][pz%2] --y (real, ky=0..15)--> --z (kz in K')--> H2[cell][px][kz][ky]
//            Kb2 column kz: H2(:,kz,ky)  --x (kx in K'), P^-3, [Q^_0 := 0]--> --x inverse (jx)--> E1[cell][jx][kz][ky]
//            Kb3 plane jx : E1(jx,:,:)   --z inverse (jz)--> --y Hermitian->real (jy)-->  Q (or f* + s Q)
// (G is stored py-fastest so that the term-loop kernel writes it coalesced; the real axis of the back transform
// is therefore y.  Inside kb1..kb3 the loop variables keep the generic names "row"/"col".)
#include <algorithm>
#include "fks_internal.cuh"
#include "fft_dev.cuh"

namespace fks {
namespace x32 {

constexpr int N = 32, K = 31, P = 48, H = 16;  // H: retained non-negative z modes 0..15
constexpr int C = N / 2 - 1;                   // mode index offset (l = i - C)

// Each short transform below is a register FFT (fft_dev.cuh): a radix-2 (n = 32) or radix-3 (n = 48) combine of
// one output class followed by a 16-point FFT.  One thread = one (pencil, class) task; classes are warp-uniform.
using fftd::dif_class;
using fftd::dif_combine;
using fftd::fft16;
using fftd::qslot;

constexpr int PL8 = 8;  // planes (or pencil groups) per CTA in kf1 / kf2 / kb3 (3 CTAs per SM: the launch bounds
                        // cap them at 85 registers; kf1 -16 %, kf2 -11 %, kb3 -2.5 % against the register-limited 2)
constexpr int PB1 = 4;  // px planes per CTA in kb1 (2 measured the same, 1 30 % slower)
constexpr int KB1_T = 72 * PB1;  // kb1 threads: (class, plane, row pair)
constexpr int PB2 = 4;  // ky columns per CTA in kb2
constexpr int RS = 17;  // padded row stride (double2) of 16-element rows
constexpr int ZS = 49;  // padded row stride (double2) of 48-element rows

// Asynchronous global -> shared copies (LDGSTS): every load of a tile is in flight at once, instead of the few a
// register-staged loop keeps outstanding (the load phase dominated these HBM/latency-bound kernels).
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// smem input adaptors: nz(i) is constant-folded after unrolling
struct InCol {  // x[i] = base[i * ld], i = 0..n-1, all present
  const double2* base; int ld;
  __device__ __forceinline__ bool nz(int) const { return true; }
  __device__ __forceinline__ double2 operator()(int i) const { return base[i * ld]; }
};
struct InModes32 {  // x[i], i = k mod 32 for k in K' (16 absent); rows stored at base[(k + C) * ld]
  const double2* base; int ld;
  __device__ __forceinline__ bool nz(int i) const { return i != 16; }
  __device__ __forceinline__ double2 operator()(int i) const { return base[(i <= 15 ? i + C : i - 17) * ld]; }
};

// ---- forward ------------------------------------------------------------------------------------------
// kf1: CTA = (cell, 8 jx planes).  z: real FFT32 per row (two reals packed per complex, FFT16, untangle),
// lz = 0..15;  y: FFT32 over jy -> ly in K'.  Out F2[cell][jx][ly][lz].
// Source cells of the fused transport for destination cell j (global) and velocity planes jx0..jx0+7:
// sx[pl] (x index of plane jx0+pl), sy[jy], sz[jz], as in the transport gather kernel.
__device__ __forceinline__ void gather_tables(const GatherSrc& g, long long j, int jx0, int* sx, int* sy, int* sz) {
  const Shift& sh = g.sh;
  const int jz = (int)(j % sh.nz), jy = (int)((j / sh.nz) % sh.ny), jxc = (int)(j / ((long long)sh.nz * sh.ny));
  const int k = threadIdx.x;
  if (k < N) {
    int b = (jy - sh.delta[1][k]) % sh.ny; if (b < 0) b += sh.ny;
    int c = (jz - sh.delta[2][k]) % sh.nz; if (c < 0) c += sh.nz;
    sy[k] = b; sz[k] = c;
  }
  if (k < PL8) {
    int a = (jxc - sh.delta[0][jx0 + k]) % sh.nx; if (a < 0) a += sh.nx;
    sx[k] = a;
  }
}

__global__ void __launch_bounds__(256, 3) kf1(const double* __restrict__ f, double2* __restrict__ F2, const GatherSrc g,
                                           int gather) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* buf = reinterpret_cast<double2*>(smem_raw);  // [8][32][RS] (rows padded: conflict-free row tasks)
  __shared__ int sx[PL8], sy[N], sz[N];
  const int tid = threadIdx.x;
  const long long cell = blockIdx.x / (N / PL8);
  const int jx0 = (blockIdx.x % (N / PL8)) * PL8;
  if (!gather) {
    const double2* src = reinterpret_cast<const double2*>(f + (cell * N + jx0) * N * N);
#pragma unroll 4
    for (int i = tid; i < PL8 * N * H; i += 256) cp16(buf + (i >> 4) * RS + (i & 15), src + i);
  } else {  // fused transport: pairs (jz, jz+1) from one source cell move as 16 bytes, others as two 8-byte copies
    gather_tables(g, g.cell0 + cell, jx0, sx, sy, sz);
    __syncthreads();
    const long long nv = (long long)N * N * N;
#pragma unroll 4
    for (int i = tid; i < PL8 * N * H; i += 256) {
      const int pl = i >> 9, jy = (i >> 4) & 31, jz = 2 * (i & 15);
      const long long row = (long long)sx[pl] * g.sh.ny + sy[jy];
      const long long s0 = row * g.sh.nz + sz[jz], s1 = row * g.sh.nz + sz[jz + 1];
      const long long off = ((long long)(jx0 + pl) * N + jy) * N + jz;
      double2* d = buf + (i >> 4) * RS + (i & 15);
      if (s0 == s1 && g.in16) {
        cp16(d, g.base + s0 * nv + off);
      } else {
        cp8(d, g.base + s0 * nv + off);
        cp8(reinterpret_cast<double*>(d) + 1, g.base + s1 * nv + off + 1);
      }
    }
  }
  cp_wait_all();
  __syncthreads();
  {  // z: thread = (plane, jy)
    double2* row = buf + tid * RS;
    double2 u[16];
#pragma unroll
    for (int n = 0; n < 16; n++) u[n] = row[n];
    fft16<-1>(u);
#pragma unroll
    for (int k = 0; k < 16; k++) {
      const double2 z = u[qslot(k)], zm = u[qslot((16 - k) & 15)];
      const double2 e = make_double2(0.5 * (z.x + zm.x), 0.5 * (z.y - zm.y));   // even-sample DFT
      const double2 o = make_double2(0.5 * (z.y + zm.y), -0.5 * (z.x - zm.x));  // odd-sample DFT
      row[k] = k == 0 ? make_double2(e.x + o.x, 0.0) : fftd::cadd(e, fftd::cmul_s<-1>(fftd::c_tw32[k], o));
    }
  }
  __syncthreads();
  {  // y: thread = (class r, plane, lz)
    const int r = tid >> 7, s = (tid >> 4) & 7, lz = tid & 15;
    InCol in{buf + s * N * RS + lz, RS};
    double2 u[16];
    if (r == 0) dif_class<2, -1, 0>(in, u); else dif_class<2, -1, 1>(in, u);
    double2* dst = F2 + ((cell * N + jx0 + s) * K) * H + lz;
#pragma unroll
    for (int q = 0; q < 16; q++) {
      const int k = 2 * q + r;
      if (k == 16) continue;
      dst[(k <= 15 ? k + C : k - 32 + C) * H] = u[qslot(q)];
    }
  }
}

// Offset of pencil pp <= 480 (lower half of the (lx,ly) plane) at lz index iz in the per-CTA block layout used by
// the hot kernel: CTA c of a cell's team of nb CTAs owns pencils [h_c, h_{c+1}), h_c = floor(481 c / nb), stored as
// [iz][pp - h_c] starting at 31*h_c.  One contiguous block per CTA -> one bulk copy.
__device__ __forceinline__ int lh_offset(int pp, int iz, int nb) {
  // member c = max{c : floor(481 c / nb) <= pp} = ceil(nb (pp + 1) / 481) - 1
  const int c = (nb * (pp + 1) + 480) / 481 - 1;
  const int h0 = (481 * c) / nb, h1 = (481 * (c + 1)) / nb;
  return K * h0 + iz * (h1 - h0) + (pp - h0);
}

// kf2: CTA = 8 consecutive (cell, ly) columns.  x: FFT32 over jx -> lx in K', times N^-3; writes f^ at +l and
// (for lz > 0) its conjugate at -l, lower-half pencils only.
__global__ void __launch_bounds__(256, 3) kf2(const double2* __restrict__ F2, double2* __restrict__ fhT, long long ncol, int nb) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* buf = reinterpret_cast<double2*>(smem_raw);  // [8][32 jx][16 lz]
  const int tid = threadIdx.x;
  const long long g0 = (long long)blockIdx.x * PL8;
#pragma unroll 4
  for (int i = tid; i < PL8 * N * H; i += 256) {
    const int p = i / (N * H), jx = (i / H) % N, lz = i % H;
    const long long g = g0 + p;
    if (g < ncol) {
      const long long cell = g / K;
      const int iy = (int)(g - cell * K);
      cp16(buf + i, F2 + ((cell * N + jx) * K + iy) * H + lz);
    }
  }
  cp_wait_all();
  __syncthreads();
  const int r = tid >> 7, p = (tid >> 4) & 7, lz = tid & 15;
  const long long g = g0 + p;
  if (g >= ncol) return;
  const long long cell = g / K;
  const int iy = (int)(g - cell * K);
  InCol in{buf + p * N * H + lz, H};
  double2 u[16];
  if (r == 0) dif_class<2, -1, 0>(in, u); else dif_class<2, -1, 1>(in, u);
  const double sc = 1.0 / (N * N * N);
  double2* out = fhT + cell * (long long)K * (K * K / 2 + 1);  // lower-half pencils only (14911 per cell)
#pragma unroll
  for (int q = 0; q < 16; q++) {
    const int k = 2 * q + r;
    if (k == 16) continue;
    const int ix = k <= 15 ? k + C : k - 32 + C;
    const double2 v = make_double2(u[qslot(q)].x * sc, u[qslot(q)].y * sc);
    const int pp = ix * K + iy, pm = (K * K - 1) - pp;  // pencil of +l and of -l
    if (pp <= K * K / 2) out[lh_offset(pp, lz + C, nb)] = v;
    if (lz > 0 && pm <= K * K / 2) out[lh_offset(pm, C - lz, nb)] = make_double2(v.x, -v.y);
  }
}

// ---- back ---------------------------------------------------------------------------------------------
// kb1: CTA = (cell, 4 px planes), 288 threads.  First axis (py, contiguous): two real rows packed as one
// complex row, FFT48, untangled on the fly (ky = 0..15);  second axis (pz): FFT48 -> kz in K'.
// Out H2[cell][px][kz][ky].
#ifndef KB1_MINB
#define KB1_MINB (8 / PB1)
#endif
__global__ void __launch_bounds__(KB1_T, KB1_MINB) kb1(const double* __restrict__ G, double2* __restrict__ H2) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // [4 planes][24 row pairs][ZS]: element py of the pair = (G(pz = 2pr, py), G(pz = 2pr+1, py)); then in
  // place the complex FFT48 of the pair
  double2* zc = reinterpret_cast<double2*>(smem_raw);
  const int tid = threadIdx.x;
  const long long cell = blockIdx.x / (P / PB1);
  const int px0 = (blockIdx.x % (P / PB1)) * PB1;
  {  // G holds each pair of z-rows interleaved: (G(2pr, py), G(2pr+1, py)) is one 16-byte element
    const double2* src = reinterpret_cast<const double2*>(G + (cell * P + px0) * P * P);
#pragma unroll 4
    for (int i = tid; i < PB1 * P * P / 2; i += KB1_T) {
      const int pr = i / P, col = i - pr * P;  // pr = s * 24 + row pair, col = py
      cp16(zc + pr * ZS + col, src + i);
    }
  }
  cp_wait_all();
  __syncthreads();
  {  // z: thread = (class r, plane, row pair)
    const int r = tid / (24 * PB1), s = (tid % (24 * PB1)) / 24, pr = tid % 24;
    double2* zrow = zc + (s * 24 + pr) * ZS;
    InCol in{zrow, 1};
    double2 u[16];
    if (r == 0) dif_combine<3, -1, 0>(in, u);
    else if (r == 1) dif_combine<3, -1, 1>(in, u);
    else dif_combine<3, -1, 2>(in, u);
    __syncthreads();  // every task has read its pair: the row may now receive its transform
    fft16<-1>(u);
#pragma unroll
    for (int q = 0; q < 16; q++) zrow[3 * q + r] = u[qslot(q)];
  }
  __syncthreads();
  if (tid < 48 * PB1) {  // y: thread = (class r, plane, kz)
    const int r = tid / (16 * PB1), s = (tid / 16) % PB1, kz = tid & 15;
    struct InUntangle {  // H1(py, kz): even py -> first row of the pair, odd py -> second row
      const double2* z; int kz;
      __device__ __forceinline__ bool nz(int) const { return true; }
      __device__ __forceinline__ double2 operator()(int i) const {
        const double2 a = z[(i >> 1) * ZS + kz], b = z[(i >> 1) * ZS + ((P - kz) % P)];
        return (i & 1) ? make_double2(0.5 * (a.y + b.y), -0.5 * (a.x - b.x)) : make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
      }
    } in{zc + s * 24 * ZS, kz};
    double2 u[16];
    if (r == 0) dif_class<3, -1, 0>(in, u);
    else if (r == 1) dif_class<3, -1, 1>(in, u);
    else dif_class<3, -1, 2>(in, u);
    double2* dst = H2 + ((cell * P + px0 + s) * K) * H + kz;
#pragma unroll
    for (int q = 0; q < 16; q++) {
      const int k = 3 * q + r;
      if (k >= 16 && k <= 32) continue;
      dst[(k <= 15 ? k + C : k - 48 + C) * H] = u[qslot(q)];
    }
  }
}

// kb2: CTA = 4 consecutive (cell, ky) columns, 192 threads.  x: FFT48 over px -> kx in K', times P^-3
// ([Q^_0 := 0]);  then inverse FFT32 over kx -> jx.  Out E1[cell][jx][ky][kz].
__global__ void __launch_bounds__(192) kb2(const double2* __restrict__ H2, double2* __restrict__ E1, long long ncol,
                                           int project_mass) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* buf = reinterpret_cast<double2*>(smem_raw);  // [4][48 px][16 kz]
  double2* qh = buf + PB2 * P * H;                      // [4][31 kx][16 kz]
  const int tid = threadIdx.x;
  const long long g0 = (long long)blockIdx.x * PB2;
#pragma unroll 4
  for (int i = tid; i < PB2 * P * H; i += 192) {
    const int p = i / (P * H), px = (i / H) % P, kz = i % H;
    const long long g = g0 + p;
    if (g < ncol) {
      const long long cell = g / K;
      const int iy = (int)(g - cell * K);
      cp16(buf + i, H2 + ((cell * P + px) * K + iy) * H + kz);
    }
  }
  cp_wait_all();
  __syncthreads();
  {
    const int r = tid >> 6, p = (tid >> 4) & 3, kz = tid & 15;
    const long long g = g0 + p;
    const int iy = (int)(g % K);
    InCol in{buf + p * P * H + kz, H};
    double2 u[16];
    if (r == 0) dif_class<3, -1, 0>(in, u);
    else if (r == 1) dif_class<3, -1, 1>(in, u);
    else dif_class<3, -1, 2>(in, u);
    const double sc = 1.0 / ((double)P * P * P);
#pragma unroll
    for (int q = 0; q < 16; q++) {
      const int k = 3 * q + r;
      if (k >= 16 && k <= 32) continue;
      const int ix = k <= 15 ? k + C : k - 48 + C;
      double2 v = make_double2(u[qslot(q)].x * sc, u[qslot(q)].y * sc);
      if (project_mass && ix == C && iy == C && kz == 0) v = make_double2(0.0, 0.0);  // A24
      qh[(p * K + ix) * H + kz] = v;
    }
  }
  __syncthreads();
  if (tid < 128) {  // inverse x: thread = (class r, column, kz)
    const int r = tid >> 6, p = (tid >> 4) & 3, kz = tid & 15;
    const long long g = g0 + p;
    if (g >= ncol) return;
    const long long cell = g / K;
    const int iy = (int)(g - cell * K);
    InModes32 in{qh + p * K * H + kz, H};
    double2 u[16];
    if (r == 0) dif_class<2, 1, 0>(in, u); else dif_class<2, 1, 1>(in, u);
    double2* dst = E1 + cell * (long long)N * K * H + iy * H + kz;
#pragma unroll
    for (int q = 0; q < 16; q++) dst[(2 * q + r) * K * H] = u[qslot(q)];
  }
}

// kb3: CTA = (cell, 8 jx planes).  z: inverse FFT32 over kz -> jz;  y: Hermitian -> real inverse FFT32 (packed
// FFT16); then Q or f* + s Q, transposed through shared memory into coalesced stores.
__global__ void __launch_bounds__(256, 3) kb3(const double2* __restrict__ E1, const double* fin, double* out,
                                           int euler, double s, const GatherSrc g, int gather, double* mpart,
                                           double L, double hv) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int sx[PL8], sy[N], sz[N];
  double2* buf = reinterpret_cast<double2*>(smem_raw);  // [8][32 rows][RS]
  const int tid = threadIdx.x;
  const long long cell = blockIdx.x / (N / PL8);
  const int jx0 = (blockIdx.x % (N / PL8)) * PL8;
  {
    const double2* src = E1 + (cell * N + jx0) * K * H;
#pragma unroll 4
    for (int i = tid; i < PL8 * K * H; i += 256) {
      const int pl = i / (K * H), rem = i % (K * H);
      cp16(buf + (pl * N + rem / H) * RS + rem % H, src + i);
    }
  }
  cp_wait_all();
  __syncthreads();
  {  // inverse y: thread = (class r, plane, kz)
    const int r = tid >> 7, pl = (tid >> 4) & 7, kz = tid & 15;
    InModes32 in{buf + pl * N * RS + kz, RS};
    double2 u[16];
    if (r == 0) dif_combine<2, 1, 0>(in, u); else dif_combine<2, 1, 1>(in, u);
    __syncthreads();  // inputs consumed: write E2(jy, kz) in place
    fft16<1>(u);
#pragma unroll
    for (int q = 0; q < 16; q++) buf[(pl * N + 2 * q + r) * RS + kz] = u[qslot(q)];
  }
  __syncthreads();
  double2 z[16];
  {  // y (Hermitian -> real): thread = (plane, jz): X[k] = E2(jz, k), k = 0..15 (X[16] = 0, X[0] taken real)
    const double2* row = buf + tid * RS;
    double2 x[16];
#pragma unroll
    for (int k = 0; k < 16; k++) x[k] = row[k];
    x[0].y = 0.0;
#pragma unroll
    for (int k = 0; k < 16; k++) {
      const double2 a = x[k];
      const double2 b = k == 0 ? make_double2(0.0, 0.0) : make_double2(x[16 - k].x, -x[16 - k].y);  // conj X[16-k]
      const double2 ev = fftd::cadd(a, b);
      const double2 od = k == 0 ? a : fftd::cmul_s<1>(fftd::c_tw32[k], fftd::csub(a, b));
      z[k] = make_double2(ev.x - od.y, ev.y + od.x);  // ev + i od
    }
    fft16<1>(z);  // z[qslot(n)] = (Q(jy = 2n, jz), Q(jy = 2n + 1, jz))
  }
  __syncthreads();  // every row has been read: the region becomes the output staging [plane][jy][OS]
  constexpr int OS = 33;  // padded jz stride (doubles): conflict-free column writes and row reads
  double* stg = reinterpret_cast<double*>(smem_raw);
  {
    const int pl = tid >> 5, jz = tid & 31;
#pragma unroll
    for (int n = 0; n < 16; n++) {
      stg[(pl * N + 2 * n) * OS + jz] = z[fftd::qslot(n)].x;
      stg[(pl * N + 2 * n + 1) * OS + jz] = z[fftd::qslot(n)].y;
    }
  }
  __syncthreads();
  const long long base = (cell * N + jx0) * N * N;
  constexpr int PER = PL8 * N * N / 256;  // 32 outputs per thread
  double fv[PER];
  if (euler && !gather) {  // all loads of f* in flight at once
#pragma unroll
    for (int k = 0; k < PER; k++) fv[k] = fin[base + tid + 256 * k];
  } else if (euler) {  // fused transport: f* gathered from the untransported input
    gather_tables(g, g.cell0 + cell, jx0, sx, sy, sz);
    __syncthreads();
    const long long nv = (long long)N * N * N;
#pragma unroll
    for (int k = 0; k < PER; k++) {
      const int i = tid + 256 * k, pl = i >> 10, jy = (i >> 5) & 31, jz = i & 31;
      const long long src = ((long long)sx[pl] * g.sh.ny + sy[jy]) * g.sh.nz + sz[jz];
      fv[k] = __ldg(g.base + src * nv + ((long long)(jx0 + pl) * N + jy) * N + jz);
    }
  }
  // moments of the written values (NEXT-1, Eq. DM_update): this CTA's partial sums of
  // phi(v) f over its 8 planes, phi = (1, v, |v|^2/2), in a fixed order (thread, warp butterfly, warps in order)
  double m[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const double vz = __dadd_rn(-L, __dmul_rn((double)(tid & 31), hv));  // v_k = -L + k h, as fks_moments
  const double wz = 0.5 * vz * vz;
#pragma unroll
  for (int k = 0; k < PER; k++) {
    const int i = tid + 256 * k, pl = i >> 10, jy = (i >> 5) & 31, jz = i & 31;
    double v = stg[(pl * N + jy) * OS + jz];
    if (euler) v = fma(s, v, fv[k]);
    out[base + i] = v;
    if (mpart) {
      const double vx = __dadd_rn(-L, __dmul_rn((double)(jx0 + pl), hv));
      const double vy = __dadd_rn(-L, __dmul_rn((double)jy, hv));
      m[0] += v;
      m[1] = fma(v, vx, m[1]);
      m[2] = fma(v, vy, m[2]);
      m[3] = fma(v, vz, m[3]);
      m[4] = fma(v, 0.5 * vx * vx + 0.5 * vy * vy + wz, m[4]);
    }
  }
  if (mpart) {
#pragma unroll
    for (int a = 0; a < 5; a++) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m[a] += __shfl_xor_sync(0xffffffffu, m[a], o);
    }
    __syncthreads();  // the staging region is free: reuse it for the per-warp partials
    double* red = reinterpret_cast<double*>(smem_raw);
    if ((tid & 31) == 0) {
#pragma unroll
      for (int a = 0; a < 5; a++) red[(tid >> 5) * 5 + a] = m[a];
    }
    __syncthreads();
    if (tid < 5) {
      double acc = 0.0;
#pragma unroll
      for (int w = 0; w < 8; w++) acc += red[w * 5 + tid];
      mpart[blockIdx.x * 5LL + tid] = acc;  // [cell][N / PL8 plane groups][5]
    }
  }
}

}  // namespace x32

// tables [t][ix][iy][iz] -> [t][lower-half block layout] (init only)
__global__ void tables_to_lh_kernel(const double2* __restrict__ in, double2* __restrict__ out, int T1, int nb) {
  using namespace x32;
  constexpr int NL = K * (K * K / 2 + 1);
  const long long total = (long long)T1 * NL;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const long long t = e / NL;
    const int r = (int)(e - t * NL);
    // invert lh_offset by scanning the nb blocks
    int c = 0;
    for (int k = 1; k < nb; k++) c += (r >= K * ((481 * k) / nb));
    const int h0 = (481 * c) / nb, nh = (481 * (c + 1)) / nb - h0;
    const int q = r - K * h0, iz = q / nh, pp = h0 + (q - iz * nh);
    out[e] = in[t * (long long)K * K * K + (long long)pp * K + iz];
  }
}

void xform32_tables_lh(const double2* ab, double2* abL, int T1, int nb) {
  tables_to_lh_kernel<<<1024, 256>>>(ab, abL, T1, nb);
}

size_t xform32_ws_bytes_per_cell() {
  using namespace x32;
  // F2 / E1: N*K*H complex; H2: P*K*H complex; f^T: K^3 complex; G: P^3 fp64
  return 16 * (size_t)(K * K * K + std::max(N * K * H, P * K * H)) + 8 * (size_t)P * P * P;
}

cudaError_t xform32_prepare() {
  using namespace x32;
  cudaError_t e = fftd::fill_twiddles();
  if (e == cudaSuccess) e = cudaFuncSetAttribute(kf1, cudaFuncAttributeMaxDynamicSharedMemorySize, PL8 * N * RS * 16);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(kf2, cudaFuncAttributeMaxDynamicSharedMemorySize, PL8 * N * H * 16);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(kb1, cudaFuncAttributeMaxDynamicSharedMemorySize, PB1 * 24 * ZS * 16);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(kb2, cudaFuncAttributeMaxDynamicSharedMemorySize, PB2 * (P + K) * H * 16);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(kb3, cudaFuncAttributeMaxDynamicSharedMemorySize, PL8 * N * RS * 16);
  // maximum shared-memory carveout: with the default split kb1 ran one CTA per SM (ncu)
  const void* ks[] = {(const void*)kf1, (const void*)kf2, (const void*)kb1, (const void*)kb2, (const void*)kb3};
  for (const void* kk : ks)
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kk, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  return e;
}

void xform32_forward(Ctx& c, const double* fin, double2* fhT, double2* scratch, long long n, int nb, cudaStream_t st,
                     const GatherSrc* gs) {
  using namespace x32;
  const long long ncol = n * K;
  GatherSrc g{};
  if (gs) g = *gs;
  kf1<<<(unsigned)(n * (N / PL8)), 256, PL8 * N * RS * 16, st>>>(fin, scratch, g, gs ? 1 : 0);
  kf2<<<(unsigned)((ncol + PL8 - 1) / PL8), 256, PL8 * N * H * 16, st>>>(scratch, fhT, ncol, nb);
  c.launches += 2;
}

void xform32_back(Ctx& c, const double* G, double2* scratch_a, double2* scratch_b, const double* fin, double* out,
                  long long n, bool euler, double s, cudaStream_t st, const GatherSrc* gs, double* mpart) {
  using namespace x32;
  const long long ncol = n * K;
  GatherSrc g{};
  if (gs) g = *gs;
  kb1<<<(unsigned)(n * (P / PB1)), KB1_T, PB1 * 24 * ZS * 16, st>>>(G, scratch_a);
  kb2<<<(unsigned)((ncol + PB2 - 1) / PB2), 192, PB2 * (P + K) * H * 16, st>>>(scratch_a, scratch_b, ncol, c.p.project_mass);
  kb3<<<(unsigned)(n * (N / PL8)), 256, PL8 * N * RS * 16, st>>>(scratch_b, fin, out, euler ? 1 : 0, s, g, gs ? 1 : 0,
                                                                  mpart, c.p.L, 2.0 * c.p.L / N);
  c.launches += 3;
}

}  // namespace fks
