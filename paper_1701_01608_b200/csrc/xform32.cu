// Forward (a2) and back (a6-a7) transforms of the N = 32, P = 48 fast path.
//
// Both use the Hermitian symmetry of real data: only the half-spectrum lz >= 0 (resp. kz >= 0) is computed and
// the other half follows by conjugation.  Each kernel owns either a plane (two axes local in shared memory)
// or a set of columns (the third axis), so one cell's transform is 2 (forward) or 3 (back) kernels with the
// compact intermediates in the workspace.  The short transforms are plain DFT sums from a twiddle table in
// shared memory (the work is < 10 % of the term loop).
//
//   forward  Kf1 plane jx : f(jx,jy,jz)  --z (real, lz=0..15)--> --y (ly in K')-->  F2[cell][jx][ly][lz]
//            Kf2 column ly: F2(:,ly,lz)  --x (lx in K'), N^-3-->  f^T[cell][lz][lx*31+ly] and its conjugate at -l
//   back     Kb1 plane px : G(px,py,pz)  --z (real, kz=0..15)--> --y (ky in K')--> H2[cell][px][ky][kz]
//            Kb2 column ky: H2(:,ky,kz)  --x (kx in K'), P^-3, [Q^_0 := 0]--> --x inverse (jx)--> E1[cell][jx][ky][kz]
//            Kb3 plane jx : E1(jx,:,:)   --y inverse (jy)--> --z Hermitian->real (jz)-->  Q (or f* + s Q)
#include <algorithm>
#include "fks_internal.cuh"

namespace fks {
namespace x32 {

constexpr int N = 32, K = 31, P = 48, H = 16;  // H: retained non-negative z modes 0..15
constexpr int C = N / 2 - 1;                   // mode index offset (l = i - C)

// e^{sign 2 pi i m / M}
__device__ __forceinline__ void fill_tw(double2* tw, int M, int sign) {
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    double s, c;
    sincospi(2.0 * m / M, &s, &c);
    tw[m] = make_double2(c, sign * s);
  }
}
__device__ __forceinline__ double2 cmac(double2 acc, double2 x, double2 w) {
  acc.x = fma(x.x, w.x, fma(-x.y, w.y, acc.x));
  acc.y = fma(x.x, w.y, fma(x.y, w.x, acc.y));
  return acc;
}
__device__ __forceinline__ int md(int a, int M) { a %= M; return a < 0 ? a + M : a; }

// ---- forward ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) kf1(const double* __restrict__ f, double2* __restrict__ F2) {
  __shared__ double sf[N * N];
  __shared__ double2 sF1[N * H];
  __shared__ double2 tw[N];
  const long long cell = blockIdx.y;
  const int jx = blockIdx.x;
  fill_tw(tw, N, -1);
  const double* src = f + (cell * N + jx) * N * N;
  for (int i = threadIdx.x; i < N * N; i += blockDim.x) sf[i] = src[i];
  __syncthreads();
  for (int o = threadIdx.x; o < N * H; o += blockDim.x) {  // F1(jy, lz), lz = 0..15
    const int jy = o / H, lz = o % H;
    double2 acc = make_double2(0.0, 0.0);
    int m = 0;
    for (int jz = 0; jz < N; jz++) {
      const double x = sf[jy * N + jz];
      acc.x = fma(x, tw[m].x, acc.x);
      acc.y = fma(x, tw[m].y, acc.y);
      m += lz; if (m >= N) m -= N;
    }
    sF1[o] = acc;
  }
  __syncthreads();
  double2* dst = F2 + (cell * N + jx) * K * H;
  for (int o = threadIdx.x; o < K * H; o += blockDim.x) {  // F2(ly, lz), ly in K'
    const int iy = o / H, lz = o % H, ly = iy - C;
    double2 acc = make_double2(0.0, 0.0);
    for (int jy = 0; jy < N; jy++) acc = cmac(acc, sF1[jy * H + lz], tw[md(ly * jy, N)]);
    dst[o] = acc;
  }
}

// Offset of pencil pp <= 480 (lower half of the (lx,ly) plane) at lz index iz in the per-CTA block layout used by
// the hot kernel: CTA c of a cell's team of nb CTAs owns pencils [h_c, h_{c+1}), h_c = floor(481 c / nb), stored as
// [iz][pp - h_c] starting at 31*h_c.  One contiguous block per CTA -> one bulk copy.
__device__ __forceinline__ int lh_offset(int pp, int iz, int nb) {
  int c = 0;
  for (int k = 1; k < nb; k++) c += (pp >= (481 * k) / nb);
  const int h0 = (481 * c) / nb, h1 = (481 * (c + 1)) / nb;
  return K * h0 + iz * (h1 - h0) + (pp - h0);
}

__global__ void __launch_bounds__(256) kf2(const double2* __restrict__ F2, double2* __restrict__ fhT, int nb) {
  __shared__ double2 s[N * H];  // F2(jx, ly fixed, lz)
  __shared__ double2 tw[N];
  const long long cell = blockIdx.y;
  const int iy = blockIdx.x, ly = iy - C;
  fill_tw(tw, N, -1);
  for (int i = threadIdx.x; i < N * H; i += blockDim.x) {
    const int jx = i / H, lz = i % H;
    s[i] = F2[((cell * N + jx) * K + iy) * H + lz];
  }
  __syncthreads();
  const double sc = 1.0 / (N * N * N);
  double2* out = fhT + cell * (long long)K * (K * K / 2 + 1);  // lower-half pencils only (14911 per cell)
  for (int o = threadIdx.x; o < K * H; o += blockDim.x) {
    const int ix = o / H, lz = o % H, lx = ix - C;
    double2 acc = make_double2(0.0, 0.0);
    for (int jx = 0; jx < N; jx++) acc = cmac(acc, s[jx * H + lz], tw[md(lx * jx, N)]);
    acc.x *= sc; acc.y *= sc;
    const int pp = ix * K + iy, pm = (K * K - 1) - pp;                        // pencil of +l and of -l
    if (pp <= K * K / 2) out[lh_offset(pp, lz + C, nb)] = acc;                                      // +l
    if (lz > 0 && pm <= K * K / 2) out[lh_offset(pm, C - lz, nb)] = make_double2(acc.x, -acc.y);    // -l
  }
}

// ---- back ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) kb1(const double* __restrict__ G, double2* __restrict__ H2) {
  __shared__ double sg[P * P];      // G(px fixed, py, pz)  18 KB
  __shared__ double2 sH1[P * H];    // H1(py, kz)  12 KB
  __shared__ double2 tw[P];
  const long long cell = blockIdx.y;
  const int px = blockIdx.x;
  fill_tw(tw, P, -1);
  const double* src = G + (cell * P + px) * P * P;
  for (int i = threadIdx.x; i < P * P; i += blockDim.x) sg[i] = src[i];
  __syncthreads();
  for (int o = threadIdx.x; o < P * H; o += blockDim.x) {
    const int py = o / H, kz = o % H;
    double2 acc = make_double2(0.0, 0.0);
    int m = 0;
    for (int pz = 0; pz < P; pz++) {
      const double x = sg[py * P + pz];
      acc.x = fma(x, tw[m].x, acc.x);
      acc.y = fma(x, tw[m].y, acc.y);
      m += kz; if (m >= P) m -= P;
    }
    sH1[o] = acc;
  }
  __syncthreads();
  double2* dst = H2 + (cell * P + px) * K * H;
  for (int o = threadIdx.x; o < K * H; o += blockDim.x) {
    const int iy = o / H, kz = o % H, ky = iy - C;
    double2 acc = make_double2(0.0, 0.0);
    for (int py = 0; py < P; py++) acc = cmac(acc, sH1[py * H + kz], tw[md(ky * py, P)]);
    dst[o] = acc;
  }
}

__global__ void __launch_bounds__(256) kb2(const double2* __restrict__ H2, double2* __restrict__ E1, int project_mass) {
  __shared__ double2 s[P * H];      // H2(px, ky fixed, kz)
  __shared__ double2 sQ[K * H];     // Q^(kx, ky fixed, kz)
  __shared__ double2 twP[P], twN[N];
  const long long cell = blockIdx.y;
  const int iy = blockIdx.x, ky = iy - C;
  fill_tw(twP, P, -1);
  fill_tw(twN, N, +1);
  for (int i = threadIdx.x; i < P * H; i += blockDim.x) {
    const int px = i / H, kz = i % H;
    s[i] = H2[((cell * P + px) * K + iy) * H + kz];
  }
  __syncthreads();
  const double sc = 1.0 / ((double)P * P * P);
  for (int o = threadIdx.x; o < K * H; o += blockDim.x) {
    const int ix = o / H, kz = o % H, kx = ix - C;
    double2 acc = make_double2(0.0, 0.0);
    for (int px = 0; px < P; px++) acc = cmac(acc, s[px * H + kz], twP[md(kx * px, P)]);
    acc.x *= sc; acc.y *= sc;
    if (project_mass && kx == 0 && ky == 0 && kz == 0) acc = make_double2(0.0, 0.0);  // A24
    sQ[o] = acc;
  }
  __syncthreads();
  double2* dst = E1 + cell * (long long)N * K * H;
  for (int o = threadIdx.x; o < N * H; o += blockDim.x) {
    const int jx = o / H, kz = o % H;
    double2 acc = make_double2(0.0, 0.0);
    for (int ix = 0; ix < K; ix++) acc = cmac(acc, sQ[ix * H + kz], twN[md((ix - C) * jx, N)]);
    dst[(jx * K + iy) * H + kz] = acc;
  }
}

__global__ void __launch_bounds__(256) kb3(const double2* __restrict__ E1, const double* fin, double* out,
                                           int euler, double s) {
  __shared__ double2 sE[K * H];     // E1(jx fixed, ky, kz)
  __shared__ double2 sE2[N * H];    // E2(jy, kz)
  __shared__ double2 twN[N];
  const long long cell = blockIdx.y;
  const int jx = blockIdx.x;
  fill_tw(twN, N, +1);
  const double2* src = E1 + (cell * N + jx) * K * H;
  for (int i = threadIdx.x; i < K * H; i += blockDim.x) sE[i] = src[i];
  __syncthreads();
  for (int o = threadIdx.x; o < N * H; o += blockDim.x) {
    const int jy = o / H, kz = o % H;
    double2 acc = make_double2(0.0, 0.0);
    for (int iy = 0; iy < K; iy++) acc = cmac(acc, sE[iy * H + kz], twN[md((iy - C) * jy, N)]);
    sE2[o] = acc;
  }
  __syncthreads();
  const long long base = (cell * N + jx) * N * N;
  for (int o = threadIdx.x; o < N * N; o += blockDim.x) {
    const int jy = o / N, jz = o % N;
    // Q = Re E2(0) + 2 Re sum_{kz=1..15} E2(kz) e^{2 pi i kz jz / N}
    double q = sE2[jy * H].x, acc = 0.0;
    int m = jz;
    for (int kz = 1; kz < H; kz++) {
      const double2 e = sE2[jy * H + kz], w = twN[m];
      acc = fma(e.x, w.x, fma(-e.y, w.y, acc));
      m += jz; if (m >= N) m -= N;
    }
    q = fma(2.0, acc, q);
    out[base + o] = euler ? fma(s, q, fin[base + o]) : q;
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

void xform32_forward(Ctx& c, const double* fin, double2* fhT, double2* scratch, long long n, int nb, cudaStream_t st) {
  using namespace x32;
  for (long long c0 = 0; c0 < n; c0 += 65535) {
    const unsigned m = (unsigned)std::min<long long>(65535, n - c0);
    kf1<<<dim3(N, m), 256, 0, st>>>(fin + c0 * N * N * N, scratch + c0 * N * K * H);
    kf2<<<dim3(K, m), 256, 0, st>>>(scratch + c0 * N * K * H, fhT + c0 * K * (K * K / 2 + 1), nb);
    c.launches += 2;
  }
}

void xform32_back(Ctx& c, const double* G, double2* scratch_a, double2* scratch_b, const double* fin, double* out,
                  long long n, bool euler, double s, cudaStream_t st) {
  using namespace x32;
  for (long long c0 = 0; c0 < n; c0 += 65535) {
    const unsigned m = (unsigned)std::min<long long>(65535, n - c0);
    kb1<<<dim3(P, m), 256, 0, st>>>(G + c0 * P * P * P, scratch_a + c0 * P * K * H);
    kb2<<<dim3(K, m), 256, 0, st>>>(scratch_a + c0 * P * K * H, scratch_b + c0 * N * K * H, c.p.project_mass);
    kb3<<<dim3(N, m), 256, 0, st>>>(scratch_b + c0 * N * K * H, fin + c0 * N * N * N, out + c0 * N * N * N,
                                     euler ? 1 : 0, s);
    c.launches += 3;
  }
}

}  // namespace fks
