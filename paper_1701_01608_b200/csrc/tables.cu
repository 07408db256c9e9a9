// K1: separated Carleman weight tables on the device (readings A1-A7, A11, A12 of DESIGN.md §3).
//
// For every retained mode l in K'^3 (xi_l = (pi/L) l) and term t:
//   hard spheres (B~ = 1, separable), t = 1 + d:
//       a_t(l) = w_d phi_R(xi_l . e_d),             phi_R(s) = 2R^2 [sin(Rs)/(Rs) - 2 sin^2(Rs/2)/(Rs)^2]
//       b_t(l) = psi_R(|xi_l - (xi_l . e_d) e_d|),  psi_R(tau) = int_0^pi phi_R(tau cos th) dth
//   Maxwell molecules (radial split, A6), t = 1 + d*M_r + i:
//       a_t(l) = w_d 2 W_i rho_i cos(rho_i xi_l . e_d)
//       b_t(l) = 2 sum_j W_j rho_j (rho_i^2 + rho_j^2)^(-1/2) J0(rho_j tau),  J0(x) = (2/pi) int_0^{pi/2} cos(x cos th) dth
//   loss (t = 0): a_0 = 1, b_0 = -sum_{t>=1} a_t b_t.
// The theta integrals use a 64-node Gauss-Legendre rule on [0, pi/2] built from sin/cos only (relative error
// ~1e-15 for R*tau <= 78, i.e. every N <= 64), so no device Bessel routine is needed.
#include <algorithm>
#include <cmath>
#include <cstring>
#include "fks_internal.cuh"

namespace fks {

constexpr int kThetaNodes = 64;
constexpr int kMaxRadial = 64;

struct TableArgs {
  int K, c;            // modes per axis, index offset (l = i - c)
  double xi_scale;     // pi / L
  double R;            // cutoff radius R_c
  int kernel, n_dirs, M_r;
  const double* dirs;  // [n_dirs][3]
  const double* w;     // [n_dirs]
  const double* rho;   // [M_r]
  const double* Wr;    // [M_r]
  const double* cij;   // [M_r][M_r] = W_j rho_j (rho_i^2 + rho_j^2)^(-1/2)
  const double* th_cos;  // [64] cos(theta_q)
  const double* th_w;    // [64] GL weights on [0, pi/2]
  double2* ab;         // [(T+1)][K^3]
};

__device__ __forceinline__ double phi_R(double s, double R) {
  double x = R * s;
  if (x == 0.0) return R * R;
  double sh = sin(0.5 * x);
  return 2.0 * R * R * (sin(x) / x - 2.0 * sh * sh / (x * x));
}

__device__ double psi_R_quad(double tau, double R, const double* th_cos, const double* th_w) {
  double acc = 0.0;
  for (int q = 0; q < kThetaNodes; q++) acc += th_w[q] * phi_R(tau * th_cos[q], R);
  return 2.0 * acc;
}

__global__ void tables_kernel(TableArgs A) {
  __shared__ double s_cos[kThetaNodes], s_w[kThetaNodes];
  for (int q = threadIdx.x; q < kThetaNodes; q += blockDim.x) { s_cos[q] = A.th_cos[q]; s_w[q] = A.th_w[q]; }
  __syncthreads();
  const long long nl = (long long)A.K * A.K * A.K;
  long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (l >= nl) return;
  int ix = (int)(l / (A.K * A.K)), iy = (int)((l / A.K) % A.K), iz = (int)(l % A.K);
  double x0 = A.xi_scale * (ix - A.c), x1 = A.xi_scale * (iy - A.c), x2 = A.xi_scale * (iz - A.c);
  double xi2 = x0 * x0 + x1 * x1 + x2 * x2;
  double loss = 0.0;
  if (A.kernel == FKS_KERNEL_HARD_SPHERES) {
    for (int d = 0; d < A.n_dirs; d++) {
      double s = x0 * A.dirs[3 * d] + x1 * A.dirs[3 * d + 1] + x2 * A.dirs[3 * d + 2];
      double tau = sqrt(fmax(xi2 - s * s, 0.0));
      double a = A.w[d] * phi_R(s, A.R);
      double b = psi_R_quad(tau, A.R, s_cos, s_w);
      A.ab[(long long)(1 + d) * nl + l] = make_double2(a, b);
      loss = fma(-a, b, loss);
    }
  } else {
    double J0[kMaxRadial];
    for (int d = 0; d < A.n_dirs; d++) {
      double s = x0 * A.dirs[3 * d] + x1 * A.dirs[3 * d + 1] + x2 * A.dirs[3 * d + 2];
      double tau = sqrt(fmax(xi2 - s * s, 0.0));
      for (int j = 0; j < A.M_r; j++) {
        double x = A.rho[j] * tau, acc = 0.0;
        for (int q = 0; q < kThetaNodes; q++) acc += s_w[q] * cos(x * s_cos[q]);
        J0[j] = acc * (2.0 / 3.14159265358979323846);
      }
      for (int i = 0; i < A.M_r; i++) {
        double a = A.w[d] * 2.0 * A.Wr[i] * A.rho[i] * cos(A.rho[i] * s);
        double b = 0.0;
        for (int j = 0; j < A.M_r; j++) b += A.cij[i * A.M_r + j] * J0[j];
        b *= 2.0;
        A.ab[(long long)(1 + d * A.M_r + i) * nl + l] = make_double2(a, b);
        loss = fma(-a, b, loss);
      }
    }
  }
  A.ab[l] = make_double2(1.0, loss);
}

// Per-term max|a_t|, max|b_t| (positive doubles order like their bit patterns).
__global__ void table_absmax_kernel(const double2* ab, long long nl, unsigned long long* mx) {
  const int t = blockIdx.y;
  unsigned long long ma = 0, mb = 0;
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < nl; l += (long long)gridDim.x * blockDim.x) {
    double2 v = ab[(long long)t * nl + l];
    ma = max(ma, (unsigned long long)__double_as_longlong(fabs(v.x)));
    mb = max(mb, (unsigned long long)__double_as_longlong(fabs(v.y)));
  }
  atomicMax(&mx[2 * t], ma);
  atomicMax(&mx[2 * t + 1], mb);
}

// Exact power-of-two balancing a_t <- kappa_t a_t, b_t <- b_t / kappa_t: the product a_t(l) b_t(m), hence Q, is
// unchanged bit for bit, but the packed transform z_t = IDFT((a_t + i b_t) f^) = A_t + i B_t then carries
// comparable magnitudes in both parts, so the rounding of one does not swamp the other (b_0 ~ 2 pi^2 R^4 vs a_0 = 1).
__global__ void table_scale_kernel(double2* ab, long long nl, const double* kappa) {
  const int t = blockIdx.y;
  const double k = kappa[t], ik = 1.0 / k;
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < nl; l += (long long)gridDim.x * blockDim.x) {
    double2 v = ab[(long long)t * nl + l];
    ab[(long long)t * nl + l] = make_double2(v.x * k, v.y * ik);
  }
}

__global__ void twiddle_kernel(double2* tw, int M) {
  int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  double s, c;
  sincospi(2.0 * m / M, &s, &c);  // e^{+2 pi i m / M}
  tw[m] = make_double2(c, s);
}

fks_status build_tables(Ctx& c) {
  const double pi = 3.14159265358979323846;
  const fks_params& p = c.p;
  if (p.kernel != FKS_KERNEL_HARD_SPHERES && p.M_radial > kMaxRadial) {
    set_error("M_radial must be <= 64");
    return FKS_ERR_UNSUPPORTED;
  }
  // directions e_d and weights w_d, d = p*n_phi + q (A11, A12)
  int nt = c.n_theta, nf = c.n_phi, nd = nt * nf;
  std::vector<double> mu(nt), st(nt), wt(nt);
  if (p.quad_rule == FKS_QUAD_GL_UNIFORM) {
    std::vector<double> x, w;
    gauss_legendre(nt, -1.0, 1.0, x, w);
    for (int i = 0; i < nt; i++) { mu[i] = x[i]; st[i] = std::sqrt(1.0 - x[i] * x[i]); wt[i] = w[i] * pi / nf; }
  } else {
    for (int i = 0; i < nt; i++) {
      double th = i * pi / nt;
      mu[i] = std::cos(th); st[i] = std::sin(th); wt[i] = pi * pi / (nt * nf) * st[i];
    }
  }
  c.dirs.assign(3 * (size_t)nd, 0.0);
  c.w.assign(nd, 0.0);
  for (int i = 0; i < nt; i++)
    for (int q = 0; q < nf; q++) {
      int d = i * nf + q;
      double ph = q * pi / nf;
      c.dirs[3 * d] = st[i] * std::cos(ph);
      c.dirs[3 * d + 1] = st[i] * std::sin(ph);
      c.dirs[3 * d + 2] = mu[i];
      c.w[d] = wt[i];
    }
  // radial rule (Maxwell molecules) and theta rule on [0, pi/2]
  int Mr = p.kernel != FKS_KERNEL_HARD_SPHERES ? p.M_radial : 1;
  std::vector<double> rho, Wr, cij(Mr * (size_t)Mr, 0.0);
  gauss_legendre(Mr, 0.0, c.Rc, rho, Wr);
  // b_t = 2 sum_j cij J0(rho_j tau) = 2 pi sum_j W_j rho_j B~(rho_i, rho_j) J0:  cij = pi W_j rho_j B~(rho_i, rho_j)
  //   Maxwell molecules B~ = (1/pi)(rho_i^2 + rho_j^2)^(-1/2);  VHS B~ = 4 C_a (rho_i^2 + rho_j^2)^((a-1)/2) (A30)
  const double vhs_C = p.vhs_C > 0.0 ? p.vhs_C : 1.0 / (4.0 * pi);
  for (int i = 0; i < Mr; i++)
    for (int j = 0; j < Mr; j++) {
      const double r2 = rho[i] * rho[i] + rho[j] * rho[j];
      cij[i * Mr + j] = p.kernel == FKS_KERNEL_VHS ? pi * Wr[j] * rho[j] * 4.0 * vhs_C * std::pow(r2, (p.vhs_alpha - 1.0) / 2.0)
                                                   : Wr[j] * rho[j] / std::sqrt(r2);
    }
  std::vector<double> th, thw, thc(kThetaNodes);
  gauss_legendre(kThetaNodes, 0.0, 0.5 * pi, th, thw);
  for (int q = 0; q < kThetaNodes; q++) thc[q] = std::cos(th[q]);

  const size_t nl = (size_t)c.K * c.K * c.K;
  double* dbuf = nullptr;
  size_t nbuf = 3 * nd + nd + 2 * Mr + Mr * Mr + 2 * kThetaNodes;
  cudaError_t e = cudaMalloc(&c.d_ab, (size_t)(c.T + 1) * nl * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc(&dbuf, nbuf * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&c.d_twN, c.N * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc(&c.d_twP, c.P * sizeof(double2));
  if (e != cudaSuccess) { cudaGetLastError(); if (dbuf) cudaFree(dbuf); return cuda_status(e, "table allocation"); }
  std::vector<double> h(nbuf);
  size_t o = 0;
  auto put = [&](const std::vector<double>& v) { size_t at = o; std::copy(v.begin(), v.end(), h.begin() + o); o += v.size(); return at; };
  size_t o_dirs = put(c.dirs), o_w = put(c.w), o_rho = put(rho), o_Wr = put(Wr), o_cij = put(cij),
         o_thc = put(thc), o_thw = put(thw);
  e = cudaMemcpy(dbuf, h.data(), nbuf * sizeof(double), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { cudaFree(dbuf); return cuda_status(e, "table upload"); }
  TableArgs A;
  A.K = c.K; A.c = c.N / 2 - 1; A.xi_scale = pi / p.L; A.R = c.Rc; A.kernel = p.kernel; A.n_dirs = nd; A.M_r = Mr;
  A.dirs = dbuf + o_dirs; A.w = dbuf + o_w; A.rho = dbuf + o_rho; A.Wr = dbuf + o_Wr; A.cij = dbuf + o_cij;
  A.th_cos = dbuf + o_thc; A.th_w = dbuf + o_thw; A.ab = c.d_ab;
  int thr = 128;
  tables_kernel<<<(unsigned)((nl + thr - 1) / thr), thr>>>(A);
  // power-of-two balancing of each term (see table_scale_kernel)
  {
    unsigned long long* d_mx = nullptr;
    double* d_kappa = nullptr;
    int nt1 = c.T + 1;
    e = cudaMalloc(&d_mx, 2 * nt1 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMalloc(&d_kappa, nt1 * sizeof(double));
    if (e != cudaSuccess) { cudaGetLastError(); cudaFree(dbuf); return cuda_status(e, "table scale allocation"); }
    cudaMemset(d_mx, 0, 2 * nt1 * sizeof(unsigned long long));
    dim3 g((unsigned)std::min<size_t>((nl + 255) / 256, 64), nt1);
    table_absmax_kernel<<<g, 256>>>(c.d_ab, (long long)nl, d_mx);
    std::vector<unsigned long long> mx(2 * nt1);
    e = cudaMemcpy(mx.data(), d_mx, mx.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    c.kappa.assign(nt1, 1.0);
    for (int t = 0; t < nt1 && e == cudaSuccess; t++) {
      double ma, mb;
      std::memcpy(&ma, &mx[2 * t], 8);
      std::memcpy(&mb, &mx[2 * t + 1], 8);
      if (ma > 0 && mb > 0) c.kappa[t] = std::ldexp(1.0, (int)std::lround(0.5 * std::log2(mb / ma)));
    }
    if (e == cudaSuccess) e = cudaMemcpy(d_kappa, c.kappa.data(), nt1 * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) table_scale_kernel<<<g, 256>>>(c.d_ab, (long long)nl, d_kappa);
    c.launches += 2;
    cudaError_t e2 = cudaDeviceSynchronize();
    cudaFree(d_mx);
    cudaFree(d_kappa);
    if (e == cudaSuccess) e = e2;
    if (e != cudaSuccess) { cudaFree(dbuf); return cuda_status(e, "table balancing"); }
  }
  twiddle_kernel<<<(c.N + 63) / 64, 64>>>(c.d_twN, c.N);
  twiddle_kernel<<<(c.P + 63) / 64, 64>>>(c.d_twP, c.P);
  c.launches += 3;
  e = cudaDeviceSynchronize();
  cudaFree(dbuf);
  return cuda_status(e, "table kernel");
}

}  // namespace fks
