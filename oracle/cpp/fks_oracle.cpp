// CPU ORACLE in plain C++17 for the FKS fast-spectral Boltzmann hot path (arXiv 1701.01608) —
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
// leg may load this library (through oracle/cpp_oracle.py).  It shares no code, header, table or constant with
// the CUDA product (paper_1701_01608_b200/) and never links it; it is also written independently of the numpy
// oracle (oracle/fks_oracle.py), against which the tests cross-check it.
//
// Plain, slow, obviously correct, fp64, in the paper's order and notation.  Citations: "P:n" = line n of
// PAPER.md (Appendix A "Boltzmann collision operator" P:1469-1632; FKS scheme P:263-390); "A<n>" = the readings
// of garbled / silent passages in DESIGN.md §3.
//
//   f^_l = N^-3 sum_j f_j e^{-2 pi i l.j/N},  l in K'^3,  K' = {-(N/2-1)..N/2-1}                 (A9, A14)
//   Q^_k = sum_{l,m in K', l+m=k} beta(l,m) f^_l f^_m,  beta(l,m) = sum_{t=0..T} a_t(l) b_t(m)    (Eq. CF1)
//   Q_j  = sum_{k in K'} Q^_k e^{2 pi i k.j/N}
//
// Two evaluations: collision_fast (the paper's "sum of A convolutions" with zero-padded P-point naive DFTs,
// A_t and B_t each transformed separately, G = sum_t A_t B_t) and collision_direct (the double sum).
// Threads: a std::thread pool over cells (cells are independent).
//
// Layouts (match oracle/fks_oracle.py): f, Q [n_cells][N][N][N] C order (kz fastest); tables a, b
// [T+1][K][K][K] with index i <-> mode l = i - (N/2 - 1); term order HS t = 1 + d, MM/VHS t = 1 + d*M_r + i.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

using cplx = std::complex<double>;
const double PI = 3.14159265358979323846264338327950288;

// ---------------------------------------------------------------------------------------------------------
// Quadratures (A2, A6, A11, A12)
// ---------------------------------------------------------------------------------------------------------

// n-point Gauss-Legendre rule on [a, b]: nodes are the roots of P_n (Newton on the three-term recurrence),
// weights 2 / ((1 - x^2) P_n'(x)^2) scaled to [a, b].
void gauss_legendre(int n, double a, double b, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int i = 0; i < n; i++) {
    double z = std::cos(PI * (i + 0.75) / (n + 0.5));  // initial guess of the i-th largest root
    double dp = 1.0;
    for (int it = 0; it < 200; it++) {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= n; k++) {
        const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      if (n == 1) { p1 = z; p0 = 1.0; }
      dp = n * (z * p1 - p0) / (z * z - 1.0);
      const double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    double p0 = 1.0, p1 = z;
    for (int k = 2; k <= n; k++) {
      const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
    if (n == 1) { p1 = z; p0 = 1.0; }
    dp = n * (z * p1 - p0) / (z * z - 1.0);
    // roots come out in decreasing order; store ascending
    x[n - 1 - i] = 0.5 * (b - a) * z + 0.5 * (b + a);
    w[n - 1 - i] = 0.5 * (b - a) * 2.0 / ((1.0 - z * z) * dp * dp);
  }
}

void split_angles(int M, int& nt, int& nf) {  // A12: n_theta = 2^ceil(log2(M)/2), n_phi = M / n_theta
  nt = 1;
  while (nt * nt < M) nt *= 2;
  if (M % nt) nt = M;
  nf = M / nt;
}

// Directions e_d on the half sphere and weights w_d, d = p*n_phi + q (A11; paper rule P:1614, P:1628-1631 with
// the spherical sin(theta) outside psi, A2).
void directions(int nt, int nf, int rule, std::vector<double>& e, std::vector<double>& w) {
  std::vector<double> mu(nt), st(nt), wt(nt);
  if (rule == 0) {
    std::vector<double> W;
    gauss_legendre(nt, -1.0, 1.0, mu, W);
    for (int p = 0; p < nt; p++) { st[p] = std::sqrt(1.0 - mu[p] * mu[p]); wt[p] = W[p] * PI / nf; }
  } else {
    for (int p = 0; p < nt; p++) {
      const double th = p * PI / nt;
      mu[p] = std::cos(th);
      st[p] = std::sin(th);
      wt[p] = PI * PI / (nt * nf) * st[p];
    }
  }
  e.assign(3 * nt * nf, 0.0);
  w.assign(nt * nf, 0.0);
  for (int p = 0; p < nt; p++)
    for (int q = 0; q < nf; q++) {
      const int d = p * nf + q;
      const double ph = q * PI / nf;
      e[3 * d] = st[p] * std::cos(ph);
      e[3 * d + 1] = st[p] * std::sin(ph);
      e[3 * d + 2] = mu[p];
      w[d] = wt[p];
    }
}

// ---------------------------------------------------------------------------------------------------------
// Separated Carleman weights (A1-A7, A30)
// ---------------------------------------------------------------------------------------------------------

// phi_R(s) = int_{-R}^{R} |rho| e^{i rho s} d rho = 2 R^2 [sin(Rs)/(Rs) - 2 sin^2(Rs/2)/(Rs)^2]   (A1)
double phi_R(double s, double R) {
  const double x = R * s;
  if (x == 0.0) return R * R;
  const double h = std::sin(0.5 * x);
  return 2.0 * R * R * (std::sin(x) / x - 2.0 * h * h / (x * x));
}
// psi_R(tau) = int_0^pi phi_R(tau cos theta) d theta = 2 pi R J_1(R tau) / tau                    (A2)
double psi_R(double tau, double R) {
  if (tau == 0.0) return PI * R * R;
  return 2.0 * PI * R * std::cyl_bessel_j(1.0, R * tau) / tau;
}

struct TableSpec {
  int N; double L; int M; int M_r; int kernel; int n_theta; int n_phi; int rule; double cutoff_ratio;
  double alpha; double C_alpha;
};

int n_terms(const TableSpec& s) {
  int nt = s.n_theta, nf = s.n_phi;
  if (nt <= 0 || nf <= 0) split_angles(s.M, nt, nf);
  return s.kernel == 0 ? nt * nf : nt * nf * s.M_r;
}

// a, b: [(T+1)][K^3].  Term t >= 1 step by step as DESIGN.md §2 / SURVEY §8(c); then the loss term t = 0:
// a_0 = 1, b_0 = -sum_{t>=1} a_t b_t.
int build_tables(const TableSpec& s, double* a, double* b) {
  const int N = s.N, K = N - 1, c = N / 2 - 1;
  if (N % 2 || N < 4) return 1;
  const double R = 2.0 / (3.0 + std::sqrt(2.0)) * s.L;                    // R = lambda L
  const double Rc = R * (s.cutoff_ratio > 0 ? s.cutoff_ratio : 1.0);      // A7
  int nt = s.n_theta, nf = s.n_phi;
  if (nt <= 0 || nf <= 0) split_angles(s.M, nt, nf);
  std::vector<double> e, w;
  directions(nt, nf, s.rule, e, w);
  const int nd = nt * nf;
  const size_t nl = (size_t)K * K * K;
  std::vector<double> rho, Wr;
  if (s.kernel != 0) gauss_legendre(s.M_r, 0.0, Rc, rho, Wr);
  const int T = n_terms(s);
  for (size_t l = 0; l < nl; l++) {
    const int ix = (int)(l / (K * K)), iy = (int)((l / K) % K), iz = (int)(l % K);
    const double xi[3] = {PI / s.L * (ix - c), PI / s.L * (iy - c), PI / s.L * (iz - c)};  // xi_l = (pi/L) l
    const double xi2 = xi[0] * xi[0] + xi[1] * xi[1] + xi[2] * xi[2];
    double loss = 0.0;
    for (int d = 0; d < nd; d++) {
      const double sd = xi[0] * e[3 * d] + xi[1] * e[3 * d + 1] + xi[2] * e[3 * d + 2];  // xi.e_d
      const double tau = std::sqrt(std::max(xi2 - sd * sd, 0.0));                        // |Pi_{e_d perp} xi|
      if (s.kernel == 0) {  // hard spheres, B~ = 1
        const int t = 1 + d;
        a[t * nl + l] = w[d] * phi_R(sd, Rc);
        b[t * nl + l] = psi_R(tau, Rc);
        loss += a[t * nl + l] * b[t * nl + l];
      } else {  // radial split (A6): MM B~ = (1/pi)(rho^2+rho'^2)^-1/2; VHS B~ = 4 C (rho^2+rho'^2)^((alpha-1)/2)
        for (int i = 0; i < s.M_r; i++) {
          const int t = 1 + d * s.M_r + i;
          double bs = 0.0;
          for (int j = 0; j < s.M_r; j++) {
            const double r2 = rho[i] * rho[i] + rho[j] * rho[j];
            const double Bt = s.kernel == 1 ? 1.0 / (PI * std::sqrt(r2))
                                            : 4.0 * s.C_alpha * std::pow(r2, 0.5 * (s.alpha - 1.0));
            bs += Wr[j] * rho[j] * Bt * std::cyl_bessel_j(0.0, rho[j] * tau);
          }
          a[t * nl + l] = w[d] * 2.0 * Wr[i] * rho[i] * std::cos(rho[i] * sd);
          b[t * nl + l] = 2.0 * PI * bs;
          loss += a[t * nl + l] * b[t * nl + l];
        }
      }
    }
    a[l] = 1.0;
    b[l] = -loss;
  }
  (void)T;
  return 0;
}

// ---------------------------------------------------------------------------------------------------------
// Naive per-axis DFTs (O(n) per output point per axis, no factorisation; A10, A14)
// ---------------------------------------------------------------------------------------------------------

// y = M x along one axis of an (n0, n1, n2) array: out[i0][i1][i2] with the transformed axis replaced.
// `E[o][i]` is the (out x in) matrix of exponentials.
void along(const std::vector<cplx>& x, int n0, int n1, int n2, int axis, const std::vector<cplx>& E, int nout,
           std::vector<cplx>& y) {
  const int nin = axis == 0 ? n0 : axis == 1 ? n1 : n2;
  const int m0 = axis == 0 ? nout : n0, m1 = axis == 1 ? nout : n1, m2 = axis == 2 ? nout : n2;
  y.assign((size_t)m0 * m1 * m2, cplx(0.0, 0.0));
  for (int i0 = 0; i0 < m0; i0++)
    for (int i1 = 0; i1 < m1; i1++)
      for (int i2 = 0; i2 < m2; i2++) {
        const int o = axis == 0 ? i0 : axis == 1 ? i1 : i2;
        cplx acc(0.0, 0.0);
        for (int j = 0; j < nin; j++) {
          const int j0 = axis == 0 ? j : i0, j1 = axis == 1 ? j : i1, j2 = axis == 2 ? j : i2;
          acc += E[(size_t)o * nin + j] * x[((size_t)j0 * n1 + j1) * n2 + j2];
        }
        y[((size_t)i0 * m1 + i1) * m2 + i2] = acc;
      }
}

// E[o][i] = exp(sign 2 pi i rows[o] cols[i] / M)
std::vector<cplx> expmat(const std::vector<int>& rows, const std::vector<int>& cols, int M, int sign) {
  std::vector<cplx> E(rows.size() * cols.size());
  for (size_t o = 0; o < rows.size(); o++)
    for (size_t i = 0; i < cols.size(); i++) {
      const long long r = ((long long)rows[o] * cols[i]) % M;
      const double ang = sign * 2.0 * PI * (double)r / M;
      E[o * cols.size() + i] = cplx(std::cos(ang), std::sin(ang));
    }
  return E;
}

std::vector<int> range(int n) { std::vector<int> v(n); for (int i = 0; i < n; i++) v[i] = i; return v; }
std::vector<int> kprime(int N) { std::vector<int> v(N - 1); for (int i = 0; i < N - 1; i++) v[i] = i - (N / 2 - 1); return v; }

struct Dft {  // the four transforms of one (N, P)
  int N, P, K;
  std::vector<cplx> fwdN, invN, invP, fwdP;
  Dft(int N_, int P_) : N(N_), P(P_), K(N_ - 1) {
    fwdN = expmat(kprime(N), range(N), N, -1);  // f^: j -> l in K'
    invN = expmat(range(N), kprime(N), N, +1);  // Q: k in K' -> j
    invP = expmat(range(P), kprime(N), P, +1);  // z(p) = sum_l Z(l) e^{2 pi i l p / P}
    fwdP = expmat(kprime(N), range(P), P, -1);  // G^: p -> k in K'
  }
  void apply3(std::vector<cplx> x, int nin, const std::vector<cplx>& E, int nout, std::vector<cplx>& y) const {
    std::vector<cplx> t1, t2;
    along(x, nin, nin, nin, 0, E, nout, t1);
    along(t1, nout, nin, nin, 1, E, nout, t2);
    along(t2, nout, nout, nin, 2, E, nout, y);
  }
};

// f^ on K'^3 (A14)
void forward_modes(const Dft& D, const double* f, std::vector<cplx>& fh) {
  const int N = D.N;
  std::vector<cplx> x((size_t)N * N * N);
  for (size_t i = 0; i < x.size(); i++) x[i] = cplx(f[i], 0.0);
  D.apply3(x, N, D.fwdN, D.K, fh);
  const double s = 1.0 / ((double)N * N * N);
  for (auto& v : fh) v *= s;
}

// One cell, the paper's algorithm:
//  1. f^ = forward_modes(f)
//  2. for t = 0..T: A_t(p) = sum_l a_t(l) f^_l e^{2 pi i l.p/P},  B_t(p) = sum_m b_t(m) f^_m e^{2 pi i m.p/P},
//     G(p) += A_t(p) B_t(p)                        ("a discrete sum of A convolutions")
//  3. Q^_k = P^-3 sum_p G(p) e^{-2 pi i k.p/P}, k in K'   (exact Galerkin for P >= 3N/2 - 2, A10)
//  4. optional Q^_0 := 0 (A24)
//  5. Q_j = sum_k Q^_k e^{2 pi i k.j/N}; Re Q returned, max |Im Q| reported (A15).
void collision_fast_cell(const Dft& D, int T1, const double* a, const double* b, int project_mass, const double* f,
                         double* Q, double* max_imag) {
  const int N = D.N, K = D.K, P = D.P;
  const size_t nl = (size_t)K * K * K, np3 = (size_t)P * P * P;
  std::vector<cplx> fh;
  forward_modes(D, f, fh);
  std::vector<cplx> G(np3, cplx(0.0, 0.0)), Za(nl), Zb(nl), A, B;
  for (int t = 0; t < T1; t++) {
    for (size_t l = 0; l < nl; l++) { Za[l] = a[t * nl + l] * fh[l]; Zb[l] = b[t * nl + l] * fh[l]; }
    D.apply3(Za, K, D.invP, P, A);
    D.apply3(Zb, K, D.invP, P, B);
    for (size_t p = 0; p < np3; p++) G[p] += A[p] * B[p];
  }
  std::vector<cplx> Gh, q;
  D.apply3(G, P, D.fwdP, K, Gh);
  const double s = 1.0 / ((double)P * P * P);
  for (auto& v : Gh) v *= s;
  const int c = N / 2 - 1;
  if (project_mass) Gh[((size_t)c * K + c) * K + c] = 0.0;
  D.apply3(Gh, K, D.invN, N, q);
  double mi = 0.0;
  for (size_t j = 0; j < q.size(); j++) { Q[j] = q[j].real(); mi = std::max(mi, std::fabs(q[j].imag())); }
  if (max_imag) *max_imag = mi;
}

// Direct O(N^6) double sum of Eq. CF1; beta(l,m) = sum_t a_t(l) b_t(m) formed per pair.
// aliased_P > 0 (N <= P < 3N/2 - 2): the aliased collocation operator, pairs with l + m = k (mod P) per axis
// (SURVEY NEXT-4 (ii)); 0 = the exact Galerkin sum.
void collision_direct_cell(const Dft& D, int T1, const double* a, const double* b, int project_mass, int aliased_P,
                           const double* f, double* Q) {
  const int N = D.N, K = D.K, c = N / 2 - 1;
  const size_t nl = (size_t)K * K * K;
  std::vector<cplx> fh;
  forward_modes(D, f, fh);
  std::vector<cplx> Qh(nl, cplx(0.0, 0.0));
  auto target = [&](int li, int mi) -> int {  // index of k = l + m in K' (or -1)
    const int l = li - c, m = mi - c;
    int k = l + m;
    if (aliased_P > 0) k = ((k + c) % aliased_P + aliased_P) % aliased_P - c;
    return (k >= -c && k <= c) ? k + c : -1;
  };
  for (size_t l = 0; l < nl; l++) {
    const int lx = (int)(l / (K * K)), ly = (int)((l / K) % K), lz = (int)(l % K);
    for (size_t m = 0; m < nl; m++) {
      const int mx = (int)(m / (K * K)), my = (int)((m / K) % K), mz = (int)(m % K);
      const int kx = target(lx, mx), ky = target(ly, my), kz = target(lz, mz);
      if (kx < 0 || ky < 0 || kz < 0) continue;
      double beta = 0.0;
      for (int t = 0; t < T1; t++) beta += a[t * nl + l] * b[t * nl + m];
      Qh[((size_t)kx * K + ky) * K + kz] += beta * fh[l] * fh[m];
    }
  }
  if (project_mass) Qh[((size_t)c * K + c) * K + c] = 0.0;
  std::vector<cplx> q;
  D.apply3(Qh, K, D.invN, N, q);
  for (size_t j = 0; j < q.size(); j++) Q[j] = q[j].real();
}

// cells [0, n) over a pool of `threads` std::threads (cells are independent)
template <class F>
void parallel_cells(long long n, int threads, F fn) {
  if (threads <= 1 || n <= 1) { for (long long i = 0; i < n; i++) fn(i); return; }
  std::atomic<long long> next(0);
  std::vector<std::thread> pool;
  const int nt = (int)std::min<long long>(threads, n);
  for (int k = 0; k < nt; k++)
    pool.emplace_back([&]() { for (long long i; (i = next.fetch_add(1)) < n;) fn(i); });
  for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

// Number of separated terms T (the loss term t = 0 is extra).
int fkso_n_terms(int N, double L, int M, int M_r, int kernel, int n_theta, int n_phi) {
  TableSpec s{N, L, M, M_r, kernel, n_theta, n_phi, 0, 1.0, 0.5, 0.0};
  return n_terms(s);
}

int fkso_gauss_legendre(int n, double a, double b, double* x, double* w) {
  std::vector<double> xv, wv;
  gauss_legendre(n, a, b, xv, wv);
  std::memcpy(x, xv.data(), n * sizeof(double));
  std::memcpy(w, wv.data(), n * sizeof(double));
  return 0;
}

int fkso_directions(int n_theta, int n_phi, int rule, double* e, double* w) {
  std::vector<double> ev, wv;
  directions(n_theta, n_phi, rule, ev, wv);
  std::memcpy(e, ev.data(), ev.size() * sizeof(double));
  std::memcpy(w, wv.data(), wv.size() * sizeof(double));
  return 0;
}

void fkso_phi_psi(const double* s, long long n, double R, double* phi, double* psi) {
  for (long long i = 0; i < n; i++) { phi[i] = phi_R(s[i], R); psi[i] = psi_R(s[i], R); }
}

int fkso_tables(int N, double L, int M, int M_r, int kernel, int n_theta, int n_phi, int rule, double cutoff_ratio,
                double alpha, double C_alpha, double* a, double* b) {
  TableSpec s{N, L, M, M_r, kernel, n_theta, n_phi, rule, cutoff_ratio, alpha, C_alpha};
  return build_tables(s, a, b);
}

void fkso_forward_modes(int N, const double* f, double* fh_re, double* fh_im) {
  Dft D(N, N);
  std::vector<cplx> fh;
  forward_modes(D, f, fh);
  for (size_t i = 0; i < fh.size(); i++) { fh_re[i] = fh[i].real(); fh_im[i] = fh[i].imag(); }
}

int fkso_collision_fast(int N, int P, int T1, const double* a, const double* b, int project_mass, const double* f,
                        double* Q, double* max_imag, long long n_cells, int threads) {
  if (N % 2 || N < 4 || P < N) return 1;
  const Dft D(N, P);
  const size_t nv = (size_t)N * N * N;
  std::vector<double> mi(std::max<long long>(n_cells, 1), 0.0);
  parallel_cells(n_cells, threads, [&](long long i) {
    collision_fast_cell(D, T1, a, b, project_mass, f + i * nv, Q + i * nv, &mi[i]);
  });
  if (max_imag) for (long long i = 0; i < n_cells; i++) max_imag[i] = mi[i];
  return 0;
}

int fkso_collision_direct(int N, int T1, const double* a, const double* b, int project_mass, int aliased_P,
                          const double* f, double* Q, long long n_cells, int threads) {
  if (N % 2 || N < 4 || N > 24) return 1;  // guarded: (N-1)^6 pairs
  const Dft D(N, N);
  const size_t nv = (size_t)N * N * N;
  parallel_cells(n_cells, threads, [&](long long i) {
    collision_direct_cell(D, T1, a, b, project_mass, aliased_P, f + i * nv, Q + i * nv);
  });
  return 0;
}

// Loss part of Q alone (used to normalise mass and parity metrics, A23/A24): Q_loss(v_j) = f_j nu_j with the
// collision frequency nu_j = sum_m B^_F(m,m) f^_m e^{2 pi i m.j/N} = sum_m (-b_0(m)) f^_m e^{...}.
void fkso_loss_part(int N, const double* b0, const double* f, double* out) {
  const Dft D(N, N);
  std::vector<cplx> fh, nu;
  forward_modes(D, f, fh);
  for (size_t l = 0; l < fh.size(); l++) fh[l] *= -b0[l];
  D.apply3(fh, D.K, D.invN, N, nu);
  for (size_t j = 0; j < nu.size(); j++) out[j] = f[j] * nu[j].real();
}

// Generic-cell bookkeeping (A16): offsets[3][N] in units of 1/(N c_den) cell, particle k
// moves (2k - N) c_num units per step; delta = floor((o + d + unit/2) / unit), o <- o + d - delta unit.
void fkso_generic_cell_advance(int N, long long c_num, long long c_den, long long* offsets, long long* delta) {
  const long long unit = (long long)N * c_den;
  for (int a = 0; a < 3; a++)
    for (int k = 0; k < N; k++) {
      const long long o = offsets[a * N + k] + (2LL * k - N) * c_num;
      const long long num = o + unit / 2;
      long long d = num / unit;
      if (num % unit != 0 && num < 0) d -= 1;  // floor division
      offsets[a * N + k] = o - d * unit;
      delta[a * N + k] = d;
    }
}

// Exact transport: out[j][k] = f[(j - delta(k)) mod (nx, ny, nz)][k], cell j = (jx ny + jy) nz + jz.
void fkso_transport(const double* f, double* out, int nx, int ny, int nz, int N, const long long* delta) {
  const size_t nv = (size_t)N * N * N;
  auto md = [](long long a, long long n) { return (int)(((a % n) + n) % n); };
  for (int jx = 0; jx < nx; jx++)
    for (int jy = 0; jy < ny; jy++)
      for (int jz = 0; jz < nz; jz++) {
        const size_t j = ((size_t)jx * ny + jy) * nz + jz;
        for (int kx = 0; kx < N; kx++)
          for (int ky = 0; ky < N; ky++)
            for (int kz = 0; kz < N; kz++) {
              const int sx = md(jx - delta[kx], nx), sy = md(jy - delta[N + ky], ny), sz = md(jz - delta[2 * N + kz], nz);
              const size_t src = ((size_t)sx * ny + sy) * nz + sz;
              const size_t k = ((size_t)kx * N + ky) * N + kz;
              out[j * nv + k] = f[src * nv + k];
            }
      }
}

// One FKS step (Eq. disc_relax; A17, A18): transport, collision, explicit Euler
// f_out = f* + s Q(f*).  offsets [3][N] are advanced in place; delta_out [3][N] receives the shifts.
int fkso_step(int N, int P, int T1, const double* a, const double* b, const double* f_in, double* f_out, int nx,
              int ny, int nz, long long c_num, long long c_den, long long* offsets, double s, int threads,
              long long* delta_out) {
  std::vector<long long> delta(3 * N);
  fkso_generic_cell_advance(N, c_num, c_den, offsets, delta.data());
  if (delta_out) std::memcpy(delta_out, delta.data(), delta.size() * sizeof(long long));
  const long long n = (long long)nx * ny * nz;
  const size_t nv = (size_t)N * N * N;
  std::vector<double> fs((size_t)n * nv), q((size_t)n * nv);
  fkso_transport(f_in, fs.data(), nx, ny, nz, N, delta.data());
  int rc = fkso_collision_fast(N, P, T1, a, b, 0, fs.data(), q.data(), nullptr, n, threads);
  if (rc) return rc;
  for (size_t i = 0; i < fs.size(); i++) f_out[i] = fs[i] + s * q[i];
  return 0;
}

}  // extern "C"
