// Generic path (any even N in [4, 64], any P >= 3N/2 - 2): the collision operator as a sequence of per-axis
// DFT passes through a device workspace, one thread per output element.  It is the correctness-first
// realisation of DESIGN.md §2 (the same arithmetic as the fused N = 32 kernel, without the FFT
// factorisation) and the path used for the c0 (N = 16) and c1 (N = 24) configurations.
//
//   forward   f (N^3 real)            -> f^ on K'^3            3 passes, scale N^-3
//   per term  Z_t = (a_t + i b_t) f^  -> z_t on the P^3 grid  3 pruned passes (K' -> P)
//             G(p) (+)= Re z_t(p) * Im z_t(p)                   [Re z_t = A_t, Im z_t = B_t]
//   back      G (P^3 real)            -> Q^ on K'^3           3 passes, scale P^-3 (Galerkin projection, A10)
//             Q^                      -> Q (N^3 real)         3 passes; optional Euler f* + s Q
#include <algorithm>
#include "fks_internal.cuh"

namespace fks {

enum InKind { IN_REAL = 0, IN_CPLX = 1, IN_CPLX_TAB = 2 };
enum OutKind { OUT_CPLX = 0, OUT_ACC_G = 1, OUT_REAL = 2 };

struct AxisArgs {
  const void* in;
  void* out;
  long long B;        // batches (all cells)
  int n_in, n_out;    // axis lengths in / out
  long long R;        // trailing stride
  int in_off, out_off;  // value = index - off
  int M, sign;        // exponent sign * 2 pi i (v_in v_out)/M
  double scale;
  const double2* tw;  // e^{+2 pi i m/M}
  const double2* ab;  // IN_CPLX_TAB: term table slice [K^3]
  long long cell_elems;  // elements of the input per cell (for the table index)
  int first;          // OUT_ACC_G: 1 = overwrite G
  const double* fstar;  // OUT_REAL with Euler
  double s;
  int euler;
};

template <int IK, int OK>
__global__ void __launch_bounds__(256) dft_axis_kernel(AxisArgs A) {
  const long long total = A.B * A.n_out * A.R;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long r = idx % A.R;
    const long long bo = idx / A.R;
    const int o = (int)(bo % A.n_out);
    const long long b = bo / A.n_out;
    const int vo = o - A.out_off;
    double sr = 0.0, si = 0.0;
    const long long base = b * A.n_in * A.R + r;
    // twiddle index m_i = (sign (i - in_off) vo) mod M, advanced incrementally (no division in the loop); the
    // table index of the input element stays within one cell along the axis
    int step = (int)(((long long)A.sign * vo) % A.M);
    if (step < 0) step += A.M;
    int m = (int)(((long long)A.sign * (-A.in_off) * vo) % A.M);
    if (m < 0) m += A.M;
    const long long tab0 = (IK == IN_CPLX_TAB) ? base % A.cell_elems : 0;
    // one accumulation chain in input order, with the same explicit FMAs as dft_tile_kernel: both variants give
    // the same bits, so results do not depend on which one a batch size (or a workspace chunk) selects
#pragma unroll 2
    for (int i = 0; i < A.n_in; i++) {
      const long long e = base + (long long)i * A.R;
      const double2 w = A.tw[m];
      m += step;
      if (m >= A.M) m -= A.M;
      double xr, xi;
      if (IK == IN_REAL) {
        xr = reinterpret_cast<const double*>(A.in)[e];
        xi = 0.0;
      } else {
        double2 x = reinterpret_cast<const double2*>(A.in)[e];
        xr = x.x; xi = x.y;
        if (IK == IN_CPLX_TAB) {
          const double2 t = A.ab[tab0 + (long long)i * A.R];  // (a, b): (a + i b)(xr + i xi)
          const double zr = fma(t.x, xr, -(t.y * xi)), zi = fma(t.x, xi, t.y * xr);
          xr = zr; xi = zi;
        }
      }
      sr = fma(xr, w.x, fma(-xi, w.y, sr));
      si = fma(xr, w.y, fma(xi, w.x, si));
    }
    sr *= A.scale;
    si *= A.scale;
    if (OK == OUT_CPLX) {
      reinterpret_cast<double2*>(A.out)[idx] = make_double2(sr, si);
    } else if (OK == OUT_ACC_G) {
      double* G = reinterpret_cast<double*>(A.out);
      G[idx] = A.first ? sr * si : fma(sr, si, G[idx]);
    } else {
      double* q = reinterpret_cast<double*>(A.out);
      q[idx] = A.euler ? fma(A.s, sr, A.fstar[idx]) : sr;
    }
  }
}

// Tiled variant: a CTA stages the inputs of 32 pencils (flattened pencil index b R + r) in shared memory once
// (the table product applied on the way in), then each warp computes two outputs at a time for its lane's
// pencil with the twiddles from a shared table.  Every input is read from global memory once instead of once per
// output (the per-output reloads bound the one-thread-per-output kernel on L1 bandwidth).  n_in <= 64, M <= 256.
constexpr int kTileIn = 64, kTileM = 256;
template <int IK, int OK>
__global__ void __launch_bounds__(256) dft_tile_kernel(AxisArgs A) {
  __shared__ double2 xs[kTileIn * 32];
  __shared__ double2 tws[kTileM];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int m = threadIdx.x; m < A.M; m += 256) tws[m] = A.tw[m];
  const long long npen = A.B * A.R;
  const long long p = (long long)blockIdx.x * 32 + lane;
  const bool okp = p < npen;
  const long long pc = okp ? p : npen - 1;
  const long long b = pc / A.R, r = pc - b * A.R;
  const long long base = b * A.n_in * A.R + r;
  const long long tab0 = (IK == IN_CPLX_TAB) ? base % A.cell_elems : 0;
  for (int i = wid; i < A.n_in; i += 8) {
    const long long e = base + (long long)i * A.R;
    double2 x;
    if (IK == IN_REAL) {
      x = make_double2(reinterpret_cast<const double*>(A.in)[e], 0.0);
    } else {
      x = reinterpret_cast<const double2*>(A.in)[e];
      if (IK == IN_CPLX_TAB) {
        const double2 t = A.ab[tab0 + (long long)i * A.R];  // (a, b): (a + i b)(xr + i xi)
        x = make_double2(fma(t.x, x.x, -(t.y * x.y)), fma(t.x, x.y, t.y * x.x));  // as dft_axis_kernel
      }
    }
    xs[i * 32 + lane] = x;
  }
  __syncthreads();
  const long long obase = b * A.n_out * A.R + r;
  auto m_start = [&](int o, int& m, int& step) {
    const int vo = o - A.out_off;
    step = (int)(((long long)A.sign * vo) % A.M);
    if (step < 0) step += A.M;
    m = (int)(((long long)A.sign * (-A.in_off) * vo) % A.M);
    if (m < 0) m += A.M;
  };
  auto emit = [&](int o, double sr, double si) {
    if (!okp || o >= A.n_out) return;
    const long long idx = obase + (long long)o * A.R;
    sr *= A.scale;
    si *= A.scale;
    if (OK == OUT_CPLX) {
      reinterpret_cast<double2*>(A.out)[idx] = make_double2(sr, si);
    } else if (OK == OUT_ACC_G) {
      double* G = reinterpret_cast<double*>(A.out);
      G[idx] = A.first ? sr * si : fma(sr, si, G[idx]);
    } else {
      double* q = reinterpret_cast<double*>(A.out);
      q[idx] = A.euler ? fma(A.s, sr, A.fstar[idx]) : sr;
    }
  };
  for (int o = wid; o < A.n_out; o += 16) {  // outputs o and o + 8 share every input load
    int m1, s1, m2, s2;
    m_start(o, m1, s1);
    m_start(o + 8, m2, s2);
    double r1 = 0.0, i1 = 0.0, r2 = 0.0, i2 = 0.0;
    for (int i = 0; i < A.n_in; i++) {
      const double2 x = xs[i * 32 + lane];
      const double2 w1 = tws[m1], w2 = tws[m2];
      r1 = fma(x.x, w1.x, fma(-x.y, w1.y, r1));
      i1 = fma(x.x, w1.y, fma(x.y, w1.x, i1));
      r2 = fma(x.x, w2.x, fma(-x.y, w2.y, r2));
      i2 = fma(x.x, w2.y, fma(x.y, w2.x, i2));
      m1 += s1; if (m1 >= A.M) m1 -= A.M;
      m2 += s2; if (m2 >= A.M) m2 -= A.M;
    }
    emit(o, r1, i1);
    emit(o + 8, r2, i2);
  }
}

__global__ void zero_mode_kernel(double2* h, long long n_cells, long long per_cell, long long at) {
  long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c < n_cells) h[c * per_cell + at] = make_double2(0.0, 0.0);
}

template <int IK, int OK>
static void launch_axis(Ctx& c, const AxisArgs& A, cudaStream_t st) {
  const long long tiles = (A.B * A.R + 31) / 32;
  if (A.n_in <= kTileIn && A.M <= kTileM && tiles >= 4LL * c.num_sms) {  // enough pencils to fill the GPU
    dft_tile_kernel<IK, OK><<<(unsigned)tiles, 256, 0, st>>>(A);
    c.launches++;
    return;
  }
  long long total = A.B * A.n_out * A.R;
  long long blocks = std::min<long long>((total + 255) / 256, (long long)c.num_sms * 16);
  dft_axis_kernel<IK, OK><<<(unsigned)std::max<long long>(blocks, 1), 256, 0, st>>>(A);
  c.launches++;
}

size_t generic_ws_bytes_per_cell(const Ctx& c) {
  size_t K = c.K, P = c.P;
  return 16 * (K * K * K + K * K * P + K * P * P) + 8 * P * P * P;
}

GenericWs generic_ws(const Ctx& c, long long n) {
  const long long K = c.K, P = c.P;
  GenericWs w;
  w.hat = reinterpret_cast<double2*>(c.d_ws);
  w.a = w.hat + n * K * K * K;
  w.b = w.a + n * K * K * P;
  w.G = reinterpret_cast<double*>(w.b + n * K * P * P);
  return w;
}

// forward transform f -> f^ into w.hat ([cell][ix][iy][iz], scaled N^-3)
void generic_forward(Ctx& c, const double* fin, long long n, cudaStream_t st) {
  const long long N = c.N, K = c.K;
  const int cm = c.N / 2 - 1;
  GenericWs w = generic_ws(c, n);
  AxisArgs A{};
  A.tw = c.d_twN; A.M = c.N; A.sign = -1; A.scale = 1.0;
  A.in = fin; A.out = w.b; A.B = n * N * N; A.n_in = N; A.n_out = K; A.R = 1; A.in_off = 0; A.out_off = cm;
  launch_axis<IN_REAL, OUT_CPLX>(c, A, st);
  A.in = w.b; A.out = w.a; A.B = n * N; A.R = K;
  launch_axis<IN_CPLX, OUT_CPLX>(c, A, st);
  A.in = w.a; A.out = w.hat; A.B = n; A.R = K * K; A.scale = 1.0 / (double)(N * N * N);
  launch_axis<IN_CPLX, OUT_CPLX>(c, A, st);
}

// back transform of w.G ([cell][px][py][pz]) to Q^ on K' (Galerkin projection), then Q (+ Euler) into out
void generic_back(Ctx& c, const double* fin, double* out, long long n, bool euler, double s, cudaStream_t st) {
  const long long N = c.N, K = c.K, P = c.P;
  const int cm = c.N / 2 - 1;
  const long long nl = K * K * K;
  GenericWs w = generic_ws(c, n);
  AxisArgs C{};
  C.tw = c.d_twP; C.M = c.P; C.sign = -1; C.scale = 1.0; C.in_off = 0; C.out_off = cm;
  C.in = w.G; C.out = w.b; C.B = n * P * P; C.n_in = P; C.n_out = K; C.R = 1;
  launch_axis<IN_REAL, OUT_CPLX>(c, C, st);
  C.in = w.b; C.out = w.a; C.B = n * P; C.R = K;
  launch_axis<IN_CPLX, OUT_CPLX>(c, C, st);
  C.in = w.a; C.out = w.hat; C.B = n; C.R = K * K; C.scale = 1.0 / ((double)P * P * P);
  launch_axis<IN_CPLX, OUT_CPLX>(c, C, st);
  if (c.p.project_mass) {  // A24: Q^_0 := 0
    zero_mode_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(w.hat, n, nl, ((long long)cm * K + cm) * K + cm);
    c.launches++;
  }
  AxisArgs D{};
  D.tw = c.d_twN; D.M = c.N; D.sign = +1; D.scale = 1.0; D.in_off = cm; D.out_off = 0;
  D.in = w.hat; D.out = w.a; D.B = n * K * K; D.n_in = K; D.n_out = N; D.R = 1;
  launch_axis<IN_CPLX, OUT_CPLX>(c, D, st);
  D.in = w.a; D.out = w.b; D.B = n * K; D.R = N;
  launch_axis<IN_CPLX, OUT_CPLX>(c, D, st);
  D.in = w.b; D.out = out; D.B = n; D.R = N * N; D.euler = euler ? 1 : 0; D.s = s; D.fstar = fin;
  launch_axis<IN_CPLX, OUT_REAL>(c, D, st);
}

fks_status generic_collision(Ctx& c, const double* fin, double* out, long long n, bool euler, double s,
                             cudaStream_t st) {
  const long long N = c.N, K = c.K, P = c.P;
  const int cm = c.N / 2 - 1;  // mode index offset: l = i - cm
  char* ws = reinterpret_cast<char*>(c.d_ws);
  double2* Rhat = reinterpret_cast<double2*>(ws);
  double2* Ra = Rhat + n * K * K * K;
  double2* Rb = Ra + n * K * K * P;
  double* G = reinterpret_cast<double*>(Rb + n * K * P * P);

  AxisArgs A{};
  c.prof.begin(1, st);
  // ---- forward: f -> f^ -----------------------------------------------------------
  A.tw = c.d_twN; A.M = c.N; A.sign = -1; A.scale = 1.0;
  A.in = fin; A.out = Rb; A.B = n * N * N; A.n_in = N; A.n_out = K; A.R = 1; A.in_off = 0; A.out_off = cm;
  launch_axis<IN_REAL, OUT_CPLX>(c, A, st);
  A.in = Rb; A.out = Ra; A.B = n * N; A.R = K;
  launch_axis<IN_CPLX, OUT_CPLX>(c, A, st);
  A.in = Ra; A.out = Rhat; A.B = n; A.R = K * K; A.scale = 1.0 / (double)(N * N * N);
  launch_axis<IN_CPLX, OUT_CPLX>(c, A, st);

  c.prof.end(1, st);
  // ---- per term: pruned inverse K' -> P, accumulate G += Re z * Im z ---------------
  c.prof.begin(2, st);
  const long long nl = K * K * K;
  for (int t = 0; t <= c.T; t++) {
    AxisArgs B{};
    B.tw = c.d_twP; B.M = c.P; B.sign = +1; B.scale = 1.0; B.in_off = cm; B.out_off = 0;
    B.in = Rhat; B.out = Ra; B.B = n * K * K; B.n_in = K; B.n_out = P; B.R = 1;
    B.ab = c.d_ab + (long long)t * nl; B.cell_elems = nl;
    launch_axis<IN_CPLX_TAB, OUT_CPLX>(c, B, st);
    B.in = Ra; B.out = Rb; B.B = n * K; B.R = P;
    launch_axis<IN_CPLX, OUT_CPLX>(c, B, st);
    B.in = Rb; B.out = G; B.B = n; B.R = P * P; B.first = (t == 0);
    launch_axis<IN_CPLX, OUT_ACC_G>(c, B, st);
  }

  c.prof.end(2, st);
  // ---- back: G -> Q^ on K' (Galerkin projection), Q^ -> Q ------------------
  c.prof.begin(3, st);
  AxisArgs C{};
  C.tw = c.d_twP; C.M = c.P; C.sign = -1; C.scale = 1.0; C.in_off = 0; C.out_off = cm;
  C.in = G; C.out = Rb; C.B = n * P * P; C.n_in = P; C.n_out = K; C.R = 1;
  launch_axis<IN_REAL, OUT_CPLX>(c, C, st);
  C.in = Rb; C.out = Ra; C.B = n * P; C.R = K;
  launch_axis<IN_CPLX, OUT_CPLX>(c, C, st);
  C.in = Ra; C.out = Rhat; C.B = n; C.R = K * K; C.scale = 1.0 / ((double)P * P * P);
  launch_axis<IN_CPLX, OUT_CPLX>(c, C, st);
  if (c.p.project_mass) {  // A24: Q^_0 := 0
    zero_mode_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(Rhat, n, nl, ((long long)cm * K + cm) * K + cm);
    c.launches++;
  }
  AxisArgs D{};
  D.tw = c.d_twN; D.M = c.N; D.sign = +1; D.scale = 1.0; D.in_off = cm; D.out_off = 0;
  D.in = Rhat; D.out = Ra; D.B = n * K * K; D.n_in = K; D.n_out = N; D.R = 1;
  launch_axis<IN_CPLX, OUT_CPLX>(c, D, st);
  D.in = Ra; D.out = Rb; D.B = n * K; D.R = N;
  launch_axis<IN_CPLX, OUT_CPLX>(c, D, st);
  D.in = Rb; D.out = out; D.B = n; D.R = N * N; D.euler = euler ? 1 : 0; D.s = s; D.fstar = fin;
  launch_axis<IN_CPLX, OUT_REAL>(c, D, st);
  c.prof.end(3, st);
  return cuda_status(cudaPeekAtLastError(), "generic collision");
}

}  // namespace fks
