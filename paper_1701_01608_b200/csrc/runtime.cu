// libfks host runtime: the C ABI of include/fks.h (validation, handle, Gauss-Legendre nodes, workspace and
// chunk planning, generic-cell transport bookkeeping).  Every compute step runs in the sm_100a kernels of
// tables.cu / generic.cu / fast32.cu / transport.cu; there is no CPU fallback.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include "fks_internal.cuh"

namespace fks {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

fks_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return FKS_OK;
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? FKS_ERR_NOMEM : FKS_ERR_CUDA;
}

// Gauss-Legendre nodes/weights on [a, b] by Newton iteration on P_n (three-term recurrence).
void gauss_legendre(int n, double a, double b, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < (n + 1) / 2; i++) {
    double z = std::cos(pi * (i + 0.75) / (n + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; it++) {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= n; k++) {
        double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      if (n == 1) { p1 = z; p0 = 1.0; }
      dp = n * (z * p1 - p0) / (z * z - 1.0);
      double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-17) break;
    }
    // recompute derivative at the converged node
    double p0 = 1.0, p1 = z;
    for (int k = 2; k <= n; k++) {
      double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
    if (n == 1) { p1 = z; p0 = 1.0; }
    dp = n * (z * p1 - p0) / (z * z - 1.0);
    double wi = 2.0 / ((1.0 - z * z) * dp * dp);
    x[i] = -z;
    x[n - 1 - i] = z;
    w[i] = wi;
    w[n - 1 - i] = wi;
  }
  if (n % 2 == 1) x[n / 2] = 0.0;
  for (int i = 0; i < n; i++) {
    x[i] = 0.5 * (b - a) * x[i] + 0.5 * (b + a);
    w[i] = 0.5 * (b - a) * w[i];
  }
}

void PhaseTimer::begin(int ph, cudaStream_t st) {
  if (!on) return;
  std::pair<cudaEvent_t, cudaEvent_t> ev;
  if (!pool.empty()) { ev = pool.back(); pool.pop_back(); }
  else { cudaEventCreate(&ev.first); cudaEventCreate(&ev.second); }
  cudaEventRecord(ev.first, st);
  used[ph].push_back(ev);
  open_phase = ph;
}

void PhaseTimer::end(int ph, cudaStream_t st) {
  if (!on || used[ph].empty()) return;
  cudaEventRecord(used[ph].back().second, st);
  open_phase = -1;
}

static fks_status check_device_ptr(const void* p, const char* name) {
  if (!p) { set_error(std::string(name) + " is NULL"); return FKS_ERR_INVALID; }
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) { cudaGetLastError(); set_error(std::string(name) + ": not a CUDA pointer"); return FKS_ERR_INVALID; }
  if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged) {
    set_error(std::string(name) + " must be a device pointer");
    return FKS_ERR_INVALID;
  }
  return FKS_OK;
}

static bool overlap(const void* a, size_t na, const void* b, size_t nb) {
  auto x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
  return x < y + nb && y < x + na;
}

static fks_status sticky_check() {
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) { cudaGetLastError(); return cuda_status(e, "asynchronous CUDA error"); }
  return FKS_OK;
}

static fks_status ensure_ws(Ctx& c, size_t bytes) {
  if (bytes <= c.ws_bytes) return FKS_OK;
  if (c.d_ws) { cudaFree(c.d_ws); c.d_ws = nullptr; c.ws_bytes = 0; }
  cudaError_t e = cudaMalloc(&c.d_ws, bytes);
  if (e != cudaSuccess) { cudaGetLastError(); return cuda_status(e, "workspace allocation"); }
  c.ws_bytes = bytes;
  return FKS_OK;
}

// Calls on one handle share its device workspace, W1 ring and team counters, so they are serialised in
// submission order across streams: a call's stream waits for the event recorded by the previous call, and the
// call records the event on its own stream when its work is enqueued (two streams must not race on
// one handle's workspace).
static fks_status order_begin(Ctx& c, cudaStream_t st) {
  if (!c.ev_done) {
    cudaError_t e = cudaEventCreateWithFlags(&c.ev_done, cudaEventDisableTiming);
    if (e != cudaSuccess) { cudaGetLastError(); return cuda_status(e, "ordering event"); }
  }
  if (!c.ev_pending) return FKS_OK;
  return cuda_status(cudaStreamWaitEvent(st, c.ev_done, 0), "stream ordering");
}
static fks_status order_end(Ctx& c, cudaStream_t st, fks_status rc) {
  if (!c.ev_done) return rc;
  fks_status r2 = cuda_status(cudaEventRecord(c.ev_done, st), "stream ordering");
  if (r2 == FKS_OK) c.ev_pending = true;
  return rc ? rc : r2;
}

static long long chunk_cells(Ctx& c, size_t per_cell, long long n_cells) {
  long long lim = c.p.max_cells_in_flight;
  if (lim <= 0) {
    // the memory query is done once per handle and per-cell size (cudaMemGetInfo costs host time on every call,
    // which small, launch-bound steps (c0) cannot afford); the workspace then stays allocated at that size
    if (c.auto_chunk <= 0 || c.auto_chunk_per_cell != per_cell) {
      size_t fr = 0, tot = 0;
      if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) { cudaGetLastError(); fr = 8ull << 30; }
      size_t budget = std::min<size_t>(fr / 3, 24ull << 30);
      c.auto_chunk = std::max<long long>(1, (long long)(budget / std::max<size_t>(per_cell, 1)));
      c.auto_chunk_per_cell = per_cell;
    }
    lim = c.auto_chunk;
  }
  return std::min(lim, n_cells);
}

// Collision (+ optional Euler) over n cells resident on the device, chunked through the workspace.
// With `gs` (fast path only) the input is not materialised: cell j's f* is gathered from gs->base by the first
// and last kernels (transport fused); `fin` is then unused and cells [gs->cell0, +n) are computed.
static fks_status run_collision(Ctx& c, const double* fin, double* out, long long n, bool euler, double s,
                                cudaStream_t st, const GatherSrc* gs = nullptr, double* U = nullptr, double* W = nullptr) {
  const bool fast = c.path == FKS_PATH_FAST;
  size_t per_cell = fast ? fast_ws_bytes_per_cell(c) : generic_ws_bytes_per_cell(c);
  long long ch = chunk_cells(c, per_cell, n);
  // more than one chunk on the N = 32 path: two workspace slots, the chunks' phases overlapped across streams (the
  // second slot is allocated only when the batch needs it; if it cannot be, the chunks run one after another)
  if (fast && ch < n && fast_pipeline_ok(c) && ensure_ws(c, 2 * per_cell * (size_t)ch) == FKS_OK) {
    const size_t nv = (size_t)c.N * c.N * c.N;
    // chunk boundaries: the first and the last chunk a quarter slot, so that the forward transform before the first
    // term-loop launch and the back transform after the last one (the two the pipeline cannot hide) are short; the
    // rest split evenly into full-slot-or-smaller chunks
    std::vector<long long> cb{0};
    const long long q4 = ch / 4;
    if (n >= 2 * q4 + ch && q4 >= 1 && !std::getenv("FKS_PIPE_NO_CARVE")) {
      cb.push_back(q4);
      const long long mid = n - 2 * q4, nm = (mid + ch - 1) / ch;
      for (long long i = 1; i <= nm; i++) cb.push_back(q4 + mid * i / nm);
      cb.push_back(n);
    } else {
      for (long long c0 = ch; c0 < n; c0 += ch) cb.push_back(c0);
      cb.push_back(n);
    }
    std::vector<PipeChunk> ck;
    for (size_t i = 0; i + 1 < cb.size(); i++) {
      const long long c0 = cb[i];
      PipeChunk q{};
      q.fin = gs ? nullptr : fin + c0 * nv;
      q.out = out + c0 * nv;
      q.n = cb[i + 1] - c0;
      q.euler = euler; q.s = s;
      if (gs) { q.has_g = true; q.g = *gs; q.g.cell0 = gs->cell0 + c0; }
      q.U = U ? U + 5 * c0 : nullptr;
      q.W = W ? W + 5 * c0 : nullptr;
      ck.push_back(q);
    }
    return fast_collision_pipelined(c, ck, ch, st);
  }
  fks_status rc = ensure_ws(c, per_cell * (size_t)ch);
  if (rc) return rc;
  const size_t nv = (size_t)c.N * c.N * c.N;
  for (long long c0 = 0; c0 < n; c0 += ch) {
    long long m = std::min(ch, n - c0);
    double* Uc = U ? U + 5 * c0 : nullptr;
    double* Wc = W ? W + 5 * c0 : nullptr;
    if (gs) {
      GatherSrc g = *gs;
      g.cell0 = gs->cell0 + c0;
      rc = fast_collision(c, nullptr, out + c0 * nv, m, euler, s, st, &g, Uc, Wc);
    } else if (fast) {
      rc = fast_collision(c, fin + c0 * nv, out + c0 * nv, m, euler, s, st, nullptr, Uc, Wc);
    } else {
      rc = generic_collision(c, fin + c0 * nv, out + c0 * nv, m, euler, s, st);
      if (!rc && (U || W)) rc = launch_macro(c, 0, out + c0 * nv, nullptr, Uc, Wc, m, 0.0, nullptr, st);
    }
    if (rc) return rc;
  }
  return cuda_status(cudaPeekAtLastError(), "collision launch");
}

static GatherSrc make_gather(const double* base, const Shift& sh, long long cell0) {
  GatherSrc g{};
  g.base = base;
  g.sh = sh;
  g.cell0 = cell0;
  g.in16 = ((uintptr_t)base & 15) == 0;
  return g;
}

static Shift advance_generic_cell(Ctx& c) {
  // Move every particle of the generic cell by v_k dt.  Units: 1/(N*cfl_den) cell; velocity
  // index k moves (2k - N)*cfl_num units per step.  delta = floor((o + d + unit/2)/unit), o <- o + d - delta*unit,
  // i.e. offsets stay in the half-open [-1/2, 1/2) cell (A16).
  Shift sh{};
  sh.nx = c.nx; sh.ny = c.ny; sh.nz = c.nz; sh.N = c.N;
  const long long unit = (long long)c.N * c.cfl_den;
  for (int a = 0; a < 3; a++) {
    for (int k = 0; k < c.N; k++) {
      long long o = c.offsets[a * c.N + k] + (2LL * k - c.N) * c.cfl_num;
      long long num = o + unit / 2;
      long long d = num >= 0 ? num / unit : -((-num + unit - 1) / unit);  // floor division
      c.offsets[a * c.N + k] = o - d * unit;
      sh.delta[a][k] = (int)d;
    }
  }
  c.last = sh;
  return sh;
}

static bool shift_is_identity(const Shift& sh) {
  for (int a = 0; a < 3; a++) {
    int n = a == 0 ? sh.nx : a == 1 ? sh.ny : sh.nz;
    for (int k = 0; k < sh.N; k++)
      if (((sh.delta[a][k] % n) + n) % n) return false;
  }
  return true;
}

}  // namespace fks

using namespace fks;

extern "C" {

const char* fks_last_error(void) { return g_last_error.c_str(); }

fks_status fks_collision_init(fks_ctx** out, int N, double L, int M_angles, int M_radial, int kernel) {
  fks_params p{};
  p.N = N; p.L = L; p.M_angles = M_angles; p.M_radial = M_radial; p.kernel = kernel;
  return fks_collision_init_ex(out, &p);
}

fks_status fks_collision_init_ex(fks_ctx** out, const fks_params* pp) {
  if (!out || !pp) { set_error("NULL argument"); return FKS_ERR_INVALID; }
  *out = nullptr;
  const fks_params& p = *pp;
  if (p.N % 2 != 0 || p.N < 4 || p.N > kMaxN) { set_error("N must be even and in [4, 64]"); return FKS_ERR_UNSUPPORTED; }
  if (!(p.L > 0.0) || !std::isfinite(p.L)) { set_error("L must be > 0"); return FKS_ERR_INVALID; }
  if (p.M_angles < 1) { set_error("M_angles must be >= 1"); return FKS_ERR_INVALID; }
  if (p.kernel != FKS_KERNEL_HARD_SPHERES && p.kernel != FKS_KERNEL_MAXWELL && p.kernel != FKS_KERNEL_VHS) {
    set_error("unknown kernel");
    return FKS_ERR_UNSUPPORTED;
  }
  if (p.kernel != FKS_KERNEL_HARD_SPHERES && p.M_radial < 1) { set_error("M_radial must be >= 1 for Maxwell molecules / VHS"); return FKS_ERR_INVALID; }
  if (p.kernel == FKS_KERNEL_VHS && !(p.vhs_alpha >= 0.0 && p.vhs_alpha <= 1.0 && p.vhs_C >= 0.0 && std::isfinite(p.vhs_C))) {
    set_error("VHS needs 0 <= vhs_alpha <= 1 and vhs_C >= 0 (0 = 1/(4 pi))");
    return FKS_ERR_INVALID;
  }
  if (p.quad_rule != FKS_QUAD_GL_UNIFORM && p.quad_rule != FKS_QUAD_PAPER_RECT) { set_error("unknown quadrature rule"); return FKS_ERR_UNSUPPORTED; }
  // 0 = default (R_c = R); otherwise R_c/R in [1, (1+sqrt2)/sqrt2]: below 1 the cutoff would truncate the
  // support of the Carleman integral (A7), above it the periodised collision partners alias
  if (!(p.cutoff_ratio == 0.0 || (p.cutoff_ratio >= 1.0 && p.cutoff_ratio <= (1.0 + std::sqrt(2.0)) / std::sqrt(2.0) + 1e-12))) {
    set_error("cutoff_ratio must be 0 (default) or in [1, (1+sqrt2)/sqrt2] (A7)"); return FKS_ERR_INVALID;
  }
  if (p.path < FKS_PATH_AUTO || p.path > FKS_PATH_FAST) { set_error("unknown path"); return FKS_ERR_UNSUPPORTED; }
  int P = p.pad > 0 ? p.pad : 3 * p.N / 2;
  // P >= 3N/2 - 2: the exact Galerkin operator (A10); N <= P < 3N/2 - 2: the aliased collocation operator
  // (l + m = k mod P; P = N is the classical collocation method)
  if (P < p.N || P > 4 * p.N) { set_error("pad must be in [N, 4N] (A10; P < 3N/2-2 is the aliased variant)"); return FKS_ERR_UNSUPPORTED; }
  int nt = p.n_theta, nf = p.n_phi;
  if (nt <= 0 || nf <= 0) {
    nt = 1 << (int)std::ceil(std::log2((double)p.M_angles) / 2.0 - 1e-12);
    if (p.M_angles % nt) nt = p.M_angles;
    nf = p.M_angles / nt;
  }
  int nd = nt * nf;
  int T = p.kernel == FKS_KERNEL_HARD_SPHERES ? nd : nd * p.M_radial;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) { cudaGetLastError(); return cuda_status(e, "no CUDA device"); }

  Ctx* c = new (std::nothrow) Ctx();
  if (!c) { set_error("host allocation failed"); return FKS_ERR_NOMEM; }
  c->p = p;
  c->N = p.N; c->K = p.N - 1; c->P = P; c->T = T;
  c->n_theta = nt; c->n_phi = nf;
  c->lambda = 2.0 / (3.0 + std::sqrt(2.0));
  c->R = c->lambda * p.L;
  c->Rc = c->R * (p.cutoff_ratio > 0.0 ? p.cutoff_ratio : 1.0);
  c->device = dev;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, dev);
  c->offsets.assign(3 * (size_t)p.N, 0);
  fks_status rc = build_tables(*c);
  if (rc) { fks_destroy(reinterpret_cast<fks_ctx*>(c)); return rc; }
  bool fast_ok = fast_available(*c);
  if (p.path == FKS_PATH_FAST && !fast_ok) {
    fks_destroy(reinterpret_cast<fks_ctx*>(c));
    set_error("fast path not instantiated for this (N, P, kernel)");
    return FKS_ERR_UNSUPPORTED;
  }
  c->path = (p.path == FKS_PATH_GENERIC || !fast_ok) ? FKS_PATH_GENERIC : FKS_PATH_FAST;
  if (c->path == FKS_PATH_FAST) {
    rc = fast_prepare(*c);
    if (rc) { fks_destroy(reinterpret_cast<fks_ctx*>(c)); return rc; }
  }
  if (std::getenv("FKS_DEBUG_PROGRESS")) {  // mapped host memory the device writes while running (hang probes)
    void* hp = nullptr;
    if (cudaHostAlloc(&hp, 4096 * 16 * sizeof(long long), cudaHostAllocMapped) == cudaSuccess) {
      std::memset(hp, 0, 4096 * 16 * sizeof(long long));
      c->prog_host = (long long*)hp;
      void* dp = nullptr;
      if (cudaHostGetDevicePointer(&dp, hp, 0) == cudaSuccess) c->prog_dev = (long long*)dp;
    } else {
      cudaGetLastError();
    }
  }
  if (std::getenv("FKS_PHASE_TIMING")) {  // debug instrumentation of the hot kernel (tools/phase_timing.py)
    if (cudaMalloc(&c->dbg, 64 * 1024 * sizeof(long long)) == cudaSuccess) cudaMemset(c->dbg, 0, 64 * 1024 * sizeof(long long));
    else { cudaGetLastError(); c->dbg = nullptr; }
  }
  rc = cuda_status(cudaDeviceSynchronize(), "table build");
  if (rc) { fks_destroy(reinterpret_cast<fks_ctx*>(c)); return rc; }
  *out = reinterpret_cast<fks_ctx*>(c);
  return FKS_OK;
}

fks_status fks_collision_batch(fks_ctx* h, const double* f, double* Q, long long n_cells, void* stream) {
  if (!h) { set_error("NULL handle"); return FKS_ERR_INVALID; }
  Ctx& c = *reinterpret_cast<Ctx*>(h);
  if (n_cells < 0) { set_error("n_cells < 0"); return FKS_ERR_INVALID; }
  if (n_cells == 0) return FKS_OK;
  fks_status rc;
  if ((rc = check_device_ptr(f, "f")) || (rc = check_device_ptr(Q, "Q"))) return rc;
  size_t bytes = (size_t)n_cells * c.N * c.N * c.N * sizeof(double);
  if (overlap(f, bytes, Q, bytes)) { set_error("Q overlaps f"); return FKS_ERR_INVALID; }
  if ((rc = sticky_check())) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if ((rc = order_begin(c, st))) return rc;
  return order_end(c, st, run_collision(c, f, Q, n_cells, false, 0.0, st));
}

fks_status fks_transport_setup(fks_ctx* h, int nx, int ny, int nz, long long cfl_num, long long cfl_den) {
  if (!h) { set_error("NULL handle"); return FKS_ERR_INVALID; }
  Ctx& c = *reinterpret_cast<Ctx*>(h);
  if (nx < 1 || ny < 1 || nz < 1) { set_error("grid dimensions must be >= 1"); return FKS_ERR_INVALID; }
  if (cfl_den < 1 || cfl_num < 0) { set_error("cfl_den must be >= 1 and cfl_num >= 0"); return FKS_ERR_INVALID; }
  if ((long long)nx * ny * nz > (1LL << 40)) { set_error("grid too large"); return FKS_ERR_INVALID; }
  if ((double)c.N * (double)cfl_den * (double)(cfl_num + 1) * 4.0 > 4e18) { set_error("CFL fraction too large"); return FKS_ERR_INVALID; }
  c.nx = nx; c.ny = ny; c.nz = nz;
  c.cfl_num = cfl_num; c.cfl_den = cfl_den;
  std::fill(c.offsets.begin(), c.offsets.end(), 0);
  c.transport_ready = true;
  c.slab = false;
  c.slab_shift_valid = false;
  c.nx_glob = nx; c.x0 = 0; c.halo = 0;
  return FKS_OK;
}

// max |delta| of any step: |displacement| <= N cfl_num units = cfl cells, offsets in [-1/2, 1/2)
static int halo_bound(long long cfl_num, long long cfl_den) { return (int)((cfl_num + cfl_den - 1) / cfl_den) + 1; }

fks_status fks_transport_setup_slab(fks_ctx* h, int nx_global, int ny, int nz, int x0, int nx_local,
                                    long long cfl_num, long long cfl_den) {
  if (!h) { set_error("NULL handle"); return FKS_ERR_INVALID; }
  Ctx& c = *reinterpret_cast<Ctx*>(h);
  if (nx_local < 1 || x0 < 0 || x0 + (long long)nx_local > nx_global) {
    set_error("slab: need 0 <= x0 and 1 <= nx_local, x0 + nx_local <= nx_global");
    return FKS_ERR_INVALID;
  }
  fks_status rc = fks_transport_setup(h, nx_local, ny, nz, cfl_num, cfl_den);
  if (rc) return rc;
  const int H = halo_bound(cfl_num, cfl_den);
  if (nx_local + 2LL * H > kMaxPlanes) { set_error("slab: nx_local + 2*halo exceeds 1024 planes"); return FKS_ERR_UNSUPPORTED; }
  c.slab = true;
  c.slab_shift_valid = false;
  c.nx_glob = nx_global; c.x0 = x0; c.halo = H;
  return FKS_OK;
}

fks_status fks_slab_halo(const fks_ctx* h, int* halo) {
  if (!h || !halo) { set_error("NULL argument"); return FKS_ERR_INVALID; }
  const Ctx& c = *reinterpret_cast<const Ctx*>(h);
  if (!c.transport_ready || !c.slab) { set_error("fks_transport_setup_slab not called"); return FKS_ERR_STATE; }
  *halo = c.halo;
  return FKS_OK;
}

fks_status fks_slab_plane_count(const fks_ctx* h, int* n_planes) {
  if (!h || !n_planes) { set_error("NULL argument"); return FKS_ERR_INVALID; }
  const Ctx& c = *reinterpret_cast<const Ctx*>(h);
  if (!c.transport_ready || !c.slab) { set_error("fks_transport_setup_slab not called"); return FKS_ERR_STATE; }
  *n_planes = c.nx + 2 * c.halo;
  return FKS_OK;
}

static fks_status slab_table(Ctx& c, const double* const* planes, double* f_out, PlaneTable& tab) {
  if (!c.transport_ready || !c.slab) { set_error("fks_transport_setup_slab not called"); return FKS_ERR_STATE; }
  if (!planes) { set_error("planes is NULL"); return FKS_ERR_INVALID; }
  fks_status rc;
  if ((rc = check_device_ptr(f_out, "f_out"))) return rc;
  const int np = c.nx + 2 * c.halo;
  const size_t plane_bytes = (size_t)c.ny * c.nz * c.N * c.N * c.N * sizeof(double);
  const size_t out_bytes = plane_bytes * c.nx;
  for (int i = 0; i < np; i++) {
    if (!planes[i]) { set_error("planes[i] is NULL"); return FKS_ERR_INVALID; }
    if ((rc = check_device_ptr(planes[i], "planes[i]"))) return rc;  // device or peer-mapped memory
    if (overlap(planes[i], plane_bytes, f_out, out_bytes)) { set_error("a source plane overlaps f_out"); return FKS_ERR_INVALID; }
    tab.p[i] = planes[i];
  }
  return FKS_OK;
}

fks_status fks_transport_step_slab(fks_ctx* h, const double* const* planes, double* f_out, void* stream) {
  if (!h) { set_error("NULL handle"); return FKS_ERR_INVALID; }
  Ctx& c = *reinterpret_cast<Ctx*>(h);
  static thread_local PlaneTable tab;
  fks_status rc;
  if ((rc = slab_table(c, planes, f_out, tab))) return rc;
  if ((rc = sticky_check())) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if ((rc = order_begin(c, st))) return rc;
  Shift sh = advance_generic_cell(c);
  c.slab_shift_valid = false;  // a later fks_step_slab_range(advance = 0) must not reuse an older step's shift
  c.prof.begin(0, st);
  rc = launch_transport_gather_slab(c, tab, f_out, sh, st);
  c.prof.end(0, st);
  return order_end(c, st, rc);
}

fks_status fks_step_slab_range(fks_ctx* h, const double* const* planes, double* f_out, double coll_scale, int lx0,
                               int lx1, int advance, void* stream) {
  if (!h) { set_error("NULL handle"); return FKS_ERR_INVALID; }
  Ctx& c = *reinterpret_cast<Ctx*>(h);
  if (!std::isfinite(coll_scale)) { set_error("coll_scale must be finite"); return FKS_ERR_INVALID; }
  static thread_local PlaneTable tab;
  fks_status rc;
  if ((rc = slab_table(c, planes, f_out, tab))) return rc;
  if (lx0 < 0 || lx1 < lx0 || lx1 > c.nx) { set_error("plane range outside [0, nx_local]"); return FKS_ERR_INVALID; }
  if (!advance && !c.slab_shift_valid) { set_error("no step in progress: the first call of a step must advance"); return FKS_ERR_STATE; }
  if ((rc = sticky_check())) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if ((rc = order_begin(c, st))) return rc;
  if (advance) {
    c.slab_shift = advance_generic_cell(c);
    c.slab_shift_valid = true;
  }
  const long long plane = (long long)c.ny * c.nz, cell0 = lx0 * plane, m = (long long)(lx1 - lx0) * plane;
  const size_t nv = (size_t)c.N * c.N * c.N;
  c.prof.begin(0, st);
  rc = launch_transport_gather_slab(c, tab, f_out, c.slab_shift, st, cell0, m);
  c.prof.end(0, st);
  if (!rc && m > 0) rc = run_collision(c, f_out + cell0 * nv, f_out + cell0 * nv, m, true, coll_scale, st);
  return order_end(c, st, rc);
}

fks_status fks_step_slab(fks_ctx* h, const double* const* planes, double* f_out, double coll_scale, void* stream) {
  if (!h) { set_error("NULL handle"); return FKS_ERR_INVALID; }
  return fks_step_slab_range(h, planes, f_out, coll_scale, 0, reinterpret_cast<Ctx*>(h)->nx, 1, stream);
}

fks_status fks_transport_step(fks_ctx* h, const double* f_in, double* f_out, void* stream) {
  if (!h) { set_error("NULL handle"); return FKS_ERR_INVALID; }
  Ctx& c = *reinterpret_cast<Ctx*>(h);
  if (!c.transport_ready) { set_error("fks_transport_setup not called"); return FKS_ERR_STATE; }
  if (c.slab) { set_error("handle is set up for a slab: use the _slab calls"); return FKS_ERR_STATE; }
  fks_status rc;
  if ((rc = check_device_ptr(f_in, "f_in")) || (rc = check_device_ptr(f_out, "f_out"))) return rc;
  long long n = (long long)c.nx * c.ny * c.nz;
  size_t bytes = (size_t)n * c.N * c.N * c.N * sizeof(double);
  if (overlap(f_in, bytes, f_out, bytes)) { set_error("f_out overlaps f_in"); return FKS_ERR_INVALID; }
  if ((rc = sticky_check())) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if ((rc = order_begin(c, st))) return rc;
  Shift sh = advance_generic_cell(c);
  c.prof.begin(0, st);
  rc = launch_transport_gather(c, f_in, f_out, sh, st);
  c.prof.end(0, st);
  return order_end(c, st, rc);
}

// fks_step and fks_step_moments: transport, collision + Euler, optional moments of f_out (U, W may be NULL)
static fks_status step_impl(fks_ctx* h, const double* f_in, double* f_out, double coll_scale, double* U, double* W,
                            void* stream) {
  if (!h) { set_error("NULL handle"); return FKS_ERR_INVALID; }
  Ctx& c = *reinterpret_cast<Ctx*>(h);
  if (!c.transport_ready) { set_error("fks_transport_setup not called"); return FKS_ERR_STATE; }
  if (c.slab) { set_error("handle is set up for a slab: use the _slab calls"); return FKS_ERR_STATE; }
  if (!std::isfinite(coll_scale)) { set_error("coll_scale must be finite"); return FKS_ERR_INVALID; }
  fks_status rc;
  if ((rc = check_device_ptr(f_in, "f_in")) || (rc = check_device_ptr(f_out, "f_out"))) return rc;
  long long n = (long long)c.nx * c.ny * c.nz;
  size_t bytes = (size_t)n * c.N * c.N * c.N * sizeof(double);
  if (overlap(f_in, bytes, f_out, bytes)) { set_error("f_out overlaps f_in"); return FKS_ERR_INVALID; }
  if (U || W) {
    const size_t mb = (size_t)n * 5 * sizeof(double);
    if ((U && (rc = check_device_ptr(U, "U"))) || (W && (rc = check_device_ptr(W, "W")))) return rc;
    if ((U && (overlap(U, mb, f_in, bytes) || overlap(U, mb, f_out, bytes))) ||
        (W && (overlap(W, mb, f_in, bytes) || overlap(W, mb, f_out, bytes))) || (U && W && overlap(U, mb, W, mb))) {
      set_error("U / W overlap f_in, f_out or each other"); return FKS_ERR_INVALID;
    }
  }
  if ((rc = sticky_check())) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if ((rc = order_begin(c, st))) return rc;
  Shift sh = advance_generic_cell(c);
  if (shift_is_identity(sh)) return order_end(c, st, run_collision(c, f_in, f_out, n, true, coll_scale, st, nullptr, U, W));
  if (c.path == FKS_PATH_FAST && !std::getenv("FKS_UNFUSED_TRANSPORT")) {  // transport fused into kf1 / kb3
    const GatherSrc g = make_gather(f_in, sh, 0);
    return order_end(c, st, run_collision(c, nullptr, f_out, n, true, coll_scale, st, &g, U, W));
  }
  // transport (exact permutation) into f_out, then collision + Euler in place on f_out
  c.prof.begin(0, st);
  rc = launch_transport_gather(c, f_in, f_out, sh, st);
  c.prof.end(0, st);
  if (!rc) rc = run_collision(c, f_out, f_out, n, true, coll_scale, st, nullptr, U, W);
  return order_end(c, st, rc);
}

fks_status fks_step(fks_ctx* h, const double* f_in, double* f_out, double coll_scale, void* stream) {
  return step_impl(h, f_in, f_out, coll_scale, nullptr, nullptr, stream);
}

fks_status fks_step_moments(fks_ctx* h, const double* f_in, double* f_out, double coll_scale, double* U, double* W,
                            void* stream) {
  if (!U && !W) { set_error("fks_step_moments: U and W are both NULL"); return FKS_ERR_INVALID; }
  return step_impl(h, f_in, f_out, coll_scale, U, W, stream);
}

static fks_status ensure_stage(Ctx& c, long long cells) {
  if (cells <= c.stage_cells) return FKS_OK;
  if (c.d_stage_in) cudaFree(c.d_stage_in);
  if (c.d_stage_out) cudaFree(c.d_stage_out);
  c.d_stage_in = c.d_stage_out = nullptr;
  c.stage_cells = 0;
  size_t bytes = (size_t)cells * c.N * c.N * c.N * sizeof(double);
  cudaError_t e = cudaMalloc(&c.d_stage_in, bytes);
  if (e == cudaSuccess) e = cudaMalloc(&c.d_stage_out, bytes);
  if (e != cudaSuccess) { cudaGetLastError(); return cuda_status(e, "staging allocation"); }
  if (!c.stage_stream) cudaStreamCreateWithFlags(&c.stage_stream, cudaStreamNonBlocking);
  c.stage_cells = cells;
  return FKS_OK;
}

fks_status fks_collision_batch_host(fks_ctx* h, const double* f_host, double* Q_host, long long n_cells) {
  if (!h) { set_error("NULL handle"); return FKS_ERR_INVALID; }
  Ctx& c = *reinterpret_cast<Ctx*>(h);
  if (n_cells < 0 || (n_cells > 0 && (!f_host || !Q_host))) { set_error("bad host buffers"); return FKS_ERR_INVALID; }
  if (n_cells == 0) return FKS_OK;
  fks_status rc;
  if ((rc = sticky_check())) return rc;
  if ((rc = ensure_stage(c, n_cells))) return rc;
  // pipelined in chunks of cells over three streams: copy-in of chunk i+1 and copy-out of chunk i-1 overlap the
  // collision of chunk i (cells are independent)
  if (!c.h2d_stream) cudaStreamCreateWithFlags(&c.h2d_stream, cudaStreamNonBlocking);
  if (!c.d2h_stream) cudaStreamCreateWithFlags(&c.d2h_stream, cudaStreamNonBlocking);
  const long long nv = (long long)c.N * c.N * c.N;
  // chunks of >= 32 MB of input (at most 32), the first and the last one with their outer quarter cut off as a
  // chunk of its own, so that only a small copy-in and copy-out stay exposed at the two ends (c2: 512 cells of
  // 256 KB -> 4 chunks + 2 quarter chunks; it was one chunk with both copies exposed)
  std::vector<long long> cb;  // chunk boundaries
  {
    const long long box_bytes = n_cells * nv * (long long)sizeof(double);
    const long long n0 = std::max(1LL, std::min({32LL, box_bytes / (32LL << 20), n_cells}));
    for (long long i = 0; i <= n0; i++) cb.push_back(n_cells * i / n0);
    if (n0 >= 3 && cb[1] - cb[0] >= 4 && !std::getenv("FKS_HOST_NO_CARVE")) {
      cb.insert(cb.begin() + 1, cb[0] + (cb[1] - cb[0]) / 4);
      const size_t e = cb.size() - 1;
      cb.insert(cb.begin() + e, cb[e] - (cb[e] - cb[e - 1]) / 4);
    }
  }
  const long long nch = (long long)cb.size() - 1;
  cudaStream_t st = c.stage_stream;
  if ((rc = order_begin(c, st)) || (rc = order_begin(c, c.h2d_stream))) return rc;
  std::vector<cudaEvent_t> eh(nch), ec(nch);
  for (long long i = 0; i < nch; i++) {
    cudaEventCreateWithFlags(&eh[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ec[i], cudaEventDisableTiming);
  }
  for (long long i = 0; i < nch && !rc; i++) {
    const long long c0 = cb[i], m = cb[i + 1] - cb[i];
    rc = cuda_status(cudaMemcpyAsync(c.d_stage_in + c0 * nv, f_host + c0 * nv, (size_t)m * nv * sizeof(double),
                                     cudaMemcpyHostToDevice, c.h2d_stream), "H2D");
    if (!rc) rc = cuda_status(cudaEventRecord(eh[i], c.h2d_stream), "event");
  }
  // N = 32: the chunks run through the chunk pipeline (each chunk's forward transform waits for its copy-in, its
  // copy-out for its back transform), as in fks_step_host
  long long cap = 0;
  for (long long i = 0; i < nch; i++) cap = std::max(cap, cb[i + 1] - cb[i]);
  const size_t pc_bytes = c.path == FKS_PATH_FAST ? fast_ws_bytes_per_cell(c) : 0;
  const bool piped = !rc && nch >= 2 && c.path == FKS_PATH_FAST && fast_pipeline_ok(c) &&
                     chunk_cells(c, pc_bytes, cap) >= cap &&
                     ensure_ws(c, 2 * pc_bytes * (size_t)cap) == FKS_OK;  // else the chunks run one by one
  if (piped) {
    std::vector<PipeChunk> pc;
    for (long long i = 0; i < nch; i++) {
      const long long c0 = cb[i], m = cb[i + 1] - cb[i];
      PipeChunk q{};
      q.fin = c.d_stage_in + c0 * nv;
      q.out = c.d_stage_out + c0 * nv;
      q.n = m;
      q.wait_before = eh[i];
      q.record_after = ec[i];
      pc.push_back(q);
    }
    if (!rc) rc = fast_collision_pipelined(c, pc, cap, st);
    for (long long i = 0; i < nch && !rc; i++) {
      const long long c0 = cb[i], m = cb[i + 1] - cb[i];
      rc = cuda_status(cudaStreamWaitEvent(c.d2h_stream, ec[i], 0), "wait compute");
      if (!rc) rc = cuda_status(cudaMemcpyAsync(Q_host + c0 * nv, c.d_stage_out + c0 * nv, (size_t)m * nv * sizeof(double),
                                                cudaMemcpyDeviceToHost, c.d2h_stream), "D2H");
    }
  }
  for (long long i = 0; i < nch && !rc && !piped; i++) {
    const long long c0 = cb[i], m = cb[i + 1] - cb[i];
    rc = cuda_status(cudaStreamWaitEvent(st, eh[i], 0), "wait H2D");
    if (!rc) rc = run_collision(c, c.d_stage_in + c0 * nv, c.d_stage_out + c0 * nv, m, false, 0.0, st);
    if (!rc) rc = cuda_status(cudaEventRecord(ec[i], st), "event");
    if (!rc) rc = cuda_status(cudaStreamWaitEvent(c.d2h_stream, ec[i], 0), "wait compute");
    if (!rc) rc = cuda_status(cudaMemcpyAsync(Q_host + c0 * nv, c.d_stage_out + c0 * nv, (size_t)m * nv * sizeof(double),
                                              cudaMemcpyDeviceToHost, c.d2h_stream), "D2H");
  }
  fks_status rs = cuda_status(cudaStreamSynchronize(c.d2h_stream), "host-buffer collision");
  cudaStreamSynchronize(st);
  cudaStreamSynchronize(c.h2d_stream);
  for (long long i = 0; i < nch; i++) { cudaEventDestroy(eh[i]); cudaEventDestroy(ec[i]); }
  c.ev_pending = false;  // everything this handle enqueued has completed
  return rc ? rc : rs;
}

// Host-buffer step, pipelined over slabs of x-planes on three streams: the input planes are copied in (the
// periodic wrap-around halo first), each slab is transported and collided as soon as the planes it gathers from
// (slab +- max |delta_x|) have landed, and each finished slab is copied back while the next one computes.
fks_status fks_step_host(fks_ctx* h, const double* f_in_host, double* f_out_host, double coll_scale) {
  if (!h) { set_error("NULL handle"); return FKS_ERR_INVALID; }
  Ctx& c = *reinterpret_cast<Ctx*>(h);
  if (!c.transport_ready) { set_error("fks_transport_setup not called"); return FKS_ERR_STATE; }
  if (c.slab) { set_error("handle is set up for a slab: use the _slab calls"); return FKS_ERR_STATE; }
  if (!f_in_host || !f_out_host) { set_error("bad host buffers"); return FKS_ERR_INVALID; }
  if (!std::isfinite(coll_scale)) { set_error("coll_scale must be finite"); return FKS_ERR_INVALID; }
  const long long n = (long long)c.nx * c.ny * c.nz;
  fks_status rc;
  if ((rc = sticky_check())) return rc;
  if ((rc = ensure_stage(c, n))) return rc;
  if (!c.h2d_stream) cudaStreamCreateWithFlags(&c.h2d_stream, cudaStreamNonBlocking);
  if (!c.d2h_stream) cudaStreamCreateWithFlags(&c.d2h_stream, cudaStreamNonBlocking);
  const long long nv = (long long)c.N * c.N * c.N;
  const long long plane = (long long)c.ny * c.nz;          // cells per x-plane (contiguous)
  const size_t pbytes = (size_t)plane * nv * sizeof(double);
  cudaStream_t st = c.stage_stream;
  if ((rc = order_begin(c, st)) || (rc = order_begin(c, c.h2d_stream))) return rc;
  const Shift sh = advance_generic_cell(c);
  int dmax = 0, dmy = 0;
  for (int k = 0; k < c.N; k++) {
    dmax = std::max(dmax, std::abs(sh.delta[0][k]));
    dmy = std::max(dmy, std::abs(sh.delta[1][k]));
  }
  const int nx = c.nx, ny = c.ny;
  // slabs: more slabs expose less of the first copy-in and the last copy-out (c3: 32 slabs of one plane;
  // measured e2e 1.71e9 with 4 slabs, 1.82e9 with 8, 1.88e9 with 16, 1.90e9 with 32); each
  // slab must be at least max|delta_x| planes wide, and the halo must not wrap onto itself
  // ... and no slab below 32 MB of input: a small box (c1: 7 MB) would otherwise pay a dozen kernel launches
  // per slab for a copy that takes microseconds
  const long long box_bytes = (long long)nx * pbytes;
  int nslab = (int)std::max(1LL, std::min(32LL, box_bytes / (32LL << 20)));
  if (const char* e = std::getenv("FKS_HOST_SLABS")) nslab = std::max(1, std::atoi(e));
  int nch = std::min(nslab, nx / std::max(1, dmax));
  if (nch < 1 || nx <= 2 * dmax) nch = 1;                  // halo too wide for slabs: one piece
  // Work chunks = (x-planes [xa, xb), y-rows [ya, yb)), a contiguous cell range each.  The first and the last
  // slab, when they are one plane of >= 16 rows, are cut into 4 row blocks: the first computation then waits only
  // for the rows it reads (its plane and its x-neighbours, its rows +- max|delta_y|) and the last copy-out is a
  // quarter plane (round 2: about 14 ms less exposed copy per c3 step).
  // A first / last slab of several planes (a slab box such as c2: 512 x 1 x 1) gives up its outer quarter (at least
  // max|delta_x| planes) as a piece of its own, for the same reason: less copy exposed at the two ends.
  struct Chunk { int xa, xb, ya, yb; };
  std::vector<std::pair<int, int>> xs;
  const int wmin = std::max(1, dmax);
  for (int i = 0; i < nch; i++) {
    const int xa = (int)((long long)nx * i / nch), xb = (int)((long long)nx * (i + 1) / nch);
    const bool carve = nch >= 3 && (i == 0 || i == nch - 1) && xb - xa >= 4 * wmin && !std::getenv("FKS_HOST_NO_CARVE");
    if (!carve) { xs.push_back({xa, xb}); continue; }
    const int w = std::max(wmin, (xb - xa) / 4);
    if (i == 0) { xs.push_back({xa, xa + w}); xs.push_back({xa + w, xb}); }
    else { xs.push_back({xa, xb - w}); xs.push_back({xb - w, xb}); }
  }
  std::vector<Chunk> ch;
  const int nxs = (int)xs.size();
  for (int i = 0; i < nxs; i++) {
    const int xa = xs[i].first, xb = xs[i].second;
    const bool split = nxs > 1 && (i == 0 || i == nxs - 1) && xb - xa == 1 && ny >= 16 && ny >= 4 * (2 * dmy + 1);
    const int parts = split ? 4 : 1;
    for (int q = 0; q < parts; q++) ch.push_back({xa, xb, (int)((long long)ny * q / parts), (int)((long long)ny * (q + 1) / parts)});
  }
  const int nk = (int)ch.size();
  std::vector<cudaEvent_t> eh(nk), ec(nk);
  for (int i = 0; i < nk; i++) {
    cudaEventCreateWithFlags(&eh[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ec[i], cudaEventDisableTiming);
  }
  // copy-in in the order of first need, at row granularity (rows are contiguous within a plane)
  std::vector<char> have((size_t)nx * ny, 0);
  const size_t rbytes = (size_t)c.nz * nv * sizeof(double);  // one y-row of one plane
  auto need_rows = [&](int p, int y0, int y1) -> fks_status {  // rows [y0, y1) of plane p (mod ny), not yet copied
    for (int y = y0; y < y1;) {
      const int yy = ((y % ny) + ny) % ny;
      if (have[(size_t)p * ny + yy]) { y++; continue; }
      int run = 0;  // contiguous uncopied rows starting at yy without wrapping
      while (y + run < y1 && yy + run < ny && !have[(size_t)p * ny + yy + run]) run++;
      for (int k = 0; k < run; k++) have[(size_t)p * ny + yy + k] = 1;
      const size_t off = ((size_t)p * ny + yy) * c.nz * nv;
      fks_status r = cuda_status(cudaMemcpyAsync(c.d_stage_in + off, f_in_host + off, run * rbytes,
                                                 cudaMemcpyHostToDevice, c.h2d_stream), "H2D");
      if (r) return r;
      y += run;
    }
    return FKS_OK;
  };
  for (int i = 0; i < nk && !rc; i++) {
    const Chunk& k = ch[i];
    const bool whole = k.ya == 0 && k.yb == ny;
    const int y0 = whole ? 0 : k.ya - dmy, y1 = whole ? ny : k.yb + dmy;
    for (int x = k.xa - (nch > 1 ? dmax : 0); x < k.xb + (nch > 1 ? dmax : 0) && !rc; x++)
      rc = need_rows(((x % nx) + nx) % nx, y0, y1);
    if (i == nk - 1)  // everything left (single-piece case: the whole box)
      for (int x = 0; x < nx && !rc; x++) rc = need_rows(x, 0, ny);
    if (!rc) rc = cuda_status(cudaEventRecord(eh[i], c.h2d_stream), "event");
  }
  const bool ident = shift_is_identity(sh);
  auto first_cell = [&](const Chunk& k) { return ((long long)k.xa * ny + k.ya) * c.nz; };
  auto cells_of = [&](const Chunk& k) {
    return (k.xb - k.xa == 1) ? (long long)(k.yb - k.ya) * c.nz : (long long)(k.xb - k.xa) * plane;
  };
  // N = 32: the pieces run through the chunk pipeline (forward / back transforms of neighbouring pieces beside
  // the term loop, fast_collision_pipelined), each piece's forward transform waiting for its own copy-in and its
  // copy-out waiting for its back transform
  const bool fused = c.path == FKS_PATH_FAST && !std::getenv("FKS_UNFUSED_TRANSPORT");
  long long cap = 0;
  for (const Chunk& k : ch) cap = std::max(cap, cells_of(k));
  const size_t pc_bytes = c.path == FKS_PATH_FAST ? fast_ws_bytes_per_cell(c) : 0;
  const bool piped = !rc && nk >= 2 && fused && fast_pipeline_ok(c) && chunk_cells(c, pc_bytes, cap) >= cap &&
                     ensure_ws(c, 2 * pc_bytes * (size_t)cap) == FKS_OK;  // else the pieces run one by one
  if (piped) {
    std::vector<PipeChunk> pc;
    for (int i = 0; i < nk && !rc; i++) {
      const long long c0 = first_cell(ch[i]);
      PipeChunk q{};
      q.fin = ident ? c.d_stage_in + c0 * nv : nullptr;
      q.out = c.d_stage_out + c0 * nv;
      q.n = cells_of(ch[i]);
      q.euler = true; q.s = coll_scale;
      if (!ident) { q.has_g = true; q.g = make_gather(c.d_stage_in, sh, c0); }
      q.wait_before = eh[i];
      q.record_after = ec[i];
      pc.push_back(q);
    }
    if (!rc) rc = fast_collision_pipelined(c, pc, cap, st);
    for (int i = 0; i < nk && !rc; i++) {
      const long long c0 = first_cell(ch[i]), m = cells_of(ch[i]);
      rc = cuda_status(cudaStreamWaitEvent(c.d2h_stream, ec[i], 0), "wait compute");
      if (!rc) rc = cuda_status(cudaMemcpyAsync(f_out_host + c0 * nv, c.d_stage_out + c0 * nv, (size_t)m * nv * sizeof(double),
                                                cudaMemcpyDeviceToHost, c.d2h_stream), "D2H");
    }
  }
  for (int i = 0; i < nk && !rc && !piped; i++) {
    const Chunk& k = ch[i];
    const long long c0 = first_cell(k);
    const long long m = cells_of(k);
    rc = cuda_status(cudaStreamWaitEvent(st, eh[i], 0), "wait H2D");
    if (!rc) {
      if (ident) rc = run_collision(c, c.d_stage_in + c0 * nv, c.d_stage_out + c0 * nv, m, true, coll_scale, st);
      else if (c.path == FKS_PATH_FAST && !std::getenv("FKS_UNFUSED_TRANSPORT")) {
        const GatherSrc g = make_gather(c.d_stage_in, sh, c0);
        rc = run_collision(c, nullptr, c.d_stage_out + c0 * nv, m, true, coll_scale, st, &g);
      } else {
        rc = launch_transport_gather(c, c.d_stage_in, c.d_stage_out, sh, st, c0, m);
        if (!rc) rc = run_collision(c, c.d_stage_out + c0 * nv, c.d_stage_out + c0 * nv, m, true, coll_scale, st);
      }
    }
    if (!rc) rc = cuda_status(cudaEventRecord(ec[i], st), "event");
    if (!rc) rc = cuda_status(cudaStreamWaitEvent(c.d2h_stream, ec[i], 0), "wait compute");
    if (!rc) rc = cuda_status(cudaMemcpyAsync(f_out_host + c0 * nv, c.d_stage_out + c0 * nv, (size_t)m * nv * sizeof(double),
                                              cudaMemcpyDeviceToHost, c.d2h_stream), "D2H");
  }
  fks_status rs = cuda_status(cudaStreamSynchronize(c.d2h_stream), "host-buffer step");
  cudaStreamSynchronize(st);
  cudaStreamSynchronize(c.h2d_stream);
  for (int i = 0; i < nk; i++) { cudaEventDestroy(eh[i]); cudaEventDestroy(ec[i]); }
  c.ev_pending = false;  // everything this handle enqueued has completed
  return rc ? rc : rs;
}

// ---- macroscopic moments and the BGK operator (macro.cu) -----------------------------------------------
static fks_status check_opt_moments(const Ctx& c, double* U, double* W, long long n, const void* f, size_t fbytes) {
  fks_status rc;
  const size_t mb = (size_t)n * 5 * sizeof(double);
  if (U && (rc = check_device_ptr(U, "U"))) return rc;
  if (W && (rc = check_device_ptr(W, "W"))) return rc;
  if (U && overlap(U, mb, f, fbytes)) { set_error("U overlaps f"); return FKS_ERR_INVALID; }
  if (W && overlap(W, mb, f, fbytes)) { set_error("W overlaps f"); return FKS_ERR_INVALID; }
  if (U && W && overlap(U, mb, W, mb)) { set_error("U overlaps W"); return FKS_ERR_INVALID; }
  (void)c;
  return FKS_OK;
}

fks_status fks_moments(fks_ctx* h, const double* f, double* U, double* W, long long n_cells, void* stream) {
  if (!h) { set_error("NULL handle"); return FKS_ERR_INVALID; }
  Ctx& c = *reinterpret_cast<Ctx*>(h);
  if (n_cells < 0) { set_error("n_cells < 0"); return FKS_ERR_INVALID; }
  if (n_cells == 0) return FKS_OK;
  if (!U && !W) { set_error("fks_moments: U and W are both NULL"); return FKS_ERR_INVALID; }
  fks_status rc;
  if ((rc = check_device_ptr(f, "f"))) return rc;
  const size_t bytes = (size_t)n_cells * c.N * c.N * c.N * sizeof(double);
  if ((rc = check_opt_moments(c, U, W, n_cells, f, bytes))) return rc;
  if ((rc = sticky_check())) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if ((rc = order_begin(c, st))) return rc;
  return order_end(c, st, launch_macro(c, 0, f, nullptr, U, W, n_cells, 0.0, nullptr, st));
}

fks_status fks_bgk_batch(fks_ctx* h, const double* f, double* Q, double nu, long long n_cells, void* stream) {
  if (!h) { set_error("NULL handle"); return FKS_ERR_INVALID; }
  Ctx& c = *reinterpret_cast<Ctx*>(h);
  if (n_cells < 0) { set_error("n_cells < 0"); return FKS_ERR_INVALID; }
  if (!std::isfinite(nu)) { set_error("nu must be finite"); return FKS_ERR_INVALID; }
  if (n_cells == 0) return FKS_OK;
  fks_status rc;
  if ((rc = check_device_ptr(f, "f")) || (rc = check_device_ptr(Q, "Q"))) return rc;
  const size_t bytes = (size_t)n_cells * c.N * c.N * c.N * sizeof(double);
  if (overlap(f, bytes, Q, bytes)) { set_error("Q overlaps f"); return FKS_ERR_INVALID; }
  if ((rc = sticky_check())) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if ((rc = order_begin(c, st))) return rc;
  return order_end(c, st, launch_macro(c, 1, f, Q, nullptr, nullptr, n_cells, nu, nullptr, st));
}

fks_status fks_bgk_step(fks_ctx* h, const double* f_in, double* f_out, double nu_dt, double* U, double* W,
                        void* stream) {
  if (!h) { set_error("NULL handle"); return FKS_ERR_INVALID; }
  Ctx& c = *reinterpret_cast<Ctx*>(h);
  if (!c.transport_ready) { set_error("fks_transport_setup not called"); return FKS_ERR_STATE; }
  if (c.slab) { set_error("handle is set up for a slab: use the _slab calls"); return FKS_ERR_STATE; }
  if (!std::isfinite(nu_dt)) { set_error("nu_dt must be finite"); return FKS_ERR_INVALID; }
  fks_status rc;
  if ((rc = check_device_ptr(f_in, "f_in")) || (rc = check_device_ptr(f_out, "f_out"))) return rc;
  const long long n = (long long)c.nx * c.ny * c.nz;
  const size_t bytes = (size_t)n * c.N * c.N * c.N * sizeof(double);
  if (overlap(f_in, bytes, f_out, bytes)) { set_error("f_out overlaps f_in"); return FKS_ERR_INVALID; }
  if ((rc = check_opt_moments(c, U, W, n, f_in, bytes))) return rc;
  if ((U && overlap(U, (size_t)n * 40, f_out, bytes)) || (W && overlap(W, (size_t)n * 40, f_out, bytes))) {
    set_error("U/W overlap f_out");
    return FKS_ERR_INVALID;
  }
  if ((rc = sticky_check())) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if ((rc = order_begin(c, st))) return rc;
  Shift sh = advance_generic_cell(c);
  return order_end(c, st, launch_macro(c, 2, f_in, f_out, U, W, n, nu_dt, &sh, st));
}

fks_status fks_get_info(const fks_ctx* h, int* P, int* T, double* R, double* lambda) {
  if (!h) { set_error("NULL handle"); return FKS_ERR_INVALID; }
  const Ctx& c = *reinterpret_cast<const Ctx*>(h);
  if (P) *P = c.P;
  if (T) *T = c.T;
  if (R) *R = c.Rc;
  if (lambda) *lambda = c.lambda;
  return FKS_OK;
}

fks_status fks_get_tables(const fks_ctx* h, double* a_host, double* b_host, double* dirs_host, double* w_host) {
  if (!h) { set_error("NULL handle"); return FKS_ERR_INVALID; }
  const Ctx& c = *reinterpret_cast<const Ctx*>(h);
  size_t nl = (size_t)c.K * c.K * c.K, n = (size_t)(c.T + 1) * nl;
  if (a_host || b_host) {
    std::vector<double2> tmp(n);
    fks_status rc = cuda_status(cudaMemcpy(tmp.data(), c.d_ab, n * sizeof(double2), cudaMemcpyDeviceToHost), "table copy");
    if (rc) return rc;
    for (size_t i = 0; i < n; i++) {
      const double k = c.kappa.empty() ? 1.0 : c.kappa[i / nl];  // undo the exact power-of-two balancing
      if (a_host) a_host[i] = tmp[i].x / k;
      if (b_host) b_host[i] = tmp[i].y * k;
    }
  }
  if (dirs_host) std::memcpy(dirs_host, c.dirs.data(), c.dirs.size() * sizeof(double));
  if (w_host) std::memcpy(w_host, c.w.data(), c.w.size() * sizeof(double));
  return FKS_OK;
}

fks_status fks_get_fast_layout(const fks_ctx* h, int* ctas_per_cell, int* concurrent_cells) {
  if (!h) { set_error("NULL handle"); return FKS_ERR_INVALID; }
  const Ctx& c = *reinterpret_cast<const Ctx*>(h);
  const bool fast = c.path == FKS_PATH_FAST;
  if (ctas_per_cell) *ctas_per_cell = fast ? c.fast_variant : 0;
  if (concurrent_cells) *concurrent_cells = fast ? c.fast_nteams : 0;
  return FKS_OK;
}

int fks_get_path(const fks_ctx* h) { return h ? reinterpret_cast<const Ctx*>(h)->path : -1; }

fks_status fks_get_last_shift(const fks_ctx* h, int* delta_host) {
  if (!h || !delta_host) { set_error("NULL argument"); return FKS_ERR_INVALID; }
  const Ctx& c = *reinterpret_cast<const Ctx*>(h);
  for (int a = 0; a < 3; a++)
    for (int k = 0; k < c.N; k++) delta_host[a * c.N + k] = c.last.delta[a][k];
  return FKS_OK;
}

fks_status fks_profile(fks_ctx* h, int enable) {
  if (!h) { set_error("NULL handle"); return FKS_ERR_INVALID; }
  reinterpret_cast<Ctx*>(h)->prof.on = enable != 0;
  return FKS_OK;
}

fks_status fks_profile_read(fks_ctx* h, double* ms, long long* count) {
  if (!h || !ms || !count) { set_error("NULL argument"); return FKS_ERR_INVALID; }
  PhaseTimer& pt = reinterpret_cast<Ctx*>(h)->prof;
  for (int ph = 0; ph < 4; ph++) {
    ms[ph] = 0.0;
    count[ph] = (long long)pt.used[ph].size();
    for (auto& ev : pt.used[ph]) {
      cudaError_t e = cudaEventSynchronize(ev.second);
      if (e != cudaSuccess) return cuda_status(e, "profile event");
      float t = 0.f;
      cudaEventElapsedTime(&t, ev.first, ev.second);
      ms[ph] += t;
      pt.pool.push_back(ev);
    }
    pt.used[ph].clear();
  }
  return FKS_OK;
}

long long fks_debug_timestamps(const fks_ctx* h, long long* host, long long n) {
  if (!h || !host) return 0;
  const Ctx& c = *reinterpret_cast<const Ctx*>(h);
  if (!c.dbg) return 0;
  n = std::min<long long>(n, 64 * 1024);
  if (cudaMemcpy(host, c.dbg, n * sizeof(long long), cudaMemcpyDeviceToHost) != cudaSuccess) { cudaGetLastError(); return 0; }
  return n;
}

// debug only (not in fks.h): host address of the mapped progress words, 0 if disabled
extern "C" long long fks_debug_progress_ptr(const fks_ctx* h) {
  return h ? (long long)reinterpret_cast<const Ctx*>(h)->prog_host : 0;
}

long long fks_launch_count(const fks_ctx* h) {
  return h ? reinterpret_cast<const Ctx*>(h)->launches : -1;
}

fks_status fks_sync(fks_ctx* h, void* stream) {
  (void)h;
  fks_status rc = cuda_status(cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream)), "stream sync");
  if (rc) return rc;
  return sticky_check();
}

void fks_destroy(fks_ctx* h) {
  if (!h) return;
  Ctx* c = reinterpret_cast<Ctx*>(h);
  if (c->d_ab) cudaFree(c->d_ab);
  if (c->d_abT) cudaFree(c->d_abT);
  if (c->d_w1) cudaFree(c->d_w1);
  if (c->d_mpart) cudaFree(c->d_mpart);
  if (c->dbg) cudaFree(c->dbg);
  if (c->prog_host) cudaFreeHost(c->prog_host);
  if (c->d_ctr) cudaFree(c->d_ctr);
  if (c->d_twN) cudaFree(c->d_twN);
  if (c->d_twP) cudaFree(c->d_twP);
  if (c->d_ws) cudaFree(c->d_ws);
  if (c->d_stage_in) cudaFree(c->d_stage_in);
  if (c->d_stage_out) cudaFree(c->d_stage_out);
  if (c->stage_stream) cudaStreamDestroy(c->stage_stream);
  if (c->h2d_stream) cudaStreamDestroy(c->h2d_stream);
  if (c->d2h_stream) cudaStreamDestroy(c->d2h_stream);
  if (c->hot_stream) cudaStreamDestroy(c->hot_stream);
  if (c->side_stream) cudaStreamDestroy(c->side_stream);
  for (cudaEvent_t ev : c->ev_pipe)
    if (ev) cudaEventDestroy(ev);
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  for (int ph = 0; ph < 4; ph++)
    for (auto& ev : c->prof.used[ph]) c->prof.pool.push_back(ev);
  for (auto& ev : c->prof.pool) { cudaEventDestroy(ev.first); cudaEventDestroy(ev.second); }
  delete c;
}

}  // extern "C"
