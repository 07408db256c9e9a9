// Internal declarations shared by the libfks translation units (host runtime + sm_100a kernels).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <string>
#include <vector>
#include "../../include/fks.h"

namespace fks {

constexpr int kMaxN = 64;

// Per-step transport shifts passed BY VALUE as a kernel parameter (snapshotted at launch, so the host can
// advance the generic cell for the next step immediately).  delta[a][k] = whole cells crossed along axis a
// by velocity index k in this step (A16).
struct Shift {
  int nx, ny, nz, N;
  int delta[3][kMaxN];
};

// CUDA-event phase timers (fks_profile).  Phases: 0 transport, 1 forward, 2 term loop (hot), 3 back.
struct PhaseTimer {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> used[4];
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pool;
  int open_phase = -1;
  void begin(int ph, cudaStream_t st);
  void end(int ph, cudaStream_t st);
};

struct Ctx {
  fks_params p{};
  int N = 0, K = 0, P = 0, T = 0;       // K = N-1 retained modes per axis; T separated terms (+1 loss)
  int n_theta = 0, n_phi = 0;
  double R = 0, Rc = 0, lambda = 0;
  int device = 0;
  int path = FKS_PATH_AUTO;             // resolved path
  // device tables: ab[t][l] = (a_t(l), b_t(l)), t = 0..T, l flattened over K'^3
  double2* d_ab = nullptr;
  double2* d_abT = nullptr;             // fast path: tables restricted to lower-half pencils, per-member blocks
  double2* d_w1 = nullptr;              // fast path: per-team L2-resident ring of z-pass outputs W1
  unsigned* d_ctr = nullptr;            // fast path: per-team produce / consume counters of the W1 ring
  int fast_kernel = 0;                  // fast path term-loop kernel (4 = hot_kernel_v4)
  int fast_variant = 12;                // fast path: CTAs per cell (team size)
  int fast_nteams = 0;                  // fast path: co-resident teams (cells in flight)
  long long* dbg = nullptr;             // debug: hot-kernel phase timestamps (env FKS_PHASE_TIMING)
  long long* prog_host = nullptr;       // debug: mapped pinned per-warp progress words (FKS_DEBUG_PROGRESS)
  long long* prog_dev = nullptr;
  std::vector<double> dirs, w;          // host copy of directions / weights
  std::vector<double> kappa;            // exact power-of-two balance per term (device tables hold a*kappa, b/kappa)
  // twiddles e^{+2 pi i m/M} for M = N and M = P
  double2* d_twN = nullptr;
  double2* d_twP = nullptr;
  // workspace
  void* d_ws = nullptr;
  size_t ws_bytes = 0;
  long long auto_chunk = 0;             // cells per workspace chunk (max_cells_in_flight = 0), computed once
  size_t auto_chunk_per_cell = 0;
  long long ws_cells = 0;
  // host-buffer path staging
  double* d_stage_in = nullptr;
  double* d_stage_out = nullptr;
  long long stage_cells = 0;
  cudaStream_t stage_stream = nullptr;
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;  // host-buffer step pipeline
  // transport state (generic cell)
  bool transport_ready = false;
  bool slab = false;                    // slab decomposition in x (fks_transport_setup_slab): this handle owns
  int nx_glob = 0, x0 = 0, halo = 0;    // global x-planes [x0, x0 + nx) of nx_glob; halo = max |delta_x|
  int nx = 0, ny = 0, nz = 0;
  long long cfl_num = 0, cfl_den = 1;
  std::vector<long long> offsets;       // [3][N] in units of 1/(N*cfl_den) cell
  Shift last{};
  long long launches = 0;
  // stream ordering across calls: every call first waits for the previous call's work on this handle (the
  // workspace, W1 ring and team counters are per handle), whatever stream either ran on
  cudaEvent_t ev_done = nullptr;
  bool ev_pending = false;
  PhaseTimer prof;
  int num_sms = 148;
  int small_ctas = 0;                   // small-N fast path (N = 16, 24): persistent CTAs (SMs x CTAs per SM)
  Shift slab_shift{};                   // fks_step_slab_range: the shift of the step in progress
  bool slab_shift_valid = false;
  double* d_mpart = nullptr;            // fks_step_moments: per-CTA partial moment sums of the last kernel
  size_t mpart_elems = 0;
  // N = 32 chunk pipeline (fast_collision_pipelined): the term-loop kernel of chunk k on a high-priority stream,
  // the forward transform of chunk k+1 and the back transform of chunk k-1 on a low-priority stream, so that they
  // run on the SMs the 12-CTA teams leave idle (148 = 12 x 12 + 4) and fill each launch's tail
  cudaStream_t hot_stream = nullptr, side_stream = nullptr;
  cudaEvent_t ev_pipe[6] = {};          // start, fwd[2], hot[2], end
  bool pipeline = true;                 // FKS_NO_PIPELINE=1 turns it off (A/B)
};

// error plumbing
void set_error(const std::string& msg);
fks_status cuda_status(cudaError_t e, const char* what);

// host quadrature (own implementation; shares nothing with the oracle)
void gauss_legendre(int n, double a, double b, std::vector<double>& x, std::vector<double>& w);

// K1 table builder (tables.cu)
fks_status build_tables(Ctx& c);

// generic path (generic.cu): Q or Euler update for n_cells cells already resident on the device.
//   out = Q(fin)                     if euler == false
//   out = fin + s * Q(fin)           if euler == true  (out may alias fin)
fks_status generic_collision(Ctx& c, const double* fin, double* out, long long n_cells, bool euler, double s,
                             cudaStream_t st);
size_t generic_ws_bytes_per_cell(const Ctx& c);
struct GenericWs { double2* hat; double2* a; double2* b; double* G; };
GenericWs generic_ws(const Ctx& c, long long n);
void generic_forward(Ctx& c, const double* fin, long long n, cudaStream_t st);
void generic_back(Ctx& c, const double* fin, double* out, long long n, bool euler, double s, cudaStream_t st);

// Transport fused into the fast path's first and last kernels: the input of cell j (chunk-local index j - cell0)
// is f*[j][k] = base[(j - delta(k)) mod grid][k], read directly from the untransported f_in.
struct GatherSrc {
  const double* base;   // f_in of the whole grid
  Shift sh;
  long long cell0;      // global index of the chunk's first cell
  int in16;             // base 16-byte aligned
};

// fast path (fast32.cu)
bool fast_available(const Ctx& c);
// U, W (optional, [n_cells][5]): moments of `out` (NEXT-1), fused into the last kernel on the N = 32 path
fks_status fast_collision(Ctx& c, const double* fin, double* out, long long n_cells, bool euler, double s,
                          cudaStream_t st, const GatherSrc* gs = nullptr, double* U = nullptr, double* W = nullptr);
size_t fast_ws_bytes_per_cell(const Ctx& c);
fks_status fast_prepare(Ctx& c);
// N = 32 only: chunks of at most `cap` cells through two workspace slots (the workspace holds 2 cap cells), the
// three phases of consecutive chunks overlapped across streams; all work is ordered after st on entry and st waits
// for all of it on return
struct PipeChunk {
  const double* fin;           // input cells (nullptr with a gather source)
  double* out;
  long long n;
  bool euler; double s;
  bool has_g; GatherSrc g;     // transport fused into the first and last kernels
  double* U; double* W;        // optional moments of `out` ([n][5])
  cudaEvent_t wait_before;     // optional: the chunk's forward transform waits for it (e.g. its input's H2D copy)
  cudaEvent_t record_after;    // optional: recorded after the chunk's back transform (e.g. for its D2H copy)
};
bool fast_pipeline_ok(const Ctx& c);
fks_status fast_collision_pipelined(Ctx& c, const std::vector<PipeChunk>& chunks, long long cap, cudaStream_t st);

// small-N fast path (small.cu): N = 16 / 24 with P = 3N/2; generic forward / back transforms around one
// persistent term-loop kernel (one CTA per (cell, z-class, term chunk) unit)
bool small_available(const Ctx& c);
size_t small_ws_bytes_per_cell(const Ctx& c);
fks_status small_prepare(Ctx& c);
fks_status small_collision(Ctx& c, const double* fin, double* out, long long n_cells, bool euler, double s,
                           cudaStream_t st, const GatherSrc* gs);

// transport gather (transport.cu)
fks_status launch_transport_gather(Ctx& c, const double* fin, double* fout, const Shift& sh, cudaStream_t st,
                                   long long cell0 = 0, long long ncells = -1);

// slab-decomposed transport (transport.cu): x-plane pointer table, plane i = global plane (x0 - halo + i) mod
// nx_glob, each [ny][nz][N^3] (local or peer memory)
constexpr int kMaxPlanes = 1024;
struct PlaneTable {
  const double* p[kMaxPlanes];
};
fks_status launch_transport_gather_slab(Ctx& c, const PlaneTable& tab, double* fout, const Shift& sh, cudaStream_t st,
                                        long long cell0 = 0, long long ncells = -1);

// moments / BGK (macro.cu): mode 0 = moments of fin into U/W, 1 = out = coef (E - fin), 2 = transport by *sh then
// out = f* + coef (E[f*] - f*).  U, W optional ([n_cells][5]).
fks_status launch_macro(Ctx& c, int mode, const double* fin, double* out, double* U, double* W, long long n_cells,
                        double coef, const Shift* sh, cudaStream_t st);
// U, W of n_cells cells from per-cell partial sums mpart[cell][parts][5] (summed in order, times dv^3)
void launch_moments_finish(Ctx& c, const double* mpart, int parts, long long n_cells, double* U, double* W,
                           cudaStream_t st);

}  // namespace fks
