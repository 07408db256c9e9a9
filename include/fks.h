/* fks.h — C ABI of libfks: the hot path of the Fast Kinetic Scheme for the 3D/3D Boltzmann equation
 * (J. Narski, arXiv 1701.01608) on one NVIDIA B200 (sm_100a), fp64.
 *
 * Citations: "P:n" = line n of the paper's PAPER.md; "A<n>" = the readings of garbled or silent passages
 * listed in DESIGN.md §3.  What the calls compute is defined in DESIGN.md §2; in short, per spatial cell j,
 *
 *   f^_l  = N^-3 sum_j f_j e^{-2 pi i l.j/N},   l in K'^3,  K' = {-(N/2-1), ..., N/2-1}
 *   Q^_k  = sum_{l,m in K', l+m=k} beta(l,m) f^_l f^_m,  beta(l,m) = sum_{t=0..T} a_t(l) b_t(m)  (Eq. CF1)
 *   Q_j   = sum_{k in K'} Q^_k e^{2 pi i k.j/N}
 *
 * with the separated Carleman weights a_t, b_t of Appendix A (hard spheres B~ = 1, or Maxwell
 * molecules by a radial split, A6) and the loss term t = 0 (a_0 = 1, b_0 = -sum_{t>=1} a_t b_t).
 *
 * Conventions (all calls):
 *  - Arrays f, Q, f_in, f_out are DEVICE pointers to fp64, owned by the caller, layout [n_cells][N][N][N]
 *    C order (kz fastest); the velocity node (kx,ky,kz) is v = -L + (kx,ky,kz)*2L/N (A13).  Spatial cell
 *    index for transport is (jx*ny + jy)*nz + jz on a periodic nx*ny*nz grid (A21).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream); every call is stream-ordered
 *    and asynchronous unless stated.  No exception crosses the ABI.
 *  - Validation errors return before any launch.  Asynchronous kernel faults surface as FKS_ERR_CUDA on the
 *    next call or on fks_sync.  fks_last_error() returns a thread-local message for the last failure.
 *  - A handle is used from one host thread at a time.  Tables are immutable after init.  Calls on one handle
 *    are serialised in submission order even across streams: each call's stream first waits for the work the
 *    previous call on the handle enqueued (an internal event), because they share the handle's workspace.
 *  - Inputs and outputs must not overlap (checked by pointer range): FKS_ERR_INVALID.
 *  - There is no CPU fallback: without a CUDA device every compute call returns FKS_ERR_CUDA.
 */
#ifndef FKS_H
#define FKS_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fks_ctx fks_ctx;

typedef enum {
  FKS_OK = 0,
  FKS_ERR_INVALID = 1,      /* bad argument, overlapping buffers, host pointer where a device pointer is needed */
  FKS_ERR_UNSUPPORTED = 2,  /* N odd, N < 4, N > 64, P < N or P > 4N, unknown kernel/rule, requested path unavailable */
  FKS_ERR_NOMEM = 3,        /* device allocation failed */
  FKS_ERR_CUDA = 4,         /* launch failure or asynchronous CUDA error (sticky errors stay sticky) */
  FKS_ERR_STATE = 5         /* e.g. fks_transport_step / fks_step before fks_transport_setup */
} fks_status;

typedef enum {
  FKS_KERNEL_HARD_SPHERES = 0,  /* B~ = 1          (B = |u|/4, A4)                 */
  FKS_KERNEL_MAXWELL = 1,       /* B~ = (1/pi)(|x|^2+|y|^2)^(-1/2)  (B = 1/(4 pi); Eq. Btilde_pl, A5) */
  FKS_KERNEL_VHS = 2            /* variable hard spheres B = C_a |u|^a, 0 <= a <= 1:
                                   B~ = 4 C_a (|x|^2+|y|^2)^(-(1-a)/2), radial split as Maxwell molecules (A30) */
} fks_kernel;

typedef enum {
  FKS_QUAD_GL_UNIFORM = 0,  /* default: Gauss-Legendre in cos(theta) x uniform phi on the half sphere (A11) */
  FKS_QUAD_PAPER_RECT = 1   /* (theta_p, phi_q) = (p pi/A1, q pi/A2), weight pi^2/(A1 A2) sin(theta_p) (A2) */
} fks_quad;

typedef enum {
  FKS_PATH_AUTO = 0,        /* fastest instantiated path for (N, P) */
  FKS_PATH_GENERIC = 1,     /* per-axis DFT kernels through device workspace, any even N in [4, 64]     */
  FKS_PATH_FAST = 2         /* fused pruned-FFT kernels (N = 32, P = 48); FKS_ERR_UNSUPPORTED elsewhere */
} fks_path;

typedef struct {
  int N;                        /* velocity points per axis, even, 4..64                                   */
  double L;                     /* half-width of the periodic velocity box [-L, L)^3; support R = lambda*L  */
  int M_angles;                 /* number of half-sphere directions (A12: n_theta = 2^ceil(log2(M)/2))      */
  int M_radial;                 /* Maxwell molecules / VHS: radial GL nodes on [0, R_c] (>= 1); HS: unused */
  int kernel;                   /* fks_kernel                                                              */
  int n_theta, n_phi;           /* 0,0 = derive from M_angles (A12)                                        */
  int quad_rule;                /* fks_quad                                                                */
  int pad;                      /* 0 = P = 3N/2 (default, A10); else explicit P in [N, 4N]: P >= 3N/2-2 is
                                   the exact Galerkin operator, P < 3N/2-2 the aliased collocation operator
                                   (pairs with l+m = k mod P; P = N: classical collocation; generic path)   */
  double cutoff_ratio;          /* Carleman cutoff R_c = ratio*R: 0 (default) or in [1, 1.7071] (A7);
                                   1 = paper-literal; ratios in (0, 1) are rejected (FKS_ERR_INVALID)        */
  int project_mass;             /* 1 = set Q^_0 := 0 exactly (A24); default 0                              */
  long long max_cells_in_flight;/* workspace limit in cells per chunk; 0 = auto.  On the N = 32 path a batch
                                   of more than one chunk uses two chunk slots (2x the workspace) so that the
                                   transforms of neighbouring chunks overlap the term loop (FKS_NO_PIPELINE=1
                                   in the environment at init turns this off)                              */
  int path;                     /* fks_path                                                                */
  double vhs_alpha;             /* FKS_KERNEL_VHS: exponent a in [0, 1]                                    */
  double vhs_C;                 /* FKS_KERNEL_VHS: C_a > 0; 0 = 1/(4 pi) (a = 0 is then Maxwell molecules) */
} fks_params;

/* Precompute the separated-kernel weight tables a_t, b_t (t = 0..T) on the device (A1-A7).
 * T = M_angles (hard spheres) or M_angles*M_radial (Maxwell molecules).  *out receives the handle (owned by
 * the caller; release with fks_destroy).  Defaults: paper-literal cutoff, GL x uniform rule, P = 3N/2. */
fks_status fks_collision_init(fks_ctx** out, int N, double L, int M_angles, int M_radial, int kernel);
fks_status fks_collision_init_ex(fks_ctx** out, const fks_params* p);

/* Q[c] = Q(f[c], f[c]) for c < n_cells (device pointers, [n_cells][N][N][N] fp64).  n_cells = 0: no-op.
 * Q must not overlap f. */
fks_status fks_collision_batch(fks_ctx* h, const double* f, double* Q, long long n_cells, void* stream);

/* Same operation on HOST buffers: chunks of cells (up to 32) are copied in, collided and copied back on three
 * streams so that the copies overlap the compute; returns when Q is written (synchronous).  Bit-identical to
 * fks_collision_batch.  Used for the end-to-end measurement. */
fks_status fks_collision_batch_host(fks_ctx* h, const double* f_host, double* Q_host, long long n_cells);

/* Configure the exact transport (A16): periodic nx*ny*nz cells of width dx, time step
 * dt = (cfl_num/cfl_den)*dx/L (rational CFL c = dt*L/dx), generic-cell offsets reset to 0 (cell centres).
 * cfl_num = 0 makes transport the identity (space-homogeneous runs).  cfl_den >= 1. */
fks_status fks_transport_setup(fks_ctx* h, int nx, int ny, int nz, long long cfl_num, long long cfl_den);

/* One exact transport step: advances the generic-cell offsets (host, O(N)) and gathers
 * f_out[j][k] = f_in[(j - delta(k)) mod (nx,ny,nz)][k] (bit-exact permutation).  f_out must not overlap f_in. */
fks_status fks_transport_step(fks_ctx* h, const double* f_in, double* f_out, void* stream);

/* One FKS time step (Eq. disc_relax; A17, A18): transport, then collision, then explicit
 * Euler: f_out = f* + coll_scale * Q(f*), f* = transported f_in, coll_scale = dt/Kn. */
fks_status fks_step(fks_ctx* h, const double* f_in, double* f_out, double coll_scale, void* stream);

/* fks_step plus the macroscopic moments of the new state (the paper's per-step moment update, Eq. DM_update
 * P:464-493): U[c] = sum_k phi(v_k) f_out[c][k] dv^3, phi = (1, v, |v|^2/2), and
 * W[c] = (rho, u, T), exactly as fks_moments defines them, for every cell c of f_out.  U and W are DEVICE arrays
 * [nx*ny*nz][5] fp64; either may be NULL, not both (FKS_ERR_INVALID); they must not overlap f_in, f_out or each
 * other.  On the N = 32 fast path the sums are reduced inside the step's last kernel (a fixed-order per-CTA
 * reduction, then one tiny kernel per chunk), otherwise by one moments pass over f_out.  f_out is bit-identical
 * to fks_step's; U, W agree with fks_moments(f_out) to rounding (different summation order). */
fks_status fks_step_moments(fks_ctx* h, const double* f_in, double* f_out, double coll_scale, double* U, double* W,
                            void* stream);

/* Host-buffer variant of fks_step (synchronous), for the end-to-end measurement.  The step is pipelined over
 * x-slabs (one plane each, up to 32; env FKS_HOST_SLABS overrides) on three streams: copy-in (wrap-around halo
 * first), transport + collision of each slab as soon as its source planes have landed, copy-out.  Pinned host
 * buffers overlap fully; pageable ones work too.  Bit-identical to fks_step. */
fks_status fks_step_host(fks_ctx* h, const double* f_in_host, double* f_out_host, double coll_scale);

/* Slab decomposition in x for one process per GPU (the paper's MPI FKS).
 * This handle owns the global x-planes [x0, x0 + nx_local) of a periodic nx_global x ny x nz grid; every rank
 * runs the same generic-cell bookkeeping (identical shifts).  Afterwards only the _slab calls below (and the
 * collision calls) are valid on the handle; fks_transport_setup returns it to a single domain. */
fks_status fks_transport_setup_slab(fks_ctx* h, int nx_global, int ny, int nz, int x0, int nx_local,
                                    long long cfl_num, long long cfl_den);

/* Halo width H = an upper bound of max |delta_x| over all steps (ceil(cfl) + 1). */
fks_status fks_slab_halo(const fks_ctx* h, int* halo);

/* Length nx_local + 2H of the `planes` table the _slab calls read (FKS_ERR_STATE before the slab setup). */
fks_status fks_slab_plane_count(const fks_ctx* h, int* n_planes);

/* One transport step of the local cells, gathering across the slab boundary directly from the owner's memory:
 * `planes` is a HOST array of nx_local + 2H DEVICE pointers; planes[i] is global x-plane (x0 - H + i) mod
 * nx_global, laid out [ny][nz][N][N][N] fp64 (this rank's own planes, or a neighbour's mapped through CUDA IPC /
 * peer access: the kernel loads them over NVLink, no separate halo exchange).  f_out: local
 * [nx_local*ny*nz][N^3]; must not overlap any plane.  The caller orders the steps across ranks: a rank may
 * overwrite a buffer only after every rank that reads it finished the previous step (e.g. one barrier per step).
 * Bit-identical to fks_transport_step on the whole grid. */
fks_status fks_transport_step_slab(fks_ctx* h, const double* const* planes, double* f_out, void* stream);

/* Slab variant of fks_step: the gather above, then collision + Euler on the local cells in place in f_out. */
fks_status fks_step_slab(fks_ctx* h, const double* const* planes, double* f_out, double coll_scale, void* stream);

/* Part of a slab step: destination x-planes [lx0, lx1) of this rank (local indices, 0 <= lx0 <= lx1 <= nx_local)
 * with the shift of the current step.  advance = 1 starts a new step (advances the generic cell, as fks_step_slab
 * does); advance = 0 continues it with the same shift (FKS_ERR_STATE if no step was started).  Destination planes
 * [H, nx_local - H) read only this rank's own planes and are never read by a neighbour, so they can run before
 * the inter-rank barrier of the step and the boundary planes after it (the paper's relaxation of interior cells
 * overlapping the exchange).  fks_step_slab = fks_step_slab_range(0, nx_local, advance = 1). */
fks_status fks_step_slab_range(fks_ctx* h, const double* const* planes, double* f_out, double coll_scale, int lx0,
                               int lx1, int advance, void* stream);

/* Macroscopic moments per cell ("ToConservative" / "ToPrimitive"):
 *   U[c] = sum_k phi(v_k) f[c][k] dv^3 = (rho, rho u_x, rho u_y, rho u_z, E),  phi = (1, v, |v|^2/2), dv = 2L/N;
 *   W[c] = (rho, u_x, u_y, u_z, T) with (3/2) rho T = E - rho |u|^2 / 2.
 * U and W are DEVICE arrays [n_cells][5] fp64; either may be NULL (not both).  rho = 0 gives non-finite u, T.
 * Direct sums (the paper's incremental Eq. DM_update gives the same numbers after transport, pin P20). */
fks_status fks_moments(fks_ctx* h, const double* f, double* U, double* W, long long n_cells, void* stream);

/* BGK operator: Q[c] = nu (E[f[c]] - f[c]), E the Maxwellian with f[c]'s (rho, u, T)
 * sampled at the velocity nodes; E = 0 for a cell with rho <= 0 or T <= 0 (A26).  Q must not overlap f. */
fks_status fks_bgk_batch(fks_ctx* h, const double* f, double* Q, double nu, long long n_cells, void* stream);

/* One FKS time step with the BGK operator (Eq. disc_relax): transport (as
 * fks_transport_step, requires fks_transport_setup; advances the generic cell), then explicit Euler
 * f_out = f* + nu_dt (E[f*] - f*), nu_dt = nu * dt.  One fused kernel: f_in is read once and f_out written
 * once.  Optional U, W ([n_cells][5], device, may be NULL) receive the moments of the transported f*
 * (the relaxation keeps them up to the velocity-grid quadrature error, P18/P22). */
fks_status fks_bgk_step(fks_ctx* h, const double* f_in, double* f_out, double nu_dt, double* U, double* W,
                        void* stream);

/* Diagnostics: padded size P, number of separated terms T (the loss term t = 0 is extra), cutoff R_c,
 * lambda = 2/(3+sqrt 2).  Any out pointer may be NULL. */
fks_status fks_get_info(const fks_ctx* h, int* P, int* T, double* R, double* lambda);

/* The path this handle runs (fks_path: FKS_PATH_GENERIC or FKS_PATH_FAST); -1 for a NULL handle. */
int fks_get_path(const fks_ctx* h);

/* Fast-path layout: CTAs per cell and cells processed concurrently by the persistent hot kernel (0, 0 on the
 * generic path).  Either out pointer may be NULL. */
fks_status fks_get_fast_layout(const fks_ctx* h, int* ctas_per_cell, int* concurrent_cells);

/* Test-only: copy the tables to host arrays a_host, b_host [(T+1)][N-1][N-1][N-1], the directions
 * dirs_host [n_dirs][3] and weights w_host [n_dirs] (n_dirs = n_theta*n_phi).  Synchronous. */
fks_status fks_get_tables(const fks_ctx* h, double* a_host, double* b_host, double* dirs_host, double* w_host);

/* Test-only (no device needed): the static per-phase task schedule of the N = 16 / 24 term-loop kernel
 * (csrc/small.cu).  Phases 0..3 = A (Z + X of y-class 2), B (Y of class 0), C (X0 + Y1), D (X1 + Y2).  Writes the
 * warp count, the Z / Y slot counts and the X slot count per y-class, cnt[4][16] (items per warp) and
 * items[4][16][12] (item = type << 5 | slot; type 0 = Z, 1 = Y, 2 = X).  Any out pointer may be NULL.
 * Returns 0, or -1 for another N. */
int fks_small_schedule(int N, int* warps, int* nzs, int* nys, int* nxs, unsigned char* cnt, unsigned char* items);

/* Test-only: the per-axis whole-cell shifts delta[3][N] of the most recent transport step (host). */
fks_status fks_get_last_shift(const fks_ctx* h, int* delta_host);

/* Instrumentation (bench.py): when enabled, CUDA events are recorded on the launch stream around each phase:
 *   0 = transport gather (a1), 1 = forward transform (a2), 2 = term loop / hot kernel (a3-a5),
 *   3 = back transform + write-back / Euler (a6-a7).
 * fks_profile_read synchronises those events and returns, per phase, the summed milliseconds ms[4] and the
 * number of timed launches count[4], then resets the accumulators. */
fks_status fks_profile(fks_ctx* h, int enable);
fks_status fks_profile_read(fks_ctx* h, double* ms, long long* count);

/* Debug: copy up to n entries of the hot-kernel phase timestamp buffer (allocated only when the environment
 * variable FKS_PHASE_TIMING is set at init); returns the number copied (0 when disabled). */
long long fks_debug_timestamps(const fks_ctx* h, long long* host, long long n);

/* Number of kernel launches issued by this handle since creation (instrumentation for the bench). */
long long fks_launch_count(const fks_ctx* h);

/* Synchronise `stream` and report any asynchronous CUDA error. */
fks_status fks_sync(fks_ctx* h, void* stream);

void fks_destroy(fks_ctx* h);
const char* fks_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* FKS_H */
