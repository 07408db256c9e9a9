// Fast path for N = 32 (P = 48): the term loop (rows a3-a5 of DESIGN.md §2) as ONE persistent sm_100a kernel.
//
// Every pruned transform is z(p) = sum_{l=-15..15} Z(l) e^{2 pi i l p/48} (pruned to the retained
// modes K' of A9), computed per output class r (p = 3q + r) as a radix-3 DIF combine of the 31 inputs followed
// by a 16-point radix-4x4 FFT held in registers (fft_dev.cuh).  The kernel itself is described above
// namespace v4 below; forward / back transforms are in xform32.cu.
#include <cooperative_groups.h>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include "fks_internal.cuh"
#include "fft_dev.cuh"

namespace fks {
namespace f32 {

constexpr int N = 32, K = 31, P = 48;
constexpr int NPEN = K * K;           // 961 (lx, ly) pencils

// ---- mbarrier + TMA bulk copies (global -> this CTA's shared memory) ----------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
               "r"(bytes) : "memory");
}
// Waiting warps are suspended by the hardware (try_wait with a suspend-time hint) until the phase completes: a
// back-off with __nanosleep over-slept by up to its last interval on every hand-off of the term loop's chains.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  uint32_t done = 0;
  unsigned spins = 0;
  while (true) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(a), "r"(parity), "r"(20000u) : "memory");
    if (done) break;
    if (++spins > (1u << 20)) asm volatile("trap;");  // never hang the GPU on a byte-count bug
  }
}
// arrive (release, CTA scope) on a barrier initialised with count 1
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
                 "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}

constexpr int W1_BUF = P * NPEN;  // complex elements per buffer (738 KB)
constexpr int LHN = K * (NPEN / 2 + 1);  // lower-half block layout: 14911 complex per cell / per term

// ======================================================================================================
// v4: decoupled warp roles.  Teams of TM = 12 CTAs per cell, ONE CTA per SM; member k owns the z-planes
// pz in [4k, 4k+4) and ~1/12 of the lower-half (lx, ly) pencils (with their mirrors (-lx, -ly)).  Per term t:
//   * 4 Z warps: products Z = (a_t + i b_t) f^ of the member's pencils (tables from L2, f^ staged once per cell
//     by TMA), then the z-pass class tasks, whose output W1(lx, ly, pz) goes to an NB-deep, L2-resident team
//     ring; published with per-buffer produce counters (zcnt), consumers acknowledge with ycnt.
//   * 6 Y warps (2 plane pairs g x 3 output classes c): TMA-copy the pair's two W1 planes, y-pass class c of
//     both planes (lanes = lx) into the class-c slot.
//   * 6 X warps (g, c): park their 32 rows (2 planes x 16 py of class c) in TMEM once, free the slot, run the
//     three px classes from TMEM and accumulate G(p) += Re z Im z in TMEM (the balanced tables make this
//     A_t B_t); G is written to HBM once per cell.
// All hand-offs are counters (shared memory inside the CTA, global across the team) or mbarriers; see
// DESIGN.md §5 for the measured variants behind this shape.
// ======================================================================================================
namespace v4 {
constexpr int TM = 12;                        // CTAs (members) per team = per cell
constexpr int PLN = P / TM;                   // 4 z-planes per member
constexpr int NB = 4;                         // W1 team buffers (Z warps run ahead by < NB terms)
// 16 warps: 6 X + 6 Y (two plane pairs) + 4 Z, <= 128 registers per thread
constexpr int GW = 6;                         // warps per YX group
constexpr int NYX = 2 * GW, NZW = 4;          // YX warps (2 groups of GW), Z warps
constexpr int NTHR = 32 * (NYX + NZW);        // 288
constexpr int NZT = 32 * NZW;                 // Z threads
constexpr int MAXH = 41;                      // max staged pencils per member (481 / 12 rounded up)
constexpr int ZSLOT = 96;                     // Z task slots per output class (>= 41 + 41)
constexpr int YB = 16 * K;                    // complex elements of one Y class buffer [16 rows][31]
constexpr int W1IN_B = NPEN * 16;             // 15376 B: one W1 plane
constexpr int YBUF_B = YB * 16;               // 7936 B
constexpr int NYSLOT = 3;                     // Y class slots per plane (one per class: Y(c) never waits for X(c'))
constexpr int PLANE_B = W1IN_B + NYSLOT * YBUF_B;  // per owned plane
constexpr int ZBLK_B = K * MAXH * 16;         // 20336 B
constexpr int OFF_Z = PLN * PLANE_B;          // 124992
constexpr int SMEM_B = OFF_Z + 3 * ZBLK_B;    // Z: products (2) + the cell's f^ block (tables are read from L2)
constexpr int CTR_STRIDE = 256;               // counter words per team (one 128-B line per counter)
// Synchronisation (exact because buffer b = tg % NB is refilled only after all consumers of its previous
// generation acknowledged it):  W1(tg) is complete when zcnt[b] == TM (tg / NB + 1);  buffer b may be
// overwritten with W1(tg) when ycnt[b] == 2 TM (tg / NB)  (2 YX groups per member).

struct Args {
  const double2* fhatT;  // [cell][LHN], 12 blocks
  const double2* tabT;   // [t][LHN], 12 blocks
  double* G;             // [cell][px][pz/2][py][pz%2]: pairs of z-rows interleaved (the back transform packs them)
  double2* W1;           // [team][NB][P][NPEN]
  unsigned* ctr;         // [team][CTR_STRIDE]: per W1 buffer b: zcnt at 32 b, ycnt at 32 (NB + b) (zeroed)
  long long n_cells;
  int T1;
  int nteams;
  long long* dbg;        // optional per-phase clock64 stamps (tools/phase_timing.py); nullptr in production
};

// Phase accounting (instrumented build variant only, tools/phase_timing_v4.py): lane 0 of the sampled warps adds
// the clock64 time of each phase of every term of one steady-state cell (the third of its team) into pt_acc[i] and
// writes the sums when that cell is done.
#ifdef FKS_V4_PHASE_TIMING
#define PT_DECL long long pt_acc[6] = {0, 0, 0, 0, 0, 0}; long long pt_last = clock64();
#define PT(i) do { const long long pt_n = clock64(); pt_acc[i] += pt_n - pt_last; pt_last = pt_n; } while (0)
#define PT_FLUSH(sel, off) do { if ((sel) && A.dbg) for (int pt_i = 0; pt_i < 6; pt_i++) \
    A.dbg[(long long)blockIdx.x * 128 + (off) + pt_i] = pt_acc[pt_i]; } while (0)
// pins a transform's results before a stamp, so that the stamp does not fall inside the transform
#define PT_HOLD(u) do { for (int pt_i = 0; pt_i < 16; pt_i += 2) \
    asm volatile("" : "+d"(u[pt_i].x), "+d"(u[pt_i].y), "+d"(u[pt_i + 1].x), "+d"(u[pt_i + 1].y) :: "memory"); } while (0)
#else
#define PT_HOLD(u) do { } while (0)
#define PT_DECL
#define PT(i) do { } while (0)
#define PT_FLUSH(sel, off) do { } while (0)
#endif

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
#ifndef FKS_POLL_NS
#define FKS_POLL_NS 2048
#endif
// Team counters are polled with relaxed loads and acquired once when the target is seen: an acquire load at GPU
// scope compiles to LDG.STRONG.GPU + CCTL.IVALL, and invalidating the SM's L1 on every poll iteration evicted the
// other warps' cached table loads and spill lines.  The interval is long (2 us): the waits are rare, and a shorter
// interval measured slower (acquire polling: 128 ns 122.2 ms, 2 us 120.0 ms; relaxed: 128 ns 121.1, 512 ns 119.8,
// 2 us 119.1 ms per 8640-cell c3 collision).
__device__ __forceinline__ void poll_ge(const unsigned* p, unsigned target) {
  unsigned spins = 0;
  while (ld_relaxed(p) < target) {
    __nanosleep(FKS_POLL_NS);
    if (++spins > (1u << 25)) asm volatile("trap;");  // never hang the GPU on a counting bug
  }
  (void)ld_acquire(p);
}
// Counter updates use fence.sc + atomicAdd: red.release.gpu (MEMBAR.ALL.GPU + RED) measured 4 % slower on the
// c3 collision (124.3 vs 119.1 ms per 8640 cells, profiles/r02_experiments.txt).
__device__ __forceinline__ int vload(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ void nbar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

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
}

// Inputs of a pruned length-48 inverse transform: modes l = -15..15 stored at base[(l + 15) * ld]; transform
// index i = l mod 48 (16..32 absent).
struct InK {
  const double2* base; int ld;
  __device__ __forceinline__ bool nz(int i) const { return i <= 15 || i >= 33; }
  __device__ __forceinline__ double2 operator()(int i) const { return base[(i <= 15 ? i + 15 : i - 33) * ld]; }
};

// Pruned inverse transform of one output class r (runtime, warp-uniform): z(3q + r) = sum_{l=-15..15} Z(l)
// e^{2 pi i l (3q + r)/48}, inputs Z(l) at base[(l + 15) * ld].  Two forms (fft_dev.cuh):
//   xform48_gt  Good-Thomas form (Y and Z warps): no inter-stage twiddles, the 16-point stage in tangent form, one
//               code path for the three classes; slot k2 ends in u[qslot(k2)] and holds z(3 pfa_q(r, k2) + r).  The
//               Z warps store slot k2 of class r to the "virtual" W1 plane v = 16 r + k2 and the Y warps to row k2
//               of their class slot; the Y and X passes do not care which pz / py a plane or row holds, so only the
//               G write-out maps them back (pz = pfa_p(v), py = pfa_p(16 c + xq)).
//   DIF         radix-3 decimation-in-frequency combine with the twiddles w48^{rm}, then FFT16; z(3q + r) ends in
//               u[qslot(q)].  The X warps (inlined, inputs from TMEM): there the Good-Thomas form measured slower.
// The choice per role is set by the instruction cache as much as by the FP64 count: the hot loops of the three roles
// share it and sit at its edge (profiles/r02_experiments.txt r2ae-r2ap).  ONE instance per warp role
// keeps the kernel's hot code small (templated per-class copies thrashed the cache: ncu no_instruction stalls).
__device__ __forceinline__ void xform48_gt(const double2* base, int ld, int r, double2 (&u)[16]) {
  // one code path for every class: class 0 is the same combine with the rotation w = 1 (the Z code is 1.1 KB smaller
  // than with a separate class-0 loop, which measured 0.4 % faster despite the extra FP64 of the class-0 tasks: the
  // kernel's hot code sits at the edge of the instruction cache)
  const double cr = (r == 0) ? 1.0 : -0.5;
  const double sg = (r == 0) ? 0.0 : ((r == 1) ? 0.86602540378443864676 : -0.86602540378443864676);
  u[0] = base[15 * ld];
#pragma unroll
  for (int m = 1; m < 16; m++) u[fftd::pfa_n2(m)] = fftd::pfa_combine(m, base[(m + 15) * ld], base[(m - 1) * ld], cr, sg);
  fftd::fft16i(u);
}
// transform index p of the Good-Thomas slot k2 of class r, v = 16 r + k2 (the Z warps' virtual W1 plane v)
__device__ __forceinline__ int pfa_p(int v) { return 3 * fftd::pfa_q(v >> 4, v & 15) + (v >> 4); }

__device__ __forceinline__ void tmem_ld16_async(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void g_accumulate(uint32_t tcol, const double2 (&u)[16]) {
  uint32_t gw[32];
  tmem_ld32(tcol, gw);
#pragma unroll
  for (int q = 0; q < 16; q++) {
    const double2 z = u[fftd::qslot(q)];
    const double acc = fma(z.x, z.y, __hiloint2double((int)gw[2 * q + 1], (int)gw[2 * q]));
    gw[2 * q] = (uint32_t)__double2loint(acc);
    gw[2 * q + 1] = (uint32_t)__double2hiint(acc);
  }
  tmem_st32(tcol, gw);
}

__global__ void __launch_bounds__(NTHR, 1) hot_kernel_v4(Args A) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t tmem_base_sh;
  __shared__ __align__(8) uint64_t bar_w1[2];
  __shared__ __align__(8) uint64_t bar_full[2][3], bar_empty[2][3];  // Y(g,c) -> X(g,c) slot hand-offs
  __shared__ __align__(8) uint64_t bar_tab, bar_fh;
  // YX groups: per-group completion counters (Y -> X per class, X -> Y slot release)
  __shared__ int s_yall[2], s_w1iss[2];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int team = blockIdx.x / TM, k = blockIdx.x - (blockIdx.x / TM) * TM;
  constexpr int NLOW = NPEN / 2 + 1;
  const int h0 = (k * NLOW) / TM, h1 = ((k + 1) * NLOW) / TM;
  const int nh = h1 - h0;
  const int nmir = (h1 == NLOW) ? nh - 1 : nh;
  double2* W1t = A.W1 + (long long)team * NB * W1_BUF;
  unsigned* zcnt = A.ctr + (long long)team * CTR_STRIDE;  // + 32 b
  unsigned* ycnt = zcnt + 32 * NB;                         // + 32 b
  // 32-bit loop state (a launch covers one workspace chunk: far fewer than 2^31 cell-terms per team); 64-bit
  // counters spilled to local memory in the YX warps and their reloads stalled the term loop
  const int ncells = (int)A.n_cells;
  const int ncell_team = (team < ncells) ? (ncells - 1 - team) / A.nteams + 1 : 0;
  const int total_tg = ncell_team * A.T1;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                 ::"r"((uint32_t)__cvta_generic_to_shared(&tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&bar_w1[0]);
    mbar_init(&bar_w1[1]);
    for (int i = 0; i < 6; i++) { mbar_init(&bar_full[0][0] + i); mbar_init(&bar_empty[0][0] + i); }
    mbar_init(&bar_tab);
    mbar_init(&bar_fh);
    s_yall[0] = s_yall[1] = 0;
    s_w1iss[0] = s_w1iss[1] = 0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tmem_base_sh;

  if (warp < NYX) {
    // --------------------------------- YX warps, X rows parked in TMEM -------------------------------------
    // 6 X warps (one per group and row class c; warps 0..5 -> (g,c) = (0,0) (0,1) (0,2) (1,2) (1,0) (1,1), lane
    // quarters 0,1,2,3,0,1) and 6 Y warps (6..11 -> (g, c) = (w-6)/3, (w-6)%3).  Per term t:
    //   Y(g,c): wait W1(t) and slot c free (X(g,c) parked term t-1); class c of the y-pass of both planes
    //           -> slot c; count yc[g][c] = t+1; the last Y warp of the group done with W1(t) prefetches W1(t+1).
    //   X(g,c): wait yc[g][c] = t+1; load its 32 rows of class c once, park them in TMEM (124 columns), free the
    //           slot (xc[g][c] = t+1), then the three px classes from TMEM with G += Re z Im z (3 x 32 columns).
    const bool isx = warp < 6;
    const int g = isx ? ((warp >= 3) ? 1 : 0) : (warp - 6) / 3;
    const int c = isx ? (warp < 3 ? warp : (warp == 3 ? 2 : warp - 4)) : (warp - 6) % 3;
    double2* pb0 = reinterpret_cast<double2*>(smem + (2 * g) * PLANE_B);
    double2* pb1 = reinterpret_cast<double2*>(smem + (2 * g + 1) * PLANE_B);
    double2* in0 = pb0;
    double2* in1 = pb1;
    auto ybuf = [&](int pl, int slot) { return (pl ? pb1 : pb0) + NPEN + slot * YB; };
    const int pz0 = PLN * k + 2 * g;
    const uint32_t tX = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(warp >= 4 && warp < 6 ? 224 : 0);
    const uint32_t tPark = tX + 96u;
    const int xp = lane >> 4, xq = lane & 15;
    auto issue_w1 = [&](int tgi) {
      const double2* src = W1t + (tgi % NB) * (long long)W1_BUF + pz0 * NPEN;
      asm volatile("fence.proxy.async.global;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect(&bar_w1[g], 2u * W1IN_B);
      bulk_g2s(in0, src, W1IN_B, &bar_w1[g]);
      bulk_g2s(in1, src + NPEN, W1IN_B, &bar_w1[g]);
    };
    auto try_issue_w1 = [&](int tz, bool block) {  // lane 0: bulk-copy W1(tz) once per group
      const int sl = g;
      if (tz >= total_tg) return;
      if (vload(&s_w1iss[sl]) > tz) return;
      if (vload(&s_yall[sl]) < 3 * tz) {
        if (!block) return;
        unsigned spins = 0;
        while (vload(&s_yall[sl]) < 3 * tz) { __nanosleep(64); if (++spins > (1u << 26)) asm volatile("trap;"); }
      }
      unsigned* zc = zcnt + 32 * (tz % NB);
      const unsigned target = (unsigned)(TM * (tz / NB + 1));
      if (block) poll_ge(zc, target);
      else if (ld_acquire(zc) < target) return;  // one acquire (a relaxed pre-check cost another L2 round trip)
      if (atomicCAS(&s_w1iss[sl], tz, tz + 1) == tz) issue_w1(tz);
    };
    uint32_t par = 0;
    int tg = 0;
#pragma unroll 1
    for (int cell = team; cell < ncells; cell += A.nteams) {
      PT_DECL
#pragma unroll 1
      for (int t = 0; t < A.T1; t++, tg++) {
        const int T = tg;
        if (!isx) {
          // ---------------- Y warp ----------------
          if (lane == 0 && c == 0) try_issue_w1(tg, true);
          mbar_wait(&bar_w1[g], par);
          if (c == 0 && lane == 0) {
            // this group's copy of W1(tg) has landed (observed through the mbarrier), so the buffer may be
            // refilled: a relaxed count suffices (a fence.sc here cost 2 % of the kernel)
            atomicAdd(ycnt + 32 * (tg % NB), 1u);
          }
          PT(0);  // Y: W1 issue / wait / ack
#pragma unroll 1
          for (int pl = 0; pl < 2; pl++) {
            double2 u[16];
            xform48_gt((pl ? in1 : in0) + (lane < K ? lane : K - 1) * K, 1, c, u);
            PT_HOLD(u);
            PT(1);  // Y: transforms
            // slot c is free once X(g, c) has parked the rows of term t - 1 (waited after the first transform, so
            // that the park overlaps it)
            if (pl == 0 && T > 0) mbar_wait(&bar_empty[g][c], (T - 1) & 1);
            PT(2);  // Y: slot wait
            if (lane < K) {
              double2* ydst = ybuf(pl, c) + lane;
#pragma unroll
              for (int q = 0; q < 16; q++) ydst[q * K] = u[fftd::qslot(q)];
            }
            PT(3);  // Y: stores
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar_full[g][c]);
          if (lane == 0 && atomicAdd(&s_yall[g], 1) + 1 == 3 * (T + 1)) try_issue_w1(tg + 1, false);  // prefetch
          PT(4);  // Y: signal / prefetch
        } else {
          // ---------------- X warp ----------------
          mbar_wait(&bar_full[g][c], T & 1);
          PT(0);  // X: wait for Y
          if (t == 0) {  // first term of the cell: zero the three G blocks
            uint32_t zw[32];
#pragma unroll
            for (int i = 0; i < 32; i++) zw[i] = 0u;
#pragma unroll 1
            for (int rx = 0; rx < 3; rx++) tmem_st32(tX + 32u * rx, zw);
          }
          {  // park the row (31 complex = 124 words) in this lane's TMEM columns, 8 values per store
            const double2* row = ybuf(xp, c) + xq * K;
#pragma unroll
            for (int ch = 0; ch < 4; ch++) {
              uint32_t w[32];
#pragma unroll
              for (int k2 = 0; k2 < 8; k2++) {
                const int i = 8 * ch + k2;
                const double2 v = (i < K) ? row[i] : make_double2(0.0, 0.0);
                w[4 * k2] = (uint32_t)__double2loint(v.x);
                w[4 * k2 + 1] = (uint32_t)__double2hiint(v.x);
                w[4 * k2 + 2] = (uint32_t)__double2loint(v.y);
                w[4 * k2 + 3] = (uint32_t)__double2hiint(v.y);
              }
              tmem_st32(tPark + 32u * ch, w);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar_empty[g][c]);  // the Y slot may be refilled
          PT(1);  // X: park
#pragma unroll 1
          for (int rx = 0; rx < 3; rx++) {
            double2 u[16];
            const double sg = (rx == 1) ? -0.86602540378443864676 : 0.86602540378443864676;
#pragma unroll
            for (int mm = 0; mm < 4; mm++) {
              uint32_t wa[16], wb[16];
              tmem_ld16_async(tPark + 16u * mm, wa);
              tmem_ld16_async(tPark + 64u + 16u * mm, wb);
              tmem_wait_ld();
#pragma unroll
              for (int k2 = 0; k2 < 4; k2++) {
                const int m = 4 * mm + k2 + 1;
                const double2 va = make_double2(__hiloint2double((int)wa[4 * k2 + 1], (int)wa[4 * k2]),
                                                __hiloint2double((int)wa[4 * k2 + 3], (int)wa[4 * k2 + 2]));
                if (mm == 3 && k2 == 3) { u[0] = va; continue; }
                const double2 vb = make_double2(__hiloint2double((int)wb[4 * k2 + 1], (int)wb[4 * k2]),
                                                __hiloint2double((int)wb[4 * k2 + 3], (int)wb[4 * k2 + 2]));
                if (rx == 0) {
                  u[m] = fftd::cadd(vb, va);
                } else {
                  double2 acc;
                  acc.x = fma(-0.5, va.x, vb.x);
                  acc.x = fma(-sg, va.y, acc.x);
                  acc.y = fma(-0.5, va.y, vb.y);
                  acc.y = fma(sg, va.x, acc.y);
                  u[m] = fftd::cmul_s<1>(fftd::c_tw48[rx * m], acc);
                }
              }
            }
            fftd::fft16<1>(u);
            g_accumulate(tX + 32u * rx, u);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          PT(2);  // X: three class tasks
          if (t == A.T1 - 1) {  // G[cell][px = 3q' + rx][pz / 2][py = 3 xq + c][pz % 2]: z-rows interleaved in
                                // pairs; the virtual plane pz0 + xp holds pz = pfa_p(pz0 + xp)
            const int pz = pfa_p(pz0 + xp);
            const int py = pfa_p(16 * c + xq);
            double* Gc = A.G + cell * (long long)(P * P * P) + (long long)(pz >> 1) * (2 * P) + (pz & 1) + 2 * py;
#pragma unroll 1
            for (int rx = 0; rx < 3; rx++) {
              uint32_t gw[32];
              tmem_ld32(tX + 32u * rx, gw);
#pragma unroll
              for (int q = 0; q < 16; q++)
                Gc[(long long)(3 * q + rx) * P * P] =
                    __hiloint2double((int)gw[2 * q + 1], (int)gw[2 * q]);
            }
          }
        }
        PT(3);  // X: G write-out (last term) / Y: -
        par ^= 1;
      }
      PT_FLUSH(lane == 0 && (warp == 6 || warp == 7 || warp == 0) && cell == team + 2 * A.nteams,
               warp == 0 ? 8 : (warp == 6 ? 0 : 32));
    }
  } else {
    // ---------------------------------------------- Z warps -----------------------------------------------
    const int zt = tid - 32 * NYX;  // 0..NZT-1
    double2* zp = reinterpret_cast<double2*>(smem + OFF_Z);
    double2* zm = reinterpret_cast<double2*>(smem + OFF_Z + ZBLK_B);
    double2* fh = reinterpret_cast<double2*>(smem + OFF_Z + 2 * ZBLK_B);  // the cell's f^ block (TMA, per cell)
    const uint32_t fblk = (uint32_t)(K * nh) * 16u;
    auto issue_fh = [&](int cl) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect(&bar_fh, fblk);
      bulk_g2s(fh, A.fhatT + cl * (long long)LHN + K * h0, fblk, &bar_fh);
    };
    if (zt == 0 && ncell_team > 0) issue_fh(team);
    uint32_t par_fh = 0;
    int tg = 0;
#pragma unroll 1
    for (int cell = team; cell < ncells; cell += A.nteams) {
      mbar_wait(&bar_fh, par_fh);
      par_fh ^= 1;
      PT_DECL
#pragma unroll 1
      for (int t = 0; t < A.T1; t++, tg++) {
        const double2* tb = A.tabT + (long long)t * LHN + K * h0;     // the member's table block (L2)
        // Warp 12 publishes W1(tg - 1) (fence + team counter) and waits for the buffer of W1(tg) to be free while
        // warps 13-15 form the products, so neither the store drain nor the poll sits on the Z warps' chain.
        if (zt < 32) {
          if (zt == 0) {
            if (tg >= 1) {
              __threadfence();
              atomicAdd(zcnt + 32 * ((tg - 1) % NB), 1u);
            }
            if (tg >= NB) poll_ge(ycnt + 32 * (tg % NB), (unsigned)(2 * TM * (tg / NB)));  // buffer free
          }
          __syncwarp();
        } else {
          // products: Z = (a + ib) f^ for the staged pencils, and for their mirrors (-lx,-ly): (a + ib) conj(f^)
          // at the reversed lz (a, b even; f real).  Element pairs {i, 30 - i} of pencil j, e = i * nh + j; i = e / nh
          // by multiply-high (exact: e nh < 2^32); every table load of a thread is issued before the first product
          constexpr int NPT = NZT - 32;                       // product threads
          constexpr int ZIT = (16 * MAXH + NPT - 1) / NPT;
          const int zq = zt - 32;
          const unsigned mdiv = 0xffffffffu / (unsigned)nh + 1u;
          const double2* __restrict__ fr = fh;  // f^ block in shared memory
          const double2* __restrict__ tr = tb;
          double2* __restrict__ pw = zp;
          double2* __restrict__ mw = zm;
          const int ne = 16 * nh;
          double2 f1[ZIT], a1[ZIT], f2[ZIT], a2[ZIT];
          int o1[ZIT], o2[ZIT];
#pragma unroll
          for (int u = 0; u < ZIT; u++) {
            const int e = min(zq + u * NPT, ne - 1);
            const int i = (int)__umulhi((unsigned)e, mdiv), j = e - i * nh;
            o1[u] = i * nh + j;
            o2[u] = (30 - i) * nh + j;
            a1[u] = __ldg(tr + o1[u]);
            a2[u] = __ldg(tr + o2[u]);
          }
#pragma unroll
          for (int u = 0; u < ZIT; u++) {
            f1[u] = fr[o1[u]];  // shared memory
            f2[u] = fr[o2[u]];
            if (zq + u * NPT < ne) {
              pw[o1[u]] = make_double2(fma(a1[u].x, f1[u].x, -a1[u].y * f1[u].y), fma(a1[u].x, f1[u].y, a1[u].y * f1[u].x));
              pw[o2[u]] = make_double2(fma(a2[u].x, f2[u].x, -a2[u].y * f2[u].y), fma(a2[u].x, f2[u].y, a2[u].y * f2[u].x));
              mw[o1[u]] = make_double2(fma(a2[u].x, f2[u].x, a2[u].y * f2[u].y), fma(-a2[u].x, f2[u].y, a2[u].y * f2[u].x));
              mw[o2[u]] = make_double2(fma(a1[u].x, f1[u].x, a1[u].y * f1[u].y), fma(-a1[u].x, f1[u].y, a1[u].y * f1[u].x));
            }
          }
        }
        PT(0);  // Z: products (warps 13-15) / publication + ring poll (warp 12)
        nbar(3, NZT);  // products complete, W1(tg - 1) published, W1(tg)'s buffer free
        if (zt == 0 && t == A.T1 - 1 && cell + A.nteams < ncells) issue_fh(cell + A.nteams);
        PT(1);  // Z: barrier
        double2* W1b = W1t + (tg % NB) * (long long)W1_BUF;
        {  // 4 Z warps: single class tasks tau = r * na + j, 2 rounds of 128 threads cover 3 na <= 246
          const int na = nh + nmir;
#pragma unroll 1
          for (int kk = zt; kk < 2 * NZT; kk += NZT) {
            if (kk - lane >= 3 * na) break;  // no active lane in this warp (warp-uniform)
            const bool act = kk < 3 * na;
            const int kc = act ? kk : 0;
            const int r = kc / na, j = kc - r * na;
            const bool mir = j >= nh;
            const int jj = mir ? j - nh : j;
            double2 u[16];
            xform48_gt((mir ? zm : zp) + jj, nh, r, u);
            if (act) {
              const int pp = mir ? (NPEN - 1) - (h0 + jj) : h0 + jj;
              // one 64-bit base per task, the plane offsets q NPEN as immediates (an int index per store cost five
              // address instructions each)
              double2* dst = W1b + (16 * r * NPEN + pp);
#pragma unroll
              for (int q = 0; q < 16; q++) dst[q * NPEN] = u[fftd::qslot(q)];  // virtual plane 16 r + q
            }
          }
        }
        nbar(3, NZT);
        PT(2);  // Z: class tasks + stores + barrier
      }
      PT_FLUSH((zt & 31) == 0 && zt < 64 && cell == team + 2 * A.nteams, zt == 0 ? 24 : 16);
    }
    if (zt == 0 && tg > 0) {  // publish the last term
      __threadfence();
      atomicAdd(zcnt + 32 * ((tg - 1) % NB), 1u);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}
}  // namespace v4

}  // namespace f32

bool fast_available(const Ctx& c) { return (c.N == 32 && c.P == 48) || small_available(c); }

size_t xform32_ws_bytes_per_cell();
cudaError_t xform32_prepare();
void xform32_tables_lh(const double2* ab, double2* abL, int T1, int nb);
void xform32_forward(Ctx& c, const double* fin, double2* fhT, double2* scratch, long long n, int nb, cudaStream_t st,
                     const GatherSrc* gs);
void xform32_back(Ctx& c, const double* G, double2* scratch_a, double2* scratch_b, const double* fin, double* out,
                  long long n, bool euler, double s, cudaStream_t st, const GatherSrc* gs, double* mpart);

size_t fast_ws_bytes_per_cell(const Ctx& c) {
  return c.N == 32 ? xform32_ws_bytes_per_cell() : small_ws_bytes_per_cell(c);
}

fks_status fast_prepare(Ctx& c) {
  if (c.N != 32) return small_prepare(c);
  using namespace f32;
  cudaError_t e = xform32_prepare();
  if (e == cudaSuccess) e = fftd::fill_twiddles();
  if (e != cudaSuccess) return cuda_status(e, "fast constants");
  int per_sm = 0;
  e = cudaFuncSetAttribute(v4::hot_kernel_v4, cudaFuncAttributeMaxDynamicSharedMemorySize, v4::SMEM_B);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, v4::hot_kernel_v4, v4::NTHR, v4::SMEM_B);
  if (e != cudaSuccess) return cuda_status(e, "hot kernel attributes");
  if (per_sm < 1) { set_error("hot kernel does not fit on one SM"); return FKS_ERR_UNSUPPORTED; }
  c.fast_kernel = 4;
  c.fast_variant = v4::TM;
  c.pipeline = std::getenv("FKS_NO_PIPELINE") == nullptr;
  c.fast_nteams = c.num_sms / v4::TM;
  if (c.fast_nteams < 1) { set_error("fewer SMs than one team"); return FKS_ERR_UNSUPPORTED; }
  // two counter sets: the chunk pipeline zeroes the set of launch k + 2 on the side stream while launch k + 1 runs
  e = cudaMalloc(&c.d_ctr, 2 * (size_t)c.fast_nteams * v4::CTR_STRIDE * sizeof(unsigned));
  if (e != cudaSuccess) { cudaGetLastError(); return cuda_status(e, "team counters"); }
  const size_t w1_elems = (size_t)c.fast_nteams * v4::NB * W1_BUF;
  const size_t n = (size_t)(c.T + 1) * LHN;
  e = cudaMalloc(&c.d_abT, n * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc(&c.d_w1, w1_elems * sizeof(double2));
  if (e != cudaSuccess) { cudaGetLastError(); return cuda_status(e, "fast path allocation"); }
  xform32_tables_lh(c.d_ab, c.d_abT, c.T + 1, c.fast_variant);
  c.launches++;
  return cuda_status(cudaDeviceSynchronize(), "fast prepare");
}

namespace {
// One workspace chunk of `cap` cells: f^T [cap][K^3] complex | scratch [cap][P*K*16] complex | G [cap][P^3] fp64
// (the back transform reuses f^T as its second scratch buffer).
struct Slot {
  double2* fhT; double2* scratch; double* G;
};
Slot slot_at(void* base, long long cap) {
  using namespace f32;
  Slot sl;
  sl.fhT = reinterpret_cast<double2*>(base);
  sl.scratch = sl.fhT + cap * K * NPEN;
  sl.G = reinterpret_cast<double*>(sl.scratch + cap * (long long)P * K * 16);
  return sl;
}

size_t ctr_set_bytes(const Ctx& c) { return (size_t)c.fast_nteams * f32::v4::CTR_STRIDE * sizeof(unsigned); }

// term-loop launch over the counter set `set`; zero_ctr: zero the set on `st` first (the pipeline zeroes it ahead on
// the side stream, so that nothing but the launch itself sits between two term-loop launches on the hot stream)
fks_status hot_launch(Ctx& c, const Slot& sl, long long n, cudaStream_t st, int set = 0, bool zero_ctr = true) {
  using namespace f32;
  const long long nt = std::min<long long>(c.fast_nteams, n);
  unsigned* ctr = c.d_ctr + (size_t)set * (ctr_set_bytes(c) / sizeof(unsigned));
  v4::Args A{sl.fhT, c.d_abT, sl.G, c.d_w1, ctr, n, c.T + 1, (int)nt, c.dbg};
  if (zero_ctr) cudaMemsetAsync(ctr, 0, ctr_set_bytes(c), st);
  void* args[] = {&A};
  // cooperative launch: the teams spin on each other's counters, so every CTA must be co-resident
  cudaError_t e = cudaLaunchCooperativeKernel((void*)v4::hot_kernel_v4, dim3((unsigned)(nt * v4::TM)),
                                              dim3(v4::NTHR), args, v4::SMEM_B, st);
  if (e != cudaSuccess) return cuda_status(e, "cooperative hot kernel launch");
  c.launches++;
  return cuda_status(cudaPeekAtLastError(), "fast hot kernel launch");
}

// moment partials of `n` cells (kb3's epilogue, N / 8 per cell)
fks_status ensure_mpart(Ctx& c, long long n) {
  const size_t need = (size_t)n * (f32::N / 8) * 5;
  if (need <= c.mpart_elems) return FKS_OK;
  if (c.d_mpart) cudaFree(c.d_mpart);
  c.d_mpart = nullptr;
  c.mpart_elems = 0;
  cudaError_t e = cudaMalloc(&c.d_mpart, need * sizeof(double));
  if (e != cudaSuccess) { cudaGetLastError(); return cuda_status(e, "moment partials"); }
  c.mpart_elems = need;
  return FKS_OK;
}

void back_chunk(Ctx& c, const Slot& sl, const double* fin, double* out, long long n, bool euler, double s,
                cudaStream_t st, const GatherSrc* gs, double* U, double* W) {
  double* mpart = (U || W) ? c.d_mpart : nullptr;  // moments of the step's output, reduced in kb3's epilogue
  xform32_back(c, sl.G, sl.scratch, sl.fhT, fin, out, n, euler, s, st, gs, mpart);
  if (mpart) launch_moments_finish(c, mpart, f32::N / 8, n, U, W, st);
}

// Cells [o, o + m) of a pipelined chunk: the transform kernels index their buffers cell-major, each with its own
// per-cell stride (f / out N^3, F2 and E1 N K H, H2 P K H complex, f^ LHN complex, G P^3, moment partials (N/8) 5).
void fwd_range(Ctx& c, const Slot& sl, const PipeChunk& q, long long o, long long m, cudaStream_t st) {
  using namespace f32;
  constexpr long long H = N / 2;
  GatherSrc g = q.g;
  if (q.has_g) g.cell0 += o;
  xform32_forward(c, q.fin ? q.fin + o * (long long)N * N * N : nullptr, sl.fhT + o * LHN, sl.scratch + o * N * K * H,
                  m, c.fast_variant, st, q.has_g ? &g : nullptr);
}
void back_range(Ctx& c, const Slot& sl, const PipeChunk& q, long long o, long long m, cudaStream_t st) {
  using namespace f32;
  constexpr long long H = N / 2, nv = (long long)N * N * N;
  GatherSrc g = q.g;
  if (q.has_g) g.cell0 += o;
  double* mpart = (q.U || q.W) ? c.d_mpart + o * (N / 8) * 5 : nullptr;
  xform32_back(c, sl.G + o * (long long)P * P * P, sl.scratch + o * P * K * H, sl.fhT + o * N * K * H,
               q.fin ? q.fin + o * nv : nullptr, q.out + o * nv, m, q.euler, q.s, st, q.has_g ? &g : nullptr, mpart);
  if (mpart) launch_moments_finish(c, mpart, N / 8, m, q.U ? q.U + 5 * o : nullptr, q.W ? q.W + 5 * o : nullptr, st);
}
// Side-stream kernels are launched over sub-ranges of at most this many cells: a term-loop launch that becomes ready
// while a side kernel is running has to wait for SMs that side CTAs keep occupying until that kernel's grid is
// dispatched, so short side grids bound the wait (FKS_PIPE_SUB cells; 0 = whole chunks)
long long pipe_sub_cells() {
  const char* e = std::getenv("FKS_PIPE_SUB");
  return e ? std::atoll(e) : 1024LL;
}
}  // namespace

fks_status fast_collision(Ctx& c, const double* fin, double* out, long long n, bool euler, double s,
                          cudaStream_t st, const GatherSrc* gs, double* U, double* W) {
  if (c.N != 32) {
    fks_status rc = small_collision(c, fin, out, n, euler, s, st, gs);
    if (!rc && (U || W)) rc = launch_macro(c, 0, out, nullptr, U, W, n, 0.0, nullptr, st);  // separate moments pass
    return rc;
  }
  const Slot sl = slot_at(c.d_ws, n);
  if (U || W) {
    fks_status rc = ensure_mpart(c, n);
    if (rc) return rc;
  }
  c.prof.begin(1, st);
  xform32_forward(c, fin, sl.fhT, sl.scratch, n, c.fast_variant, st, gs);
  c.prof.end(1, st);
  c.prof.begin(2, st);
  fks_status rc = hot_launch(c, sl, n, st);
  c.prof.end(2, st);
  if (rc) return rc;
  c.prof.begin(3, st);
  back_chunk(c, sl, fin, out, n, euler, s, st, gs, U, W);
  c.prof.end(3, st);
  return cuda_status(cudaPeekAtLastError(), "fast collision");
}

bool fast_pipeline_ok(const Ctx& c) { return c.N == 32 && c.P == 48 && c.pipeline; }

// Chunks k = 0..nc-1 alternate between two workspace slots.  Stream order (host issue order fwd0, fwd1, then per k:
// hot(k), back(k), fwd(k+2)):
//   hot stream  (highest priority): [wait fwd(k)] hot(k) [record hot(k)]
//   side stream (lowest priority):  fwd(0) fwd(1) back(0) fwd(2) back(1) fwd(3) ... back(nc-1)
// back(k) waits for hot(k); fwd(k+2) reuses slot k % 2 after back(k) on the same stream, and hot(k+2) waits for
// fwd(k+2), so every hazard on a slot is ordered.  The 12-CTA teams of the term-loop kernel occupy 144 of the 148
// SMs; the transforms of the neighbouring chunks run on the other 4 (and on the SMs each team frees at the end of a
// launch), while the priority puts the next term-loop launch's CTAs first whenever SMs free up.  A chunk may name
// an event its forward transform waits for (its input's host copy) and one recorded after its back transform.
fks_status fast_collision_pipelined(Ctx& c, const std::vector<PipeChunk>& ck, long long cap, cudaStream_t st) {
  using namespace f32;
  cudaError_t e = cudaSuccess;
  if (!c.hot_stream) {
    int lo = 0, hi = 0;
    e = cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (std::getenv("FKS_PIPE_NOPRIO")) hi = lo;  // experiment: both streams at the default priority
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&c.hot_stream, cudaStreamNonBlocking, hi);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&c.side_stream, cudaStreamNonBlocking, lo);
    for (int i = 0; i < 6 && e == cudaSuccess; i++) e = cudaEventCreateWithFlags(&c.ev_pipe[i], cudaEventDisableTiming);
    if (e != cudaSuccess) { cudaGetLastError(); return cuda_status(e, "pipeline streams"); }
    if (std::getenv("FKS_L2_PERSIST")) {  // experiment: keep the W1 ring L2-resident against the side streams
      int maxwin = 0, maxpers = 0;
      cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, c.device);
      cudaDeviceGetAttribute(&maxpers, cudaDevAttrMaxPersistingL2CacheSize, c.device);
      const size_t w1b = (size_t)c.fast_nteams * v4::NB * W1_BUF * sizeof(double2);
      const size_t win = std::min<size_t>(w1b, (size_t)maxwin);
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min<size_t>(win, (size_t)maxpers));
      cudaStreamAttrValue av{};
      av.accessPolicyWindow.base_ptr = c.d_w1;
      av.accessPolicyWindow.num_bytes = win;
      av.accessPolicyWindow.hitRatio = 1.0f;
      av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cudaStreamSetAttribute(c.hot_stream, cudaStreamAttributeAccessPolicyWindow, &av);
      cudaGetLastError();
      fprintf(stderr, "FKS_L2_PERSIST: window %zu of %zu B, persisting limit %d, max window %d\n", win, w1b, maxpers, maxwin);
    }
  }
  bool mom = false;
  for (const PipeChunk& k : ck) mom = mom || k.U || k.W;
  if (mom) {
    fks_status rc = ensure_mpart(c, cap);
    if (rc) return rc;
  }
  cudaStream_t hs = c.hot_stream, ss = c.side_stream;
  cudaEvent_t ev_start = c.ev_pipe[0], ev_end = c.ev_pipe[5];
  cudaEvent_t* ev_f = c.ev_pipe + 1;
  cudaEvent_t* ev_h = c.ev_pipe + 3;
  const size_t slot_bytes = fast_ws_bytes_per_cell(c) * (size_t)cap;
  Slot sl[2] = {slot_at(c.d_ws, cap), slot_at(static_cast<char*>(c.d_ws) + slot_bytes, cap)};
  const long long nc = (long long)ck.size();
  const long long sub = pipe_sub_cells() > 0 ? pipe_sub_cells() : cap;
  auto fwd = [&](long long k) {
    const PipeChunk& q = ck[k];
    cudaError_t r = q.wait_before ? cudaStreamWaitEvent(ss, q.wait_before, 0) : cudaSuccess;
    if (r != cudaSuccess) return r;
    c.prof.begin(1, ss);
    for (long long o = 0; o < q.n; o += sub) fwd_range(c, sl[k & 1], q, o, std::min(sub, q.n - o), ss);
    c.prof.end(1, ss);
    return cudaEventRecord(ev_f[k & 1], ss);
  };
  const bool ctr_ahead = std::getenv("FKS_PIPE_HOT_MEMSET") == nullptr;
  fks_status hot_rc = FKS_OK;
  e = cudaEventRecord(ev_start, st);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(ss, ev_start, 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(hs, ev_start, 0);
  if (e == cudaSuccess && ctr_ahead) e = cudaMemsetAsync(c.d_ctr, 0, 2 * ctr_set_bytes(c), ss);
  if (e == cudaSuccess) e = fwd(0);
  if (e == cudaSuccess && nc > 1) e = fwd(1);
  for (long long k = 0; k < nc && e == cudaSuccess; k++) {
    const PipeChunk& q = ck[k];
    e = cudaStreamWaitEvent(hs, ev_f[k & 1], 0);
    if (e != cudaSuccess) break;
    c.prof.begin(2, hs);
    fks_status rc = hot_launch(c, sl[k & 1], q.n, hs, (int)(k & 1), !ctr_ahead);
    c.prof.end(2, hs);
    if (rc) { hot_rc = rc; break; }
    e = cudaEventRecord(ev_h[k & 1], hs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ss, ev_h[k & 1], 0);
    if (e != cudaSuccess) break;
    c.prof.begin(3, ss);
    for (long long o = 0; o < q.n; o += sub) back_range(c, sl[k & 1], q, o, std::min(sub, q.n - o), ss);
    c.prof.end(3, ss);
    if (q.record_after) e = cudaEventRecord(q.record_after, ss);
    // counter set k % 2 is free (launch k is done: back k waited for it); launch k + 2 waits for fwd(k + 2) below
    if (e == cudaSuccess && ctr_ahead && k + 2 < nc)
      e = cudaMemsetAsync(c.d_ctr + (size_t)(k & 1) * (ctr_set_bytes(c) / sizeof(unsigned)), 0, ctr_set_bytes(c), ss);
    if (e == cudaSuccess && k + 2 < nc) e = fwd(k + 2);
  }
  // join: the side stream's last work (back(nc-1)) follows the last term-loop launch; st waits for both streams
  // (also after an error part-way, so that no work enqueued here outlives the call's ordering on st)
  const cudaError_t e_join = e;
  if (e_join != cudaSuccess) cudaGetLastError();
  cudaError_t ej = cudaEventRecord(ev_end, ss);
  if (ej == cudaSuccess) ej = cudaStreamWaitEvent(st, ev_end, 0);
  if (ej == cudaSuccess) ej = cudaEventRecord(ev_end, hs);
  if (ej == cudaSuccess) ej = cudaStreamWaitEvent(st, ev_end, 0);
  if (hot_rc) return hot_rc;
  if (e_join != cudaSuccess) return cuda_status(e_join, "collision pipeline");
  if (ej != cudaSuccess) { cudaGetLastError(); return cuda_status(ej, "collision pipeline join"); }
  return cuda_status(cudaPeekAtLastError(), "fast collision pipeline");
}

}  // namespace fks
