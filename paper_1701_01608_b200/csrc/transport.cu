// K5: exact FKS transport as a gather (reading A16).
//   f_out[j][k] = f_in[(j - delta(k)) mod (nx, ny, nz)][k],  delta(k) = (delta_x[kx], delta_y[ky], delta_z[kz])
// The whole-cell shifts come from the host-side generic-cell bookkeeping (runtime.cu) and are passed by value.
// A bit-exact permutation: every element is copied, never combined.
#include "fks_internal.cuh"

namespace fks {

// One CTA per destination cell j, 256 threads; thread t handles kz = t % N of velocity rows (kx, ky) taken
// 256/N at a time.  The source cell of every (axis, velocity index) is resolved once per CTA in shared memory
// (no 64-bit division in the copy loop); a warp reads a few contiguous runs (one per distinct delta_z).
__global__ void __launch_bounds__(256) transport_gather_kernel(const double* __restrict__ fin,
                                                               double* __restrict__ fout, Shift sh, long long cell0) {
  __shared__ int sx[kMaxN], sy[kMaxN], sz[kMaxN];
  const int N = sh.N;
  const long long nv = (long long)N * N * N;
  const long long j = cell0 + blockIdx.x;
  const int jz = (int)(j % sh.nz), jy = (int)((j / sh.nz) % sh.ny);
  const int jx = (int)(j / ((long long)sh.nz * sh.ny));
  if (threadIdx.x < N) {
    const int k = threadIdx.x;
    int a = (jx - sh.delta[0][k]) % sh.nx; if (a < 0) a += sh.nx;
    int b = (jy - sh.delta[1][k]) % sh.ny; if (b < 0) b += sh.ny;
    int c = (jz - sh.delta[2][k]) % sh.nz; if (c < 0) c += sh.nz;
    sx[k] = a; sy[k] = b; sz[k] = c;
  }
  __syncthreads();
  const int rows_per_it = 256 / N;
  const int kz = threadIdx.x % N, rr = threadIdx.x / N;
  if (rr >= rows_per_it) return;
  const int czz = sz[kz];
  double* dst = fout + j * nv;
  for (int row = rr; row < N * N; row += rows_per_it) {
    const int kx = row / N, ky = row - (row / N) * N;
    const long long src = ((long long)sx[kx] * sh.ny + sy[ky]) * sh.nz + czz;
    const long long k = (long long)row * N + kz;
    dst[k] = __ldg(&fin[src * nv + k]);
  }
}

fks_status launch_transport_gather(Ctx& c, const double* fin, double* fout, const Shift& sh, cudaStream_t st,
                                   long long cell0, long long ncells) {
  const long long cells = (long long)sh.nx * sh.ny * sh.nz;
  if (ncells < 0) ncells = cells - cell0;  // destination cells [cell0, cell0 + ncells); sources anywhere in fin
  if (ncells <= 0) return FKS_OK;
  if (ncells > 0x7fffffffLL) { set_error("transport: too many cells"); return FKS_ERR_INVALID; }
  transport_gather_kernel<<<(unsigned)ncells, 256, 0, st>>>(fin, fout, sh, cell0);
  c.launches++;
  return cuda_status(cudaPeekAtLastError(), "transport gather");
}

// Slab variant: this rank owns the global x-planes [x0, x0 + nx_loc); the source plane of
// every velocity comes from a pointer table covering [x0 - halo, x0 + nx_loc + halo) (mod nx_glob), so cells near
// the slab edge gather directly from the neighbour's memory (peer loads over NVLink when the table holds peer
// pointers) instead of through a separate halo exchange.  Same copy order and bit-exact result as the
// single-domain gather.
__global__ void __launch_bounds__(256) transport_gather_slab_kernel(const PlaneTable tab, double* __restrict__ fout,
                                                                    Shift sh, int x0, int nx_glob, int halo,
                                                                    long long cell0) {
  __shared__ int sx[kMaxN], sy[kMaxN], sz[kMaxN];
  const int N = sh.N;
  const long long nv = (long long)N * N * N;
  const long long j = cell0 + blockIdx.x;  // local destination cell (jx_loc * ny + jy) * nz + jz
  const int jz = (int)(j % sh.nz), jy = (int)((j / sh.nz) % sh.ny);
  const int jx = x0 + (int)(j / ((long long)sh.nz * sh.ny));  // global plane
  if (threadIdx.x < N) {
    const int k = threadIdx.x;
    // table index of the source plane: ((jx - delta) - (x0 - halo)) mod nx_glob, in [0, nx_loc + 2 halo)
    int a = (jx - sh.delta[0][k] - (x0 - halo)) % nx_glob; if (a < 0) a += nx_glob;
    int b = (jy - sh.delta[1][k]) % sh.ny; if (b < 0) b += sh.ny;
    int c = (jz - sh.delta[2][k]) % sh.nz; if (c < 0) c += sh.nz;
    sx[k] = a; sy[k] = b; sz[k] = c;
  }
  __syncthreads();
  const int rows_per_it = 256 / N;
  const int kz = threadIdx.x % N, rr = threadIdx.x / N;
  if (rr >= rows_per_it) return;
  const int czz = sz[kz];
  double* dst = fout + j * nv;
  for (int row = rr; row < N * N; row += rows_per_it) {
    const int kx = row / N, ky = row - (row / N) * N;
    const double* plane = tab.p[sx[kx]];
    const long long src = (long long)sy[ky] * sh.nz + czz;
    const long long k = (long long)row * N + kz;
    dst[k] = plane[src * nv + k];
  }
}

fks_status launch_transport_gather_slab(Ctx& c, const PlaneTable& tab, double* fout, const Shift& sh, cudaStream_t st,
                                        long long cell0, long long ncells) {
  if (ncells < 0) ncells = (long long)c.nx * c.ny * c.nz - cell0;  // local destination cells [cell0, cell0 + ncells)
  if (ncells <= 0) return FKS_OK;
  if (ncells > 0x7fffffffLL) { set_error("transport: too many cells"); return FKS_ERR_INVALID; }
  transport_gather_slab_kernel<<<(unsigned)ncells, 256, 0, st>>>(tab, fout, sh, c.x0, c.nx_glob, c.halo, cell0);
  c.launches++;
  return cuda_status(cudaPeekAtLastError(), "transport gather (slab)");
}

}  // namespace fks
