// K5: exact FKS transport as a gather (reading A16).
//   f_out[j][k] = f_in[(j - delta(k)) mod (nx, ny, nz)][k],  delta(k) = (delta_x[kx], delta_y[ky], delta_z[kz])
// The whole-cell shifts come from the host-side generic-cell bookkeeping (runtime.cu) and are passed by value.
// A bit-exact permutation: every element is copied, never combined.
#include "fks_internal.cuh"

namespace fks {

__global__ void __launch_bounds__(256) transport_gather_kernel(const double* __restrict__ fin,
                                                               double* __restrict__ fout, Shift sh) {
  const int N = sh.N;
  const long long nv = (long long)N * N * N;
  const long long total = (long long)sh.nx * sh.ny * sh.nz * nv;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long k = idx % nv, j = idx / nv;
    const int kx = (int)(k / (N * N)), ky = (int)((k / N) % N), kz = (int)(k % N);
    const int jz = (int)(j % sh.nz), jy = (int)((j / sh.nz) % sh.ny);
    const long long jx = j / ((long long)sh.nz * sh.ny);
    long long sx = (jx - sh.delta[0][kx]) % sh.nx; if (sx < 0) sx += sh.nx;
    int sy = (jy - sh.delta[1][ky]) % sh.ny; if (sy < 0) sy += sh.ny;
    int sz = (jz - sh.delta[2][kz]) % sh.nz; if (sz < 0) sz += sh.nz;
    const long long src = (sx * sh.ny + sy) * sh.nz + sz;
    fout[idx] = __ldg(&fin[src * nv + k]);
  }
}

fks_status launch_transport_gather(Ctx& c, const double* fin, double* fout, const Shift& sh, cudaStream_t st) {
  long long total = (long long)sh.nx * sh.ny * sh.nz * c.N * c.N * c.N;
  long long blocks = (total + 255) / 256;
  if (blocks > (long long)c.num_sms * 32) blocks = (long long)c.num_sms * 32;
  transport_gather_kernel<<<(unsigned)blocks, 256, 0, st>>>(fin, fout, sh);
  c.launches++;
  return cuda_status(cudaPeekAtLastError(), "transport gather");
}

}  // namespace fks
