// Fast path placeholder: the fused N = 32 kernels are added in a later commit.
#include "fks_internal.cuh"
namespace fks {
bool fast_available(const Ctx&) { return false; }
size_t fast_ws_bytes_per_cell(const Ctx&) { return 0; }
fks_status fast_prepare(Ctx&) { return FKS_ERR_UNSUPPORTED; }
fks_status fast_collision(Ctx&, const double*, double*, long long, bool, double, cudaStream_t) {
  set_error("fast path not built");
  return FKS_ERR_UNSUPPORTED;
}
}  // namespace fks
