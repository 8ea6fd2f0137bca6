// Tiled 3D half-step kernels (placeholder until the z-marching kernel lands).
#include "hlf_internal.cuh"

namespace hlfk {
bool tiled3d_supported(int) { return false; }
int launch_half_tiled3d(int, HalfKind, const HalfParams&, cudaStream_t) { return -1; }
}  // namespace hlfk
