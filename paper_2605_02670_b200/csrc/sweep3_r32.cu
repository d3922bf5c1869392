// Warp-specialised recover kernel instances (sweep3_impl.cuh): K5, sample tile 32, TL = 1..7.
#include "sweep3_impl.cuh"

namespace grf {
namespace sweep3 {
cudaError_t launch_r32(int tl, sweep::Args a, cudaStream_t st) { return launch_tl(tl, a, st); }
}  // namespace sweep3
}  // namespace grf
