// Sweep kernel instances (sweep_impl.cuh): K5 recover with the correction-node interior steps,
// sample mapping V0, node tiles TL = 1..7.
#include "sweep_impl.cuh"

namespace grf {
namespace sweep {
cudaError_t launch_r0k(int tl, Args a, cudaStream_t st) { return launch_v<true, 0, true>(tl, a, st); }
}  // namespace sweep
}  // namespace grf
