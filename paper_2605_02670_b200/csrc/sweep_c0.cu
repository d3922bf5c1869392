// Sweep kernel instances (sweep_impl.cuh): K3 condense, sample mapping V0, node tiles TL = 1..7.
#include "sweep_impl.cuh"

namespace grf {
namespace sweep {
cudaError_t launch_c0(int tl, Args a, cudaStream_t st) { return launch_v<false, 0>(tl, a, st); }
}  // namespace sweep
}  // namespace grf
