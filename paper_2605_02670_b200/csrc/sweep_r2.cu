// Sweep kernel instances (sweep_impl.cuh): K5 recover, sample mapping V2, node tiles TL = 1..10.
#include "sweep_impl.cuh"

namespace grf {
namespace sweep {
cudaError_t launch_r2(int tl, Args a, cudaStream_t st) { return launch_v<true, 2>(tl, a, st); }
}  // namespace sweep
}  // namespace grf
