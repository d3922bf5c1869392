// Sweep kernel instances (sweep_impl.cuh): K5 recover, sample mapping V2, node tiles TL = 1..10.
// Plans with a correction node (Args::nk, edge_setup.cu) take the NK instances of sweep_r2k.cu.
#include "sweep_impl.cuh"

namespace grf {
namespace sweep {
cudaError_t launch_r2k(int tl, Args a, cudaStream_t st);
cudaError_t launch_r2(int tl, Args a, cudaStream_t st) {
    if (a.nk) return launch_r2k(tl, a, st);
    return launch_v<true, 2, false>(tl, a, st);
}
}  // namespace sweep
}  // namespace grf
