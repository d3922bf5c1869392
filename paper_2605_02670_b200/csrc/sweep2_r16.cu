// Warp-specialised sweep kernel instances (sweep2_impl.cuh): K5 recover, sample tile 16 (2 samples
// per lane), node tiles TL = 1..7 (one file per instance family so nvcc compiles them in parallel).
#include "sweep2_impl.cuh"

namespace grf {
namespace sweep2 {
cudaError_t launch_r16(int tl, sweep::Args a, cudaStream_t st) { return launch_tl<true, 2>(tl, a, st); }
}  // namespace sweep2
}  // namespace grf
