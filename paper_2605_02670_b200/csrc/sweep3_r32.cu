// Warp-specialised recover kernel instances (sweep3_impl.cuh): K5, sample tile 32, TL = 1..7.
#include "sweep3_impl.cuh"

namespace grf {
namespace sweep3 {
cudaError_t launch_r32(int tl, sweep::Args a, cudaStream_t st) {
    switch (tl) {
        case 1: return launch<1>(a, st);
        case 2: return launch<2>(a, st);
        case 3: return launch<3>(a, st);
        case 4: return launch<4>(a, st);
        case 5: return launch<5>(a, st);
        case 6: return launch<6>(a, st);
        case 7: return launch<7>(a, st);
        default: return cudaErrorInvalidValue;
    }
}
}  // namespace sweep3
}  // namespace grf
