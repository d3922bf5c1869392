// Warp-specialised condense kernel instances (sweep3_impl.cuh): K3, sample tile 32, TL = 1..7.
#include "sweep3_impl.cuh"

namespace grf {
namespace sweep3 {
cudaError_t launch_c32(int tl, sweep::Args a, cudaStream_t st) {
    switch (tl) {
        case 1: return launch_c<1>(a, st);
        case 2: return launch_c<2>(a, st);
        case 3: return launch_c<3>(a, st);
        case 4: return launch_c<4>(a, st);
        case 5: return launch_c<5>(a, st);
        case 6: return launch_c<6>(a, st);
        case 7: return launch_c<7>(a, st);
        default: return cudaErrorInvalidValue;
    }
}
}  // namespace sweep3
}  // namespace grf
