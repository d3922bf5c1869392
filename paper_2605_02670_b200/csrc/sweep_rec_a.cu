// K5 recover instances of the sweep kernel (sweep_impl.cuh), node tiles TL = 1..6.
#include "sweep_impl.cuh"

namespace grf {
namespace sweep {

cudaError_t recover_tl_a(int tl, Args a, cudaStream_t st) {
    switch (tl) {
        case 1: return launch_tl<1, true>(a, st);
        case 2: return launch_tl<2, true>(a, st);
        case 3: return launch_tl<3, true>(a, st);
        case 4: return launch_tl<4, true>(a, st);
        case 5: return launch_tl<5, true>(a, st);
        case 6: return launch_tl<6, true>(a, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace sweep
}  // namespace grf
