// K5 recover instances of the sweep kernel (sweep_impl.cuh), node tiles TL = 7..12.
#include "sweep_impl.cuh"

namespace grf {
namespace sweep {

cudaError_t recover_tl_b(int tl, Args a, cudaStream_t st) {
    switch (tl) {
        case 7: return launch_tl<7, true>(a, st);
        case 8: return launch_tl<8, true>(a, st);
        case 9: return launch_tl<9, true>(a, st);
        case 10: return launch_tl<10, true>(a, st);
        case 11: return launch_tl<11, true>(a, st);
        case 12: return launch_tl<12, true>(a, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace sweep
}  // namespace grf
