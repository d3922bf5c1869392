// K3 condense instances of the sweep kernel (sweep_impl.cuh), one per node tile TL.
#include "sweep_impl.cuh"

namespace grf {
namespace sweep {

cudaError_t condense_tl(int tl, Args a, cudaStream_t st) {
    switch (tl) {
        case 1: return launch_tl<1, false>(a, st);
        case 2: return launch_tl<2, false>(a, st);
        case 3: return launch_tl<3, false>(a, st);
        case 4: return launch_tl<4, false>(a, st);
        case 5: return launch_tl<5, false>(a, st);
        case 6: return launch_tl<6, false>(a, st);
        case 7: return launch_tl<7, false>(a, st);
        case 8: return launch_tl<8, false>(a, st);
        case 9: return launch_tl<9, false>(a, st);
        case 10: return launch_tl<10, false>(a, st);
        case 11: return launch_tl<11, false>(a, st);
        case 12: return launch_tl<12, false>(a, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace sweep
}  // namespace grf
