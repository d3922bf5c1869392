// K3 / K5 host-side dispatch: plan node tiling (Lp, TL, rounds) and the launch of the
// sweep kernel instance for it (kernel and mapping: sweep_impl.cuh).
#include <cstdlib>

#include "grf_internal.h"
#include "sweep_impl.cuh"

namespace grf {
namespace sweep {
cudaError_t launch_c0(int tl, Args a, cudaStream_t st);
cudaError_t launch_r0k(int tl, Args a, cudaStream_t st);
cudaError_t launch_r1k(int tl, Args a, cudaStream_t st);
cudaError_t launch_r2k(int tl, Args a, cudaStream_t st);
}  // namespace sweep
namespace sweep2 {
cudaError_t launch_c16(int tl, sweep::Args a, cudaStream_t st);
cudaError_t launch_c32(int tl, sweep::Args a, cudaStream_t st);
cudaError_t launch_r16(int tl, sweep::Args a, cudaStream_t st);
cudaError_t launch_r32(int tl, sweep::Args a, cudaStream_t st);
}  // namespace sweep2
namespace sweep3 {
cudaError_t launch_r32(int tl, sweep::Args a, cudaStream_t st);
cudaError_t launch_c32(int tl, sweep::Args a, cudaStream_t st);
}  // namespace sweep3

namespace {
constexpr int TL_MAX = 7;  // nodes per lane of the sweep kernels (register tile)

sweep::Args make_args(const DevGraph& g, const DevPlan& p, int64_t S, const double* W, double* out,
                      const double* uG, int32_t* counter) {
    sweep::Args a{};
    a.g = g;
    a.L = p.L;
    a.Lp = p.Lp;
    a.rounds = p.rounds;
    a.cL = p.cL;
    a.cI = p.cI;
    a.kappa2 = p.kappa * p.kappa;
    a.mass = p.mass;
    a.mu = p.mu;
    a.gam = p.gam;
    a.S = S;
    a.W = W;
    a.out = out;
    a.uG = uG;
    a.counter = counter;
    a.nk = 1;  // plan_tiling leaves slot L free: edge_setup.cu writes the correction node there
    static const int ablate = [] {
        const char* v = getenv("GRF_ABLATE");
        return v ? atoi(v) : 0;
    }();
    a.ablate = ablate;
    return a;
}
}  // namespace

int device_sms() {
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (cache[dev] <= 0) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = n > 0 ? n : 148;
    }
    return cache[dev];
}

int32_t sample_tile_log2(int64_t S) {
    switch (sweep::variant_for(S)) {
        case sweep::V2: return 5;
        case sweep::V1: return 4;
        default: return 0;
    }
}

// L nodes plus the correction node (slot L) in rounds of 32 x TL nodes, TL <= TL_MAX
void plan_tiling(int32_t L, int32_t* Lp, int32_t* tl, int32_t* rounds) {
    const int q0 = (L + 1 + sweep::NLT - 1) / sweep::NLT;
    const int r = (q0 + TL_MAX - 1) / TL_MAX;
    const int t = (q0 + r - 1) / r;
    *rounds = r;
    *tl = t;
    *Lp = sweep::NLT * t * r;
}

cudaError_t launch_condense(const DevGraph& g, const DevPlan& p, int64_t n_samples, const double* W, double* ends,
                            int32_t* counter, cudaStream_t st) {
    const sweep::Args a = make_args(g, p, n_samples, W, ends, nullptr, counter);
    switch (sweep::variant_for(n_samples)) {
        case sweep::V2:  // sweep3's condense is the default; sweep2's stays selectable (GRF_ABLATE bit 128)
            return a.ablate & 128 ? sweep2::launch_c32(p.TL, a, st) : sweep3::launch_c32(p.TL, a, st);
        case sweep::V1: return sweep2::launch_c16(p.TL, a, st);
        default: return sweep::launch_c0(p.TL, a, st);
    }
}

bool recover_out_write_only(const DevGraph& g, const DevPlan& p, int64_t n_samples) {
    sweep::Args a = make_args(g, p, n_samples, nullptr, nullptr, nullptr, nullptr);
    if (a.ablate) return false;
    int32_t fits = 0;
    a.fits_out = &fits;
    cudaError_t e = cudaSuccess;
    switch (sweep::variant_for(n_samples)) {
        case sweep::V2: e = sweep3::launch_r32(p.TL, a, nullptr); break;
        case sweep::V1: e = sweep::launch_r1k(p.TL, a, nullptr); break;
        default: e = sweep::launch_r0k(p.TL, a, nullptr); break;
    }
    return e == cudaSuccess && fits != 0;
}

cudaError_t launch_recover(const DevGraph& g, const DevPlan& p, int64_t n_samples, const double* W, double* u,
                           const double* uG, int32_t* counter, cudaStream_t st) {
    const sweep::Args a = make_args(g, p, n_samples, W, u, uG, counter);
    switch (sweep::variant_for(n_samples)) {
        case sweep::V2:
            // sweep3 (warp-specialised around the sweep_impl register tile) is the default; the
            // earlier designs stay selectable for design studies (GRF_ABLATE bits 8, 16)
            if (a.ablate & 8) return sweep2::launch_r32(p.TL, a, st);
            if (a.ablate & 16) return sweep::launch_r2k(p.TL, a, st);
            return sweep3::launch_r32(p.TL, a, st);
        case sweep::V1: return a.ablate & 8 ? sweep2::launch_r16(p.TL, a, st) : sweep::launch_r1k(p.TL, a, st);
        default: return sweep::launch_r0k(p.TL, a, st);
    }
}

}  // namespace grf

namespace grf {
namespace {
// vertex values of the sample (P313-324): u_v = sum_l u_G^{(l)}(v); one thread per (s, v),
// a sequential sum over l in node order
__global__ void vertex_sum_kernel(int64_t S, int32_t V, int64_t N, int64_t NI, int32_t L, int32_t csl,
                                  const double* __restrict__ uG, double* __restrict__ u) {
    // thread per (tile, v, sample-in-tile): consecutive threads read consecutive samples
    const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int cs = 1 << csl;
    const int64_t tiles = (S + cs - 1) >> csl;
    if (x >= tiles * V * cs) return;
    const int si = (int)(x & (cs - 1));
    const int64_t tv = x >> csl;
    const int64_t tile = tv / V, v = tv - tile * V;
    const int64_t s = (tile << csl) + si;
    if (s >= S) return;
    const double* src = uG + ((tile * V + v) * (int64_t)L << csl) + si;
    double acc = 0.0;
    for (int l = 0; l < L; ++l) acc += src[(int64_t)l << csl];
    u[s * N + NI + v] = acc;
}
}  // namespace

cudaError_t launch_vertex_sum(const DevGraph& g, const DevPlan& p, int64_t n_samples, const double* uG, double* u,
                              cudaStream_t st) {
    const int32_t csl = sample_tile_log2(n_samples);
    const int64_t tiles = (n_samples + (1 << csl) - 1) >> csl;
    const int64_t threads = (tiles * g.V) << csl;
    vertex_sum_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(n_samples, g.V, g.N, g.NI, p.L, csl, uG, u);
    return cudaGetLastError();
}

}  // namespace grf
