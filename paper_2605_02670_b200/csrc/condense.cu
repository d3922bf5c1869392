// K3: condensed vertex right-hand side  (PAPER.md P197-239).
//
//     g_v^{(l,s)} = W_v - sum_{(e,end) at v} (A_GI^{(l,e)} A_II^{(l,e)}^{-1} W_{I,e})_end
//                 = W_v + (c_L/h_e) * w_end,     w = A_II^{-1} W_{I,e}   (A_GI = b = -c_L/h_e)
//
// w_end is the end value of the Thomas solve (P215-228).  Only the end facing v is
// needed, so each (vertex, incident edge end) runs ONE forward elimination toward v:
//   v = edge_v (right end, needs w_m):  y_1 = W_1, y_i = W_i - (b/d'_{i-1}) y_{i-1}, w_m = y_m / d'_m
//   v = edge_u (left end,  needs w_1):  the same recurrence over the reversed interior
//     (A_II is persymmetric Toeplitz, so its reversal has the same pivots d'_i).
// Every interior DOF is swept once per edge end = twice per (l, s, e), 2 FMA-chains total.
//
// Mapping: CTA = (vertex v, tile of samples), thread = quadrature node l (lanes read the
// node-minor pivot table coalesced; W is a warp-broadcast).  Each thread carries ST
// samples at once (ST independent chains share every pivot load).  The incident ends are
// summed in CSR order -> deterministic.  Output g[(s*V + v)*L + l] (coalesced over l).
#include "grf_internal.h"

namespace grf {
namespace {

constexpr int ST = 4;

__global__ void __launch_bounds__(256) condense_kernel(DevGraph g, int32_t L, const double* __restrict__ cLt,
                                                       const double* __restrict__ invd, int64_t S,
                                                       const double* __restrict__ W, double* __restrict__ gu) {
    const int v = blockIdx.x;
    const int64_t s0 = (int64_t)blockIdx.y * ST;
    const int ns = (int)((S - s0) < ST ? (S - s0) : ST);
    const int k0 = g.inc_ptr[v], k1 = g.inc_ptr[v + 1];
    for (int l = threadIdx.x; l < L; l += blockDim.x) {
        const double cL = cLt[l];
        double acc[ST];
#pragma unroll
        for (int j = 0; j < ST; ++j) acc[j] = (j < ns) ? W[(s0 + j) * g.N + g.NI + v] : 0.0;
        for (int k = k0; k < k1; ++k) {
            const int code = g.inc[k];
            const int e = code >> 1;
            const int m = g.m[e];
            if (m == 0) continue;
            const double h = g.h[e];
            const double b = -cL / h;
            const int64_t off = g.off[e];
            const double* Wp[ST];
#pragma unroll
            for (int j = 0; j < ST; ++j) Wp[j] = W + (s0 + (j < ns ? j : 0)) * g.N + off;
            // walk direction: toward v.  right end: i = 0..m-1; left end: i = m-1..0
            const bool right = (code & 1);
            const int64_t istep = right ? 1 : -1;
            int64_t idx = right ? 0 : (m - 1);
            double y[ST];
#pragma unroll
            for (int j = 0; j < ST; ++j) y[j] = __ldg(Wp[j] + idx);
            const double* piv = invd + off * L + l;
            for (int i = 1; i < m; ++i) {
                const double mu = b * __ldg(piv + (int64_t)(i - 1) * L);
                idx += istep;
#pragma unroll
                for (int j = 0; j < ST; ++j) y[j] = __ldg(Wp[j] + idx) - mu * y[j];
            }
            const double idm = __ldg(piv + (int64_t)(m - 1) * L);
            const double beta = cL / h;
#pragma unroll
            for (int j = 0; j < ST; ++j) acc[j] += beta * (y[j] * idm);
        }
#pragma unroll
        for (int j = 0; j < ST; ++j)
            if (j < ns) gu[((s0 + j) * g.V + v) * L + l] = acc[j];
    }
}

}  // namespace

void launch_condense(const DevGraph& g, const DevPlan& p, int64_t n_samples, const double* W, double* gu,
                     cudaStream_t st) {
    int threads = ((p.L + 31) / 32) * 32;
    if (threads > 256) threads = 256;
    dim3 grid(g.V, (unsigned)((n_samples + ST - 1) / ST));
    condense_kernel<<<grid, threads, 0, st>>>(g, p.L, p.cL, p.invd, n_samples, W, gu);
}

}  // namespace grf
