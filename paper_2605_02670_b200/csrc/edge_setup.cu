// K2: per-(quadrature node, edge) setup  (PAPER.md P166-195, P204-213, P298).
//
// Local operator A^{(l,e)} = c_I M^{(e)} + c_L (kappa^2 M^{(e)} + G^{(e)})  (P168-179 with
// SURVEY §8c Q3/Q7).  With lumped mass and a uniform mesh on the edge the interior block
// is Toeplitz tridiagonal:
//     a = (c_I + kappa^2 c_L) h_e + 2 c_L / h_e,    b = -c_L / h_e,
// each end carries share = (c_I + kappa^2 c_L) h_e / 2 + c_L / h_e of A_GG, and couples to
// its adjacent interior node with coefficient b (A_GI, P185).
//
// Thomas factorisation of A_II (P187-194 [eq:thomas_coefficients]):
//     d'_1 = a,  d'_lo,i = b / d'_{i-1},  d'_i = a - d'_lo,i b
// stored as invd[(off_e + i - 1) * L + l] = 1 / d'_i (node-minor: a warp of nodes reads
// one 256-B line per i in K3/K5).
//
// Local Schur complement (P204-213 [eq:local_reduced_schur]):
//     S^{(l,e)} = A_GG - A_GI A_II^{-1} A_IG = [[s_d, s_o], [s_o, s_d]],
//     s_d = share - b^2 (A_II^{-1})_{11},  s_o = -b^2 (A_II^{-1})_{1m}
// where, from the same pivots (forward/back substitution on e_m, P215-228):
//     (A_II^{-1})_{mm} = 1/d'_m = (A_II^{-1})_{11}   (Toeplitz => persymmetric)
//     (A_II^{-1})_{1m} = (1/d'_m) prod_{i<m} (-b / d'_i).
// Edges without interior (m = 0) couple their ends directly: s_d = share, s_o = b.
// The NN preconditioner (P298) needs S_e^{-1} = [[p_d, p_o], [p_o, p_d]],
// p_d = s_d / det, p_o = -s_o / det, det = s_d^2 - s_o^2.
//
// This replaces the paper's per-PCG-iteration Thomas sweeps of the Dirichlet step
// (P253) and of the permuted full-edge Neumann system (P269-292) by these exact 2x2
// blocks: the same numerical vectors (P242 "yields the exact same numerical vector"),
// O(|E|) per PCG iteration instead of O(N).
#include "grf_internal.h"

namespace grf {
namespace {

__global__ void edge_setup_kernel(DevGraph g, int32_t L, const double* __restrict__ cIt,
                                  const double* __restrict__ cLt, double kappa2, double* __restrict__ invd,
                                  double4* __restrict__ sig) {
    const int e = blockIdx.x;
    const double h = g.h[e];
    const int m = g.m[e];
    const int64_t off = g.off[e];
    for (int l = threadIdx.x; l < L; l += blockDim.x) {
        const double cI = cIt[l], cL = cLt[l];
        const double mass = cI + kappa2 * cL;
        const double stiff = cL / h;
        const double a = mass * h + 2.0 * stiff;
        const double b = -stiff;
        const double share = mass * h * 0.5 + stiff;
        double sd, so;
        if (m == 0) {
            sd = share;
            so = b;
        } else {
            double d = a;
            double id = 1.0 / d;
            invd[off * L + l] = id;
            double prod = 1.0;  // prod_{i<m} (-b / d'_i)
            for (int i = 1; i < m; ++i) {
                prod *= -b * id;
                const double lo = b * id;    // d'_lo,i+1 = b / d'_i
                d = a - lo * b;
                id = 1.0 / d;
                invd[(off + i) * L + l] = id;
            }
            const double b2 = b * b;
            sd = share - b2 * id;
            so = -b2 * (prod * id);
        }
        const double det = sd * sd - so * so;
        sig[(int64_t)l * g.E + e] = make_double4(sd, so, sd / det, -so / det);
    }
}

}  // namespace

void launch_edge_setup(const DevGraph& g, DevPlan& p, cudaStream_t st) {
    int threads = ((p.L + 31) / 32) * 32;
    if (threads > 256) threads = 256;
    edge_setup_kernel<<<g.E, threads, 0, st>>>(g, p.L, p.cI, p.cL, p.kappa * p.kappa, p.invd,
                                               reinterpret_cast<double4*>(p.sig));
}

}  // namespace grf
