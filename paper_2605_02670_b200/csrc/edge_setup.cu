// K2: per-(quadrature node, edge) setup  (PAPER.md P166-195, P204-213, P298).
//
// Local operator A^{(l,e)} = c_I M^{(e)} + c_L (kappa^2 M^{(e)} + G^{(e)})  (P168-179 with
// SURVEY §8c Q3/Q7).  With lumped mass and a uniform mesh on the edge the interior block
// is Toeplitz tridiagonal:
//     a = (c_I + kappa^2 c_L) h_e + 2 c_L / h_e,    b = -c_L / h_e,
// each end carries share = (c_I + kappa^2 c_L) h_e / 2 + c_L / h_e of A_GG, and couples to
// its adjacent interior node with coefficient b (A_GI, P185).
//
// Thomas factorisation of A_II (P187-194 [eq:thomas_coefficients], thomas.cuh):
//     d'_1 = a,  d'_lo,i = b / d'_{i-1},  d'_i = a - d'_lo,i b
// K3/K5 (sweep_impl.cuh) use them through two node-minor tables [(toff_e + t) * Lp + l]
// (one set of rows per class of edges with identical (m_e, h_e), written by its representative)
// (row padded to the sweep tiling Lp >= L with zeros, which makes padded nodes inert):
//     mu_t = d'_lo,t = b / d'_{t-1} (mu_1 = 0),  g_t = 1 / (d'_t + d'_{m+1-t} - a)
// (g_t is the diagonal of A_II^{-1}; see sweep_impl.cuh for the twisted-factorisation use).
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
#include "thomas.cuh"

namespace grf {
namespace {

__global__ void edge_setup_kernel(DevGraph g, int32_t L, int32_t Lp, const double* __restrict__ cIt,
                                  const double* __restrict__ cLt, double kappa2, int32_t mass, double* __restrict__ mu_t,
                                  double* __restrict__ gam_t, double4* __restrict__ sig) {
    const int e = blockIdx.x;
    const double h = g.h[e];
    const int m = g.m[e];
    // the class representative writes the shared table rows; every edge computes its Schur block
    const bool rep = g.tab_rep[e] != 0;
    double* tmu = mu_t + g.toff[e] * Lp;
    double* tgam = gam_t + g.toff[e] * Lp;
    if (rep) {
        for (int l = L + threadIdx.x; l < Lp; l += blockDim.x) {  // padded nodes: inert zeros
            for (int t = 0; t < m; ++t) tmu[(int64_t)t * Lp + l] = tgam[(int64_t)t * Lp + l] = 0.0;
        }
    }
    for (int l = threadIdx.x; l < L; l += blockDim.x) {
        const double cI = cIt[l], cL = cLt[l];
        const EdgeCoef c = edge_coef(cI, cL, kappa2, h, mass);
        const double share = c.share;
        double sd, so;
        if (m == 0) {
            sd = share;
            so = c.b;
        } else {
            // pivots d'_t (stored temporarily in the g table) and multipliers mu_t
            double inv = 0.0;
            double prod = 1.0;  // prod_{t=1}^{m-1} (-mu_t) = prod_{i<m} (-b / d'_i)
            for (int t = 0; t < m; ++t) {
                const double mu = thomas_step(c, inv);
                if (rep) {
                    tmu[(int64_t)t * Lp + l] = mu;
                    tgam[(int64_t)t * Lp + l] = c.a - mu * c.b;  // d'_t, the same expression thomas_step inverted
                }
                if (t > 0) prod *= -mu;
            }
            // twisted-factorisation diagonal g_t = (A_II^{-1})_tt = 1 / (d'_t + d'_{m+1-t} - a), computed in
            // mirrored pairs (t, m-1-t) so the in-place overwrite of the pivots is safe
            for (int t = 0; rep && t <= (m - 1) / 2; ++t) {
                const int tm = m - 1 - t;
                const double gv = 1.0 / (tgam[(int64_t)t * Lp + l] + tgam[(int64_t)tm * Lp + l] - c.a);
                tgam[(int64_t)t * Lp + l] = gv;
                tgam[(int64_t)tm * Lp + l] = gv;
            }
            const double b2 = c.b * c.b;
            sd = share - b2 * inv;          // (A_II^{-1})_11 = 1 / d'_m
            so = -b2 * (prod * inv);        // (A_II^{-1})_1m
        }
        const double det = sd * sd - so * so;
        sig[(int64_t)l * g.E + e] = make_double4(sd, so, sd / det, -so / det);
    }
    // correction node (K5's interior steps, sweep_impl.cuh "body_mid"): the padded slot l = L gets
    // mu = 0 and g_t = -G_t / 2 with G_t = sum_{l<L} g_t for the interior rows 1 <= t <= m-2 (0 on
    // the end rows), so its chains carry the noise itself and its two contributions remove G_i W_i
    // once from every interior position.  With several node rounds the slot lies in the last one
    // and corrects the sum over all of them (the rounds only partition the sum over l).
    if (rep && L < Lp && m > 2) {
        __syncthreads();  // all g rows of this class written
        for (int t = 1 + threadIdx.x; t <= m - 2; t += blockDim.x) {
            double G = 0.0;
            for (int l = 0; l < L; ++l) G += tgam[(int64_t)t * Lp + l];
            tgam[(int64_t)t * Lp + L] = -0.5 * G;
        }
    }
}

}  // namespace

void launch_edge_setup(const DevGraph& g, DevPlan& p, cudaStream_t st) {
    int threads = ((p.L + 31) / 32) * 32;
    if (threads > 256) threads = 256;
    edge_setup_kernel<<<g.E, threads, 0, st>>>(g, p.L, p.Lp, p.cI, p.cL, p.kappa * p.kappa, p.mass, p.mu, p.gam,
                                               reinterpret_cast<double4*>(p.sig));
}

}  // namespace grf
