// Thomas recurrences of PAPER.md P187-228 for the Toeplitz interior block of one edge,
// evaluated on the fly (no pivot table):
//
//   a = (c_I + kappa^2 c_L) h_e + 2 c_L / h_e,   b = -c_L / h_e          (P166-185, K2)
//   d'_1 = a,   d'_lo,i = b / d'_{i-1},   d'_i = a - d'_lo,i b           ([eq:thomas_coefficients])
//   forward  y_1 = f_1,  y_i = f_i - d'_lo,i y_{i-1}                      (P217-221)
//   backward w_m = y_m / d'_m,  w_i = (y_i - b w_{i+1}) / d'_i            (P222-228)
//
// One "step" advances the pivot state (inv_prev = 1/d'_{i-1}, 0 before the first node,
// which makes d'_lo,1 = 0 and d'_1 = a) and returns mu = d'_lo,i and 1/d'_i.  The pivots
// depend only on (l, e, i), so a thread carrying ST samples of the same (l, e) computes
// them once for all ST chains.
#pragma once

namespace grf {

struct EdgeCoef {
    double a, b, beta, share;  // beta = -b (end coupling), share = one end's part of A_GG
};

// Local operator of edge e at node l: c_I M_e + c_L (kappa^2 M_e + G_e), M_e lumped (mass = 0:
// h per interior node, h/2 per end, P137-145) or consistent (mass = 1: 2h/3 diagonal, h/6
// off-diagonal, h/3 per end, P129-136).
__host__ __device__ __forceinline__ EdgeCoef edge_coef(double cI, double cL, double kappa2, double h, int mass = 0) {
    const double mc = cI + kappa2 * cL;
    const double stiff = cL / h;
    if (mass == 0) return EdgeCoef{mc * h + 2.0 * stiff, -stiff, stiff, mc * h * 0.5 + stiff};
    const double b = mc * (h / 6.0) - stiff;
    return EdgeCoef{mc * (2.0 * h / 3.0) + 2.0 * stiff, b, -b, mc * (h / 3.0) + stiff};
}

// advance: given inv_prev = 1/d'_{i-1} (0 at i = 1) return mu_i = b / d'_{i-1} and 1/d'_i
__device__ __forceinline__ double thomas_step(const EdgeCoef& c, double& inv_prev) {
    const double mu = c.b * inv_prev;
    const double d = c.a - mu * c.b;
    inv_prev = __drcp_rn(d);
    return mu;
}

}  // namespace grf
