// K5: interior recovery + quadrature accumulation  (PAPER.md P300-324).
//
//     A_II^{(l,e)} u_I^{(l,e)} = W_{I,e} - A_IG^{(l,e)} u_G^{(l,e)}      (P306-311 [eq:internal_recovery])
// The right-hand side is W_I with its first / last entries raised by (c_L/h_e) u_left /
// u_right (A_IG = b = -c_L/h_e, P310), solved with the cached Thomas pivots (forward
// substitution y_i = f_i - (b/d'_{i-1}) y_{i-1}, back substitution
// w_i = (y_i - b w_{i+1}) / d'_i, P215-228), then u = sum_l u^{(l)} (P313-324).
// Vertex values u_v = sum_l u_G^{(l)}[v] are written by the CTA of the edge end that
// "owns" v (its first incidence), so every output element has exactly one writer.
//
// Mapping (fused over quadrature nodes, nothing per-node goes back to HBM):
//   CTA = (edge e, tile of ST samples), thread = node l, ST chains per thread.
//   Forward sweep over the edge keeps only every C-th y (checkpoints, local memory);
//   the backward sweep walks segments right to left, recomputes the segment's C
//   forward values into registers from its checkpoint, back-substitutes them, and
//   reduces each DOF's value over l (warp shuffles + one smem pass across warps)
//   straight into the output.  The recomputation repeats the identical operations,
//   so the result is bit-identical to a plain Thomas sweep.
// In place: the output array holds W on entry (grf_sample generates W into it) and u
// on exit; a segment is overwritten only after every thread has re-read its W.
#include "grf_internal.h"

namespace grf {
namespace {

constexpr int C = 8;          // segment length (registers per chain)
constexpr int ST = 2;         // samples per thread
constexpr int MAXSEG = 128;   // => interior length <= C * MAXSEG

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void __launch_bounds__(1024) recover_kernel(DevGraph g, int32_t L, const double* __restrict__ cLt,
                                                       const double* __restrict__ invd, int64_t S,
                                                       double* __restrict__ Wu, const double* __restrict__ gu) {
    extern __shared__ double red[];  // [nwarp][ST][C]
    const int e = blockIdx.x;
    const int64_t s0 = (int64_t)blockIdx.y * ST;
    const int ns = (int)((S - s0) < ST ? (S - s0) : ST);
    const int l = threadIdx.x;
    const bool act = l < L;
    const int lc = act ? l : (L - 1);
    const int nwarp = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int V = g.V;
    const int m = g.m[e];
    const int64_t off = g.off[e];
    const double h = g.h[e];
    const int vu = g.eu[e], vv = g.ev[e];
    const double cL = cLt[lc];
    const double beta = cL / h;  // = -b
    const double b = -beta;

    double uL[ST], uR[ST];
    const double* Wrow[ST];
#pragma unroll
    for (int j = 0; j < ST; ++j) {
        const int64_t s = s0 + (j < ns ? j : 0);
        uL[j] = gu[(s * V + vu) * (int64_t)L + lc];
        uR[j] = gu[(s * V + vv) * (int64_t)L + lc];
        Wrow[j] = Wu + s * g.N + off;
    }

    // vertex values owned by this edge: u_v = sum_l u_G^{(l)}[v]
#pragma unroll
    for (int side = 0; side < 2; ++side) {
        const int vert = side ? vv : vu;
        if (g.owner[vert] != 2 * e + side) continue;  // uniform over the block
#pragma unroll
        for (int j = 0; j < ST; ++j) {
            double t = warp_sum(act ? (side ? uR[j] : uL[j]) : 0.0);
            if (lane == 0) red[warp * ST + j] = t;
        }
        __syncthreads();
        if (threadIdx.x < ns) {
            double t = 0.0;
            for (int w = 0; w < nwarp; ++w) t += red[w * ST + threadIdx.x];
            Wu[(s0 + threadIdx.x) * g.N + g.NI + vert] = t;
        }
        __syncthreads();
    }
    if (m == 0) return;

    const double* piv = invd + off * L + lc;
    const int nseg = (m + C - 1) / C;
    double ck[MAXSEG][ST];
    double y[ST];
#pragma unroll
    for (int j = 0; j < ST; ++j) y[j] = 0.0;
    // forward substitution with checkpoints y_{kC}
    for (int k = 0; k < nseg; ++k) {
#pragma unroll
        for (int j = 0; j < ST; ++j) ck[k][j] = y[j];
        const int i0 = k * C;
        const int len = (m - i0) < C ? (m - i0) : C;
        for (int c = 0; c < len; ++c) {
            const int i = i0 + c;
            const double mu = (i == 0) ? 0.0 : b * __ldg(piv + (int64_t)(i - 1) * L);
#pragma unroll
            for (int j = 0; j < ST; ++j) {
                double f = __ldg(Wrow[j] + i);
                if (i == 0) f += beta * uL[j];
                if (i == m - 1) f += beta * uR[j];
                y[j] = f - mu * y[j];
            }
        }
    }
    // backward substitution, segment by segment, right to left
    double wn[ST];
#pragma unroll
    for (int j = 0; j < ST; ++j) wn[j] = 0.0;
    for (int k = nseg - 1; k >= 0; --k) {
        const int i0 = k * C;
        const int len = (m - i0) < C ? (m - i0) : C;
        double ys[C][ST];
        double iv[C];
        double prev_iv = (i0 == 0) ? 0.0 : __ldg(piv + (int64_t)(i0 - 1) * L);
        double yp[ST];
#pragma unroll
        for (int j = 0; j < ST; ++j) yp[j] = ck[k][j];
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (c < len) {
                const int i = i0 + c;
                iv[c] = __ldg(piv + (int64_t)i * L);
                const double mu = (i == 0) ? 0.0 : b * prev_iv;
                prev_iv = iv[c];
#pragma unroll
                for (int j = 0; j < ST; ++j) {
                    double f = __ldg(Wrow[j] + i);
                    if (i == 0) f += beta * uL[j];
                    if (i == m - 1) f += beta * uR[j];
                    ys[c][j] = f - mu * yp[j];
                    yp[j] = ys[c][j];
                }
            }
        }
#pragma unroll
        for (int c = C - 1; c >= 0; --c) {
            if (c < len) {
#pragma unroll
                for (int j = 0; j < ST; ++j) {
                    const double w = (ys[c][j] - b * wn[j]) * iv[c];
                    wn[j] = w;
                    ys[c][j] = w;
                }
            }
        }
        // sum over nodes l
#pragma unroll
        for (int c = 0; c < C; ++c) {
#pragma unroll
            for (int j = 0; j < ST; ++j) {
                const double t = warp_sum((act && c < len) ? ys[c][j] : 0.0);
                if (lane == 0) red[(warp * ST + j) * C + c] = t;
            }
        }
        __syncthreads();
        for (int t = threadIdx.x; t < ns * len; t += blockDim.x) {
            const int j = t / len, c = t - j * len;
            double acc = 0.0;
            for (int w = 0; w < nwarp; ++w) acc += red[(w * ST + j) * C + c];
            Wu[(s0 + j) * g.N + off + i0 + c] = acc;
        }
        __syncthreads();
    }
}

}  // namespace

int32_t recover_max_interior() { return C * MAXSEG; }
int32_t max_nodes_per_block() { return 1024; }

cudaError_t launch_recover(const DevGraph& g, const DevPlan& p, int64_t n_samples, double* Wu, const double* gu,
                           cudaStream_t st) {
    const int threads = ((p.L + 31) / 32) * 32;
    const size_t smem = sizeof(double) * (threads / 32) * ST * C;
    dim3 grid(g.E, (unsigned)((n_samples + ST - 1) / ST));
    recover_kernel<<<grid, threads, smem, st>>>(g, p.L, p.cL, p.invd, n_samples, Wu, gu);
    return cudaGetLastError();
}

}  // namespace grf
