// K3 (condense) and K5 (recover + quadrature sum): the per-edge Thomas work of PAPER.md
// P187-239 and P300-324, batched over (quadrature node l) x (sample s) x (edge e).
//
// For one edge, node l and right-hand side f (length m), the interior block
// A_II = tridiag(b, a, b) (Toeplitz) is eliminated from both ends:
//   left  (P217-221):  Y_1 = f_1,  Y_i = f_i - mu_i Y_{i-1},   mu_i = b / d'_{i-1}
//   right (same pivots, A_II persymmetric):  Z_m = f_m,  Z_i = f_i - mu_{m+1-i} Z_{i+1}
// and the Thomas solution is the twisted-factorisation combination of the two sweeps
//   (A_II^{-1} f)_i = g_i (Y_i + Z_i - f_i),   g_i = 1 / (d'_i + d'_{m+1-i} - a)
// (equal, up to rounding, to forward + back substitution P215-228: both are exact
// LU-type eliminations of the same system).  Because Y_i - f_i = -mu_i Y_{i-1}, the
// left sweep contributes kap_i Y_{i-1} (kap_i = -g_i mu_i) and the right sweep g_i Z_i to
// position i: NO intermediate vector has to be stored -- each sweep adds straight into
// the result.  At step t the left chain is at position t and the right chain at m+1-t,
// and both use the same (mu_t, g_t, kap_t) (g is symmetric).
//
//   K3 condense (f = W_I):        w_m = g_m Y_m,  w_1 = g_1 Z_1   -> ends[((s*E+e)*2+end)*L + l]
//   K5 recover  (f = W_I + (c_L/h_e)(u_left e_1 + u_right e_m), P306-311):
//                                 u_i = sum_l g_i (Y_i + Z_i - f_i)  (+ vertex values sum_l u_G)
//
// Mapping: an item = (edge, tile of SL samples), pulled from a longest-edge-first queue.
// lane = (sample, node sub-lane), warp = group of NLW*LL nodes; every thread carries
// NLW nodes x 2 chains in registers.  The per-(l, t) coefficients are staged into shared
// memory IB steps at a time and read as warp broadcasts; per-warp partial sums over the
// thread's nodes are combined across warps through shared memory in fixed order
// (deterministic) and added into the output (first visit writes, second adds).
#include "grf_internal.h"

namespace grf {
namespace {

constexpr int IB = 8;          // steps per staging / reduction block
constexpr int MAXW = 16;       // warps per CTA

struct SweepArgs {
    DevGraph g;
    int32_t L;
    const double* cL;
    const double* mu;   // [(off+t)*L + l]
    const double* gam;
    const double* kap;
    int64_t S;
    const double* W;    // [s*N + dof]
    double* out;        // condense: ends; recover: u [s*N + dof]
    const double* uG;   // recover: [(s*V + v)*L + l]
    WorkQueue wq;
    int32_t nwarps;     // warps per CTA (node groups per round)
};

template <int SL>
struct Lanes {
    static constexpr int LL = 32 / SL;  // node sub-lanes per warp
};

// Shared memory layout (doubles):
//   coef [3][IB][LR]                 staged mu/gam/kap for this round's LR nodes
//   part [2*IB][P][SL+1]             per (row, partial, sample) sums, P = nwarps*LL
template <int NLW, int SL, bool REC>
__global__ void __launch_bounds__(MAXW * 32) sweep_kernel(SweepArgs A) {
    constexpr int LL = Lanes<SL>::LL;
    extern __shared__ double smem[];
    __shared__ int item_sh;
    const DevGraph& g = A.g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sl = lane % SL, ll = lane / SL;
    const int nwarps = A.nwarps;
    const int P = nwarps * LL;
    const int LR = nwarps * NLW * LL;           // nodes per round
    const int L = A.L;
    const int rounds = (L + LR - 1) / LR;
    double* coef = smem;                          // 3*IB*LR
    double* part = smem + 3 * IB * LR;            // 2*IB*P*(SL+1)
    const int64_t N = g.N;
    const int V = g.V;

    for (;;) {
        if (tid == 0) item_sh = atomicAdd(A.wq.counter, 1);
        __syncthreads();
        const int it = item_sh;
        __syncthreads();
        if (it >= A.wq.n_items) break;
        const int e = g.edge_order[it / A.wq.chunks];
        const int64_t s0 = (int64_t)(it % A.wq.chunks) * SL;
        const int64_t s = s0 + sl;
        const bool sact = s < A.S;
        const int64_t sc = sact ? s : (A.S - 1);
        const int m = g.m[e];
        const int64_t off = g.off[e];
        const double h = g.h[e];
        const int vu = g.eu[e], vv = g.ev[e];
        const double* Wrow = A.W + sc * N + off;

        for (int rd = 0; rd < rounds; ++rd) {
            const int lbase = rd * LR + warp * (NLW * LL) + ll;  // node of chain k: lbase + k*LL
            double Y[NLW], Z[NLW];
            // ---------------- recover: vertex values owned by this edge (sum over l of u_G)
            if (REC) {
                const bool ownL = g.owner[vu] == 2 * e, ownR = g.owner[vv] == 2 * e + 1;
                if (ownL || ownR) {
                    double a0 = 0.0, a1 = 0.0;
#pragma unroll
                    for (int k = 0; k < NLW; ++k) {
                        const int l = lbase + k * LL;
                        if (l < L) {
                            a0 += A.uG[(sc * V + vu) * (int64_t)L + l];
                            a1 += A.uG[(sc * V + vv) * (int64_t)L + l];
                        }
                    }
                    const int pidx = warp * LL + ll;
                    part[(0 * P + pidx) * (SL + 1) + sl] = a0;
                    part[(1 * P + pidx) * (SL + 1) + sl] = a1;
                    __syncthreads();
                    for (int o = tid; o < 2 * SL; o += blockDim.x) {
                        const int side = o / SL, j = o % SL;
                        double t = 0.0;
                        for (int p = 0; p < P; ++p) t += part[(side * P + p) * (SL + 1) + j];
                        const int64_t so = s0 + j;
                        if (so < A.S && (side ? ownR : ownL)) {
                            double* dst = A.out + so * N + g.NI + (side ? vv : vu);
                            *dst = rd == 0 ? t : *dst + t;
                        }
                    }
                    __syncthreads();
                }
            }
            if (m == 0) {
                if (!REC) {
#pragma unroll
                    for (int k = 0; k < NLW; ++k) {
                        const int l = lbase + k * LL;
                        if (l < L && sact) {
                            double* o = A.out + (s * g.E + e) * 2 * (int64_t)L + l;
                            o[0] = 0.0;
                            o[L] = 0.0;
                        }
                    }
                }
                continue;
            }
#pragma unroll
            for (int k = 0; k < NLW; ++k) Y[k] = Z[k] = 0.0;
            const double* mu_e = A.mu + off * L + rd * LR;
            const double* gam_e = A.gam + off * L + rd * LR;
            const double* kap_e = A.kap + off * L + rd * LR;
            const int lr_here = (L - rd * LR) < LR ? (L - rd * LR) : LR;
            const int lo = warp * (NLW * LL) + ll;  // local node index of chain 0 in the staged block

            for (int t0 = 0; t0 < m; t0 += IB) {
                const int nb = (m - t0) < IB ? (m - t0) : IB;
                // stage coefficients for steps [t0, t0+nb) of this round's nodes (zero past L:
                // such chains then contribute nothing)
                __syncthreads();
                for (int x = tid; x < nb * LR; x += blockDim.x) {
                    const int tt = x / LR, lc = x - tt * LR;
                    const bool ok = lc < lr_here;
                    const int64_t src = (int64_t)(t0 + tt) * L + lc;
                    coef[(0 * IB + tt) * LR + lc] = ok ? __ldg(mu_e + src) : 0.0;
                    if (REC) {
                        coef[(1 * IB + tt) * LR + lc] = ok ? __ldg(gam_e + src) : 0.0;
                        coef[(2 * IB + tt) * LR + lc] = ok ? __ldg(kap_e + src) : 0.0;
                    }
                }
                __syncthreads();
                for (int tt = 0; tt < nb; ++tt) {
                    const int t = t0 + tt;
                    const double wl = __ldg(Wrow + t);
                    const double wr = __ldg(Wrow + (m - 1 - t));
                    const double* cmu = coef + (0 * IB + tt) * LR + lo;
                    double accL = 0.0, accR = 0.0;
                    if (REC) {
                        const double* cg = coef + (1 * IB + tt) * LR + lo;
                        const double* ck = coef + (2 * IB + tt) * LR + lo;
                        const bool first = (t == 0), last = (t == m - 1);
                        if (first || last) {
                            // boundary rows: f_1 += (c_L/h) u_left, f_m += (c_L/h) u_right  (P310)
#pragma unroll
                            for (int k = 0; k < NLW; ++k) {
                                const int l = lbase + k * LL;
                                double ul = 0.0, ur = 0.0;
                                if (l < L) {
                                    const double beta = A.cL[l] / h;
                                    ul = beta * A.uG[(sc * V + vu) * (int64_t)L + l];
                                    ur = beta * A.uG[(sc * V + vv) * (int64_t)L + l];
                                }
                                double fl = wl, fr = wr;
                                if (first) {
                                    fl += ul;
                                    fr += ur;
                                }
                                if (last) {
                                    fl += ur;
                                    fr += ul;
                                }
                                const double c_mu = cmu[k * LL], c_g = cg[k * LL], c_k = ck[k * LL];
                                accL += c_k * Y[k];
                                Y[k] = fl - c_mu * Y[k];
                                Z[k] = fr - c_mu * Z[k];
                                accR += c_g * Z[k];
                            }
                        } else {
#pragma unroll
                            for (int k = 0; k < NLW; ++k) {
                                const double c_mu = cmu[k * LL], c_g = cg[k * LL], c_k = ck[k * LL];
                                accL += c_k * Y[k];     // left sweep: kap_t Y_{t-1} -> position t
                                Y[k] = wl - c_mu * Y[k];
                                Z[k] = wr - c_mu * Z[k];
                                accR += c_g * Z[k];     // right sweep: g_t Z -> position m-1-t
                            }
                        }
                        const int pidx = warp * LL + ll;
                        part[((tt)*P + pidx) * (SL + 1) + sl] = accL;
                        part[((IB + tt) * P + pidx) * (SL + 1) + sl] = accR;
                    } else {
#pragma unroll
                        for (int k = 0; k < NLW; ++k) {
                            const double c_mu = cmu[k * LL];
                            Y[k] = wl - c_mu * Y[k];
                            Z[k] = wr - c_mu * Z[k];
                        }
                    }
                }
                if (REC) {
                    __syncthreads();
                    // Each position i is visited by the left sweep at step i and by the right sweep at
                    // step m-1-i; visits are processed per IB block, left rows before right rows, so
                    // the first visit is the smaller (block, phase) pair.
                    // left-sweep rows: positions t0..t0+nb-1
                    for (int o = tid; o < nb * SL; o += blockDim.x) {
                        const int tt = o / SL, j = o % SL;
                        double acc = 0.0;
                        for (int p = 0; p < P; ++p) acc += part[(tt * P + p) * (SL + 1) + j];
                        const int64_t so = s0 + j;
                        if (so < A.S) {
                            const int i = t0 + tt;
                            double* dst = A.out + so * N + off + i;
                            const bool first = (rd == 0) && (i / IB <= (m - 1 - i) / IB);
                            *dst = first ? acc : *dst + acc;
                        }
                    }
                    __syncthreads();
                    // right-sweep rows: positions m-1-t
                    for (int o = tid; o < nb * SL; o += blockDim.x) {
                        const int tt = o / SL, j = o % SL;
                        double acc = 0.0;
                        for (int p = 0; p < P; ++p) acc += part[((IB + tt) * P + p) * (SL + 1) + j];
                        const int64_t so = s0 + j;
                        if (so < A.S) {
                            const int i = m - 1 - (t0 + tt);
                            double* dst = A.out + so * N + off + i;
                            const bool first = (rd == 0) && ((m - 1 - i) / IB < i / IB);
                            *dst = first ? acc : *dst + acc;
                        }
                    }
                }
            }
            if (!REC) {
                // w_m = g_m Y_m (left sweep end), w_1 = g_1 Z_1 (right sweep end); g_1 = g_m
#pragma unroll
                for (int k = 0; k < NLW; ++k) {
                    const int l = lbase + k * LL;
                    if (l < L && sact) {
                        const double g1 = __ldg(A.gam + off * L + l);
                        double* o = A.out + (s * g.E + e) * 2 * (int64_t)L + l;
                        o[0] = g1 * Z[k];
                        o[L] = g1 * Y[k];
                    }
                }
            }
        }
    }
}

template <int NLW, int SL, bool REC>
cudaError_t launch_sweep(SweepArgs a, cudaStream_t st) {
    constexpr int LL = Lanes<SL>::LL;
    int nw = (a.L + NLW * LL - 1) / (NLW * LL);
    if (nw > MAXW) nw = MAXW;
    a.nwarps = nw;
    const int LR = nw * NLW * LL;
    const int P = nw * LL;
    const size_t smem = sizeof(double) * ((size_t)3 * IB * LR + (size_t)2 * IB * P * (SL + 1));
    cudaError_t e = cudaFuncSetAttribute(sweep_kernel<NLW, SL, REC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(a.wq.counter, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return e;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_kernel<NLW, SL, REC>, nw * 32, smem);
    if (per_sm < 1) per_sm = 1;
    int blocks = 148 * per_sm;
    if (blocks > a.wq.n_items) blocks = a.wq.n_items;
    sweep_kernel<NLW, SL, REC><<<blocks, nw * 32, smem, st>>>(a);
    return cudaGetLastError();
}

template <bool REC>
cudaError_t dispatch(SweepArgs a, cudaStream_t st) {
    // sample lanes per warp: as many samples as the call has, up to 32
    if (a.S >= 32) return launch_sweep<16, 32, REC>(a, st);
    if (a.S >= 16) return launch_sweep<16, 16, REC>(a, st);
    if (a.S >= 8) return launch_sweep<8, 8, REC>(a, st);
    if (a.S >= 4) return launch_sweep<8, 4, REC>(a, st);
    if (a.S >= 2) return launch_sweep<8, 2, REC>(a, st);
    return launch_sweep<8, 1, REC>(a, st);
}

int sample_lanes(int64_t S) {
    return S >= 32 ? 32 : S >= 16 ? 16 : S >= 8 ? 8 : S >= 4 ? 4 : S >= 2 ? 2 : 1;
}

}  // namespace

WorkQueue make_work_queue(const DevGraph& g, int64_t n_samples, int32_t* counter) {
    WorkQueue q;
    q.counter = counter;
    q.samples_per_item = sample_lanes(n_samples);
    q.chunks = (int)((n_samples + q.samples_per_item - 1) / q.samples_per_item);
    q.n_items = g.E * q.chunks;
    return q;
}

cudaError_t launch_condense(const DevGraph& g, const DevPlan& p, int64_t n_samples, const double* W, double* ends,
                            WorkQueue wq, cudaStream_t st) {
    SweepArgs a{g, p.L, p.cL, p.mu, p.gam, p.kap, n_samples, W, ends, nullptr, wq, 0};
    return dispatch<false>(a, st);
}

cudaError_t launch_recover(const DevGraph& g, const DevPlan& p, int64_t n_samples, const double* W, double* u,
                           const double* uG, WorkQueue wq, cudaStream_t st) {
    SweepArgs a{g, p.L, p.cL, p.mu, p.gam, p.kap, n_samples, W, u, uG, wq, 0};
    return dispatch<true>(a, st);
}

int32_t recover_max_interior() { return 1 << 30; }
int32_t max_nodes_per_block() { return 1 << 20; }

}  // namespace grf
