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
// Mapping: a warp owns one (edge, tile of SL samples) and ALL quadrature nodes: lane =
// (sample sl, node sub-lane ll), LL = 32/SL sub-lanes, and each thread carries the NLW
// consecutive nodes ll*NLW .. ll*NLW+NLW-1 (2 chains each) in registers.  The sum over l is
// an in-thread sum over the thread's nodes plus log2(LL) warp shuffles -- no cross-warp
// reduction, no partial-sum buffers.  The warps of a CTA work on the same edge (different
// sample tiles), so the per-(l, t) coefficients are staged once per CTA in shared memory,
// IB steps at a time with cp.async, double buffered, and read as (near-)broadcasts.  Each
// warp keeps its edge's output tile in shared memory and writes it to HBM once, coalesced.
// Edges are handed out longest first through an atomic work queue.
#include <cuda_pipeline.h>

#include <cstdlib>

#include "grf_internal.h"

namespace grf {
namespace {

constexpr int NWARP = 8;     // warps per CTA
constexpr int OTILE_DOUBLES_PER_WARP = 640;  // smem output tile per warp: m * SL <= 640

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
    int32_t rounds;     // node rounds (L > NLW*LL only)
};

__device__ __forceinline__ void cp8(double* dst, const double* src) { __pipeline_memcpy_async(dst, src, 8); }

// smem node stride per sub-lane: NLW rounded so that the LL sub-lanes' LDS.128 hit
// disjoint banks (stride in doubles = 2, 6, 10 or 14 mod 16) and stays 16-byte aligned
template <int NLW>
struct Stride {
    static constexpr int e = (NLW + 1) / 2 * 2;
    static constexpr int v = (e % 4 == 2) ? e : e + 2;
};

// Shared memory (doubles):
//   coef [2][IB][NT][LP]      staged mu (, gam, kap); LP = LL * stride padded node slots
//   wbuf [2][IB][2][NWARP*SL]  staged W (left position t, right position m-1-t) for the CTA's samples
//   g1   [LP]                  condense: g_1 row
//   otile[NWARP][m][SL]        recover: per-warp output tile (edges with m * SL <= OTILE_DOUBLES_PER_WARP)
template <int NLW, int SL>
struct Geo {
    static constexpr int LL = 32 / SL;
    static constexpr int LP = LL * Stride<NLW>::v;
    static constexpr int IB = LP > 320 ? 4 : 8;  // steps per staging block (smem budget)
};

template <int NLW, int SL, bool REC>
__global__ void __launch_bounds__(NWARP * 32) sweep_kernel(SweepArgs A) {
    constexpr int LL = 32 / SL;
    constexpr int NT = REC ? 3 : 1;
    constexpr int NS = Stride<NLW>::v;
    constexpr int LP = LL * NS;
    constexpr int IB = Geo<NLW, SL>::IB;
    constexpr int CS = NWARP * SL;  // samples per CTA item
    extern __shared__ double smem[];
    __shared__ int item_sh;
    const DevGraph& g = A.g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sl = lane % SL, ll = lane / SL;
    const int L = A.L;
    double* coef = smem;                        // 2*IB*NT*LP
    double* wbuf = coef + 2 * IB * NT * LP;     // 2*IB*2*CS
    double* g1b = wbuf + 2 * IB * 2 * CS;       // LP
    double* otile = g1b + LP + warp * OTILE_DOUBLES_PER_WARP;
    const int64_t N = g.N;
    const int V = g.V;

    for (;;) {
        if (tid == 0) item_sh = atomicAdd(A.wq.counter, 1);
        __syncthreads();
        const int it = item_sh;
        __syncthreads();
        if (it >= A.wq.n_items) break;
        const int e = g.edge_order[it / A.wq.chunks];
        const int64_t c0 = (int64_t)(it % A.wq.chunks) * CS;  // first sample of the CTA item
        const int64_t s = c0 + warp * SL + sl;
        const bool sact = s < A.S;
        const int64_t sc = sact ? s : (A.S - 1);
        const int m = g.m[e];
        const int64_t off = g.off[e];
        const double h = g.h[e];
        const int vu = g.eu[e], vv = g.ev[e];
        const bool in_smem = REC && (m * SL <= OTILE_DOUBLES_PER_WARP);
        const int ncs = (int)((A.S - c0) < CS ? (A.S - c0) : CS);  // live samples of the item

        for (int rd = 0; rd < A.rounds; ++rd) {
            if (rd > 0) __syncthreads();
            const int lbase = rd * LL * NLW + ll * NLW;  // node of chain k: lbase + k
            const int lr0 = rd * LL * NLW;
            const int lr_here = (L - lr0) < LL * NLW ? (L - lr0) : LL * NLW;
            // ---------------- recover: vertex values owned by this edge (u_v = sum_l u_G)
            if (REC) {
                const bool ownL = g.owner[vu] == 2 * e, ownR = g.owner[vv] == 2 * e + 1;
                if (ownL || ownR) {
                    double a0 = 0.0, a1 = 0.0;
#pragma unroll
                    for (int k = 0; k < NLW; ++k) {
                        const int l = lbase + k;
                        if (l < L && l < lr0 + lr_here) {
                            a0 += A.uG[(sc * V + vu) * (int64_t)L + l];
                            a1 += A.uG[(sc * V + vv) * (int64_t)L + l];
                        }
                    }
#pragma unroll
                    for (int o = SL; o < 32; o <<= 1) {
                        a0 += __shfl_xor_sync(0xffffffffu, a0, o);
                        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
                    }
                    if (ll == 0 && sact) {
                        if (ownL) {
                            double* d = A.out + s * N + g.NI + vu;
                            *d = rd == 0 ? a0 : *d + a0;
                        }
                        if (ownR) {
                            double* d = A.out + s * N + g.NI + vv;
                            *d = rd == 0 ? a1 : *d + a1;
                        }
                    }
                }
                if (m > 0) {  // u_G at both ends is read at the first and the last step: warm L2
                    for (int k = 0; k < NLW; k += 4) {
                        const int l = lbase + k;
                        if (l < L) {
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(A.uG + (sc * V + vu) * (int64_t)L + l));
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(A.uG + (sc * V + vv) * (int64_t)L + l));
                        }
                    }
                }
            }
            if (m == 0) {
                if (!REC) {
#pragma unroll
                    for (int k = 0; k < NLW; ++k) {
                        const int l = lbase + k;
                        if (l < L && sact) {
                            double* o = A.out + (s * g.E + e) * 2 * (int64_t)L + l;
                            o[0] = 0.0;
                            o[L] = 0.0;
                        }
                    }
                }
                continue;
            }
            double Y[NLW], Z[NLW];
#pragma unroll
            for (int k = 0; k < NLW; ++k) Y[k] = Z[k] = 0.0;
            const int nblk = (m + IB - 1) / IB;

            // asynchronous staging of block b into buffer b&1: coefficients for the round's nodes
            // (node lc of the round goes to sub-lane lc / NLW, slot lc % NLW), and W of the CTA's samples
            auto stage = [&](int b) {
                const int t0 = b * IB;
                const int nb = (m - t0) < IB ? (m - t0) : IB;
                double* cb = coef + (b & 1) * IB * NT * LP;
                for (int x = tid; x < IB * LL * NLW; x += NWARP * 32) {
                    const int tt = x / (LL * NLW), lc = x % (LL * NLW);
                    const int slot = (lc / NLW) * NS + lc % NLW;
                    const bool ok = tt < nb && lc < lr_here;
                    const int64_t src = (off + t0 + tt) * (int64_t)L + lr0 + lc;
#pragma unroll
                    for (int tb = 0; tb < NT; ++tb) {
                        double* dst = cb + (tt * NT + tb) * LP + slot;
                        const double* tab = tb == 0 ? A.mu : (tb == 1 ? A.gam : A.kap);
                        if (ok)
                            cp8(dst, tab + src);
                        else
                            *dst = 0.0;  // nodes past L (and steps past m) contribute nothing
                    }
                }
                if (!REC && b == 0) {  // g_1 (= g_m) row for the end values
                    for (int lc = tid; lc < LL * NLW; lc += NWARP * 32) {
                        const int slot = (lc / NLW) * NS + lc % NLW;
                        if (lc < lr_here)
                            cp8(g1b + slot, A.gam + off * (int64_t)L + lr0 + lc);
                        else
                            g1b[slot] = 0.0;
                    }
                }
                double* wb = wbuf + (b & 1) * IB * 2 * CS;
                for (int x = tid; x < 2 * CS * IB; x += NWARP * 32) {
                    const int side = x / (CS * IB), r = x % (CS * IB);
                    const int j = r / IB, tt = r % IB;
                    if (tt < nb) {
                        const int pos = side ? (m - 1 - t0 - tt) : (t0 + tt);
                        double* dst = wb + (tt * 2 + side) * CS + j;
                        if (j < ncs)
                            cp8(dst, A.W + (c0 + j) * N + off + pos);
                        else
                            *dst = 0.0;
                    }
                }
                __pipeline_commit();
            };

            // recovery boundary rows (P310): f_1 += (c_L/h) u_left, f_m += (c_L/h) u_right
            auto bnd = [&](int k, double& ul, double& ur) {
                const int l = lbase + k;
                ul = ur = 0.0;
                if (l < L && l < lr0 + lr_here) {
                    const double beta = A.cL[l] / h;
                    ul = beta * A.uG[(sc * V + vu) * (int64_t)L + l];
                    ur = beta * A.uG[(sc * V + vv) * (int64_t)L + l];
                }
            };

            stage(0);
            for (int b = 0; b < nblk; ++b) {
                const int t0 = b * IB;
                const int nb = (m - t0) < IB ? (m - t0) : IB;
                __pipeline_wait_prior(0);
                __syncthreads();  // block b visible; everyone is done with block b-1's buffer
                if (b + 1 < nblk) stage(b + 1);
                const double* cb = coef + (b & 1) * IB * NT * LP + ll * NS;
                const double* wb = wbuf + (b & 1) * IB * 2 * CS + warp * SL + sl;
                for (int tt = 0; tt < nb; ++tt) {
                    const int t = t0 + tt;
                    const double wl = wb[(tt * 2 + 0) * CS];
                    const double wr = wb[(tt * 2 + 1) * CS];
                    const double* cmu = cb + (tt * NT + 0) * LP;
                    if (REC) {
                        const double* cg = cb + (tt * NT + 1) * LP;
                        const double* ck = cb + (tt * NT + 2) * LP;
                        double aL0 = 0.0, aL1 = 0.0, aL2 = 0.0, aR0 = 0.0, aR1 = 0.0, aR2 = 0.0;
                        if (t == 0 || t == m - 1) {
#pragma unroll
                            for (int k = 0; k < NLW; ++k) {
                                double ul, ur;
                                bnd(k, ul, ur);
                                double fl = wl, fr = wr;
                                if (t == 0) {
                                    fl += ul;
                                    fr += ur;
                                }
                                if (t == m - 1) {
                                    fl += ur;
                                    fr += ul;
                                }
                                aL0 += ck[k] * Y[k];
                                Y[k] = fl - cmu[k] * Y[k];
                                Z[k] = fr - cmu[k] * Z[k];
                                aR0 += cg[k] * Z[k];
                            }
                        } else {
#pragma unroll
                            for (int k = 0; k < NLW; ++k) {
                                double& aL = (k % 3 == 0) ? aL0 : (k % 3 == 1 ? aL1 : aL2);
                                double& aR = (k % 3 == 0) ? aR0 : (k % 3 == 1 ? aR1 : aR2);
                                aL += ck[k] * Y[k];  // left sweep: kap_t Y_{t-1} -> position t
                                Y[k] = wl - cmu[k] * Y[k];
                                Z[k] = wr - cmu[k] * Z[k];
                                aR += cg[k] * Z[k];  // right sweep: g_t Z -> position m-1-t
                            }
                        }
                        double cl = aL0 + aL1 + aL2, cr = aR0 + aR1 + aR2;
#pragma unroll
                        for (int o = SL; o < 32; o <<= 1) {  // sum over the node sub-lanes
                            cl += __shfl_xor_sync(0xffffffffu, cl, o);
                            cr += __shfl_xor_sync(0xffffffffu, cr, o);
                        }
                        // position i gets its left part at step i and its right part at step m-1-i;
                        // the earlier visit writes, the later adds (the middle: left then right)
                        if (ll == 0) {
                            const int il = t, ir = m - 1 - t;
                            const bool fl1 = rd == 0 && il <= m - 1 - il;
                            const bool fr1 = rd == 0 && ir > m - 1 - ir;
                            if (in_smem) {
                                double* dl = otile + il * SL + sl;
                                *dl = fl1 ? cl : *dl + cl;
                                double* dr = otile + ir * SL + sl;
                                *dr = fr1 ? cr : *dr + cr;
                            } else if (sact) {
                                double* dl = A.out + s * N + off + il;
                                *dl = fl1 ? cl : *dl + cl;
                                double* dr = A.out + s * N + off + ir;
                                *dr = fr1 ? cr : *dr + cr;
                            }
                        }
                    } else {
#pragma unroll
                        for (int k = 0; k < NLW; ++k) {
                            Y[k] = wl - cmu[k] * Y[k];
                            Z[k] = wr - cmu[k] * Z[k];
                        }
                    }
                }
            }
            if (!REC) {
                // w_m = g_m Y_m (left sweep end), w_1 = g_1 Z_1 (right sweep end); g_1 = g_m
#pragma unroll
                for (int k = 0; k < NLW; ++k) {
                    const int l = lbase + k;
                    if (l < L && l < lr0 + lr_here && sact) {
                        const double g1 = g1b[ll * NS + k];
                        double* o = A.out + (s * g.E + e) * 2 * (int64_t)L + l;
                        o[0] = g1 * Z[k];
                        o[L] = g1 * Y[k];
                    }
                }
            }
        }
        if (in_smem && m > 0) {
            __syncwarp();
            // the warp's SL samples, positions contiguous per sample row
            for (int o = lane; o < m * SL; o += 32) {
                const int j = o / m, i = o - j * m;
                const int64_t sj = c0 + warp * SL + j;
                if (sj < A.S) A.out[sj * N + off + i] = otile[i * SL + j];
            }
        }
    }
}

template <int NLW, int SL, bool REC>
cudaError_t launch_sweep(SweepArgs a, cudaStream_t st) {
    constexpr int LL = 32 / SL;
    constexpr int NT = REC ? 3 : 1;
    constexpr int LP = LL * Stride<NLW>::v;
    constexpr int IB = Geo<NLW, SL>::IB;
    constexpr int CS = NWARP * SL;
    a.rounds = (a.L + LL * NLW - 1) / (LL * NLW);
    a.wq.samples_per_item = CS;
    a.wq.chunks = (int)((a.S + CS - 1) / CS);
    a.wq.n_items = a.g.E * a.wq.chunks;
    const size_t smem = sizeof(double) * ((size_t)2 * IB * NT * LP + (size_t)2 * IB * 2 * CS + LP +
                                          (REC ? (size_t)NWARP * OTILE_DOUBLES_PER_WARP : 0));
    cudaError_t e = cudaFuncSetAttribute(sweep_kernel<NLW, SL, REC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(a.wq.counter, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return e;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_kernel<NLW, SL, REC>, NWARP * 32, smem);
    if (per_sm < 1) per_sm = 1;
    int blocks = 148 * per_sm;
    if (blocks > a.wq.n_items) blocks = a.wq.n_items;
    sweep_kernel<NLW, SL, REC><<<blocks, NWARP * 32, smem, st>>>(a);
    return cudaGetLastError();
}

// node sub-lanes LL (= 32/SL) and nodes per thread NLW for this (L, S): as few node
// sub-lanes as keep NLW <= 28 (more samples per warp), but no more sample lanes than samples
template <bool REC>
cudaError_t dispatch(SweepArgs a, cudaStream_t st) {
    int ll = 1;
    while (ll < 32 && (a.L + ll - 1) / ll > 28) ll *= 2;
    while (ll < 32 && 32 / ll > a.S) ll *= 2;
    const int need = (a.L + ll - 1) / ll;
    const int nlw = need <= 8 ? 8 : (need <= 16 ? 16 : 28);
#define GRF_SW(NL, SLV) \
    if (nlw == NL && 32 / ll == SLV) return launch_sweep<NL, SLV, REC>(a, st);
    GRF_SW(8, 32) GRF_SW(16, 32) GRF_SW(28, 32)
    GRF_SW(8, 16) GRF_SW(16, 16) GRF_SW(28, 16)
    GRF_SW(8, 8) GRF_SW(16, 8) GRF_SW(28, 8)
    GRF_SW(8, 4) GRF_SW(16, 4) GRF_SW(28, 4)
    GRF_SW(8, 2) GRF_SW(16, 2) GRF_SW(28, 2)
    GRF_SW(8, 1) GRF_SW(16, 1) GRF_SW(28, 1)
#undef GRF_SW
    return cudaErrorInvalidValue;
}

}  // namespace

WorkQueue make_work_queue(const DevGraph& g, int64_t n_samples, int32_t* counter) {
    WorkQueue q;  // the item shape (edge, samples per CTA) is fixed by the launcher
    q.counter = counter;
    (void)g;
    (void)n_samples;
    return q;
}

cudaError_t launch_condense(const DevGraph& g, const DevPlan& p, int64_t n_samples, const double* W, double* ends,
                            WorkQueue wq, cudaStream_t st) {
    SweepArgs a{g, p.L, p.cL, p.mu, p.gam, p.kap, n_samples, W, ends, nullptr, wq, 1};
    return dispatch<false>(a, st);
}

cudaError_t launch_recover(const DevGraph& g, const DevPlan& p, int64_t n_samples, const double* W, double* u,
                           const double* uG, WorkQueue wq, cudaStream_t st) {
    SweepArgs a{g, p.L, p.cL, p.mu, p.gam, p.kap, n_samples, W, u, uG, wq, 1};
    return dispatch<true>(a, st);
}

int32_t recover_max_interior() { return 1 << 30; }
int32_t max_nodes_per_block() { return 1 << 20; }

}  // namespace grf
