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
// NLW nodes x 2 chains in registers.  The per-(l, t) coefficients and the W tile are
// staged into shared memory IB steps at a time with cp.async, double buffered (block
// b+1 loads while block b computes), and read as warp broadcasts.  Per-warp partial sums
// over the thread's nodes are combined across warps in fixed order (deterministic) into
// an output tile kept in shared memory for the whole edge (written to HBM once,
// coalesced); edges too long for the tile fall back to read-modify-write in global memory.
#include <cuda_pipeline.h>

#include <cstdlib>

#include "grf_internal.h"

namespace grf {
namespace {

constexpr int MAXW = 16;       // warps per CTA
constexpr int OTILE_BYTES = 48 * 1024;

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
    int32_t mtile;      // recover: edges with m <= mtile keep their output tile in smem
};

template <int SL>
struct Lanes {
    static constexpr int LL = 32 / SL;  // node sub-lanes per warp
};

__device__ __forceinline__ void cp8(double* dst, const double* src) { __pipeline_memcpy_async(dst, src, 8); }

// Shared memory layout (doubles), NT = number of coefficient tables (1 condense, 3 recover):
//   coef [2][NT][IB][LR]   staged mu (, gam, kap) for this round's LR nodes, double buffered
//   wbuf [2][2][IB][SL+1]  staged W: [buffer][left/right positions][step][sample]
//   part [2][2*IB][P][SL+1] per (row, partial, sample) sums, P = nwarps*LL, double buffered (recover)
//   otile[mtile][SL+1]     the edge's output tile                                  (recover)
template <int NLW, int SL, bool REC, int IB, int MAXT>
__global__ void __launch_bounds__(MAXT) sweep_kernel(SweepArgs A) {
    constexpr int LL = Lanes<SL>::LL;
    constexpr int NT = REC ? 3 : 1;
    constexpr int SP = SL + 1;
    constexpr int NBUF = REC ? 2 : 3;  // staging buffers (prefetch distance NBUF-1 blocks)
    extern __shared__ double smem[];
    __shared__ int item_sh;
    const DevGraph& g = A.g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sl = lane % SL, ll = lane / SL;
    const int nwarps = A.nwarps;
    const int P = nwarps * LL;
    const int LR = nwarps * NLW * LL;  // nodes per round
    const int L = A.L;
    const int rounds = (L + LR - 1) / LR;
    double* coef = smem;                                 // 2*NT*IB*LR
    double* wbuf = coef + NBUF * NT * IB * LR;           // NBUF*2*IB*SP
    double* part = wbuf + NBUF * 2 * IB * SP;            // 2*IB*P*SP     (REC)
    double* g1buf = part;                                // LR             (condense: g_1 row)
    double* otile = part + (REC ? 4 * IB * P * SP : 0);  // mtile*SP      (REC; part is double buffered)
    const int64_t N = g.N;
    const int V = g.V;
    const int pidx = warp * LL + ll;

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
        const int ns = (int)((A.S - s0) < SL ? (A.S - s0) : SL);
        const int m = g.m[e];
        const int64_t off = g.off[e];
        const double h = g.h[e];
        const int vu = g.eu[e], vv = g.ev[e];
        const double* Wtile = A.W + s0 * N + off;
        const bool in_smem = REC && (m <= A.mtile);
        if (REC && m > 0) {  // u_G at both ends is needed at the first and last step: warm L2 now
            for (int l = 4 * (warp * LL + ll); l < L; l += 4 * nwarps * LL) {  // one 32-B sector each
                asm volatile("prefetch.global.L2 [%0];" ::"l"(A.uG + (sc * V + vu) * (int64_t)L + l));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(A.uG + (sc * V + vv) * (int64_t)L + l));
            }
        }

        for (int rd = 0; rd < rounds; ++rd) {
            if (rd > 0) __syncthreads();  // staging buffers of the previous round are free
            const int lbase = rd * LR + warp * (NLW * LL) + ll;  // node of chain k: lbase + k*LL
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
                    part[(0 * P + pidx) * SP + sl] = a0;
                    part[(1 * P + pidx) * SP + sl] = a1;
                    __syncthreads();
                    for (int o = tid; o < 2 * SL; o += blockDim.x) {
                        const int side = o / SL, j = o % SL;
                        double t = 0.0;
                        for (int p = 0; p < P; ++p) t += part[(side * P + p) * SP + j];
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
            double Y[NLW], Z[NLW];
#pragma unroll
            for (int k = 0; k < NLW; ++k) Y[k] = Z[k] = 0.0;
            const int lr_here = (L - rd * LR) < LR ? (L - rd * LR) : LR;
            const int lo = warp * (NLW * LL) + ll;  // local node index of chain 0 in the staged block
            const int nblk = (m + IB - 1) / IB;

            // asynchronous staging of block b into buffer b&1 (division-free index math)
            auto stage = [&](int b) {
                const int t0 = b * IB;
                const int nb = (m - t0) < IB ? (m - t0) : IB;
                double* cb = coef + (b % NBUF) * NT * IB * LR;
                const int64_t row0 = (off + t0) * (int64_t)L + rd * LR;
                for (int lc = tid; lc < LR; lc += blockDim.x) {
                    const bool okl = lc < lr_here;
#pragma unroll
                    for (int tt = 0; tt < IB; ++tt) {
                        const bool ok = okl && tt < nb;
                        const int64_t src = row0 + (int64_t)tt * L + lc;
#pragma unroll
                        for (int tb = 0; tb < NT; ++tb) {
                            double* dst = cb + (tb * IB + tt) * LR + lc;
                            const double* tab = tb == 0 ? A.mu : (tb == 1 ? A.gam : A.kap);
                            if (ok)
                                cp8(dst, tab + src);
                            else
                                *dst = 0.0;  // nodes past L (and steps past m) contribute nothing
                        }
                    }
                }
                if (!REC && b == 0) {  // g_1 (= g_m) row for the end values, staged with block 0
                    for (int lc = tid; lc < LR; lc += blockDim.x) {
                        if (lc < lr_here)
                            cp8(g1buf + lc, A.gam + off * (int64_t)L + rd * LR + lc);
                        else
                            g1buf[lc] = 0.0;
                    }
                }
                double* wb = wbuf + (b % NBUF) * 2 * IB * SP;
                for (int x = tid; x < 2 * IB * SL; x += blockDim.x) {
                    const int side = x / (IB * SL), r = x % (IB * SL);
                    const int j = r / IB, tt = r % IB;
                    if (tt < nb) {
                        const int pos = side ? (m - 1 - t0 - tt) : (t0 + tt);
                        double* dst = wb + (side * IB + tt) * SP + j;
                        if (j < ns)
                            cp8(dst, Wtile + (int64_t)j * N + pos);
                        else
                            *dst = 0.0;
                    }
                }
                __pipeline_commit();
            };

            // prefetch NBUF-1 blocks ahead; one commit group per block (empty groups past the end).
            // Per block: wait for block b, one barrier (b visible to all; every thread is done with
            // block b-1, whose buffer is restaged next), then issue block b+NBUF-1 and compute b.
#pragma unroll
            for (int b = 0; b < NBUF - 1; ++b) {
                if (b < nblk) stage(b);
                else __pipeline_commit();
            }
            // fold the per-warp partial sums of block bp into the output (deferred by one block so
            // that it needs no barrier of its own).  Position i is visited by the left sweep at
            // step i and by the right sweep at step m-1-i; left rows are folded before right rows,
            // so the first visit is the smaller (block, phase) pair.  Only near the edge midpoint
            // can one block hold both visits of a position: then the two phases are separated.
            auto fold = [&](int bp) {
                const int t0p = bp * IB;
                const int nbp = (m - t0p) < IB ? (m - t0p) : IB;
                const double* pb = part + (bp & 1) * 2 * IB * P * SP;
                const bool overlap = (t0p + nbp > m - t0p - nbp) && (m - 1 - t0p >= t0p);
                for (int side = 0; side < 2; ++side) {
                    if (side == 1 && overlap) __syncthreads();
                    for (int o = tid; o < IB * SL; o += blockDim.x) {
                        const int j = o / IB, tt = o % IB;
                        if (tt >= nbp) continue;
                        double acc = 0.0;
                        for (int q = 0; q < P; ++q) acc += pb[((side * IB + tt) * P + q) * SP + j];
                        const int i = side ? (m - 1 - (t0p + tt)) : (t0p + tt);
                        const int bi = i / IB, bm = (m - 1 - i) / IB;
                        const bool first = (rd == 0) && (side ? (bm < bi) : (bi <= bm));
                        if (in_smem) {
                            double* dst = otile + i * SP + j;
                            *dst = first ? acc : *dst + acc;
                        } else if (s0 + j < A.S) {
                            double* dst = A.out + (s0 + j) * N + off + i;
                            *dst = first ? acc : *dst + acc;
                        }
                    }
                }
            };
            for (int b = 0; b < nblk; ++b) {
                const int t0 = b * IB;
                const int nb = (m - t0) < IB ? (m - t0) : IB;
                __pipeline_wait_prior(NBUF - 2);
                __syncthreads();
                if (b + NBUF - 1 < nblk) stage(b + NBUF - 1);
                else __pipeline_commit();
                if (REC && b > 0) fold(b - 1);
                double* pw = part + (b & 1) * 2 * IB * P * SP;
                const double* cb = coef + (b % NBUF) * NT * IB * LR;
                const double* wb = wbuf + (b % NBUF) * 2 * IB * SP;
                for (int tt = 0; tt < nb; ++tt) {
                    const int t = t0 + tt;
                    const double wl = wb[tt * SP + sl];
                    const double wr = wb[(IB + tt) * SP + sl];
                    const double* cmu = cb + tt * LR + lo;
                    if (REC) {
                        const double* cg = cb + (IB + tt) * LR + lo;
                        const double* ck = cb + (2 * IB + tt) * LR + lo;
                        double aL0 = 0.0, aL1 = 0.0, aR0 = 0.0, aR1 = 0.0;
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
                                aL0 += c_k * Y[k];
                                Y[k] = fl - c_mu * Y[k];
                                Z[k] = fr - c_mu * Z[k];
                                aR0 += c_g * Z[k];
                            }
                        } else {
#pragma unroll
                            for (int k = 0; k < NLW; k += 2) {
                                const double m0 = cmu[k * LL], g0 = cg[k * LL], k0 = ck[k * LL];
                                const double m1 = cmu[(k + 1) * LL], g1 = cg[(k + 1) * LL], k1 = ck[(k + 1) * LL];
                                aL0 += k0 * Y[k];  // left sweep: kap_t Y_{t-1} -> position t
                                aL1 += k1 * Y[k + 1];
                                Y[k] = wl - m0 * Y[k];
                                Y[k + 1] = wl - m1 * Y[k + 1];
                                Z[k] = wr - m0 * Z[k];
                                Z[k + 1] = wr - m1 * Z[k + 1];
                                aR0 += g0 * Z[k];  // right sweep: g_t Z -> position m-1-t
                                aR1 += g1 * Z[k + 1];
                            }
                        }
                        pw[(tt * P + pidx) * SP + sl] = aL0 + aL1;
                        pw[((IB + tt) * P + pidx) * SP + sl] = aR0 + aR1;
                    } else {
#pragma unroll
                        for (int k = 0; k < NLW; ++k) {
                            const double c_mu = cmu[k * LL];
                            Y[k] = wl - c_mu * Y[k];
                            Z[k] = wr - c_mu * Z[k];
                        }
                    }
                }
            }
            if (REC) {
                __syncthreads();
                fold(nblk - 1);
            }
            if (!REC) {
                // w_m = g_m Y_m (left sweep end), w_1 = g_1 Z_1 (right sweep end); g_1 = g_m
#pragma unroll
                for (int k = 0; k < NLW; ++k) {
                    const int l = lbase + k * LL;
                    if (l < L && sact) {
                        const double g1 = g1buf[lo + k * LL];
                        double* o = A.out + (s * g.E + e) * 2 * (int64_t)L + l;
                        o[0] = g1 * Z[k];
                        o[L] = g1 * Y[k];
                    }
                }
            }
        }
        if (in_smem && m > 0) {
            __syncthreads();
            for (int o = tid; o < m * ns; o += blockDim.x) {
                const int j = o / m, i = o - j * m;
                A.out[(s0 + j) * N + off + i] = otile[i * SP + j];
            }
        }
    }
}

template <int NLW, int SL, bool REC, int IB, int MAXT = MAXW * 32>
cudaError_t launch_sweep(SweepArgs a, cudaStream_t st) {
    constexpr int LL = Lanes<SL>::LL;
    constexpr int NT = REC ? 3 : 1;
    int nw = (a.L + NLW * LL - 1) / (NLW * LL);
    if (nw > MAXT / 32) nw = MAXT / 32;
    a.nwarps = nw;
    const int LR = nw * NLW * LL;
    const int P = nw * LL;
    constexpr int NBUF = REC ? 2 : 3;
    size_t base = (size_t)NBUF * NT * IB * LR + (size_t)NBUF * 2 * IB * (SL + 1);
    base += REC ? (size_t)4 * IB * P * (SL + 1) : (size_t)LR;
    a.mtile = REC ? (int)(OTILE_BYTES / (sizeof(double) * (SL + 1))) : 0;
    size_t smem = sizeof(double) * (base + (REC ? (size_t)a.mtile * (SL + 1) : 0));
    if (REC && smem > 220 * 1024) {  // no room for the smem output tile
        a.mtile = 0;
        smem = sizeof(double) * base;
    }
    cudaError_t e = cudaFuncSetAttribute(sweep_kernel<NLW, SL, REC, IB, MAXT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(a.wq.counter, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return e;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_kernel<NLW, SL, REC, IB, MAXT>, nw * 32, smem);
    if (per_sm < 1) per_sm = 1;
    int blocks = 148 * per_sm;
    if (blocks > a.wq.n_items) blocks = a.wq.n_items;
    sweep_kernel<NLW, SL, REC, IB, MAXT><<<blocks, nw * 32, smem, st>>>(a);
    return cudaGetLastError();
}

template <bool REC>
cudaError_t dispatch(SweepArgs a, cudaStream_t st) {
    // steps per staging block (tuning knob GRF_SWEEP_IB for experiments; default 8 / 16)
    static const int ib_env = [] {
        const char* e = getenv("GRF_SWEEP_IB");
        return e ? atoi(e) : 0;
    }();
    const int ib = REC ? 8 : (ib_env ? ib_env : 16);  // recover: smem holds partials + output tile
    // sample lanes per warp: as many samples as the call has, up to 32
    if (a.S >= 32) {
        if (REC) return launch_sweep<32, 32, REC, 8, 256>(a, st);  // 32 nodes x 2 chains per thread
        if (ib == 32) return launch_sweep<16, 32, REC, 32>(a, st);
        if (ib == 16) return launch_sweep<16, 32, REC, 16>(a, st);
        return launch_sweep<16, 32, REC, 8>(a, st);
    }
    if (a.S >= 16) return launch_sweep<16, 16, REC, 8>(a, st);
    if (a.S >= 8) return launch_sweep<8, 8, REC, 8>(a, st);
    if (a.S >= 4) return launch_sweep<8, 4, REC, 8>(a, st);
    if (a.S >= 2) return launch_sweep<8, 2, REC, 8>(a, st);
    return launch_sweep<8, 1, REC, 8>(a, st);
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
    SweepArgs a{g, p.L, p.cL, p.mu, p.gam, p.kap, n_samples, W, ends, nullptr, wq, 0, 0};
    return dispatch<false>(a, st);
}

cudaError_t launch_recover(const DevGraph& g, const DevPlan& p, int64_t n_samples, const double* W, double* u,
                           const double* uG, WorkQueue wq, cudaStream_t st) {
    SweepArgs a{g, p.L, p.cL, p.mu, p.gam, p.kap, n_samples, W, u, uG, wq, 0, 0};
    return dispatch<true>(a, st);
}

int32_t recover_max_interior() { return 1 << 30; }
int32_t max_nodes_per_block() { return 1 << 20; }

}  // namespace grf
