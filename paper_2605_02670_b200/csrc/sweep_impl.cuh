// K3 (condense) and K5 (recover + quadrature sum): the per-edge Thomas work of PAPER.md
// P187-239 and P300-324, batched over (quadrature node l) x (sample s) x (edge e).
//
// For one edge, node l and right-hand side f (length m), the interior block
// A_II = tridiag(b, a, b) (Toeplitz) is eliminated from both ends with the
// paper's Thomas multipliers (P187-221):
//   left  sweep:  Y_0 = f_0,      Y_t = f_t - mu_t Y_{t-1},       mu_t = b / d'_{t-1}, mu_0 = 0
//   right sweep:  Z_0 = f_{m-1},  Z_t = f_{m-1-t} - mu_t Z_{t-1}  (same pivots: A_II persymmetric)
// and the Thomas solution is the twisted-factorisation combination of the two sweeps
//   (A_II^{-1} f)_i = g_i (Y_i + Z_{m-1-i} - f_i),   g_i = 1 / (d'_i + d'_{m-1-i} - a)
// (equal, up to rounding, to forward + back substitution P215-228: both are exact LU-type
// eliminations of the same system).  Because Y_i - f_i = -mu_i Y_{i-1}, position i receives
// -g_i mu_i Y_{i-1} from the left sweep (at step i) and g_i Z (from the right sweep, at step
// m-1-i; g is symmetric, so step t uses g_t for both).  No intermediate vector is stored.
//
//   K3 condense (f = W_I):  w_1 = g_0 Z_{m-1},  w_m = g_0 Y_{m-1}   -> ends[((s*E+e)*2+end)*L + l]
//   K5 recover  (f = W_I + (c_L/h_e)(u_left e_1 + u_right e_m), P306-311):
//                           u_i = sum_l (A_II^{(l)})^{-1} f^{(l)}     -> u[s*N + off + i]
//
// Mapping (register tiles).  A CTA works on one item = (edge e, tile of CS samples) and on
// all quadrature nodes, in `rounds` node rounds of 32*TL nodes.  Its threads form a
// 32 (l-threads) x NST (s-threads) grid; each thread carries TL nodes x TS samples x
// 2 chains in registers, so every staged coefficient feeds TS samples and every staged
// noise value feeds TL nodes.  A warp is LW l-lanes x (32/LW) s-lanes (lane = sl*LW + ll);
// there are NWL = 32/LW l-warps and NWS s-warps.  l-thread lt owns the node pairs
// (2 lt + 64 q, +1), q < TL/2, and for odd TL the node 64 (TL/2) + lt, so a warp's
// coefficient loads are conflict-free LDS.128 broadcasts over its s-lanes.
//
// Staging.  Per block of IB steps the node-minor tables mu, g [(toff_e + t) * Lp + l] are
// brought into shared memory by the bulk-copy engine (cp.async.bulk + mbarrier transaction
// count; one thread issues), and the noise of the CTA's samples by per-lane cp.async;
// both double buffered, one __syncthreads per block.
//
// Recover sum over l.  Per step each thread has 2*TS partial sums (left/right x samples)
// over its TL nodes; a shuffle reduce-scatter over the warp's LW l-lanes leaves one value
// per lane, which goes to a per-block partial buffer [IB][NWL][2][CS]; after the next
// barrier the partials are folded over the NWL l-warps in fixed order into an output tile
// [CS][m|1] kept in shared memory for the whole item (or, for edges too long for the tile,
// straight into u with read-add-write).  Every sum has a fixed order: results are
// bitwise reproducible for a given launch shape.
#pragma once

#include <cuda_pipeline.h>

#include "grf_internal.h"
#include "thomas.cuh"

namespace grf {
namespace sweep {

constexpr int IB = 8;          // steps per staging block
constexpr int NLT = 32;        // l-threads per CTA: a node round is 32 * TL nodes
constexpr size_t SMEM_MAX = 227 * 1024;

struct Args {
    DevGraph g;
    int32_t L, Lp;          // nodes; padded table row (multiple of 32 * TL * rounds)
    int32_t rounds;         // node rounds (Lp = rounds * 32 * TL)
    const double* cL;       // [Lp] c_L per node (zero padded)
    const double* cI;       // [L] c_I per node
    double kappa2;
    int32_t mass;           // 0 lumped, 1 consistent: the end coupling -b of A_IG (thomas.cuh edge_coef)
    const double* mu;       // [(off + t) * Lp + l]
    const double* gam;      // [(off + t) * Lp + l]
    int64_t S;
    const double* W;        // [s * N + dof]
    double* out;            // condense: ends; recover: u [s * N + dof]
    const double* uG;       // recover: [(s * V + v) * L + l]
    int32_t* counter;       // work-queue counter (zeroed by the launcher)
    int32_t chunks;         // sample tiles per edge
    int32_t n_items;        // E * chunks
    int32_t tile_ms;        // recover: max (m | 1) the shared-memory output tile holds (0: none)
    int32_t nk;             // recover: 1 if slot L is the correction node (edge_setup.cu; L < Lp)
    int32_t nst, nps;       // sweep3 recover: data / partial ring depths in use (set by its launch)
    int32_t* fits_out;      // recover, host-side query (no launch): 1 if every edge fits the output tile
    int32_t ablate;         // design studies only (env GRF_ABLATE, default 0), wrong results by construction:
                            // sweep2 bits 1 no output reduction, 2 no u_G loads, 4 no data waits; sweep3
                            // bits 32 no partial stores, 64 no u_G loads; kernel choice bits 8, 16, 128 (sweep.cu)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// global -> shared bulk copy (TMA engine, no tensor map); bytes multiple of 16, both 16B aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// the same wait for warps that are off the critical path (producers, fold warps): the thread may be
// suspended for up to `ns` nanoseconds per try instead of spinning on the issue slots it shares
// with the compute warps
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns = 1000) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAITS_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAITS_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(ns)
        : "memory");
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Compile-time shape of one kernel instance.
template <int TL, int TS, int LW, int NWS, bool REC>
struct Cfg {
    static constexpr int NWL = 32 / LW;             // l-warps
    static constexpr int SLW = 32 / LW;             // s-lanes per warp
    static constexpr int NT = 32 * NWL * NWS;       // threads per CTA
    static constexpr int CS = NWS * SLW * TS;       // samples per item (= the sample tile of ends / uG)
    static constexpr int CSL = CS == 32 ? 5 : (CS == 16 ? 4 : (CS == 8 ? 3 : (CS == 4 ? 2 : (CS == 2 ? 1 : 0))));
    static constexpr int NTAB = REC ? 2 : 1;        // staged tables: mu (, g)
    static constexpr int RN = NLT * TL;             // nodes per round
    // steps per staging block; the 1-warp (1-sample) instances stage less so more CTAs fit an SM
    static constexpr int IBK = TS == 1 ? (REC ? 8 : 16) : (REC ? 8 : 32);
    // recover with TS = 4: sample slot j of a thread is sample (j ^ sig(lane)); this makes
    // the reduce-scatter over the 8 l-lanes select-free (see reduce_store)
    static constexpr bool PERM = REC && TS == 4;
    static constexpr int NC = PERM ? 2 : 1;         // staged noise copies: natural, pair-swapped
    static constexpr size_t COEF = (size_t)2 * NTAB * IBK * RN * sizeof(double);
    static constexpr size_t WB = (size_t)2 * IBK * 2 * NC * CS * sizeof(double);
    static constexpr size_t PART = REC ? (size_t)2 * IBK * NWL * 2 * CS * sizeof(double) : 0;
    static constexpr size_t FIXED = 64 + COEF + WB + PART;
    static constexpr int WEL = IBK * 2 * NC * CS;   // staged noise elements per block
    static_assert(REC ? ((TS == 4 && (LW == 8 || LW == 4)) || (TS == 1 && LW == 32)) : true, "recover reduce shapes");
    static_assert((CS & (CS - 1)) == 0, "CS must be a power of two");
};

template <int TL, int TS, int LW, int NWS, bool REC, bool NK>
__global__ void __launch_bounds__(Cfg<TL, TS, LW, NWS, REC>::NT) sweep_kernel(Args A) {
    using C = Cfg<TL, TS, LW, NWS, REC>;
    constexpr int NWL = C::NWL, SLW = C::SLW, NT = C::NT, CS = C::CS, CSL = C::CSL, NTAB = C::NTAB, RN = C::RN;
    constexpr int IBK = C::IBK, NC = C::NC;
    constexpr bool PERM = C::PERM;
    constexpr int NP = TL / 2;               // node pairs per thread
    constexpr bool ODD = (TL & 1) != 0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ll = lane % LW, sl = lane / LW;
    const int lw = warp % NWL, sw = warp / NWL;
    const int lt = lw * LW + ll;             // l-thread 0..31
    const int st0 = (sw * SLW + sl) * TS;    // first sample (within the item) of this thread
    const int sig = PERM ? (((ll & 1) << 1) | ((ll >> 1) & 1)) : 0;
    const DevGraph& g = A.g;
    const int64_t N = g.N;
    const int L = A.L, Lp = A.Lp;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);           // [2]
    int* item_sh = reinterpret_cast<int*>(smem_raw + 16);           // [2] work-queue indices
    double* coef = reinterpret_cast<double*>(smem_raw + 64);         // [2][NTAB][IBK][RN]
    double* wbuf = coef + 2 * NTAB * IBK * RN;                       // [2][IBK][2][NC][CS]
    double* part = wbuf + 2 * IBK * 2 * NC * CS;                     // [2][IBK][NWL][2][CS] (REC)
    double* cLs = part + (REC ? 2 * IBK * NWL * 2 * CS : 0);         // [Lp] c_L (REC)
    double* otile = cLs + (REC ? A.Lp : 0);                          // [CS][tile_ms] (REC)

    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (REC)
        for (int i = tid; i < A.Lp; i += NT) cLs[i] = A.cL[i];  // zero padded past L
    __syncthreads();
    uint32_t phases = 0u;  // bit b: parity of the next completion of bar[b]

    // node slot (within a round) of this thread's node n (0..TL-1)
    auto slot = [&](int n) -> int { return (n < 2 * NP) ? (2 * lt + 64 * (n >> 1) + (n & 1)) : (64 * NP + lt); };

    // work queue, one item ahead: the index of the next item is fetched when the current one starts
    // and published at its end barrier, so the atomic's latency never stalls the CTA
    if (tid == 0) item_sh[0] = atomicAdd(A.counter, 1);
    __syncthreads();
    for (int cur = 0;; cur ^= 1) {
        const int it = item_sh[cur];
        if (it >= A.n_items) break;
        int next = 0;
        if (tid == 0) next = atomicAdd(A.counter, 1);
        const int e = g.edge_order[it / A.chunks];
        const int64_t c0 = (int64_t)(it % A.chunks) * CS;
        const int m = g.m[e];
        const int64_t off = g.off[e];
        const int64_t toff = g.toff[e];  // Thomas-table rows of the edge's (m, h) class
        const double h = g.h[e];
        const double inv_h = 1.0 / h;
        const int vu = g.eu[e], vv = g.ev[e];
        // coupling of node l's boundary rows to the vertex values: c_L/h (lumped), -b (consistent)
        auto beta_of = [&](int l) -> double {
            if (l >= L) return 0.0;
            return A.mass ? edge_coef(A.cI[l], A.cL[l], A.kappa2, h, 1).beta : cLs[l] * inv_h;
        };
        const int ms = m | 1;
        const bool in_tile = REC && ms <= A.tile_ms;
        int64_t sidx[TS];  // sample of slot j (clamped for loads; writes check c0 + st0 + (j ^ sig) < S)
#pragma unroll
        for (int j = 0; j < TS; ++j) {
            const int64_t s = c0 + st0 + (j ^ sig);
            sidx[j] = s < A.S ? s : A.S - 1;
        }
        // u_G of the edge's two vertices for this thread's samples: node l at uGu[j][l << CSL]
        // (layout [tile][v][l][cs], grf_internal.h) -- base pointers once per item
        const double* uGu[REC ? TS : 1];
        const double* uGv[REC ? TS : 1];
        if (REC) {
#pragma unroll
            for (int j = 0; j < TS; ++j) {
                uGu[j] = A.uG + ug_index(sidx[j], vu, 0, L, g.V, CSL);
                uGv[j] = A.uG + ug_index(sidx[j], vv, 0, L, g.V, CSL);
            }
        }

        if (m == 0 && !REC) {  // no interior: zero end values (ends layout [tile][l][code][CS], grf_internal.h)
            const int64_t tile = it % A.chunks;
            for (int x = tid; x < L * 2 * CS; x += NT) {
                const int l = x / (2 * CS), r = x % (2 * CS);
                A.out[((tile * L + l) * 2 * (int64_t)g.E + 2 * e) * CS + r] = 0.0;
            }
        }
        const int nblk = (m + IBK - 1) / IBK;

        for (int rd = 0; rd < (m == 0 ? 0 : A.rounds); ++rd) {
            const int rb = rd * RN;  // first node of the round
            double Y[TL][TS], Z[TL][TS];
            double g0[REC ? 1 : TL];
            if (REC) {
                // boundary rows (P310): f_0 += (c_L/h) u_left, f_{m-1} += (c_L/h) u_right; both
                // enter the chains at step 0 (mu_0 = 0).  The raw u_G loads are issued here and
                // scaled by beta after block 0's barrier (scale_boundary), so their latency
                // overlaps the staging of block 0.
#pragma unroll
                for (int n = 0; n < TL; ++n) {
                    const int l = rb + slot(n);
                    const bool ok = l < L;
#pragma unroll
                    for (int j = 0; j < TS; ++j) {
                        Y[n][j] = ok ? uGu[j][l << CSL] : 0.0;
                        Z[n][j] = ok ? uGv[j][l << CSL] : 0.0;
                    }
                }
            } else {
#pragma unroll
                for (int n = 0; n < TL; ++n) {
                    const int l = rb + slot(n);
                    g0[n] = l < L ? A.gam[toff * (int64_t)Lp + l] : 0.0;  // g_0 = g_{m-1} for the end values
#pragma unroll
                    for (int j = 0; j < TS; ++j) Y[n][j] = Z[n][j] = 0.0;
                }
            }

            auto stage = [&](int b) {
                const int t0 = b * IBK;
                const int nb = (m - t0) < IBK ? (m - t0) : IBK;
                const int buf = b & 1;
                if (tid == 0) {
                    fence_proxy_async();
                    constexpr uint32_t row = RN * sizeof(double);
                    mbar_expect_tx(&bar[buf], (uint32_t)(NTAB * nb) * row);
#pragma unroll
                    for (int tb = 0; tb < NTAB; ++tb) {
                        const double* tab = (tb == 0 ? A.mu : A.gam) + (toff + t0) * (int64_t)Lp + rb;
                        double* dst = coef + (buf * NTAB + tb) * IBK * RN;
                        if (A.rounds == 1) {
                            bulk_g2s(dst, tab, (uint32_t)nb * row, &bar[buf]);
                        } else {
                            for (int tt = 0; tt < nb; ++tt) bulk_g2s(dst + tt * RN, tab + tt * (int64_t)Lp, row, &bar[buf]);
                        }
                    }
                }
                // noise of the item's samples at left positions t0+tt and right positions m-1-t0-tt;
                // copy c = 1 holds the samples pair-swapped (sample s ^ 1 at index s)
                double* wb = wbuf + buf * IBK * 2 * NC * CS;
#pragma unroll
                for (int k = 0; k < (C::WEL + NT - 1) / NT; ++k) {
                    const int x = tid + k * NT;
                    if (x < C::WEL) {
                        const int tt = x % IBK, r = x / IBK;
                        const int s = r % CS, r2 = r / CS;
                        const int c = r2 % NC, side = r2 / NC;
                        if (tt < nb) {
                            int64_t sg = c0 + (c ? (s ^ 1) : s);
                            if (sg >= A.S) sg = A.S - 1;
                            const int pos = side ? (m - 1 - t0 - tt) : (t0 + tt);
                            __pipeline_memcpy_async(wb + ((tt * 2 + side) * NC + c) * CS + s, A.W + sg * N + off + pos,
                                                    8);
                        }
                    }
                }
                __pipeline_commit();
            };

            // fold block b's partial sums (over the NWL l-warps, fixed order) into the output.
            // Step t adds its left value to position t and its right value to position m-1-t;
            // a thread takes step t together with its mirror step m-1-t when both lie in this
            // block, so no two threads touch one position within a fold.
            auto fold = [&](int b) {
                const int t0 = b * IBK;
                const int nb = (m - t0) < IBK ? (m - t0) : IBK;
                const double* pb = part + (b & 1) * IBK * NWL * 2 * CS;
                auto psum = [&](int tt, int side, int s) {  // pairwise tree over the l-warps (fixed order)
                    double v[NWL];
#pragma unroll
                    for (int q = 0; q < NWL; ++q) v[q] = pb[((tt * NWL + q) * 2 + side) * CS + s];
#pragma unroll
                    for (int w = 1; w < NWL; w <<= 1) {
#pragma unroll
                        for (int q = 0; q + w < NWL; q += 2 * w) v[q] += v[q + w];
                    }
                    return v[0];
                };
                auto put = [&](int s, int p, double v, bool first) {
                    if (in_tile) {
                        double* d = otile + s * ms + p;
                        *d = first ? v : *d + v;
                    } else if (c0 + s < A.S) {
                        double* d = A.out + (c0 + s) * N + off + p;
                        *d = first ? v : *d + v;
                    }
                };
                for (int x = tid; x < nb * CS; x += NT) {
                    const int s = x % CS, tt = x / CS;
                    const int t = t0 + tt, tm = m - 1 - t;
                    const bool mirror_here = tm >= t0 && tm < t0 + nb;
                    if (mirror_here && tm < t) continue;  // handled with the mirror step
                    const double vl = psum(tt, 0, s), vr = psum(tt, 1, s);
                    if (tm == t) {
                        put(s, t, vl + vr, rd == 0);
                    } else if (mirror_here) {  // both visits of positions t and tm are in this block
                        const int ttm = tm - t0;
                        put(s, t, vl + psum(ttm, 1, s), rd == 0);
                        put(s, tm, vr + psum(ttm, 0, s), rd == 0);
                    } else {
                        const bool first = rd == 0 && t < tm;  // first visit of both t and tm is at min(t, tm)
                        put(s, t, vl, first);
                        put(s, tm, vr, first);
                    }
                }
            };

            stage(0);
            for (int b = 0; b < nblk; ++b) {
                const int t0 = b * IBK;
                const int nb = (m - t0) < IBK ? (m - t0) : IBK;
                const int buf = b & 1;
                mbar_wait(&bar[buf], (phases >> buf) & 1u);
                phases ^= 1u << buf;
                __pipeline_wait_prior(0);
                __syncthreads();  // block b staged and visible; block b-1 buffers and partials free/complete
                if (b + 1 < nblk) stage(b + 1);
                if (REC && b == 0) {  // Y = beta u_left, Z = beta u_right (both ends for m = 1)
#pragma unroll
                    for (int n = 0; n < TL; ++n) {
                        const double bt = beta_of(rb + slot(n));
#pragma unroll
                        for (int j = 0; j < TS; ++j) {
                            const double ul = Y[n][j], ur = Z[n][j];
                            Y[n][j] = bt * (m == 1 ? ul + ur : ul);
                            Z[n][j] = bt * (m == 1 ? ul + ur : ur);
                        }
                    }
                }
                const double* cmu = coef + (buf * NTAB + 0) * IBK * RN;
                const double* cga = coef + (buf * NTAB + 1) * IBK * RN;
                const double* wb = wbuf + buf * IBK * 2 * NC * CS;

                // noise of this thread's slots at step tt (left and right positions)
                auto load_w = [&](int tt, double (&wl)[TS], double (&wr)[TS]) {
                    if (TS == 1) {
                        wl[0] = wb[(tt * 2 + 0) * NC * CS + st0];
                        wr[0] = wb[(tt * 2 + 1) * NC * CS + st0];
                    } else {
                        const int cp = PERM ? (sig & 1) : 0, px = PERM ? (sig >> 1) : 0;
#pragma unroll
                        for (int q = 0; q < TS / 2; ++q) {
                            const int o = st0 + 2 * (q ^ px);
                            const double2 a = *reinterpret_cast<const double2*>(wb + ((tt * 2 + 0) * NC + cp) * CS + o);
                            const double2 c = *reinterpret_cast<const double2*>(wb + ((tt * 2 + 1) * NC + cp) * CS + o);
                            wl[2 * q] = a.x;
                            wl[2 * q + 1] = a.y;
                            wr[2 * q] = c.x;
                            wr[2 * q + 1] = c.y;
                        }
                    }
                };

                if (!REC) {
                    // step tt+1's multipliers and noise are loaded into registers while step tt's
                    // FMAs run (the last step re-loads its own row: no read past the block)
                    double wln[TS], wrn[TS], mon = 0.0;
                    double2 m2n[NP > 0 ? NP : 1];
                    auto ld = [&](int tt) {
                        load_w(tt, wln, wrn);
                        const double* rmu = cmu + tt * RN;
#pragma unroll
                        for (int q = 0; q < NP; ++q) m2n[q] = *reinterpret_cast<const double2*>(rmu + 2 * lt + 64 * q);
                        if (ODD) mon = rmu[64 * NP + lt];
                    };
                    ld(0);
#pragma unroll 2
                    for (int tt = 0; tt < nb; ++tt) {
                        double wl[TS], wr[TS], mo = mon;
                        double2 m2[NP > 0 ? NP : 1];
#pragma unroll
                        for (int j = 0; j < TS; ++j) {
                            wl[j] = wln[j];
                            wr[j] = wrn[j];
                        }
#pragma unroll
                        for (int q = 0; q < NP; ++q) m2[q] = m2n[q];
                        ld(tt + 1 < nb ? tt + 1 : tt);
#pragma unroll
                        for (int q = 0; q < NP; ++q) {
#pragma unroll
                            for (int j = 0; j < TS; ++j) {
                                Y[2 * q][j] = fma(-m2[q].x, Y[2 * q][j], wl[j]);
                                Z[2 * q][j] = fma(-m2[q].x, Z[2 * q][j], wr[j]);
                                Y[2 * q + 1][j] = fma(-m2[q].y, Y[2 * q + 1][j], wl[j]);
                                Z[2 * q + 1][j] = fma(-m2[q].y, Z[2 * q + 1][j], wr[j]);
                            }
                        }
                        if (ODD) {
#pragma unroll
                            for (int j = 0; j < TS; ++j) {
                                Y[TL - 1][j] = fma(-mo, Y[TL - 1][j], wl[j]);
                                Z[TL - 1][j] = fma(-mo, Z[TL - 1][j], wr[j]);
                            }
                        }
                    }
                } else {
                    // generic step: left chain gives -g mu Y_{t-1} = g (Y_t - f_t) to position t, right
                    // chain g Z to m-1-t.  With the correction node (A.nk) the left chain gives g Y_t
                    // instead (no g*mu product): the node's g_t = -G_t/2 and Y = Z = noise remove the
                    // sum over nodes of g_t f_t, half through each chain (edge_setup.cu)
                    auto body_mid = [&](int tt, double (&aL)[TS], double (&aR)[TS]) {
                        double wl[TS], wr[TS];
                        load_w(tt, wl, wr);
                        const double* rmu = cmu + tt * RN;
                        const double* rga = cga + tt * RN;
#pragma unroll
                        for (int j = 0; j < TS; ++j) aL[j] = aR[j] = 0.0;
                        if constexpr (NK) {
#pragma unroll
                            for (int q = 0; q < NP; ++q) {
                                const double2 m2 = *reinterpret_cast<const double2*>(rmu + 2 * lt + 64 * q);
                                const double2 g2 = *reinterpret_cast<const double2*>(rga + 2 * lt + 64 * q);
#pragma unroll
                                for (int j = 0; j < TS; ++j) {
                                    Y[2 * q][j] = fma(-m2.x, Y[2 * q][j], wl[j]);
                                    aL[j] = fma(g2.x, Y[2 * q][j], aL[j]);
                                    Z[2 * q][j] = fma(-m2.x, Z[2 * q][j], wr[j]);
                                    aR[j] = fma(g2.x, Z[2 * q][j], aR[j]);
                                    Y[2 * q + 1][j] = fma(-m2.y, Y[2 * q + 1][j], wl[j]);
                                    aL[j] = fma(g2.y, Y[2 * q + 1][j], aL[j]);
                                    Z[2 * q + 1][j] = fma(-m2.y, Z[2 * q + 1][j], wr[j]);
                                    aR[j] = fma(g2.y, Z[2 * q + 1][j], aR[j]);
                                }
                            }
                            if (ODD) {
                                const double mu = rmu[64 * NP + lt], gg = rga[64 * NP + lt];
#pragma unroll
                                for (int j = 0; j < TS; ++j) {
                                    Y[TL - 1][j] = fma(-mu, Y[TL - 1][j], wl[j]);
                                    aL[j] = fma(gg, Y[TL - 1][j], aL[j]);
                                    Z[TL - 1][j] = fma(-mu, Z[TL - 1][j], wr[j]);
                                    aR[j] = fma(gg, Z[TL - 1][j], aR[j]);
                                }
                            }
                        } else {
#pragma unroll
                            for (int q = 0; q < NP; ++q) {
                                const double2 m2 = *reinterpret_cast<const double2*>(rmu + 2 * lt + 64 * q);
                                const double2 g2 = *reinterpret_cast<const double2*>(rga + 2 * lt + 64 * q);
                                const double k0 = g2.x * m2.x, k1 = g2.y * m2.y;
#pragma unroll
                                for (int j = 0; j < TS; ++j) {
                                    aL[j] = fma(-k0, Y[2 * q][j], aL[j]);
                                    Y[2 * q][j] = fma(-m2.x, Y[2 * q][j], wl[j]);
                                    Z[2 * q][j] = fma(-m2.x, Z[2 * q][j], wr[j]);
                                    aR[j] = fma(g2.x, Z[2 * q][j], aR[j]);
                                    aL[j] = fma(-k1, Y[2 * q + 1][j], aL[j]);
                                    Y[2 * q + 1][j] = fma(-m2.y, Y[2 * q + 1][j], wl[j]);
                                    Z[2 * q + 1][j] = fma(-m2.y, Z[2 * q + 1][j], wr[j]);
                                    aR[j] = fma(g2.y, Z[2 * q + 1][j], aR[j]);
                                }
                            }
                            if (ODD) {
                                const double mu = rmu[64 * NP + lt], gg = rga[64 * NP + lt];
                                const double nk = gg * mu;
#pragma unroll
                                for (int j = 0; j < TS; ++j) {
                                    aL[j] = fma(-nk, Y[TL - 1][j], aL[j]);
                                    Y[TL - 1][j] = fma(-mu, Y[TL - 1][j], wl[j]);
                                    Z[TL - 1][j] = fma(-mu, Z[TL - 1][j], wr[j]);
                                    aR[j] = fma(gg, Z[TL - 1][j], aR[j]);
                                }
                            }
                        }
                    };
                    // step 0: mu_0 = 0, Y_0 = f_0 (W + the preloaded boundary term), no left contribution
                    auto body_first = [&](double (&aL)[TS], double (&aR)[TS]) {
                        double wl[TS], wr[TS];
                        load_w(0, wl, wr);
                        const double* rga = cga;
#pragma unroll
                        for (int j = 0; j < TS; ++j) aL[j] = aR[j] = 0.0;
#pragma unroll
                        for (int n = 0; n < TL; ++n) {
                            const double gg = rga[slot(n)];
#pragma unroll
                            for (int j = 0; j < TS; ++j) {
                                Y[n][j] += wl[j];
                                Z[n][j] += wr[j];
                                aR[j] = fma(gg, Z[n][j], aR[j]);
                            }
                        }
                    };
                    // step m-1 (m >= 2): the left chain reaches position m-1 (f += beta u_right), the right
                    // chain position 0 (f += beta u_left)
                    auto body_last = [&](int tt, double (&aL)[TS], double (&aR)[TS]) {
                        double wl[TS], wr[TS];
                        load_w(tt, wl, wr);
                        const double* rmu = cmu + tt * RN;
                        const double* rga = cga + tt * RN;
#pragma unroll
                        for (int j = 0; j < TS; ++j) aL[j] = aR[j] = 0.0;
#pragma unroll
                        for (int n = 0; n < TL; ++n) {
                            const int sn = slot(n);
                            const int l = rb + sn;
                            const bool ok = l < L;
                            const double beta = beta_of(l);
                            const double mu = rmu[sn], gg = rga[sn];
                            const double nk = gg * mu;
#pragma unroll
                            for (int j = 0; j < TS; ++j) {
                                const double ul = ok ? uGu[j][l << CSL] : 0.0;
                                const double ur = ok ? uGv[j][l << CSL] : 0.0;
                                aL[j] = fma(-nk, Y[n][j], aL[j]);
                                Y[n][j] = fma(beta, ur, fma(-mu, Y[n][j], wl[j]));
                                Z[n][j] = fma(beta, ul, fma(-mu, Z[n][j], wr[j]));
                                aR[j] = fma(gg, Z[n][j], aR[j]);
                            }
                        }
                    };
                    // sum the step's partials over the warp's l-lanes and store them for the fold
                    double* pb = part + buf * IBK * NWL * 2 * CS + lw * 2 * CS + st0 + sig;
                    auto reduce_store = [&](double (&aL)[TS], double (&aR)[TS], int tt) {
                        if (TS == 4) {
                            // slot j holds sample j ^ sig; sig bit 1 = ll bit 0, sig bit 0 = ll bit 1, so the
                            // partner's slots {2,3} (xor 1) and slot 1 (xor 2) are this lane's slots {0,1} / 0
                            aL[0] += __shfl_xor_sync(0xffffffffu, aL[2 % TS], 1);
                            aL[1 % TS] += __shfl_xor_sync(0xffffffffu, aL[3 % TS], 1);
                            aR[0] += __shfl_xor_sync(0xffffffffu, aR[2 % TS], 1);
                            aR[1 % TS] += __shfl_xor_sync(0xffffffffu, aR[3 % TS], 1);
                            aL[0] += __shfl_xor_sync(0xffffffffu, aL[1 % TS], 2);
                            aR[0] += __shfl_xor_sync(0xffffffffu, aR[1 % TS], 2);
                            if (LW == 8) {
                                aL[0] += __shfl_xor_sync(0xffffffffu, aL[0], 4);
                                aR[0] += __shfl_xor_sync(0xffffffffu, aR[0], 4);
                            }
                            if ((ll & 4) == 0) {
                                pb[tt * NWL * 2 * CS] = aL[0];
                                pb[tt * NWL * 2 * CS + CS] = aR[0];
                            }
                        } else {
#pragma unroll
                            for (int o = 16; o >= 1; o >>= 1) {
                                aL[0] += __shfl_xor_sync(0xffffffffu, aL[0], o);
                                aR[0] += __shfl_xor_sync(0xffffffffu, aR[0], o);
                            }
                            if (ll == 0) {
                                pb[tt * NWL * 2 * CS] = aL[0];
                                pb[tt * NWL * 2 * CS + CS] = aR[0];
                            }
                        }
                    };
                    // software pipeline: the reduction of step tt-1 is independent of step tt's FMAs, so
                    // the scheduler overlaps the shuffle latency with them
                    const bool last_here = (t0 + nb == m) && (m > 1);
                    if (last_here && nb > 1) {  // the last step re-reads both vertices' u_G: pull it into L1 now
#pragma unroll
                        for (int n = 0; n < TL; ++n) {
                            const int l = rb + slot(n);
                            if (l < L) {
#pragma unroll
                                for (int j = 0; j < TS; ++j) {
                                    asm volatile("prefetch.global.L1 [%0];" ::"l"(uGu[j] + (l << CSL)));
                                    asm volatile("prefetch.global.L1 [%0];" ::"l"(uGv[j] + (l << CSL)));
                                }
                            }
                        }
                    }
                    const int tend = last_here ? nb - 1 : nb;
                    double pL[TS], pR[TS];
                    bool pend = false;
                    int tt = 0;
                    if (t0 == 0) {
                        body_first(pL, pR);
                        tt = 1;
                        pend = true;
                    } else if (tend > 0) {
                        body_mid(0, pL, pR);
                        tt = 1;
                        pend = true;
                    }
                    // steps in pairs with alternating partial registers (no register copies)
                    for (; tt + 1 < tend; tt += 2) {
                        double aL[TS], aR[TS];
                        body_mid(tt, aL, aR);
                        reduce_store(pL, pR, tt - 1);
                        body_mid(tt + 1, pL, pR);
                        reduce_store(aL, aR, tt);
                    }
                    if (tt < tend) {
                        double aL[TS], aR[TS];
                        body_mid(tt, aL, aR);
                        reduce_store(pL, pR, tt - 1);
#pragma unroll
                        for (int j = 0; j < TS; ++j) {
                            pL[j] = aL[j];
                            pR[j] = aR[j];
                        }
                        ++tt;
                    }
                    if (last_here) {
                        double aL[TS], aR[TS];
                        body_last(nb - 1, aL, aR);
                        if (pend) reduce_store(pL, pR, nb - 2);
#pragma unroll
                        for (int j = 0; j < TS; ++j) {
                            pL[j] = aL[j];
                            pR[j] = aR[j];
                        }
                        pend = true;
                    }
                    if (pend) reduce_store(pL, pR, nb - 1);
                    // block b-1's partials are complete since this block's barrier and are not
                    // overwritten before the next one: fold them while other warps still compute
                    if (b > 0) fold(b - 1);
                }
            }
            if (REC) {
                __syncthreads();
                fold(nblk - 1);
            } else {
                // w_1 = g_0 Z (right sweep end, position 0), w_m = g_0 Y (left sweep end); g_0 = g_{m-1}.
                // ends layout [tile][l][code][CS]: the item's 2 codes x CS samples are contiguous per l;
                // slots past S land in the tile's padding (never read)
                const int64_t tile = it % A.chunks;
#pragma unroll
                for (int n = 0; n < TL; ++n) {
                    const int l = rb + slot(n);
                    if (l < L) {
                        double* o = A.out + ((tile * L + l) * 2 * (int64_t)g.E + 2 * e) * CS + st0;
                        if (TS % 2 == 0) {  // 16-byte stores: st0 and CS are multiples of TS
#pragma unroll
                            for (int j = 0; j < TS; j += 2) {
                                *reinterpret_cast<double2*>(o + j) = make_double2(g0[n] * Z[n][j], g0[n] * Z[n][j + 1 < TS ? j + 1 : j]);
                                *reinterpret_cast<double2*>(o + CS + j) =
                                    make_double2(g0[n] * Y[n][j], g0[n] * Y[n][j + 1 < TS ? j + 1 : j]);
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < TS; ++j) {
                                o[j] = g0[n] * Z[n][j];
                                o[CS + j] = g0[n] * Y[n][j];
                            }
                        }
                    }
                }
            }
        }
        if (in_tile) {
            __syncthreads();
            const float inv_m = 1.0f / (float)m;  // x / m without an integer division (exact after the fix-up)
            for (int x = tid; x < CS * m; x += NT) {
                int s = (int)((float)x * inv_m);
                s -= (s * m > x);
                s += ((s + 1) * m <= x);
                const int p = x - s * m;
                if (c0 + s < A.S) A.out[(c0 + s) * N + off + p] = otile[s * ms + p];
            }
        }
        if (tid == 0) item_sh[cur ^ 1] = next;
        __syncthreads();  // next index visible; output tile and staging buffers free
    }
}

// One instance: threads = NT, items = E * ceil(S / CS), persistent CTAs over an atomic queue.
// NK (recover only): the interior steps use the correction-node form (A.nk, edge_setup.cu).
template <int TL, int TS, int LW, int NWS, bool REC, bool NK>
cudaError_t launch(Args a, cudaStream_t st) {
    using C = Cfg<TL, TS, LW, NWS, REC>;
    a.chunks = (int32_t)((a.S + C::CS - 1) / C::CS);
    a.n_items = a.g.E * a.chunks;
    size_t smem = C::FIXED + (REC ? (size_t)a.Lp * sizeof(double) : 0);
    a.tile_ms = 0;
    if (REC) {
        // the output tile holds edges with (m | 1) <= tile_ms; sized for the longest edge if it fits
        const int want = a.g.max_m | 1;
        const size_t room = SMEM_MAX > smem ? SMEM_MAX - smem : 0;
        const int fit = (int)(room / ((size_t)C::CS * sizeof(double)));
        a.tile_ms = want <= fit ? want : (fit >= 1 ? ((fit - 1) | 1) : 0);
        smem += (size_t)C::CS * a.tile_ms * sizeof(double);
        if (a.fits_out) {  // query only: does the output leave the kernel by plain tile stores?
            *a.fits_out = a.tile_ms >= want;
            return cudaSuccess;
        }
    }
    cudaError_t e = cudaFuncSetAttribute(sweep_kernel<TL, TS, LW, NWS, REC, NK>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(a.counter, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return e;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_kernel<TL, TS, LW, NWS, REC, NK>, C::NT, smem);
    if (per_sm < 1) per_sm = 1;
    int blocks = (a.g.n_sm > 0 ? a.g.n_sm : 148) * per_sm;
    if (blocks > a.n_items) blocks = a.n_items;
    sweep_kernel<TL, TS, LW, NWS, REC, NK><<<blocks, C::NT, smem, st>>>(a);
    return cudaGetLastError();
}

// Sample mapping (the node tile TL is fixed by the plan's Lp):
//   V2: TS = 4, LW = 8, NWS = 2  (CTA = 4 l-warps x 2 s-warps, 32 samples per item)   S >= 17
//       (recover: LW = 4, NWS = 1 -- CTA = 8 l-warps of 4 l-lanes x 8 s-lanes, same 32 samples:
//        two shuffle levels per step instead of three, the fold sums 8 warp partials)
//   V1: TS = 4, LW = 8, NWS = 1  (CTA = 4 l-warps, 16 samples per item)               9 <= S <= 16
//   V0: TS = 1, LW = 32, NWS = 1 (CTA = 1 warp, 1 sample per item)                    S <= 8
enum Variant { V0 = 0, V1 = 1, V2 = 2 };
inline Variant variant_for(int64_t S) { return S >= 17 ? V2 : (S >= 9 ? V1 : V0); }

template <bool REC, int V, bool NK = false>
cudaError_t launch_v(int tl, Args a, cudaStream_t st) {
    constexpr int TS = V == V0 ? 1 : 4;
    constexpr int LW = V == V0 ? 32 : ((REC && V == V2) ? 4 : 8);
    constexpr int NWS = (V == V2 && !REC) ? 2 : 1;
    switch (tl) {
        case 1: return launch<1, TS, LW, NWS, REC, NK>(a, st);
        case 2: return launch<2, TS, LW, NWS, REC, NK>(a, st);
        case 3: return launch<3, TS, LW, NWS, REC, NK>(a, st);
        case 4: return launch<4, TS, LW, NWS, REC, NK>(a, st);
        case 5: return launch<5, TS, LW, NWS, REC, NK>(a, st);
        case 6: return launch<6, TS, LW, NWS, REC, NK>(a, st);
        case 7: return launch<7, TS, LW, NWS, REC, NK>(a, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace sweep
}  // namespace grf
