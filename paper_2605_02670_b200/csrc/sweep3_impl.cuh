// K5 recover + quadrature sum (PAPER.md P300-324) and K3 condense (P197-239) for sample tiles of
// 32 samples, warp-specialised.  Recover (sweep3_kernel):
//   * consumers (warps 0-7, 232 registers): 8 l-warps of CL l-lanes x 32/CL s-lanes; a thread
//     carries TLT = 4 TL / CL nodes x CL samples x 2 chains (56 chains at TL = 7) through the
//     correction-node interior steps; per step the partial sums over its nodes are reduced over
//     the warp's CL l-lanes by a select-free shuffle reduce-scatter (sample slot j of a lane holds
//     sample j ^ sig(lane): one level for CL = 2, the default; two for CL = 4, the mapping of
//     sweep_impl.cuh's V2 instance, GRF_ABLATE bit 256) and stored per l-warp into an NPS-deep
//     ring of partial buffers (pfull / pempty mbarriers);
//   * warp 8 (producer) streams the coefficient rows (bulk copies) and the noise (cp.async) into
//     an NST-deep ring of stages (full / empty mbarriers), as in sweep2_impl.cuh;
//   * warps 9-11 (fold warps) add the 8 l-warp partials of every block in fixed order into the
//     item's output tile [CS][m|1] (or into u for edges too long for it) and write the tile out
//     at the item's end; the ring depths give way to the tile (launch).
// No block-wide barrier anywhere after the prologue: the consumers wait only for staged data
// and for a free partial buffer, the fold warps for complete partials.  Results are bitwise
// reproducible (fixed shuffle and fold orders).  Condense (sweep3c_kernel, further below):
// chains only, the producer warpgroup streams the stages, every consumer writes its own end
// values.
#pragma once

#include "sweep2_impl.cuh"

namespace grf {
namespace sweep3 {

using sweep::Args;
using sweep::bulk_g2s;
using sweep::fence_proxy_async;
using sweep::mbar_expect_tx;
using sweep::mbar_init;
using sweep::mbar_wait;
using sweep::mbar_wait_sleep;
using sweep::smem_u32;
using sweep2::cp_async8;
using sweep2::cpasync_arrive_noinc;
using sweep2::ItemDesc;
using sweep2::mbar_arrive;

constexpr int NCW = 8;       // consumer (l-)warps
constexpr int NFW = 3;       // fold warps
constexpr int TS = 4, LW = 4, SLW = 8, NWL = 8;
constexpr int CS = SLW * TS;  // 32 samples per item
constexpr int CSL = 5;
constexpr int NT = (NCW + 4) * 32;
constexpr int IBK = 8;       // steps per stage
constexpr int NST = 3;       // data ring depth (max; A.nst in use, see launch)
constexpr bool K5_GLATE = true;   // g rows loaded after the chain updates (config 3 K5 5.69 -> 5.66 ms)
constexpr int K5_SLMAX = 6;       // straight-line full blocks for TL <= K5_SLMAX
constexpr int NPS = 2;       // partial ring depth (max; A.nps in use: 1 when that lets the output tile fit)
constexpr int NC = 2;        // noise copies: natural, pair-swapped
constexpr int WROW = CS + 4; // skewed noise row
constexpr int WEL = IBK * 2 * NC * WROW;
constexpr int PEL = IBK * NWL * 2 * CS;  // partial doubles per partial stage
constexpr size_t HDR = 1024;

// what the fold warps need to know about a block (written by consumer warp 0 with its partials)
struct BlockDesc {
    int32_t it, m, t0, nb, rd, last;  // last: the item's final block (fold warps write the tile out)
    int64_t off, c0;
};

template <int TL>
struct Cfg {
    static constexpr int RN = 32 * TL;
    static constexpr size_t STAGE1 = (size_t)(2 * IBK * RN + WEL) * sizeof(double);  // one data stage
    static constexpr size_t PART1 = (size_t)PEL * sizeof(double);                     // one partial stage
};

template <int TL, int NSTT, int CL>
__global__ void __launch_bounds__(NT, 1) sweep3_kernel(Args A) {
    using C = Cfg<TL>;
    constexpr int RN = C::RN;
    constexpr int NP = TL / 2;
    constexpr bool ODD = (TL & 1) != 0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const DevGraph& g = A.g;
    const int64_t N = g.N;
    const int L = A.L, Lp = A.Lp;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);     // [NST]
    uint64_t* empty = full + NST;                                // [NST]
    uint64_t* pfull = empty + NST;                               // [NPS]
    uint64_t* pempty = pfull + NPS;                              // [NPS]
    ItemDesc* header = reinterpret_cast<ItemDesc*>(pempty + NPS);  // [NST]
    BlockDesc* phdr = reinterpret_cast<BlockDesc*>(header + NST);  // [NPS]
    constexpr int nst = NSTT;
    const int nps = A.nps;
    double* coef = reinterpret_cast<double*>(smem_raw + HDR);   // [nst][2][IBK][RN]
    double* wbuf = coef + nst * 2 * IBK * RN;                    // [nst][IBK][2 side][NC][WROW]
    double* part = wbuf + nst * WEL;                             // [nps][IBK][NWL][2][CS]
    double* cLs = part + nps * PEL;                              // [Lp] c_L
    double* otile = cLs + Lp;                                    // [CS][tile_ms]

    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 33);    // producer lane 0's expect_tx arrive + 32 cp.async arrivals
            mbar_init(&empty[s], NCW);  // one release per consumer warp
        }
        for (int s = 0; s < NPS; ++s) {
            mbar_init(&pfull[s], NCW);   // every l-warp's partials of the block
            mbar_init(&pempty[s], NFW);  // every fold warp done with them
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < Lp; i += NT) cLs[i] = A.cL[i];  // zero padded past L
    __syncthreads();

    // ------------------------------------------------------------------------------------ producer
    if (warp >= NCW) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
        if (warp == NCW) {
            int stage = 0;
            uint32_t use = 0;
            ItemDesc cur{};
            auto produce = [&](int item_hdr, int64_t c0, int m, int64_t off, int64_t toff, int rd, int t0, int nb) {
                mbar_wait_sleep(&empty[stage], ((use >> stage) & 1u) ^ 1u);
                if (lane == 0) {
                    header[stage] = cur;
                    header[stage].it = item_hdr;
                    fence_proxy_async();
                    mbar_expect_tx(&full[stage], (uint32_t)(2 * nb * RN * sizeof(double)));
                }
                __syncwarp();
                if (nb > 0) {
                    double* cdst = coef + stage * 2 * IBK * RN;
                    if (A.rounds == 1) {
                        if (lane < 2)
                            bulk_g2s(cdst + lane * IBK * RN, (lane == 0 ? A.mu : A.gam) + (toff + t0) * (int64_t)Lp,
                                     (uint32_t)(nb * RN * sizeof(double)), &full[stage]);
                    } else {
                        for (int x = lane; x < 2 * nb; x += 32) {
                            const int tb = x / nb, tt = x % nb;
                            bulk_g2s(cdst + (tb * IBK + tt) * RN,
                                     (tb == 0 ? A.mu : A.gam) + (toff + t0 + tt) * (int64_t)Lp + rd * RN,
                                     (uint32_t)(RN * sizeof(double)), &full[stage]);
                        }
                    }
                    // 4 noise rows (side, copy, sample) per lane
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int row = lane + 32 * q;
                        const int side = row & 1, c = (row >> 1) & 1, s = row >> 2;
                        int64_t sg = c0 + (c ? (s ^ 1) : s);
                        if (sg >= A.S) sg = A.S - 1;
                        const double* src = A.W + sg * N + off + (side ? (m - 1 - t0) : t0);
                        const int dstep = side ? -1 : 1;
                        double* dst = wbuf + stage * WEL + (side * NC + c) * WROW + s;
                        for (int tt = 0; tt < nb; ++tt) cp_async8(dst + tt * 2 * NC * WROW, src + dstep * tt);
                    }
                }
                cpasync_arrive_noinc(&full[stage]);
                use ^= 1u << stage;
                stage = stage + 1 == nst ? 0 : stage + 1;
            };
            for (;;) {
                int it = 0;
                if (lane == 0) it = atomicAdd(A.counter, 1);
                it = __shfl_sync(0xffffffffu, it, 0);
                if (it >= A.n_items) {
                    produce(-1, 0, 0, 0, 0, 0, 0, 0);
                    break;
                }
                const int e = g.edge_order[it / A.chunks];
                const int m = g.m[e];
                if (m == 0) continue;  // nothing to recover: the vertex values come from vertex_sum
                const int64_t c0 = (int64_t)(it % A.chunks) * CS;
                const int64_t off = g.off[e], toff = g.toff[e];
                cur.it = it;
                cur.e = e;
                cur.m = m;
                cur.vu = g.eu[e];
                cur.vv = g.ev[e];
                cur.off = off;
                cur.toff = toff;
                cur.h = g.h[e];
                if (lane < 2) {  // the consumers' round-start u_G rows of this item: into L2 now
                    const int v = lane ? cur.vv : cur.vu;
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                     A.uG + (((it % A.chunks) * g.V + v) * (int64_t)L << CSL)),
                                 "r"((uint32_t)(L * CS * sizeof(double)))
                                 : "memory");
                }
                for (int rd = 0; rd < A.rounds; ++rd)
                    for (int t0 = 0; t0 < m; t0 += IBK) produce(it, c0, m, off, toff, rd, t0, min(IBK, m - t0));
            }
            return;
        }
        // ---------------------------------------------------------------------------- fold warps
        const int ftid = tid - (NCW + 1) * 32;  // 0 .. NFW*32-1
        auto fbar = []() { asm volatile("bar.sync 2, 96;" ::: "memory"); };
        int ps = 0;
        uint32_t puse = 0;
        for (;;) {
            mbar_wait_sleep(&pfull[ps], (puse >> ps) & 1u);
            const BlockDesc bd = phdr[ps];
            if (bd.it < 0) break;
            const int m = bd.m, t0 = bd.t0, nb = bd.nb, rd = bd.rd;
            const int ms = m | 1;
            const bool in_tile = ms <= A.tile_ms;
            const double* pb = part + ps * PEL;
            // step t adds its left value to position t and its right value to position m-1-t; a thread
            // takes step t together with its mirror step m-1-t when both lie in this block, so no two
            // threads touch one position within a fold; the fold order over l-warps is a fixed tree
            auto psum = [&](int tt, int side, int s) {
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
                } else if (bd.c0 + s < A.S) {
                    double* d = A.out + (bd.c0 + s) * N + bd.off + p;
                    *d = first ? v : *d + v;
                }
            };
            for (int x = ftid; x < nb * CS; x += NFW * 32) {
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
            // every fold warp is done with this block before any of them folds the next one (a
            // position's two visits may lie in different blocks and different fold warps)
            fbar();
            if (lane == 0) mbar_arrive(&pempty[ps]);  // the partials are consumed (the tile is ours)
            puse ^= 1u << ps;
            ps = ps + 1 == nps ? 0 : ps + 1;
            if (bd.last && in_tile) {  // the item's output tile -> u (coalesced), then reusable
                for (int x = ftid; x < CS * m; x += NFW * 32) {
                    const int s = x / m, p = x - s * m;
                    if (bd.c0 + s < A.S) A.out[(bd.c0 + s) * N + bd.off + p] = otile[s * ms + p];
                }
                fbar();
            }
        }
        return;
    }

    // ------------------------------------------------------------------------------------ consumers
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
    // consumer mapping: CL l-lanes x (32 / CL) s-lanes per warp, TSC = CL samples and TLT nodes per
    // thread (CL = 4: the sweep_impl.cuh V2 tile; CL = 2: twice the nodes per thread, one
    // reduce-scatter level instead of two)
    constexpr int LWC = CL, TSC = CL, NLT = NWL * CL, TLT = RN / NLT, NPT = TLT / 2;
    constexpr bool ODDT = (TLT & 1) != 0;
    static_assert(TLT * NLT == RN, "node slots");
    const int ll = lane % LWC, sl = lane / LWC;
    const int lw = warp;                    // l-warp
    const int lt = lw * LWC + ll;           // l-thread 0..NLT-1
    const int st0 = sl * TSC;                // first sample (within the item) of this thread
    const int sig = CL == 4 ? (((ll & 1) << 1) | ((ll >> 1) & 1)) : ll;  // sample slot j holds sample j ^ sig
    int stage = 0, ps = 0;
    uint32_t use = 0, puse = 0;
    auto acquire = [&]() { mbar_wait(&full[stage], (use >> stage) & 1u); };
    auto release = [&]() {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        use ^= 1u << stage;
        stage = stage + 1 == nst ? 0 : stage + 1;
    };
    auto slot = [&](int n) -> int { return (n < 2 * NPT) ? (2 * lt + 2 * NLT * (n >> 1) + (n & 1)) : (2 * NLT * NPT + lt); };

    for (;;) {
        acquire();
        const ItemDesc d = header[stage];
        const int it = d.it;
        if (it < 0) {
            // end of the work: tell the fold warps (they wait on the next partial stage)
            mbar_wait(&pempty[ps], ((puse >> ps) & 1u) ^ 1u);
            if (warp == 0 && lane == 0) phdr[ps].it = -1;
            __syncwarp();
            if (lane == 0) mbar_arrive(&pfull[ps]);
            break;
        }
        const int e = d.e;
        const int64_t c0 = (int64_t)(it % A.chunks) * CS;
        const int m = d.m;
        const int64_t toff = d.toff;
        const double h = d.h;
        const double inv_h = 1.0 / h;
        const int vu = d.vu, vv = d.vv;
        (void)e;
        auto beta_of = [&](int l) -> double {
            if (l >= L) return 0.0;
            return A.mass ? edge_coef(A.cI[l], A.cL[l], A.kappa2, h, 1).beta : cLs[l] * inv_h;
        };
        int64_t sidx[TSC];  // sample of slot j (clamped for loads)
#pragma unroll
        for (int j = 0; j < TSC; ++j) {
            const int64_t s = c0 + st0 + (j ^ sig);
            sidx[j] = s < A.S ? s : A.S - 1;
        }
        const double* uGu[TSC];
        const double* uGv[TSC];
#pragma unroll
        for (int j = 0; j < TSC; ++j) {
            uGu[j] = A.uG + ug_index(sidx[j], vu, 0, L, g.V, CSL);
            uGv[j] = A.uG + ug_index(sidx[j], vv, 0, L, g.V, CSL);
        }
        const int nblk = (m + IBK - 1) / IBK;
        for (int rd = 0; rd < A.rounds; ++rd) {
            const int rb = rd * RN;
            if (rd > 0) acquire();
            double Y[TLT][TSC], Z[TLT][TSC];
            // boundary rows (P310): Y = beta u_left, Z = beta u_right enter at step 0 (mu_0 = 0)
#pragma unroll
            for (int n = 0; n < TLT; ++n) {
                const int l = rb + slot(n);
                const bool ok = l < L;
                const double bt = beta_of(l);
#pragma unroll
                for (int j = 0; j < TSC; ++j) {
                    const bool ld = ok && !(A.ablate & 64);
                    const double ul = ld ? uGu[j][l << CSL] : 0.0, ur = ld ? uGv[j][l << CSL] : 0.0;
                    Y[n][j] = bt * (m == 1 ? ul + ur : ul);
                    Z[n][j] = bt * (m == 1 ? ul + ur : ur);
                }
            }
            for (int b = 0; b < nblk; ++b) {
                if (b > 0) acquire();
                const int t0 = b * IBK;
                const int nb = min(IBK, m - t0);
                const double* cmu = coef + stage * 2 * IBK * RN;
                const double* cga = cmu + IBK * RN;
                const double* wb = wbuf + stage * WEL;
                // a free partial buffer (the fold warps are at most NPS blocks behind)
                mbar_wait(&pempty[ps], ((puse >> ps) & 1u) ^ 1u);
                double* pbase = part + ps * PEL;
                if (warp == 0 && lane == 0) {
                    BlockDesc bd;
                    bd.it = it;
                    bd.m = m;
                    bd.t0 = t0;
                    bd.nb = nb;
                    bd.rd = rd;
                    bd.last = (rd == A.rounds - 1) && (b == nblk - 1);
                    bd.off = d.off;
                    bd.c0 = c0;
                    phdr[ps] = bd;
                }
                auto load_w = [&](int tt, double (&wl)[TSC], double (&wr)[TSC]) {
                    const int cp = sig & 1, px = sig >> 1;
#pragma unroll
                    for (int q = 0; q < TSC / 2; ++q) {
                        const int o = st0 + 2 * (q ^ px);
                        const double2 a = *reinterpret_cast<const double2*>(wb + ((tt * 2 + 0) * NC + cp) * WROW + o);
                        const double2 c = *reinterpret_cast<const double2*>(wb + ((tt * 2 + 1) * NC + cp) * WROW + o);
                        wl[2 * q] = a.x;
                        wl[2 * q + 1] = a.y;
                        wr[2 * q] = c.x;
                        wr[2 * q + 1] = c.y;
                    }
                };
                // interior step: correction-node form (both chains contribute g X_t)
                auto body_mid = [&](int tt, double (&aL)[TSC], double (&aR)[TSC]) {
                    double wl[TSC], wr[TSC];
                    load_w(tt, wl, wr);
                    const double* rmu = cmu + tt * RN;
                    const double* rga = cga + tt * RN;
#pragma unroll
                    for (int j = 0; j < TSC; ++j) aL[j] = aR[j] = 0.0;
                    // all chain updates first, then the accumulations (each uses a chain value computed
                    // >= TLT*TSC*2 FMAs earlier: no back-to-back DFMA dependencies)
                    double2 g2s[NPT > 0 ? NPT : 1];
#pragma unroll
                    for (int q = 0; q < NPT; ++q) {
                        const double2 m2 = *reinterpret_cast<const double2*>(rmu + 2 * lt + 2 * NLT * q);
                        if (!K5_GLATE) g2s[q] = *reinterpret_cast<const double2*>(rga + 2 * lt + 2 * NLT * q);
#pragma unroll
                        for (int j = 0; j < TSC; ++j) {
                            Y[2 * q][j] = fma(-m2.x, Y[2 * q][j], wl[j]);
                            Z[2 * q][j] = fma(-m2.x, Z[2 * q][j], wr[j]);
                            Y[2 * q + 1][j] = fma(-m2.y, Y[2 * q + 1][j], wl[j]);
                            Z[2 * q + 1][j] = fma(-m2.y, Z[2 * q + 1][j], wr[j]);
                        }
                    }
                    if (K5_GLATE) {
#pragma unroll
                        for (int q = 0; q < NPT; ++q) g2s[q] = *reinterpret_cast<const double2*>(rga + 2 * lt + 2 * NLT * q);
                    }
                    double go = 0.0;
                    if (ODDT) {
                        const double mu = rmu[2 * NLT * NPT + lt];
                        go = rga[2 * NLT * NPT + lt];
#pragma unroll
                        for (int j = 0; j < TSC; ++j) {
                            Y[TLT - 1][j] = fma(-mu, Y[TLT - 1][j], wl[j]);
                            Z[TLT - 1][j] = fma(-mu, Z[TLT - 1][j], wr[j]);
                        }
                    }
#pragma unroll
                    for (int q = 0; q < NPT; ++q) {
#pragma unroll
                        for (int j = 0; j < TSC; ++j) {
                            aL[j] = fma(g2s[q].x, Y[2 * q][j], aL[j]);
                            aR[j] = fma(g2s[q].x, Z[2 * q][j], aR[j]);
                            aL[j] = fma(g2s[q].y, Y[2 * q + 1][j], aL[j]);
                            aR[j] = fma(g2s[q].y, Z[2 * q + 1][j], aR[j]);
                        }
                    }
                    if (ODDT) {
#pragma unroll
                        for (int j = 0; j < TSC; ++j) {
                            aL[j] = fma(go, Y[TLT - 1][j], aL[j]);
                            aR[j] = fma(go, Z[TLT - 1][j], aR[j]);
                        }
                    }
                };
                // step 0: mu_0 = 0, Y_0 = f_0 (W + the preloaded boundary term), no left contribution
                auto body_first = [&](double (&aL)[TSC], double (&aR)[TSC]) {
                    double wl[TSC], wr[TSC];
                    load_w(0, wl, wr);
#pragma unroll
                    for (int j = 0; j < TSC; ++j) aL[j] = aR[j] = 0.0;
#pragma unroll
                    for (int n = 0; n < TLT; ++n) {
                        const double gg = cga[slot(n)];
#pragma unroll
                        for (int j = 0; j < TSC; ++j) {
                            Y[n][j] += wl[j];
                            Z[n][j] += wr[j];
                            aR[j] = fma(gg, Z[n][j], aR[j]);
                        }
                    }
                };
                // step m-1 (m >= 2): the left chain reaches position m-1 (f += beta u_right), the right
                // chain position 0 (f += beta u_left)
                auto body_last = [&](int tt, double (&aL)[TSC], double (&aR)[TSC]) {
                    double wl[TSC], wr[TSC];
                    load_w(tt, wl, wr);
                    const double* rmu = cmu + tt * RN;
                    const double* rga = cga + tt * RN;
#pragma unroll
                    for (int j = 0; j < TSC; ++j) aL[j] = aR[j] = 0.0;
#pragma unroll
                    for (int n = 0; n < TLT; ++n) {
                        const int sn = slot(n);
                        const int l = rb + sn;
                        const bool ok = l < L;
                        const double beta = beta_of(l);
                        const double mu = rmu[sn], gg = rga[sn];
                        const double nk = gg * mu;
#pragma unroll
                        for (int j = 0; j < TSC; ++j) {
                            const double ul = ok ? uGu[j][l << CSL] : 0.0;
                            const double ur = ok ? uGv[j][l << CSL] : 0.0;
                            aL[j] = fma(-nk, Y[n][j], aL[j]);
                            Y[n][j] = fma(beta, ur, fma(-mu, Y[n][j], wl[j]));
                            Z[n][j] = fma(beta, ul, fma(-mu, Z[n][j], wr[j]));
                            aR[j] = fma(gg, Z[n][j], aR[j]);
                        }
                    }
                };
                double* pb = pbase + lw * 2 * CS + st0 + sig;
                // sum the step's partials over the warp's CL l-lanes (select-free reduce-scatter: slot j
                // holds sample j ^ sig) and store them for the fold warps
                auto reduce_store = [&](double (&aL)[TSC], double (&aR)[TSC], int tt) {
                    if constexpr (CL == 4) {
                        aL[0] += __shfl_xor_sync(0xffffffffu, aL[2], 1);
                        aL[1] += __shfl_xor_sync(0xffffffffu, aL[3], 1);
                        aR[0] += __shfl_xor_sync(0xffffffffu, aR[2], 1);
                        aR[1] += __shfl_xor_sync(0xffffffffu, aR[3], 1);
                        aL[0] += __shfl_xor_sync(0xffffffffu, aL[1], 2);
                        aR[0] += __shfl_xor_sync(0xffffffffu, aR[1], 2);
                    } else {
                        aL[0] += __shfl_xor_sync(0xffffffffu, aL[1], 1);
                        aR[0] += __shfl_xor_sync(0xffffffffu, aR[1], 1);
                    }
                    if (!(A.ablate & 32)) {
                        pb[tt * NWL * 2 * CS] = aL[0];
                        pb[tt * NWL * 2 * CS + CS] = aR[0];
                    }
                };
                const bool last_here = (t0 + nb == m) && (m > 1);
                if (last_here && nb > 1) {  // the last step re-reads both vertices' u_G: pull it into L1
#pragma unroll
                    for (int n = 0; n < TLT; ++n) {
                        const int l = rb + slot(n);
                        if (l < L) {
#pragma unroll
                            for (int j = 0; j < TSC; ++j) {
                                asm volatile("prefetch.global.L1 [%0];" ::"l"(uGu[j] + (l << CSL)));
                                asm volatile("prefetch.global.L1 [%0];" ::"l"(uGv[j] + (l << CSL)));
                            }
                        }
                    }
                }
                const int tend = last_here ? nb - 1 : nb;
                double pL[TSC], pR[TSC];
                if (TL <= K5_SLMAX && t0 > 0 && !last_here && nb == IBK) {
                    // a full interior block (most blocks): the same step sequence as below, written
                    // straight-line so the next step's shared-memory loads can be scheduled under
                    // the current step's FMAs.  Only for TL <= 6: with the TL = 7 register tile the
                    // longer live ranges cost more than they hide (measured: config 5, TL = 6, K5
                    // 11.6 -> 11.0 ms; config 3, TL = 7, 5.69 -> 6.14 ms)
                    double aL[TSC], aR[TSC];
                    body_mid(0, pL, pR);
#pragma unroll
                    for (int u = 1; u + 1 < IBK; u += 2) {
                        body_mid(u, aL, aR);
                        reduce_store(pL, pR, u - 1);
                        body_mid(u + 1, pL, pR);
                        reduce_store(aL, aR, u);
                    }
                    body_mid(IBK - 1, aL, aR);
                    reduce_store(pL, pR, IBK - 2);
                    reduce_store(aL, aR, IBK - 1);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&pfull[ps]);
                    puse ^= 1u << ps;
                    ps = ps + 1 == nps ? 0 : ps + 1;
                    release();
                    continue;
                }
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
                // steps in pairs with alternating partial registers (no register copies); the
                // reduction of step tt-1 is issued under step tt's FMAs
                for (; tt + 1 < tend; tt += 2) {
                    double aL[TSC], aR[TSC];
                    body_mid(tt, aL, aR);
                    reduce_store(pL, pR, tt - 1);
                    body_mid(tt + 1, pL, pR);
                    reduce_store(aL, aR, tt);
                }
                if (tt < tend) {
                    double aL[TSC], aR[TSC];
                    body_mid(tt, aL, aR);
                    reduce_store(pL, pR, tt - 1);
#pragma unroll
                    for (int j = 0; j < TSC; ++j) {
                        pL[j] = aL[j];
                        pR[j] = aR[j];
                    }
                    ++tt;
                }
                if (last_here) {
                    double aL[TSC], aR[TSC];
                    body_last(nb - 1, aL, aR);
                    if (pend) reduce_store(pL, pR, nb - 2);
#pragma unroll
                    for (int j = 0; j < TSC; ++j) {
                        pL[j] = aL[j];
                        pR[j] = aR[j];
                    }
                    pend = true;
                }
                if (pend) reduce_store(pL, pR, nb - 1);
                // hand the block's partials to the fold warps, the staged data back to the producer
                __syncwarp();
                if (lane == 0) mbar_arrive(&pfull[ps]);
                puse ^= 1u << ps;
                ps = ps + 1 == nps ? 0 : ps + 1;
                release();
            }
        }
    }
}

// ------------------------------------------------------------------------------------------------
// K3 condense (P197-239) with the same decomposition: the register tile and thread mapping of
// sweep_impl.cuh's condense V2 instance (4 l-warps of 8 l-lanes x 4 s-lanes, 2 s-warps: the 8
// l-lanes of a warp share each staged coefficient pair, so a coefficient load is one shared-memory
// wavefront), chains only; the producer warpgroup streams the stages as in sweep2_impl.cuh (its
// four warps split the noise rows); no fold, no barriers: every consumer thread writes its own end
// values w_1 = g_0 Z, w_m = g_0 Y after a round's last block.
namespace cond {
constexpr int LWc = 8, SLWc = 4, NWLc = 4, NWSc = 2;
constexpr int IBKd = 28, NSTd = 3;  // steps per stage x ring depth (config 3: 16 x 4 2.04 ms, 24 x 3 2.00, 28 x 3 2.00)
constexpr int WROWc = CS + 4;
constexpr size_t HDRc = 512;
}  // namespace cond

template <int TL, int IBKc, int NSTc>
__global__ void __launch_bounds__(NT, 1) sweep3c_kernel(Args A) {
    using namespace cond;
    constexpr int WELc = IBKc * 2 * WROWc;  // [IBK][2 side][WROW]
    constexpr int RN = 32 * TL;
    constexpr int NP = TL / 2;
    constexpr bool ODD = (TL & 1) != 0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const DevGraph& g = A.g;
    const int64_t N = g.N;
    const int L = A.L, Lp = A.Lp;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);         // [NSTc]
    uint64_t* empty = full + NSTc;                                   // [NSTc]
    ItemDesc* header = reinterpret_cast<ItemDesc*>(empty + NSTc);   // [NSTc]
    double* coef = reinterpret_cast<double*>(smem_raw + HDRc);       // [NSTc][IBKc][RN] (mu)
    double* wbuf = coef + NSTc * IBKc * RN;                          // [NSTc][IBKc][2][WROWc]

    if (tid == 0) {
        for (int s = 0; s < NSTc; ++s) {
            mbar_init(&full[s], 129);  // the expect_tx arrive + the 128 producer threads' cp.async arrivals
            mbar_init(&empty[s], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp >= NCW) {  // ------------------------------------------------------------ producer warpgroup
        asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
        const int ptid = tid - NCW * 32;
        volatile int* qbox = reinterpret_cast<volatile int*>(header + NSTc);
        auto pbar = []() { asm volatile("bar.sync 1, 128;" ::: "memory"); };
        int stage = 0;
        uint32_t use = 0;
        ItemDesc cur{};
        auto produce = [&](int item_hdr, int64_t c0, int m, int64_t off, int64_t toff, int rd, int t0, int nb) {
            sweep::mbar_wait_sleep(&empty[stage], ((use >> stage) & 1u) ^ 1u);
            if (ptid == 0) {
                header[stage] = cur;
                header[stage].it = item_hdr;
                fence_proxy_async();
                mbar_expect_tx(&full[stage], (uint32_t)(nb * RN * sizeof(double)));
            }
            pbar();
            if (nb > 0) {
                double* cdst = coef + stage * IBKc * RN;
                if (A.rounds == 1) {
                    if (ptid == 0)
                        bulk_g2s(cdst, A.mu + (toff + t0) * (int64_t)Lp, (uint32_t)(nb * RN * sizeof(double)),
                                 &full[stage]);
                } else {
                    for (int tt = ptid; tt < nb; tt += 128)
                        bulk_g2s(cdst + tt * RN, A.mu + (toff + t0 + tt) * (int64_t)Lp + rd * RN,
                                 (uint32_t)(RN * sizeof(double)), &full[stage]);
                }
                if (ptid < 2 * CS) {  // noise row (side, sample) of this thread
                    const int side = ptid & 1, s = ptid >> 1;
                    int64_t sg = c0 + s;
                    if (sg >= A.S) sg = A.S - 1;
                    const double* src = A.W + sg * N + off + (side ? (m - 1 - t0) : t0);
                    const int dstep = side ? -1 : 1;
                    double* dst = wbuf + stage * WELc + side * WROWc + s;
#pragma unroll 4
                    for (int tt = 0; tt < nb; ++tt) cp_async8(dst + tt * 2 * WROWc, src + dstep * tt);
                }
            }
            cpasync_arrive_noinc(&full[stage]);
            use ^= 1u << stage;
            stage = stage + 1 == NSTc ? 0 : stage + 1;
        };
        for (;;) {
            if (ptid == 0) *qbox = atomicAdd(A.counter, 1);
            pbar();
            const int it = *qbox;
            pbar();
            if (it >= A.n_items) {
                produce(-1, 0, 0, 0, 0, 0, 0, 0);
                break;
            }
            const int e = g.edge_order[it / A.chunks];
            const int m = g.m[e];
            const int64_t c0 = (int64_t)(it % A.chunks) * CS;
            const int64_t off = g.off[e], toff = g.toff[e];
            cur.it = it;
            cur.e = e;
            cur.m = m;
            cur.vu = g.eu[e];
            cur.vv = g.ev[e];
            cur.off = off;
            cur.toff = toff;
            cur.h = g.h[e];
            if (m == 0) {  // one empty stage: the consumers write zero end values
                produce(it, c0, m, off, toff, 0, 0, 0);
                continue;
            }
            for (int rd = 0; rd < A.rounds; ++rd)
                for (int t0 = 0; t0 < m; t0 += IBKc) produce(it, c0, m, off, toff, rd, t0, min(IBKc, m - t0));
        }
        return;
    }

    // ---------------------------------------------------------------------------------- consumers
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
    const int ll = lane % LWc, sl = lane / LWc;
    const int lw = warp % NWLc, sw = warp / NWLc;
    const int lt = lw * LWc + ll;             // l-thread 0..31
    const int st0 = (sw * SLWc + sl) * TS;   // first sample (within the item) of this thread
    int stage = 0;
    uint32_t use = 0;
    auto acquire = [&]() { mbar_wait(&full[stage], (use >> stage) & 1u); };
    auto release = [&]() {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        use ^= 1u << stage;
        stage = stage + 1 == NSTc ? 0 : stage + 1;
    };
    auto slot = [&](int n) -> int { return (n < 2 * NP) ? (2 * lt + 64 * (n >> 1) + (n & 1)) : (64 * NP + lt); };
    for (;;) {
        acquire();
        const ItemDesc d = header[stage];
        const int it = d.it;
        if (it < 0) break;
        const int e = d.e;
        const int64_t tile = it % A.chunks;
        const int m = d.m;
        const int64_t toff = d.toff;
        if (m == 0) {  // no interior: zero end values (ends [tile][l][code][CS])
#pragma unroll
            for (int n = 0; n < TL; ++n) {
                const int l = slot(n);
                for (int rb = 0; rb < A.rounds * RN; rb += RN) {
                    if (rb + l < L) {
                        double* o = A.out + ((tile * L + rb + l) * 2 * (int64_t)g.E + 2 * e) * CS + st0;
                        *reinterpret_cast<double2*>(o) = make_double2(0.0, 0.0);
                        *reinterpret_cast<double2*>(o + 2) = make_double2(0.0, 0.0);
                        *reinterpret_cast<double2*>(o + CS) = make_double2(0.0, 0.0);
                        *reinterpret_cast<double2*>(o + CS + 2) = make_double2(0.0, 0.0);
                    }
                }
            }
            release();
            continue;
        }
        const int nblk = (m + IBKc - 1) / IBKc;
        for (int rd = 0; rd < A.rounds; ++rd) {
            const int rb = rd * RN;
            if (rd > 0) acquire();
            double Y[TL][TS], Z[TL][TS], g0[TL];
#pragma unroll
            for (int n = 0; n < TL; ++n) {
                const int l = rb + slot(n);
                // g_0 = g_{m-1} for the end values, loaded now (volatile: not sunk to the round's end)
                double gv = 0.0;
                if (l < L) asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(gv) : "l"(A.gam + toff * (int64_t)Lp + l));
                g0[n] = gv;
#pragma unroll
                for (int j = 0; j < TS; ++j) Y[n][j] = Z[n][j] = 0.0;
            }
            for (int b = 0; b < nblk; ++b) {
                if (b > 0) acquire();
                const int nb = min(IBKc, m - b * IBKc);
                const double* cmu = coef + stage * IBKc * RN;
                const double* wb = wbuf + stage * WELc;
                auto step = [&](int tt) {
                    const double2 wl01 = *reinterpret_cast<const double2*>(wb + (tt * 2 + 0) * WROWc + st0);
                    const double2 wl23 = *reinterpret_cast<const double2*>(wb + (tt * 2 + 0) * WROWc + st0 + 2);
                    const double2 wr01 = *reinterpret_cast<const double2*>(wb + (tt * 2 + 1) * WROWc + st0);
                    const double2 wr23 = *reinterpret_cast<const double2*>(wb + (tt * 2 + 1) * WROWc + st0 + 2);
                    const double wl[TS] = {wl01.x, wl01.y, wl23.x, wl23.y};
                    const double wr[TS] = {wr01.x, wr01.y, wr23.x, wr23.y};
                    const double* rmu = cmu + tt * RN;
#pragma unroll
                    for (int q = 0; q < NP; ++q) {
                        const double2 m2 = *reinterpret_cast<const double2*>(rmu + 2 * lt + 64 * q);
#pragma unroll
                        for (int j = 0; j < TS; ++j) {
                            Y[2 * q][j] = fma(-m2.x, Y[2 * q][j], wl[j]);
                            Z[2 * q][j] = fma(-m2.x, Z[2 * q][j], wr[j]);
                            Y[2 * q + 1][j] = fma(-m2.y, Y[2 * q + 1][j], wl[j]);
                            Z[2 * q + 1][j] = fma(-m2.y, Z[2 * q + 1][j], wr[j]);
                        }
                    }
                    if (ODD) {
                        const double mu = rmu[64 * NP + lt];
#pragma unroll
                        for (int j = 0; j < TS; ++j) {
                            Y[TL - 1][j] = fma(-mu, Y[TL - 1][j], wl[j]);
                            Z[TL - 1][j] = fma(-mu, Z[TL - 1][j], wr[j]);
                        }
                    }
                };
                if (nb == IBKc) {
#pragma unroll
                    for (int tt = 0; tt < IBKc; ++tt) step(tt);
                } else {
                    for (int tt = 0; tt < nb; ++tt) step(tt);
                }
                release();
            }
            // w_1 = g_0 Z (right sweep end, position 0), w_m = g_0 Y (left sweep end); g_0 = g_{m-1}.
            // The products go into the (now dead) chain registers and are stored from there: fresh
            // product registers were allocated over the sources of the previous node's stores, and
            // every product then waited for those stores to release them
#pragma unroll
            for (int n = 0; n < TL; ++n) {
#pragma unroll
                for (int j = 0; j < TS; ++j) {
                    Z[n][j] *= g0[n];
                    Y[n][j] *= g0[n];
                }
            }
#pragma unroll
            for (int n = 0; n < TL; ++n) {
                const int l = rb + slot(n);
                if (l < L) {
                    double* o = A.out + ((tile * L + l) * 2 * (int64_t)g.E + 2 * e) * CS + st0;
                    *reinterpret_cast<double2*>(o) = make_double2(Z[n][0], Z[n][1]);
                    *reinterpret_cast<double2*>(o + 2) = make_double2(Z[n][2], Z[n][3]);
                    *reinterpret_cast<double2*>(o + CS) = make_double2(Y[n][0], Y[n][1]);
                    *reinterpret_cast<double2*>(o + CS + 2) = make_double2(Y[n][2], Y[n][3]);
                }
            }
        }
    }
}

template <int TL, int IBKc, int NSTc>
cudaError_t launch_c_k(Args a, cudaStream_t st) {
    using namespace cond;
    constexpr int WELc = IBKc * 2 * WROWc;
    const size_t smem = HDRc + (size_t)NSTc * IBKc * 32 * TL * sizeof(double) + (size_t)NSTc * WELc * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(sweep3c_kernel<TL, IBKc, NSTc>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(a.counter, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return e;
    int blocks = a.g.n_sm > 0 ? a.g.n_sm : 148;
    if (blocks > a.n_items) blocks = a.n_items;
    sweep3c_kernel<TL, IBKc, NSTc><<<blocks, NT, smem, st>>>(a);
    return cudaGetLastError();
}

template <int TL>
cudaError_t launch_c(Args a, cudaStream_t st) {
    using namespace cond;
    a.chunks = (int32_t)((a.S + CS - 1) / CS);
    a.n_items = a.g.E * a.chunks;
    return launch_c_k<TL, IBKd, NSTd>(a, st);
}


template <int TL>
cudaError_t launch(Args a, cudaStream_t st) {
    using C = Cfg<TL>;
    a.chunks = (int32_t)((a.S + CS - 1) / CS);
    a.n_items = a.g.E * a.chunks;
    // the output tile holds edges with (m | 1) <= tile_ms, sized for the longest edge if it fits; the
    // ring depths (data nst, partials nps) give way to it: edges past the tile are folded into u in
    // global memory, a read-modify-write per visit, far slower than a shallower ring.  Preference:
    // (3, 2), (2, 2), (3, 1), (2, 1).
    const int want = a.g.max_m | 1;
    auto base_for = [&](int nst, int nps) {
        return HDR + nst * C::STAGE1 + nps * C::PART1 + (size_t)a.Lp * sizeof(double);
    };
    auto fit_for = [&](int nst, int nps) {
        const size_t b = base_for(nst, nps);
        const size_t room = sweep::SMEM_MAX > b ? sweep::SMEM_MAX - b : 0;
        return (int)(room / ((size_t)CS * sizeof(double)));
    };
    static const int depth[4][2] = {{NST, NPS}, {2, NPS}, {NST, 1}, {2, 1}};
    a.nst = NST;
    a.nps = NPS;
    for (const auto& d : depth) {
        if (fit_for(d[0], d[1]) >= want) {
            a.nst = d[0];
            a.nps = d[1];
            break;
        }
    }
    size_t smem = base_for(a.nst, a.nps);
    const int fit = fit_for(a.nst, a.nps);
    a.tile_ms = want <= fit ? want : (fit >= 1 ? ((fit - 1) | 1) : 0);
    smem += (size_t)CS * a.tile_ms * sizeof(double);
    if (a.fits_out) {  // query only (no launch): every edge's output leaves by plain tile stores
        *a.fits_out = a.tile_ms >= want;
        return cudaSuccess;
    }
    // the ring depth is a template constant (the stage offsets fold into the addressing)
    // consumer mapping CL = 2 l-lanes per warp (one reduce-scatter level) unless GRF_ABLATE bit 256
    const bool cl4 = (a.ablate & 256) != 0;
    auto kern = a.nst == NST ? (cl4 ? sweep3_kernel<TL, NST, 4> : sweep3_kernel<TL, NST, 2>)
                             : (cl4 ? sweep3_kernel<TL, 2, 4> : sweep3_kernel<TL, 2, 2>);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(a.counter, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return e;
    int blocks = a.g.n_sm > 0 ? a.g.n_sm : 148;
    if (blocks > a.n_items) blocks = a.n_items;
    kern<<<blocks, NT, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace sweep3
}  // namespace grf
