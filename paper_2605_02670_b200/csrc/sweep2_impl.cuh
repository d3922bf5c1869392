// K3 (condense) and K5 (recover + quadrature sum), warp-specialised kernels for sample tiles of
// 16 and 32 samples (calls with >= 9 samples).  The arithmetic is the one of sweep_impl.cuh:
// the twisted (two-sided) Thomas elimination of the Toeplitz interior block of every edge,
// node and sample (PAPER.md P187-239 condensation, P300-311 recovery), summed over the
// quadrature nodes (P313-324); see that file's header for the recurrences, the correction node
// and the table layout [(toff_e + t) * Lp + l].
//
// Decomposition (one CTA per SM, persistent, 12 warps):
//   * warps 8-11 form the producer warpgroup; it gives its registers away (setmaxnreg) and its
//     first warp walks the work queue (items = (edge, tile of CS samples), longest edge first)
//     and, per block of IBK steps, streams the round's rows of the coefficient tables (mu [, g])
//     with the bulk-copy engine and the item's noise with cp.async into an NST-deep ring of
//     stages guarded by "full" / "empty" mbarriers;
//   * warps 0-7 are consumers (232 registers each): every warp owns TS samples of the item and
//     ALL RN = 32 TL nodes of a round -- lane = 32 l-lanes x TL nodes -- so the sum over the
//     nodes is a warp-local shuffle reduce-scatter: no shared partial sums, no folds, no block
//     barriers; a consumer only waits for staged data and releases a stage with one arrive.
// Recover sum over l, per step: a lane holds, for its TL nodes and TS samples, the own-side
// chain contribution (aA) and the other side's (aB).  Lanes 16-31 run the mirrored problem
// ("side flip": their own chain is the right sweep), so the first reduce level keeps aA and
// sends aB with no select; the next log2(TS) levels halve the samples through a per-lane sample
// permutation (slot j holds sample j ^ perm); the remaining levels sum fully.  The right-side
// total is forwarded to the left-side lane of the same sample, which alone writes both
// positions t and m-1-t of its sample (first visit stores, second visit adds), so all writes
// to a position come from one lane in program order: no hazards, no warp barriers.  Outputs
// go to the warp's rows of a per-item shared-memory tile (written out coalesced at the item's
// end) or, for edges too long for it, straight to u.  The reduction of step t-1 is issued after
// step t's FMAs (software pipeline).  Every sum has a fixed order: bitwise reproducible results.
#pragma once

#include "sweep_impl.cuh"

namespace grf {
namespace sweep2 {

using sweep::Args;
using sweep::bulk_g2s;
using sweep::fence_proxy_async;
using sweep::mbar_expect_tx;
using sweep::mbar_init;
using sweep::mbar_wait;
using sweep::mbar_wait_sleep;
using sweep::smem_u32;

constexpr int NCW = 8;  // consumer warps


__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// arrive on `bar` once all of this thread's prior cp.async copies have landed (count pre-set)
__device__ __forceinline__ void cpasync_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// The item a stage belongs to, written by the producer (which loads the edge's metadata anyway)
// so that consumers start an item from shared memory instead of a chain of dependent global loads.
struct ItemDesc {
    int32_t it, e, m, vu, vv, pad;
    int64_t off, toff;
    double h;
};

// Output accesses of the writer lanes (generic addresses: the shared output tile, or u itself for
// edges too long for it), predicated and branch-free so the scheduler can interleave them with
// the next step's FMAs.  Volatile asm WITHOUT a memory clobber: they stay in program order among
// themselves (a position's two visits come from one lane) while the staged-coefficient loads
// remain free to move across them.
__device__ __forceinline__ double ld_if(const double* p, bool pr) {
    double v = 0.0;
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q ld.f64 %0, [%1]; }" : "+d"(v) : "l"(p), "r"((unsigned)pr));
    return v;
}
__device__ __forceinline__ void st_if(double* p, double v, bool pr) {
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.f64 [%0], %1; }" ::"l"(p), "d"(v), "r"((unsigned)pr));
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

template <int TL, int TS, bool REC>
struct Cfg {
    static constexpr int CS = NCW * TS;             // samples per item (sample tile of ends / uG)
    static constexpr int CSL = CS == 32 ? 5 : 4;
    static constexpr int LGTS = TS == 4 ? 2 : 1;
    static constexpr int NT = (NCW + 4) * 32;       // consumers + the producer warpgroup
    static constexpr int RN = 32 * TL;              // nodes per round
    static constexpr int NTAB = REC ? 2 : 1;        // staged tables: mu (, g)
    static constexpr int NC = REC ? 2 : 1;          // noise copies: natural (, pair-swapped)
    static constexpr int IBK = REC ? 8 : 16;        // steps per stage
    static constexpr int NST = REC ? 3 : 4;         // ring depth
    static constexpr int WROW = CS + 4;             // a staged noise row (skewed: the (side, copy) rows read
                                                    // together fall into different shared-memory banks)
    static constexpr int WEL = IBK * 2 * NC * WROW; // staged noise doubles per stage
    static constexpr size_t HDR = 512;              // mbarriers, stage headers (item descriptors)
    static constexpr size_t COEF = (size_t)NST * NTAB * IBK * RN * sizeof(double);
    static constexpr size_t WB = (size_t)NST * WEL * sizeof(double);
    static constexpr size_t FIXED = HDR + COEF + WB;
    static_assert(TS == 2 || TS == 4, "2 or 4 samples per lane");
    static_assert(NST * (8 + 8 + 48) + 16 <= (int)HDR, "header room");
    static_assert(2 * NC * CS <= 128, "one noise row per producer thread");
};

template <int TL, int TS, bool REC>
__global__ void __launch_bounds__(Cfg<TL, TS, REC>::NT, 1) sweep2_kernel(Args A) {
    using C = Cfg<TL, TS, REC>;
    constexpr int CS = C::CS, CSL = C::CSL, RN = C::RN, NTAB = C::NTAB, NC = C::NC, IBK = C::IBK, NST = C::NST;
    constexpr int NP = TL / 2;
    constexpr bool ODD = (TL & 1) != 0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const DevGraph& g = A.g;
    const int64_t N = g.N;
    const int L = A.L, Lp = A.Lp;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);         // [NST]
    uint64_t* empty = full + NST;                                    // [NST]
    ItemDesc* header = reinterpret_cast<ItemDesc*>(empty + NST);    // [NST] item of the stage (it = -1: end)
    double* coef = reinterpret_cast<double*>(smem_raw + C::HDR);     // [NST][NTAB][IBK][RN]
    double* wbuf = coef + NST * NTAB * IBK * RN;                     // [NST][IBK][2 side][NC][WROW]
    double* cLs = wbuf + NST * C::WEL;                               // [Lp] c_L (REC)
    double* otile = cLs + (REC ? Lp : 0);                            // [NCW][TS][tile_ms] (REC)

    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 129);   // the expect_tx arrive + the 128 producer threads' cp.async arrivals
            mbar_init(&empty[s], NCW);  // one release per consumer warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (REC)
        for (int i = tid; i < Lp; i += C::NT) cLs[i] = A.cL[i];  // zero padded past L
    __syncthreads();

    // ------------------------------------------------------------------------------------ producer
    // All four warps of the producer warpgroup (one per SM sub-partition, so the copy issue
    // load is spread evenly over the schedulers) walk the same stage sequence: warp NCW takes the
    // queue and broadcasts the item through shared memory (named barrier 1 over the warpgroup);
    // every producer thread owns one (sample, copy, side) noise row per stage and its lane 0 in
    // warp NCW issues the coefficient bulk copies.
    if (warp >= NCW) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
        const int ptid = tid - NCW * 32;  // 0..127
        volatile int* qbox = reinterpret_cast<volatile int*>(header + NST);  // queue broadcast slot
        auto pbar = []() { asm volatile("bar.sync 1, 128;" ::: "memory"); };
        int stage = 0;
        uint32_t use = 0;  // bit s: parity of stage s's current use
        ItemDesc cur{};
        constexpr int NROW = 2 * NC * CS;  // noise rows per stage (<= 128)
        auto produce = [&](int item_hdr, int64_t c0, int m, int64_t off, int64_t toff, int rd, int t0, int nb) {
            mbar_wait_sleep(&empty[stage], ((use >> stage) & 1u) ^ 1u);
            if (ptid == 0) {
                header[stage] = cur;
                header[stage].it = item_hdr;
                fence_proxy_async();
                mbar_expect_tx(&full[stage], (uint32_t)(NTAB * nb * RN * sizeof(double)));
            }
            pbar();  // the expect_tx arrive precedes every copy's completion
            if (nb > 0) {
                double* cdst = coef + stage * NTAB * IBK * RN;
                if (A.rounds == 1) {  // rows are contiguous: one copy per table
                    if (ptid < NTAB)
                        bulk_g2s(cdst + ptid * IBK * RN, (ptid == 0 ? A.mu : A.gam) + (toff + t0) * (int64_t)Lp,
                                 (uint32_t)(nb * RN * sizeof(double)), &full[stage]);
                } else {
                    for (int x = ptid; x < NTAB * nb; x += 128) {
                        const int tb = x / nb, tt = x % nb;
                        bulk_g2s(cdst + (tb * IBK + tt) * RN,
                                 (tb == 0 ? A.mu : A.gam) + (toff + t0 + tt) * (int64_t)Lp + rd * RN,
                                 (uint32_t)(RN * sizeof(double)), &full[stage]);
                    }
                }
                // noise row (side, copy, sample) of this thread: the nb positions t0+tt (left) or
                // m-1-t0-tt (right); copy 1 holds the samples pair-swapped (sample s ^ 1 at index s)
                if (ptid < NROW) {
                    const int side = ptid & 1, c = (ptid >> 1) % NC, s = (ptid >> 1) / NC;
                    int64_t sg = c0 + (c ? (s ^ 1) : s);
                    if (sg >= A.S) sg = A.S - 1;
                    const double* src = A.W + sg * N + off + (side ? (m - 1 - t0) : t0);
                    const int dstep = side ? -1 : 1;
                    double* dst = wbuf + stage * C::WEL + (side * NC + c) * C::WROW + s;
#pragma unroll 4
                    for (int tt = 0; tt < nb; ++tt) cp_async8(dst + tt * 2 * NC * C::WROW, src + dstep * tt);
                }
            }
            cpasync_arrive_noinc(&full[stage]);
            use ^= 1u << stage;
            stage = stage + 1 == NST ? 0 : stage + 1;
        };
        for (;;) {
            if (ptid == 0) *qbox = atomicAdd(A.counter, 1);
            pbar();
            const int it = *qbox;
            pbar();  // everyone has read the slot before it is rewritten
            if (it >= A.n_items) {
                produce(-1, 0, 0, 0, 0, 0, 0, 0);
                break;
            }
            const int e = g.edge_order[it / A.chunks];
            const int m = g.m[e];
            if (REC && m == 0) continue;  // nothing to recover: the vertex values come from vertex_sum
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
            if (REC && ptid < 2) {  // the consumers' round-start u_G rows of this item: into L2 now
                const int v = ptid ? cur.vv : cur.vu;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.uG + (((it % A.chunks) * g.V + v) * (int64_t)L << CSL)),
                             "r"((uint32_t)(L * CS * sizeof(double))) : "memory");
            }
            if (m == 0) {  // condense: one empty stage, the consumers write zero end values
                produce(it, c0, m, off, toff, 0, 0, 0);
                continue;
            }
            for (int rd = 0; rd < A.rounds; ++rd)
                for (int t0 = 0; t0 < m; t0 += IBK) produce(it, c0, m, off, toff, rd, t0, min(IBK, m - t0));
        }
        return;
    }

    // ------------------------------------------------------------------------------------ consumers
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
    // lane roles (recover): side flip = lane bit 4; sample permutation from the next log2(TS)
    // bits; the lane on side 0 whose remaining (full-reduction) bits are 0 writes its sample
    constexpr int FULLMASK = (1 << (4 - C::LGTS)) - 1;
    const int side = REC ? (lane >> 4) & 1 : 0;
    const int perm = REC ? (lane >> (4 - C::LGTS)) & (TS - 1) : 0;
    const bool writer = REC && (lane & (16 | FULLMASK)) == 0;
    const int s_w = warp * TS;  // the warp's first sample within the item
    int stage = 0;
    uint32_t use = 0;
    auto acquire = [&]() {
        if (!(A.ablate & 4)) mbar_wait(&full[stage], (use >> stage) & 1u);
    };
    auto release = [&]() {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        use ^= 1u << stage;
        stage = stage + 1 == NST ? 0 : stage + 1;
    };
    // node (within a round) of this lane's register slot n
    auto slot = [&](int n) -> int { return (n < 2 * NP) ? (2 * lane + 64 * (n >> 1) + (n & 1)) : (64 * NP + lane); };
    double* wtile = otile + warp * TS * (REC ? A.tile_ms : 0);  // this warp's rows of the output tile

    for (;;) {
        acquire();
        const ItemDesc d = header[stage];
        const int it = d.it;
        if (it < 0) break;
        const int e = d.e;
        const int64_t tile = it % A.chunks;
        const int64_t c0 = tile * CS;
        const int m = d.m;
        const int64_t off = d.off;
        const int64_t toff = d.toff;
        const double h = d.h;
        const double inv_h = 1.0 / h;
        const int vu = d.vu, vv = d.vv;
        if (!REC && m == 0) {  // no interior: zero end values (ends [tile][l][code][CS])
            for (int x = lane; x < L * 2 * TS; x += 32) {
                const int l = x / (2 * TS), r = x % (2 * TS);
                A.out[((tile * L + l) * 2 * (int64_t)g.E + 2 * e + r / TS) * CS + s_w + r % TS] = 0.0;
            }
            release();
            continue;
        }
        auto beta_of = [&](int l) -> double {
            if (l >= L) return 0.0;
            return A.mass ? edge_coef(A.cI[l], A.cL[l], A.kappa2, h, 1).beta : cLs[l] * inv_h;
        };
        const int ms = m | 1;
        const bool in_tile = REC && ms <= A.tile_ms;
        // the writer's output row: its row of the warp's tile, or u itself for long edges
        const int s_own = s_w + perm;  // the sample this lane holds in slot 0 after the reduction
        double* orow = REC ? (in_tile ? wtile + perm * ms : A.out + (c0 + s_own) * N + off) : nullptr;
        const bool wr_ok = writer && (in_tile || c0 + s_own < A.S);
        // u_G of the own / other vertex (layout [tile][v][l][cs]): node l, slot j at
        // uGo[(l << CSL) + sample-in-tile of slot j] (the last tile's padded slots read sample S-1)
        const int v_own = side ? vv : vu, v_oth = side ? vu : vv;
        const double* uGo = REC ? A.uG + ((tile * g.V + v_own) * (int64_t)L << CSL) : nullptr;
        const double* uGt = REC ? A.uG + ((tile * g.V + v_oth) * (int64_t)L << CSL) : nullptr;
        const int s_lim = (int)(A.S - 1 - c0 < CS - 1 ? A.S - 1 - c0 : CS - 1);
        auto sit = [&](int j) { return min(s_w + (j ^ perm), s_lim); };
        const int nblk = (m + IBK - 1) / IBK;
        for (int rd = 0; rd < A.rounds; ++rd) {
            const int rb = rd * RN;
            if (rd > 0) acquire();
            double X[TL][TS], Q[TL][TS];  // own-side chain (A) and other-side chain (B)
            double g0[REC ? 1 : TL];
            if (REC) {
                // boundary rows (P310): the own chain starts from beta u_own, the other from beta u_other
#pragma unroll
                for (int n = 0; n < TL; ++n) {
                    const int l = rb + slot(n);
                    const double bt = beta_of(l);
                    const bool ok = l < L;
#pragma unroll
                    for (int j = 0; j < TS; ++j) {
                        const double uo = ok && !(A.ablate & 2) ? uGo[(l << CSL) + sit(j)] : 0.0;
                        const double ut = ok && !(A.ablate & 2) ? uGt[(l << CSL) + sit(j)] : 0.0;
                        X[n][j] = bt * (m == 1 ? uo + ut : uo);
                        Q[n][j] = bt * (m == 1 ? uo + ut : ut);
                    }
                }
            } else {
#pragma unroll
                for (int n = 0; n < TL; ++n) {
                    const int l = rb + slot(n);
                    // g_0 = g_{m-1} for the end values, loaded now (volatile: not sunk to the round's end)
                    double gv = 0.0;
                    if (l < L) asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(gv) : "l"(A.gam + toff * (int64_t)Lp + l));
                    g0[n] = gv;
#pragma unroll
                    for (int j = 0; j < TS; ++j) X[n][j] = Q[n][j] = 0.0;
                }
            }
            // pending (reduced next step) contributions of the previous step and its index
            double pA[REC ? TS : 1];
            int pt = -1;
            // first reduce level right after a step: the side flip (aA += the partner's aB)
            auto flip = [&](double (&xA)[TS], double (&xB)[TS]) {
#pragma unroll
                for (int j = 0; j < TS; ++j) xA[j] += __shfl_xor_sync(0xffffffffu, xB[j], 16);
            };
            // the remaining levels over the 32 l-lanes and the writes (see header), one step later
            auto flush = [&](double (&xA)[REC ? TS : 1], int t) {
                if (REC && !(A.ablate & 1)) {
#pragma unroll
                    for (int h2 = 0; h2 < C::LGTS; ++h2) {  // halving levels (sample-slot permutation)
                        const int half = TS >> (h2 + 1);
#pragma unroll
                        for (int j = 0; j < half; ++j) xA[j] += __shfl_xor_sync(0xffffffffu, xA[j + half], 8 >> h2);
                    }
#pragma unroll
                    for (int o = 8 >> C::LGTS; o >= 1; o >>= 1) xA[0] += __shfl_xor_sync(0xffffffffu, xA[0], o);
                    const double vR = __shfl_xor_sync(0xffffffffu, xA[0], 16);  // right total of this sample
                    // position t takes the left total, m-1-t the right one; the first visit of a
                    // position (round 0, the outer half of the steps) stores, the second adds
                    const int tm = m - 1 - t;
                    const bool first = rd == 0 && t <= tm;
                    const double vl = t == tm ? xA[0] + vR : xA[0];
                    const bool w2 = wr_ok && t != tm;
                    st_if(orow + t, ld_if(orow + t, wr_ok && !first) + vl, wr_ok);
                    st_if(orow + tm, ld_if(orow + tm, w2 && !first) + vR, w2);
                }
            };
            for (int b = 0; b < nblk; ++b) {
                if (b > 0) acquire();
                const int t0 = b * IBK;
                const int nb = min(IBK, m - t0);
                const double* cmu = coef + stage * NTAB * IBK * RN;
                const double* cga = cmu + IBK * RN;
                const double* wb = wbuf + stage * C::WEL;
                // noise of this lane's slots at step tt (own side, other side)
                auto load_w = [&](int tt, double (&wa)[TS], double (&wo)[TS]) {
                    const int cp = perm & 1, px = perm >> 1;
#pragma unroll
                    for (int q = 0; q < TS / 2; ++q) {
                        const int o = s_w + 2 * (q ^ px);
                        const double2 a = *reinterpret_cast<const double2*>(wb + ((tt * 2 + side) * NC + cp) * C::WROW + o);
                        const double2 c =
                            *reinterpret_cast<const double2*>(wb + ((tt * 2 + (side ^ 1)) * NC + cp) * C::WROW + o);
                        wa[2 * q] = a.x;
                        wa[2 * q + 1] = a.y;
                        wo[2 * q] = c.x;
                        wo[2 * q + 1] = c.y;
                    }
                };
                if constexpr (!REC) {
                    // chains only; the end values are taken after the last block of the round
                    auto step = [&](int tt) {
                        double wa[TS], wo[TS];
                        load_w(tt, wa, wo);
                        const double* rmu = cmu + tt * RN;
#pragma unroll
                        for (int q = 0; q < NP; ++q) {
                            const double2 m2 = *reinterpret_cast<const double2*>(rmu + 2 * lane + 64 * q);
#pragma unroll
                            for (int j = 0; j < TS; ++j) {
                                X[2 * q][j] = fma(-m2.x, X[2 * q][j], wa[j]);
                                Q[2 * q][j] = fma(-m2.x, Q[2 * q][j], wo[j]);
                                X[2 * q + 1][j] = fma(-m2.y, X[2 * q + 1][j], wa[j]);
                                Q[2 * q + 1][j] = fma(-m2.y, Q[2 * q + 1][j], wo[j]);
                            }
                        }
                        if (ODD) {
                            const double mu = rmu[64 * NP + lane];
#pragma unroll
                            for (int j = 0; j < TS; ++j) {
                                X[TL - 1][j] = fma(-mu, X[TL - 1][j], wa[j]);
                                Q[TL - 1][j] = fma(-mu, Q[TL - 1][j], wo[j]);
                            }
                        }
                    };
                    if (nb == IBK) {
#pragma unroll
                        for (int tt = 0; tt < IBK; ++tt) step(tt);
                    } else {
                        for (int tt = 0; tt < nb; ++tt) step(tt);
                    }
                } else {
                    // interior step (correction-node form: both chains contribute g X_t)
                    auto body_mid = [&](int tt, double (&aA)[TS], double (&aB)[TS]) {
                        double wa[TS], wo[TS];
                        load_w(tt, wa, wo);
                        const double* rmu = cmu + tt * RN;
                        const double* rga = cga + tt * RN;
#pragma unroll
                        for (int j = 0; j < TS; ++j) aA[j] = aB[j] = 0.0;
#pragma unroll
                        for (int q = 0; q < NP; ++q) {
                            const double2 m2 = *reinterpret_cast<const double2*>(rmu + 2 * lane + 64 * q);
                            const double2 g2 = *reinterpret_cast<const double2*>(rga + 2 * lane + 64 * q);
#pragma unroll
                            for (int j = 0; j < TS; ++j) {
                                X[2 * q][j] = fma(-m2.x, X[2 * q][j], wa[j]);
                                aA[j] = fma(g2.x, X[2 * q][j], aA[j]);
                                Q[2 * q][j] = fma(-m2.x, Q[2 * q][j], wo[j]);
                                aB[j] = fma(g2.x, Q[2 * q][j], aB[j]);
                                X[2 * q + 1][j] = fma(-m2.y, X[2 * q + 1][j], wa[j]);
                                aA[j] = fma(g2.y, X[2 * q + 1][j], aA[j]);
                                Q[2 * q + 1][j] = fma(-m2.y, Q[2 * q + 1][j], wo[j]);
                                aB[j] = fma(g2.y, Q[2 * q + 1][j], aB[j]);
                            }
                        }
                        if (ODD) {
                            const double mu = rmu[64 * NP + lane], gg = rga[64 * NP + lane];
#pragma unroll
                            for (int j = 0; j < TS; ++j) {
                                X[TL - 1][j] = fma(-mu, X[TL - 1][j], wa[j]);
                                aA[j] = fma(gg, X[TL - 1][j], aA[j]);
                                Q[TL - 1][j] = fma(-mu, Q[TL - 1][j], wo[j]);
                                aB[j] = fma(gg, Q[TL - 1][j], aB[j]);
                            }
                        }
                        flip(aA, aB);
                    };
                    // step 0 (mu_0 = 0): chains += noise; the left chain contributes nothing, the
                    // right chain g_0 X_0 (to position m-1)
                    auto body_first = [&](double (&aA)[TS], double (&aB)[TS]) {
                        double wa[TS], wo[TS];
                        load_w(0, wa, wo);
#pragma unroll
                        for (int j = 0; j < TS; ++j) aA[j] = aB[j] = 0.0;
#pragma unroll
                        for (int n = 0; n < TL; ++n) {
                            const double gg = cga[slot(n)];
                            const double gA = side ? gg : 0.0, gB = side ? 0.0 : gg;  // own chain is right iff side
#pragma unroll
                            for (int j = 0; j < TS; ++j) {
                                X[n][j] += wa[j];
                                Q[n][j] += wo[j];
                                aA[j] = fma(gA, X[n][j], aA[j]);
                                aB[j] = fma(gB, Q[n][j], aB[j]);
                            }
                        }
                        flip(aA, aB);
                    };
                    // step m-1 (m >= 2): the left chain reaches position m-1 (f += beta u_right) and
                    // gives -g mu X_{t-1}; the right chain reaches position 0 (f += beta u_left) and
                    // gives g X_t.  Own chain A is left iff side == 0; each chain's far-end vertex is
                    // the other chain's start vertex.
                    auto body_last = [&](int tt, double (&aA)[TS], double (&aB)[TS]) {
                        double wa[TS], wo[TS];
                        load_w(tt, wa, wo);
                        const double* rmu = cmu + tt * RN;
                        const double* rga = cga + tt * RN;
#pragma unroll
                        for (int j = 0; j < TS; ++j) aA[j] = aB[j] = 0.0;
#pragma unroll
                        for (int n = 0; n < TL; ++n) {
                            const int sn = slot(n);
                            const int l = rb + sn;
                            const bool ok = l < L;
                            const double bt = beta_of(l);
                            const double mu = rmu[sn], gg = rga[sn];
                            const double nk = gg * mu;
#pragma unroll
                            for (int j = 0; j < TS; ++j) {
                                const double uo = ok ? uGo[(l << CSL) + sit(j)] : 0.0;
                                const double ut = ok ? uGt[(l << CSL) + sit(j)] : 0.0;
                                const double xa = fma(bt, ut, fma(-mu, X[n][j], wa[j]));
                                const double xb = fma(bt, uo, fma(-mu, Q[n][j], wo[j]));
                                if (side) {  // A = right chain, B = left chain
                                    aB[j] = fma(-nk, Q[n][j], aB[j]);
                                    aA[j] = fma(gg, xa, aA[j]);
                                } else {
                                    aA[j] = fma(-nk, X[n][j], aA[j]);
                                    aB[j] = fma(gg, xb, aB[j]);
                                }
                                X[n][j] = xa;
                                Q[n][j] = xb;
                            }
                        }
                        flip(aA, aB);
                    };
                    if (t0 > 0 && t0 + IBK < m) {
                        // a full interior block: steps in pairs with alternating pending registers
                        // (compile-time step offsets, no register copies)
#pragma unroll
                        for (int tt = 0; tt < IBK; tt += 2) {
                            double aA[TS], aB[TS];
                            body_mid(tt, aA, aB);
                            flush(pA, pt);
                            body_mid(tt + 1, pA, aB);
                            flush(aA, t0 + tt);
                            pt = t0 + tt + 1;
                        }
                    } else {
                        const bool last_here = (t0 + nb == m) && (m > 1);
                        if (last_here && nb > 1) {  // the last step re-reads both vertices' u_G: pull it into L1
#pragma unroll
                            for (int n = 0; n < TL; ++n) {
                                const int l = rb + slot(n);
                                if (l < L) {
#pragma unroll
                                    for (int j = 0; j < TS; ++j) {
                                        asm volatile("prefetch.global.L1 [%0];" ::"l"(uGo + (l << CSL) + sit(j)));
                                        asm volatile("prefetch.global.L1 [%0];" ::"l"(uGt + (l << CSL) + sit(j)));
                                    }
                                }
                            }
                        }
                        const int tend = last_here ? nb - 1 : nb;
                        // each step: body + side flip; the previous step's remaining levels and
                        // writes after it (pending sums in pA)
                        auto next = [&](double (&aA)[TS], int t) {
                            if (pt >= 0) flush(pA, pt);
#pragma unroll
                            for (int j = 0; j < TS; ++j) pA[j] = aA[j];
                            pt = t;
                        };
                        int tt = 0;
                        if (t0 == 0) {
                            double aA[TS], aB[TS];
                            body_first(aA, aB);
                            next(aA, 0);
                            tt = 1;
                        }
                        for (; tt < tend; ++tt) {
                            double aA[TS], aB[TS];
                            body_mid(tt, aA, aB);
                            next(aA, t0 + tt);
                        }
                        if (last_here) {
                            double aA[TS], aB[TS];
                            body_last(nb - 1, aA, aB);
                            next(aA, m - 1);
                        }
                    }
                }
                release();
            }
            if constexpr (REC) {
                if (pt >= 0) flush(pA, pt);
            } else {
                // w_1 = g_0 Q (right sweep end, position 0), w_m = g_0 X (left sweep end); g_0 = g_{m-1}.
                // ends layout [tile][l][code][CS]: slots past S land in the tile's padding (never read)
#pragma unroll
                for (int n = 0; n < TL; ++n) {
                    const int l = rb + slot(n);
                    if (l < L) {
                        double* o = A.out + ((tile * L + l) * 2 * (int64_t)g.E + 2 * e) * CS + s_w;
#pragma unroll
                        for (int j = 0; j < TS; j += 2) {
                            *reinterpret_cast<double2*>(o + j) = make_double2(g0[n] * Q[n][j], g0[n] * Q[n][j + 1]);
                            *reinterpret_cast<double2*>(o + CS + j) = make_double2(g0[n] * X[n][j], g0[n] * X[n][j + 1]);
                        }
                    }
                }
            }
        }
        if (in_tile) {  // the warp's TS sample rows of the tile -> u (coalesced)
            __syncwarp();
#pragma unroll
            for (int j = 0; j < TS; ++j) {
                const int64_t s = c0 + s_w + j;
                if (s < A.S) {
                    const uint32_t src = smem_u32(wtile + j * ms);
                    double* dst = A.out + s * N + off;
                    for (int p = lane; p < m; p += 32) dst[p] = lds_f64(src + 8u * p);
                }
            }
            __syncwarp();
        }
    }
}

// One instance: persistent CTAs (one per SM) over the atomic queue of E * ceil(S / CS) items.
template <int TL, int TS, bool REC>
cudaError_t launch(Args a, cudaStream_t st) {
    using C = Cfg<TL, TS, REC>;
    a.chunks = (int32_t)((a.S + C::CS - 1) / C::CS);
    a.n_items = a.g.E * a.chunks;
    size_t smem = C::FIXED + (REC ? (size_t)a.Lp * sizeof(double) : 0);
    a.tile_ms = 0;
    if (REC) {
        // the output tile holds edges with (m | 1) <= tile_ms; sized for the longest edge if it fits
        const int want = a.g.max_m | 1;
        const size_t room = sweep::SMEM_MAX > smem ? sweep::SMEM_MAX - smem : 0;
        const int fit = (int)(room / ((size_t)C::CS * sizeof(double)));
        a.tile_ms = want <= fit ? want : (fit >= 1 ? ((fit - 1) | 1) : 0);
        smem += (size_t)C::CS * a.tile_ms * sizeof(double);
    }
    cudaError_t e = cudaFuncSetAttribute(sweep2_kernel<TL, TS, REC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(a.counter, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return e;
    int blocks = a.g.n_sm > 0 ? a.g.n_sm : 148;
    if (blocks > a.n_items) blocks = a.n_items;
    sweep2_kernel<TL, TS, REC><<<blocks, C::NT, smem, st>>>(a);
    return cudaGetLastError();
}

template <bool REC, int TS>
cudaError_t launch_tl(int tl, Args a, cudaStream_t st) {
    switch (tl) {
        case 1: return launch<1, TS, REC>(a, st);
        case 2: return launch<2, TS, REC>(a, st);
        case 3: return launch<3, TS, REC>(a, st);
        case 4: return launch<4, TS, REC>(a, st);
        case 5: return launch<5, TS, REC>(a, st);
        case 6: return launch<6, TS, REC>(a, st);
        case 7: return launch<7, TS, REC>(a, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace sweep2
}  // namespace grf
