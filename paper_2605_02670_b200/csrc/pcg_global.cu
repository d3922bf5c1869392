// K4 global-memory variant of the batched NN-PCG for large vertex sets (V > 4096, config 4:
// V = 1e5).  Same operators and stopping rule as pcg.cu (PAPER.md P111-118, P241-298; the
// per-node tables DS/OS (Dirichlet step) and DM/OM (Neumann step) of pcg_tables_kernel).
//
// One cooperative persistent launch per sample tile of CS samples solves all L x CS systems
// (l, s) of the tile together.  Vertices are handled in breadth-first POSITIONS p (g.vorder,
// built at graph creation): work vectors are node-major, position, then sample:
// vec[(l * V + p) * CS + s], and the operator tables ops_pos are position-ordered CSR
// [DS (V) | DM (V) | DJ (V) | OS (2E) | OM (2E)] per node, so the CS threads of a vertex share
// its coefficients, every neighbour gather is one contiguous CS-double run, and a vertex's
// neighbours lie at nearby positions (their rows are reused from L2 instead of HBM).  Only
// the rhs read and the u_G write map positions back to vertices.  Per iteration two phases separated by grid
// barriers (standard PCG, fused so that each vector is streamed once per phase):
//   phase 1:  p' = z + beta p;  q = S p'  (neighbour p' formed on the fly from z, p);  p'.q
//   phase 2:  r' = r - alpha q;  x += alpha p';  z = M^{-1} r' (neighbour r' on the fly);
//             r'.r', r'.z
// p and r are double buffered (old values stay readable for the on-the-fly neighbours).
// Dot products: per (node, 256-vertex block) partials, reduced in fixed vertex-block order by
// the last block to arrive for that node (threadfence + arrival counter), so results are
// deterministic.  A node whose CS systems have all converged is skipped; the loop ends when
// no node is active or after max_iter iterations.
#include <algorithm>
#include <cmath>
#include <cooperative_groups.h>

#include "grf_internal.h"

namespace cg = cooperative_groups;

namespace grf {
namespace {

constexpr int GT = 256;  // threads per CTA = vertices per item
constexpr int NB = 4;    // neighbours gathered per batch (loads issued together)

struct GArgs {
    DevGraph g;
    int32_t L;
    const double* ops;    // ops_pos (position-ordered CSR tables)
    PcgParams prm;
    int64_t S;
    int32_t csl;
    int64_t tile;         // sample tile solved by this launch
    const double* rhs;    // [tile][l][cs][v] (grf_internal.h)
    double* uG;           // [tile][v][l][cs]
    int32_t* iters;       // [s * L + l]
    double* relres;
    double *x, *r0, *r1, *p0, *p1, *q, *z;   // [L][V][CS]
    double *alpha, *beta, *rz, *gg, *rr;    // [L][CS]
    int32_t* done;                          // [L][CS]
    int32_t* its;                           // [L][CS]
    int32_t* node_active;                   // [L]
    int32_t* n_active;                      // [1]
    int32_t* fin;                           // [L] iteration at which the node converged (-1: none)
    double* part;                           // [L][nvb][2][CS]
    int32_t* cnt;                           // [L] arrival counters (zero between phases)
    int32_t group;                          // nodes solved together (their work vectors stay L2-resident)
    int32_t vpi;                            // vertices per item (multiple of GT / CS)
};


// Threads: SP samples of one vertex each (SP = 2 for sample tiles of 16 or 32: double2
// accesses) -- thread t of a CTA owns samples s = SP * (t % TPV) .. + SP - 1 of vertex sub-row
// t / TPV (TPV = CS / SP threads per vertex); an item = (node l, block of VPI vertices) walked in
// sub-chunks of GT / TPV vertices, so a thread keeps only a few values (small register footprint,
// many resident warps for the latency of the neighbour gathers), and the TPV threads of a vertex
// read one contiguous CS-double run of each vector and share the vertex's operator coefficients.
constexpr int VPI_MAX = 256;  // vertices per item (at most): per-node partials have ceil(V / vpi) rows

template <int CS>
struct Lanes {
    static constexpr int SP = CS >= 2 ? 2 : 1;  // samples per thread
    static constexpr int TPV = CS / SP;         // threads per vertex
    static constexpr int VBK = GT / TPV;        // vertices per sub-chunk
};

template <int SP>
struct Vec {
    double v[SP];
};
template <int SP>
__device__ __forceinline__ Vec<SP> ldv(const double* p) {
    Vec<SP> r;
    if constexpr (SP == 2) {
        const double2 t = *reinterpret_cast<const double2*>(p);
        r.v[0] = t.x;
        r.v[1] = t.y;
    } else {
        r.v[0] = *p;
    }
    return r;
}
template <int SP>
__device__ __forceinline__ void stv(double* p, const Vec<SP>& a) {  // streaming store: keep L2 for the gathers
    if constexpr (SP == 2) {
        __stcs(reinterpret_cast<double2*>(p), make_double2(a.v[0], a.v[1]));
    } else {
        __stcs(p, a.v[0]);
    }
}

// Sum K x SP per-thread values over the CTA's vertices into red as [warp][k][s] rows summed over
// warps: tot(k, s) for this CTA, written to part[l][vb][k][s] by threads tid < K * CS.
template <int CS, int K>
__device__ __forceinline__ void cta_partials(const double (&v)[K][Lanes<CS>::SP], double* red, double* dst) {
    using LN = Lanes<CS>;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) {
#pragma unroll
        for (int j = 0; j < LN::SP; ++j) {
            double t = v[k][j];
#pragma unroll
            for (int o = 16; o >= LN::TPV && o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);  // over vertex lanes
            if (lane < (LN::TPV < 32 ? LN::TPV : 32)) red[(warp * K + k) * CS + (lane % LN::TPV) * LN::SP + j] = t;
        }
    }
    __syncthreads();
    if (tid < K * CS) {
        const int k = tid / CS, s = tid % CS;
        double t = 0.0;
        for (int w = 0; w < GT / 32; ++w) t += red[(w * K + k) * CS + s];
        dst[tid] = t;
    }
}

// Reduce the per-thread values into part[l][vb][k][s]; the last CTA of node l to arrive reduces the
// node's rows (columns in parallel, each in fixed order) and runs finish(l, totals) with
// totals[k * CS + s] in shared memory (all threads of that CTA).
template <int CS, int K, class Finish>
__device__ void block_partials(const GArgs& A, int l, int vb, int nvb, const double (&v)[K][Lanes<CS>::SP],
                               double* red, Finish&& finish) {
    const int tid = threadIdx.x;
    __shared__ int last;
    double* pb = A.part + ((int64_t)l * nvb + vb) * 2 * CS;
    cta_partials<CS, K>(v, red, pb);
    if (tid < K * CS) __threadfence();
    __syncthreads();
    if (tid == 0) last = (atomicAdd(&A.cnt[l], 1) == nvb - 1);
    __syncthreads();
    if (last) {
        __threadfence();
        constexpr int NCOL = K * CS;
        constexpr int TPC = GT / NCOL;
        const int col = tid / TPC, sub = tid % TPC;
        double t = 0.0;
        if (col < NCOL) {
            const double* pc = A.part + (int64_t)l * nvb * 2 * CS + col;
            for (int b = sub; b < nvb; b += TPC) t += pc[(int64_t)b * 2 * CS];
        }
        __syncthreads();  // red is reused
        red[tid] = t;
        __syncthreads();
        if (tid < NCOL) {
            double u = 0.0;
            for (int q = 0; q < TPC; ++q) u += red[tid * TPC + q];
            red[GT + tid] = u;
        }
        __syncthreads();
        finish(l, red + GT);
        __syncthreads();
        if (tid == 0) A.cnt[l] = 0;
    }
    __syncthreads();
}

// Iteration phases: each item only writes its partial row (no arrival counter); after a grid
// barrier one CTA per active node reduces the node's rows in the same fixed order as the
// last-arriving CTA of block_partials does and runs finish(l, totals).
template <int CS, int K>
__device__ void item_partials(const GArgs& A, int l, int vb, int nvb, const double (&v)[K][Lanes<CS>::SP],
                              double* red) {
    cta_partials<CS, K>(v, red, A.part + ((int64_t)l * nvb + vb) * 2 * CS);
    __syncthreads();  // red is reused by the next item
}

template <int CS, int K, class Finish>
__device__ void node_reduce(const GArgs& A, int l, int nvb, double* red, Finish&& finish) {
    const int tid = threadIdx.x;
    constexpr int NCOL = K * CS;
    constexpr int TPC = GT / NCOL;
    const int col = tid / TPC, sub = tid % TPC;
    double t = 0.0;
    if (col < NCOL) {
        const double* pc = A.part + (int64_t)l * nvb * 2 * CS + col;
        for (int b = sub; b < nvb; b += TPC) t += pc[(int64_t)b * 2 * CS];
    }
    red[tid] = t;
    __syncthreads();
    if (tid < NCOL) {
        double u = 0.0;
        for (int q = 0; q < TPC; ++q) u += red[tid * TPC + q];
        red[GT + tid] = u;
    }
    __syncthreads();
    finish(l, red + GT);
    __syncthreads();
}

// p_k of iteration k lives in p1 for even k, p0 for odd k (po / pn swap after every iteration)
__device__ __forceinline__ bool p_in_p1(int k) { return (k & 1) == 0; }

template <int CS>
__global__ void __launch_bounds__(GT, 4) pcg_global_kernel(GArgs A) {
    using LN = Lanes<CS>;
    constexpr int SP = LN::SP, VBK = LN::VBK;
    using VS = Vec<SP>;
    cg::grid_group grid = cg::this_grid();
    constexpr int RED = (GT + 2 * CS) > ((GT / 32) * 2 * CS) ? (GT + 2 * CS) : ((GT / 32) * 2 * CS);
    __shared__ double red[RED];
    const DevGraph& g = A.g;
    const int V = g.V, L = A.L;
    const int64_t E2 = 2 * (int64_t)g.E;
    const int VPI = A.vpi;
    const int nvb = (V + VPI - 1) / VPI;
    const int tid = threadIdx.x, s = (tid % LN::TPV) * SP, vl = tid / LN::TPV;
    const int64_t stride = 3 * (int64_t)V + 2 * E2;  // position table per node
    const int64_t s0 = A.tile << A.csl;
    double *po, *pn, *ro, *rn;
    const double tol2c = A.prm.rtol * A.prm.rtol;

    // the vertex of sub-chunk c of item vb for this thread (or -1: none)
    auto vert = [&](int vb, int c) { const int v = vb * VPI + c * VBK + vl; return v < V ? v : -1; };
    auto vzero = [] {
        VS r;
#pragma unroll
        for (int j = 0; j < SP; ++j) r.v[j] = 0.0;
        return r;
    };

    // Node groups are solved one after the other (the launcher currently uses one group of all
    // nodes: per-group barriers outweighed the L2 residency they buy on config 4).
    for (int l0 = 0; l0 < L; l0 += A.group) {
    po = A.p0;
    pn = A.p1;
    ro = A.r0;
    rn = A.r1;
    const int lg = (L - l0) < A.group ? (L - l0) : A.group;
    const int64_t items = (int64_t)lg * nvb;
    if (blockIdx.x == 0 && tid == 0) *A.n_active = 0;  // all blocks have left the previous group's loop
    // ---- init a: r = g, x = 0, p = 0; gg = g.g
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        const int l = l0 + (int)(it / nvb), vb = (int)(it % nvb);
        const int64_t lb = (int64_t)l * V * CS;  // node l's [V][CS] slab
        double acc[1][SP] = {};
        for (int c = 0; c < VPI / VBK; ++c) {
            const int v = vert(vb, c);
            if (v < 0) continue;
            const int e = v * CS + s;  // offset within node l's [V][CS] slab (32-bit)
            VS gv;
#pragma unroll
            for (int j = 0; j < SP; ++j) {
                const int64_t sg = s0 + s + j;
                gv.v[j] = sg < A.S ? A.rhs[rhs_index(sg, l, g.vorder[v], L, V, A.csl)] : 0.0;
                acc[0][j] = fma(gv.v[j], gv.v[j], acc[0][j]);
            }
            stv(ro + lb + e, gv);
            stv(A.x + lb + e, vzero());
            stv(po + lb + e, vzero());
        }
        block_partials<CS, 1>(A, l, vb, nvb, acc, red, [&](int ln, const double* tot) {
            if (tid < CS) {
                const double t = tot[tid];
                A.gg[ln * CS + tid] = t;
                A.rr[ln * CS + tid] = t;
                A.done[ln * CS + tid] = !(t > 0.0) || (s0 + tid >= A.S);
                A.its[ln * CS + tid] = 0;
                A.beta[ln * CS + tid] = 0.0;
                A.alpha[ln * CS + tid] = 0.0;  // phase 1 of iteration 0 adds alpha p_{-1} = 0 to x
            }
            if (tid == 0) A.fin[ln] = -1;
        });
    }
    grid.sync();
    // ---- init b: z = M^{-1} r; rz
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        const int l = l0 + (int)(it / nvb), vb = (int)(it % nvb);
        const int64_t lb = (int64_t)l * V * CS;  // node l's [V][CS] slab
        const double* const ro_l = ro + lb;
        const double* tab = A.ops + l * stride;
        double acc[1][SP] = {};
        for (int c = 0; c < VPI / VBK; ++c) {
            const int v = vert(vb, c);
            if (v < 0) continue;
            const int e = v * CS + s;  // offset within node l's [V][CS] slab (32-bit)
            const VS rv = ldv<SP>(ro_l + e);
            VS zv;
            if (A.prm.precond == 0) {
                const double d = tab[V + v];
#pragma unroll
                for (int j = 0; j < SP; ++j) zv.v[j] = d * rv.v[j];
                for (int k = g.gp_ptr[v]; k < g.gp_ptr[v + 1]; ++k) {
                    const double cf = tab[3 * (int64_t)V + E2 + k];
                    const VS ro_o = ldv<SP>(ro_l + g.gp_other[k] * CS + s);
#pragma unroll
                    for (int j = 0; j < SP; ++j) zv.v[j] = fma(cf, ro_o.v[j], zv.v[j]);
                }
            } else {
                const double d = A.prm.precond == 1 ? tab[2 * V + v] : 1.0;
#pragma unroll
                for (int j = 0; j < SP; ++j) zv.v[j] = d * rv.v[j];
            }
            stv(A.z + lb + e, zv);
#pragma unroll
            for (int j = 0; j < SP; ++j) acc[0][j] = fma(rv.v[j], zv.v[j], acc[0][j]);
        }
        block_partials<CS, 1>(A, l, vb, nvb, acc, red, [&](int ln, const double* tot) {
            if (tid < CS) A.rz[ln * CS + tid] = tot[tid];
            if (tid == 0) {
                int act = 0;
                for (int q = 0; q < CS; ++q) act |= !A.done[ln * CS + q];
                A.node_active[ln] = act;
                if (act) atomicAdd(A.n_active, 1);
            }
        });
    }
    grid.sync();

    int iters_run = 0;
    for (int iter = 0; iter < A.prm.max_iter; ++iter) {
        if (*(volatile int32_t*)A.n_active == 0) break;
        iters_run = iter + 1;
        // ---- phase 1: x += alpha_{k-1} p_{k-1};  p' = z + beta p, q = S p', p'.q -> alpha
        for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
            const int l = l0 + (int)(it / nvb), vb = (int)(it % nvb);
            if (!A.node_active[l]) continue;  // block-uniform
            const int64_t lb = (int64_t)l * V * CS;  // node l's [V][CS] slab
            const double* const po_l = po + lb;
            const double* const z_l = A.z + lb;
            const double* tab = A.ops + l * stride;
            double bt[SP], alo[SP];
#pragma unroll
            for (int j = 0; j < SP; ++j) {
                bt[j] = A.beta[l * CS + s + j];
                alo[j] = A.alpha[l * CS + s + j];
            }
            double acc[1][SP] = {};
            for (int c = 0; c < VPI / VBK; ++c) {
                const int v = vert(vb, c);
                if (v < 0) continue;
                const int e = v * CS + s;  // offset within node l's [V][CS] slab (32-bit)
                const VS p_old = ldv<SP>(po_l + e), z_own = ldv<SP>(z_l + e), x_old = ldv<SP>(A.x + lb + e);
                const double dS = tab[v];
                VS pv, qv, xv;
#pragma unroll
                for (int j = 0; j < SP; ++j) {
                    pv.v[j] = fma(bt[j], p_old.v[j], z_own.v[j]);
                    qv.v[j] = dS * pv.v[j];
                    xv.v[j] = fma(alo[j], p_old.v[j], x_old.v[j]);
                }
                // neighbours in chunks of NB: indices and coefficients first, then every vector load,
                // then the FMAs (many loads in flight per thread; padding slots read the own row)
                const int kb = g.gp_ptr[v], ke = g.gp_ptr[v + 1];
                for (int k0 = kb; k0 < ke; k0 += NB) {
                    int ob[NB];
                    double cf[NB];
                    VS a[NB], b[NB];
#pragma unroll
                    for (int j = 0; j < NB; ++j) {
                        const bool ok = k0 + j < ke;
                        ob[j] = (ok ? g.gp_other[k0 + j] : v) * CS + s;
                        cf[j] = ok ? tab[3 * (int64_t)V + k0 + j] : 0.0;
                    }
#pragma unroll
                    for (int j = 0; j < NB; ++j) {
                        a[j] = ldv<SP>(po_l + ob[j]);
                        b[j] = ldv<SP>(z_l + ob[j]);
                    }
#pragma unroll
                    for (int j = 0; j < NB; ++j) {
#pragma unroll
                        for (int i = 0; i < SP; ++i) qv.v[i] = fma(cf[j], fma(bt[i], a[j].v[i], b[j].v[i]), qv.v[i]);
                    }
                }
                stv(pn + lb + e, pv);
                stv(A.q + lb + e, qv);
                stv(A.x + lb + e, xv);
#pragma unroll
                for (int j = 0; j < SP; ++j) acc[0][j] = fma(pv.v[j], qv.v[j], acc[0][j]);
            }
            item_partials<CS, 1>(A, l, vb, nvb, acc, red);
        }
        grid.sync();
        for (int l = l0 + blockIdx.x; l < l0 + lg; l += gridDim.x) {
            if (!A.node_active[l]) continue;  // block-uniform
            node_reduce<CS, 1>(A, l, nvb, red, [&](int ln, const double* tot) {
                if (tid < CS) {
                    const double pq = tot[tid];
                    if (!(pq > 0.0)) A.done[ln * CS + tid] = 1;  // p = 0 (underflowed rhs)
                    A.alpha[ln * CS + tid] = A.done[ln * CS + tid] ? 0.0 : A.rz[ln * CS + tid] / pq;
                }
            });
        }
        grid.sync();
        // ---- phase 2: r' = r - alpha q, z = M^{-1} r', r'.r', r'.z -> beta, convergence
        //      (x takes alpha p' in the next phase 1, or in the write-out)
        for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
            const int l = l0 + (int)(it / nvb), vb = (int)(it % nvb);
            if (!A.node_active[l]) continue;
            const int64_t lb = (int64_t)l * V * CS;  // node l's [V][CS] slab
            const double* const ro_l = ro + lb;
            const double* const q_l = A.q + lb;
            const double* tab = A.ops + l * stride;
            double al[SP];
#pragma unroll
            for (int j = 0; j < SP; ++j) al[j] = A.alpha[l * CS + s + j];
            double acc[2][SP] = {};
            for (int c = 0; c < VPI / VBK; ++c) {
                const int v = vert(vb, c);
                if (v < 0) continue;
                const int e = v * CS + s;  // offset within node l's [V][CS] slab (32-bit)
                const VS q_own = ldv<SP>(q_l + e), r_own = ldv<SP>(ro_l + e);
                VS rv, zv;
#pragma unroll
                for (int j = 0; j < SP; ++j) rv.v[j] = fma(-al[j], q_own.v[j], r_own.v[j]);
                if (A.prm.precond == 0) {
                    const double d = tab[V + v];
#pragma unroll
                    for (int j = 0; j < SP; ++j) zv.v[j] = d * rv.v[j];
                    const int kb = g.gp_ptr[v], ke = g.gp_ptr[v + 1];
                    for (int k0 = kb; k0 < ke; k0 += NB) {
                        int ob[NB];
                        double cf[NB];
                        VS a[NB], b[NB];
#pragma unroll
                        for (int j = 0; j < NB; ++j) {
                            const bool ok = k0 + j < ke;
                            ob[j] = (ok ? g.gp_other[k0 + j] : v) * CS + s;
                            cf[j] = ok ? tab[3 * (int64_t)V + E2 + k0 + j] : 0.0;
                        }
#pragma unroll
                        for (int j = 0; j < NB; ++j) {
                            a[j] = ldv<SP>(q_l + ob[j]);
                            b[j] = ldv<SP>(ro_l + ob[j]);
                        }
#pragma unroll
                        for (int j = 0; j < NB; ++j) {
#pragma unroll
                            for (int i = 0; i < SP; ++i) zv.v[i] = fma(cf[j], fma(-al[i], a[j].v[i], b[j].v[i]), zv.v[i]);
                        }
                    }
                } else {
                    const double d = A.prm.precond == 1 ? tab[2 * V + v] : 1.0;
#pragma unroll
                    for (int j = 0; j < SP; ++j) zv.v[j] = d * rv.v[j];
                }
                stv(rn + lb + e, rv);
                stv(A.z + lb + e, zv);
#pragma unroll
                for (int j = 0; j < SP; ++j) {
                    acc[0][j] = fma(rv.v[j], rv.v[j], acc[0][j]);
                    acc[1][j] = fma(rv.v[j], zv.v[j], acc[1][j]);
                }
            }
            item_partials<CS, 2>(A, l, vb, nvb, acc, red);
        }
        grid.sync();
        for (int l = l0 + blockIdx.x; l < l0 + lg; l += gridDim.x) {
            if (!A.node_active[l]) continue;  // block-uniform
            node_reduce<CS, 2>(A, l, nvb, red, [&](int ln, const double* tot) {
                if (tid < CS) {
                    const int sy = ln * CS + tid;
                    const double rr = tot[tid], rzn = tot[CS + tid];
                    if (!A.done[sy]) {
                        A.its[sy] += 1;
                        A.rr[sy] = rr;
                        if (rr <= tol2c * A.gg[sy]) A.done[sy] = 1;
                        A.beta[sy] = A.done[sy] ? 0.0 : rzn / A.rz[sy];
                        A.rz[sy] = rzn;
                    } else {
                        A.beta[sy] = 0.0;
                    }
                }
                __syncthreads();
                if (tid == 0) {
                    int act = 0;
                    for (int q = 0; q < CS; ++q) act |= !A.done[ln * CS + q];
                    if (!act) {
                        A.node_active[ln] = 0;
                        A.fin[ln] = iter;  // p' of this iteration: its last alpha p' goes to x at the write-out
                        atomicSub(A.n_active, 1);
                    }
                }
            });
        }
        grid.sync();
        double* t = po;
        po = pn;
        pn = t;
        t = ro;
        ro = rn;
        rn = t;
    }
    // ---- write u_G = x + alpha_last p_last, iteration counts and final relative residuals
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        const int l = l0 + (int)(it / nvb), vb = (int)(it % nvb);
        const int kl = A.node_active[l] ? iters_run - 1 : A.fin[l];  // the node's last iteration (-1: none)
        const double* pl = (kl < 0 ? A.p0 : (p_in_p1(kl) ? A.p1 : A.p0)) + (int64_t)l * V * CS;
        double al[SP];
#pragma unroll
        for (int j = 0; j < SP; ++j) al[j] = kl < 0 ? 0.0 : A.alpha[l * CS + s + j];
        for (int c = 0; c < VPI / VBK; ++c) {
            const int v = vert(vb, c);
            if (v < 0) continue;
            const int e = v * CS + s;
            const VS xv = ldv<SP>(A.x + (int64_t)l * V * CS + e);
#pragma unroll
            for (int j = 0; j < SP; ++j) {
                const int64_t sg = s0 + s + j;
                if (sg >= A.S) continue;
                const double xo = al[j] != 0.0 ? fma(al[j], pl[e + j], xv.v[j]) : xv.v[j];
                A.uG[ug_index(sg, g.vorder[v], l, L, V, A.csl)] = xo;
            }
        }
        if (vb == 0 && tid < CS && s0 + tid < A.S) {
            const int sy = l * CS + tid;
            A.iters[(s0 + tid) * L + l] = A.its[sy];
            A.relres[(s0 + tid) * L + l] = A.gg[sy] > 0.0 ? sqrt(A.rr[sy] / A.gg[sy]) : 0.0;
        }
    }
    grid.sync();  // before the next group resets n_active
    }
}

template <int CS>
cudaError_t launch_cs(GArgs a, int64_t n_tiles, cudaStream_t st) {
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcg_global_kernel<CS>, GT, 0);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorLaunchOutOfResources;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = sms * per_sm;
    // node groups: all nodes together.  (Solving L2-sized groups one after the other was measured
    // on config 4: the per-group grid barriers cost more than the HBM traffic they save.)
    a.group = a.L;
    // vertices per item: enough items per phase for about two per CTA
    const int vbk = Lanes<CS>::VBK;
    a.vpi = VPI_MAX;
    while (a.vpi > vbk && (int64_t)a.group * ((a.g.V + a.vpi - 1) / a.vpi) < 2 * (int64_t)blocks) a.vpi /= 2;
    if (a.vpi < vbk) a.vpi = vbk;
    for (int64_t t = 0; t < n_tiles; ++t) {
        a.tile = t;
        e = cudaMemsetAsync(a.n_active, 0, sizeof(int32_t), st);
        if (e != cudaSuccess) return e;
        e = cudaMemsetAsync(a.cnt, 0, sizeof(int32_t) * a.L, st);
        if (e != cudaSuccess) return e;
        void* args[] = {&a};
        e = cudaLaunchCooperativeKernel((const void*)pcg_global_kernel<CS>, dim3(blocks), dim3(GT), args, 0, st);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// Position-ordered CSR tables of the two PCG operators (same values as pcg_tables_kernel in
// pcg.cu, P247-298): DS_p = sum of the incident local Schur diagonals, OS_k = their off-diagonal,
// DM_p = sum of the inverse blocks' diagonals / d_v^2, OM_k = off-diagonal / (d_v d_o), DJ = 1/diag S.
__global__ void pcg_tables_pos_kernel(DevGraph g, int32_t L, const double4* __restrict__ sig, double* __restrict__ ops) {
    const int V = g.V, E = g.E;
    const int64_t E2 = 2 * (int64_t)E, stride = 3 * (int64_t)V + 2 * E2;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < (int64_t)L * V;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int l = (int)(x / V), p = (int)(x - (int64_t)l * V);
        const int v = g.vorder[p];
        const double4* sg = sig + (int64_t)l * E;
        double* t = ops + l * stride;
        const double idv = g.inv_deg[v];
        double ds = 0.0, dm = 0.0, diag = 0.0;
        for (int k = g.gp_ptr[p]; k < g.gp_ptr[p + 1]; ++k) {
            const double4 c = sg[g.gp_code[k] >> 1];
            const int op = g.gp_other[k];
            ds += c.x;
            dm += c.z;
            t[3 * (int64_t)V + k] = c.y;
            t[3 * (int64_t)V + E2 + k] = c.w * idv * g.inv_deg[g.vorder[op]];
            diag += c.x + (op == p ? c.y : 0.0);
        }
        t[p] = ds;
        t[V + p] = dm * idv * idv;
        t[2 * V + p] = 1.0 / diag;
    }
}

// vertices per sub-chunk = the smallest item (Lanes<CS>::VBK)
int vbk_min(int64_t cs) { return cs == 1 ? Lanes<1>::VBK : (cs == 16 ? Lanes<16>::VBK : Lanes<32>::VBK); }

}  // namespace

void launch_pcg_tables_pos(const DevGraph& g, const DevPlan& p, cudaStream_t st) {
    const int64_t n = (int64_t)p.L * g.V;
    if (n == 0) return;
    int blocks = (int)((n + 255) / 256);
    if (blocks > g.n_sm * 8) blocks = g.n_sm * 8;
    pcg_tables_pos_kernel<<<blocks, 256, 0, st>>>(g, p.L, reinterpret_cast<const double4*>(p.sig), p.ops_pos);
}

size_t pcg_global_ws_bytes(const DevGraph& g, int32_t L, int64_t n_samples) {
    const int64_t cs = (int64_t)1 << sample_tile_log2(n_samples);
    const int64_t nvb = (g.V + vbk_min(cs) - 1) / vbk_min(cs);  // rows for the smallest item size
    size_t b = 7 * sizeof(double) * (size_t)L * g.V * cs;      // x, r0, r1, p0, p1, q, z
    b += 5 * sizeof(double) * (size_t)L * cs;                  // alpha, beta, rz, gg, rr
    b += 2 * sizeof(int32_t) * (size_t)L * cs;                 // done, its
    b += sizeof(int32_t) * (size_t)(L + 1);                    // node_active, n_active
    b += sizeof(double) * (size_t)L * nvb * 2 * cs;            // partials
    b += 2 * sizeof(int32_t) * (size_t)L;                      // counters, fin
    return b + 16 * 256;
}

cudaError_t launch_pcg_global(const DevGraph& g, const DevPlan& p, int64_t n_samples, const PcgParams& prm,
                              const double* rhs, double* uG, int32_t* iters, double* relres, void* ws,
                              cudaStream_t st) {
    const int32_t csl = sample_tile_log2(n_samples);
    const int64_t cs = (int64_t)1 << csl;
    const int64_t L = p.L;
    const int64_t nvb = (g.V + vbk_min(cs) - 1) / vbk_min(cs);
    char* b = static_cast<char*>(ws);
    auto take = [&](size_t bytes) {
        char* r = b;
        b += (bytes + 255) & ~size_t(255);
        return r;
    };
    GArgs a{};
    a.g = g;
    a.L = p.L;
    a.ops = p.ops_pos;
    a.prm = prm;
    a.S = n_samples;
    a.csl = csl;
    a.rhs = rhs;
    a.uG = uG;
    a.iters = iters;
    a.relres = relres;
    const size_t vec = sizeof(double) * (size_t)L * g.V * cs;
    a.x = (double*)take(vec);
    a.r0 = (double*)take(vec);
    a.r1 = (double*)take(vec);
    a.p0 = (double*)take(vec);
    a.p1 = (double*)take(vec);
    a.q = (double*)take(vec);
    a.z = (double*)take(vec);
    const size_t sys = (size_t)L * cs;
    a.alpha = (double*)take(sizeof(double) * sys);
    a.beta = (double*)take(sizeof(double) * sys);
    a.rz = (double*)take(sizeof(double) * sys);
    a.gg = (double*)take(sizeof(double) * sys);
    a.rr = (double*)take(sizeof(double) * sys);
    a.done = (int32_t*)take(sizeof(int32_t) * sys);
    a.its = (int32_t*)take(sizeof(int32_t) * sys);
    a.node_active = (int32_t*)take(sizeof(int32_t) * L);
    a.n_active = (int32_t*)take(sizeof(int32_t));
    a.part = (double*)take(sizeof(double) * (size_t)L * nvb * 2 * cs);
    a.cnt = (int32_t*)take(sizeof(int32_t) * L);
    a.fin = (int32_t*)take(sizeof(int32_t) * L);
    const int64_t n_tiles = (n_samples + cs - 1) / cs;
    switch (cs) {
        case 1: return launch_cs<1>(a, n_tiles, st);
        case 16: return launch_cs<16>(a, n_tiles, st);
        case 32: return launch_cs<32>(a, n_tiles, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace grf
