// K4: batched matrix-free PCG on the vertex Schur systems  (PAPER.md P111-118, P241-298).
//
//     S^{(l)} u_G = g,   S^{(l)} = sum_e R_e^T S^{(l,e)} R_e        (P113-116, P244 [eq:goal_func_1])
//
// Dirichlet step (P247-258): y = S p evaluated edge-locally; with the exact 2x2 local
// Schur blocks of K2, (S p)_v = sum_{(e,end) at v} (s_d p_v + s_o p_other).
// Neumann step (P260-298): z = D^{-1} (sum_e R_e^T S_e^{-1} R_e) D^{-1} r, i.e.
//     r~ = r / d (eq:distribute_dv), delta = S_e^{-1} r~ per edge, z_v = (1/d_v) sum delta
// (eq:induced_displacements); D_vv = d_v = incident edge ends.
// A loop edge has other == v, so both its ends add to v (sum of all 4 entries, Q18).
// Stopping rule: ||r_k||_2 <= rtol ||g||_2, x_0 = 0.
//
// Both operators are applied in the same "diagonal + incidence slots" form, from per-node
// tables built once per plan (pcg_tables_kernel).  The incidence lists are padded to the
// ELL width W (max degree rounded up to a power of two; padding slots point at v with a
// zero coefficient), so every (vertex, slot) loop is fully unrolled with independent loads:
//     (S p)_v      = DS_v p_v + sum_j OS_jv p_{o_jv},     DS_v = sum s_d,   OS = s_o
//     (M^{-1} r)_v = DM_v r_v + sum_j OM_jv r_{o_jv},     DM_v = d_v^-2 sum p_d,
//                                                         OM = p_o / (d_v d_o)
//     Jacobi:        DJ_v r_v,                            DJ_v = 1 / diag(S)_v
//     condensed rhs  g_v = W_v + sum_j GK_jv w_{c_jv},    GK = c_L / h_e     (P233-239, Q6)
//
// Mapping: CTA = (node l, chunk of samples) split into independent thread groups (named
// barriers) that share the node's tables, staged once in shared memory.  Each group solves
// batches of SB samples: r and p are [V][SB] in shared memory, x/q/z live in registers of
// the vertex's owner thread, and one group reduction (a single barrier) per dot product
// carries all SB values.  Each sample has its own alpha/beta and stops at its own
// convergence.  g is read from the assembled rhs (K4a, assemble_rhs_kernel);
// u_G is written to uG[(s*V + v)*L + l].
#include <cstdlib>

#include "grf_internal.h"
#include "thomas.cuh"

namespace grf {
namespace {

constexpr int PCG_THREADS = 512;
constexpr size_t SMEM_LIMIT = 220 * 1024;

// per node l: [DS (V) | DM (V) | DJ (V) | OS (W*V) | OM (W*V) | GK (W*V)], slot-major [j][v]
__host__ __device__ inline int64_t table_stride(int V, int W) { return 3 * (int64_t)V + 3 * (int64_t)W * V; }

__global__ void pcg_tables_kernel(DevGraph g, int32_t L, const double* __restrict__ cIt,
                                  const double* __restrict__ cLt, double kappa2, int32_t mass,
                                  const double4* __restrict__ sig, double* __restrict__ ops) {
    const int V = g.V, E = g.E;
    const int64_t stride = ops_stride(g), ns = ops_nslots(g);
    const int slots = g.csr ? 0 : g.ell_w;  // ELL: also write the padding slots
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < (int64_t)L * V;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int l = (int)(x / V), v = (int)(x - (int64_t)l * V);
        const double4* sg = sig + (int64_t)l * E;
        double* t = ops + l * stride;
        double* DS = t;
        double* DM = DS + V;
        double* DJ = DM + V;
        double* OS = DJ + V;
        double* OM = OS + ns;
        double* GK = OM + ns;
        const double idv = g.inv_deg[v];
        const double cL = cLt[l];
        const int dg = g.inc_ptr[v + 1] - g.inc_ptr[v];
        double ds = 0.0, dm = 0.0, diag = 0.0;
        for (int j = 0; j < (slots > dg ? slots : dg); ++j) {
            const int64_t sj = ops_slot(g, v, j);
            if (j < dg) {
                const int e = ops_code(g, sj) >> 1;
                const double4 c = sg[e];
                const int o = ops_other(g, sj);
                ds += c.x;
                dm += c.z;
                OS[sj] = c.y;
                OM[sj] = c.w * idv * g.inv_deg[o];
                GK[sj] = mass ? edge_coef(cIt[l], cL, kappa2, g.h[e], 1).beta : cL / g.h[e];  // -b (A_GI)
                diag += c.x + (o == v ? c.y : 0.0);
            } else {
                OS[sj] = OM[sj] = GK[sj] = 0.0;
            }
        }
        DS[v] = ds;
        DM[v] = dm * idv * idv;
        DJ[v] = 1.0 / diag;
    }
}

// named barrier for one thread group (ids 1..15; id 0 is __syncthreads)
__device__ __forceinline__ void group_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Group-wide sum of NV doubles per thread, broadcast back.  One barrier per call: the
// partials go to buffer `flip`, and consecutive calls alternate buffers, so a buffer is
// rewritten only after every thread has passed the next call's barrier.
template <int GT, int NV>
__device__ __forceinline__ void group_sum(double (&v)[NV], double* red /* [2][GT/32][NV] */, int& flip, int bar_id) {
    constexpr int NW = GT / 32;
    const int lane = threadIdx.x & 31, w = (threadIdx.x % GT) >> 5;
    double* rb = red + flip * NW * NV;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        double t = v[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) rb[w * NV + j] = t;
    }
    group_bar(bar_id, GT);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < NW; ++q) t += rb[q * NV + j];
        v[j] = t;
    }
    flip ^= 1;
}

// group-wide max of NV non-negative doubles per thread (same buffering as group_sum)
template <int GT, int NV>
__device__ __forceinline__ void group_max(double (&v)[NV], double* red, int& flip, int bar_id) {
    constexpr int NW = GT / 32;
    const int lane = threadIdx.x & 31, w = (threadIdx.x % GT) >> 5;
    double* rb = red + flip * NW * NV;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        double t = v[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, o));
        if (lane == 0) rb[w * NV + j] = t;
    }
    group_bar(bar_id, GT);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < NW; ++q) t = fmax(t, rb[q * NV + j]);
        v[j] = t;
    }
    flip ^= 1;
}

template <int GT, int SB, int VPT, int W, bool STAGED>
__global__ void __launch_bounds__(PCG_THREADS) pcg_kernel(DevGraph g, int32_t L, const double* __restrict__ ops,
                                                          PcgParams prm, int64_t S, int32_t spc, int32_t csl,
                                                          const double* __restrict__ rhs, double* __restrict__ uG, int32_t* __restrict__ iters,
                                                          double* __restrict__ relres) {
    constexpr int NG = PCG_THREADS / GT;
    constexpr int NW = GT / 32;
    extern __shared__ double sm[];
    __shared__ double red_all[NG][2 * NW * 2 * SB];
    const int V = g.V;
    const int64_t stride = table_stride(V, W);
    const int l = blockIdx.x;
    const int tid = threadIdx.x;
    const int gid = tid / GT, gt = tid % GT;
    const int bar_id = 1 + gid;
    double* r = sm + (size_t)gid * 2 * V * SB;  // [V][SB] per group
    double* p = r + (size_t)V * SB;            // [V][SB] per group
    double* red = red_all[gid];
    int flip = 0;
    const double* tab = ops + l * stride;
    const int* eo = g.ell_other;
    const int* ec = g.ell_code;
    if (STAGED) {  // node tables + ELL index arrays into shared memory, once per CTA
        double* st = sm + (size_t)NG * 2 * V * SB;
        int* so = reinterpret_cast<int*>(st + stride);
        int* sc = so + W * V;
        for (int64_t i = tid; i < stride; i += PCG_THREADS) st[i] = tab[i];
        for (int i = tid; i < W * V; i += PCG_THREADS) {
            so[i] = g.ell_other[i];
            sc[i] = g.ell_code[i];
        }
        tab = st;
        eo = so;
        ec = sc;
    }
    __syncthreads();
    const double* DS = tab;
    const double* DM = DS + V;
    const double* DJ = DM + V;
    const double* OS = DJ + V;
    const double* OM = OS + (size_t)W * V;

    // y = D x + sum_j O_j x_{o_j} over the owner's vertices, for SB samples (x = r or p in smem)
    auto apply = [&](const double* D, const double* O, const double* xs, double (&y)[VPT][SB]) {
#pragma unroll
        for (int a = 0; a < VPT; ++a) {
            const int v = gt + a * GT;
            if (v < V) {
                const double d = D[v];
#pragma unroll
                for (int j = 0; j < SB; ++j) y[a][j] = d * xs[v * SB + j];
#pragma unroll
                for (int s = 0; s < W; ++s) {
                    const double c = O[s * V + v];
                    const double* xo = xs + eo[s * V + v] * SB;
#pragma unroll
                    for (int j = 0; j < SB; ++j) y[a][j] += c * xo[j];
                }
            }
        }
    };
    // z = M^{-1} r (Neumann step); needs r of neighbours: callers barrier first
    auto precond = [&](double (&z)[VPT][SB]) {
        if (prm.precond == 0) {
            apply(DM, OM, r, z);
        } else {
#pragma unroll
            for (int a = 0; a < VPT; ++a) {
                const int v = gt + a * GT;
                if (v < V) {
                    const double d = prm.precond == 1 ? DJ[v] : 1.0;
#pragma unroll
                    for (int j = 0; j < SB; ++j) z[a][j] = d * r[v * SB + j];
                }
            }
        }
    };

    const int64_t c0 = (int64_t)blockIdx.y * spc;
    const int64_t c1 = (c0 + spc) < S ? (c0 + spc) : S;
    for (int64_t s0 = c0 + (int64_t)gid * SB; s0 < c1; s0 += (int64_t)NG * SB) {
        const int ns = (int)((c1 - s0) < SB ? (c1 - s0) : SB);
        double x[VPT][SB], q[VPT][SB];
        double gg[SB];
#pragma unroll
        for (int j = 0; j < SB; ++j) gg[j] = 0.0;
        // ---- condensed rhs g, x = 0, r = g; a rhs whose squared norm is near the fp64 range limits is
        // rescaled by a power of two (see pcg_warp.cu: exact, and it keeps the iteration away from
        // underflow for rhs that decayed to ~1e-300) -- a second pass only on that rare path
#pragma unroll
        for (int a = 0; a < VPT; ++a) {
            const int v = gt + a * GT;
#pragma unroll
            for (int j = 0; j < SB; ++j) x[a][j] = 0.0;
            if (v < V) {
#pragma unroll
                for (int j = 0; j < SB; ++j) {
                    const int64_t s = s0 + (j < ns ? j : 0);
                    double gv = rhs[rhs_index(s, l, v, L, V, csl)];
                    if (j >= ns) gv = 0.0;
                    r[v * SB + j] = gv;
                    gg[j] += gv * gv;
                }
            }
        }
        group_sum<GT, SB>(gg, red, flip, bar_id);  // (barrier: r complete)
        double sup[SB];  // exact powers of two
        bool rescale = false;
#pragma unroll
        for (int j = 0; j < SB; ++j) {
            sup[j] = 1.0;
            rescale = rescale || (gg[j] > 0.0 && (gg[j] < 0x1p-900 || gg[j] > 0x1p900));
        }
        if (rescale) {  // group-uniform (gg is the group sum)
            double gmax[SB];
#pragma unroll
            for (int j = 0; j < SB; ++j) gmax[j] = 0.0;
#pragma unroll
            for (int a = 0; a < VPT; ++a) {
                const int v = gt + a * GT;
                if (v < V) {
#pragma unroll
                    for (int j = 0; j < SB; ++j) gmax[j] = fmax(gmax[j], fabs(r[v * SB + j]));
                }
            }
            group_max<GT, SB>(gmax, red, flip, bar_id);
            double sdown[SB];
#pragma unroll
            for (int j = 0; j < SB; ++j) {
                int e = 0;
                if (gmax[j] > 0.0) frexp(gmax[j], &e);
                e = e < -1000 ? -1000 : (e > 1000 ? 1000 : e);
                sdown[j] = ldexp(1.0, -e);
                sup[j] = ldexp(1.0, e);
                gg[j] = 0.0;
            }
#pragma unroll
            for (int a = 0; a < VPT; ++a) {
                const int v = gt + a * GT;
                if (v < V) {
#pragma unroll
                    for (int j = 0; j < SB; ++j) {
                        const double gv = r[v * SB + j] * sdown[j];
                        r[v * SB + j] = gv;
                        gg[j] += gv * gv;
                    }
                }
            }
            group_sum<GT, SB>(gg, red, flip, bar_id);
        }
        double rz[SB], tol2[SB], rrj[SB];
        bool done[SB];
        int its[SB];
        {
            double z[VPT][SB];
            precond(z);
#pragma unroll
            for (int j = 0; j < SB; ++j) rz[j] = 0.0;
#pragma unroll
            for (int a = 0; a < VPT; ++a) {
                const int v = gt + a * GT;
                if (v < V) {
#pragma unroll
                    for (int j = 0; j < SB; ++j) {
                        p[v * SB + j] = z[a][j];
                        rz[j] += r[v * SB + j] * z[a][j];
                    }
                }
            }
            group_sum<GT, SB>(rz, red, flip, bar_id);  // (barrier: p complete)
        }
        bool all_done = true;
#pragma unroll
        for (int j = 0; j < SB; ++j) {
            tol2[j] = prm.rtol * prm.rtol * gg[j];
            done[j] = !(gg[j] > 0.0);
            its[j] = 0;
            rrj[j] = gg[j];
            all_done = all_done && done[j];
        }
        int it = 0;
        while (!all_done && it < prm.max_iter) {
            ++it;
            // ---- q = S p (Dirichlet step) and p.q
            apply(DS, OS, p, q);
            double pq[SB];
#pragma unroll
            for (int j = 0; j < SB; ++j) pq[j] = 0.0;
#pragma unroll
            for (int a = 0; a < VPT; ++a) {
                const int v = gt + a * GT;
                if (v < V) {
#pragma unroll
                    for (int j = 0; j < SB; ++j) pq[j] += p[v * SB + j] * q[a][j];
                }
            }
            group_sum<GT, SB>(pq, red, flip, bar_id);
            double alpha[SB];
#pragma unroll
            for (int j = 0; j < SB; ++j) {
                if (!(pq[j] > 0.0)) done[j] = true;  // p = 0 (underflowed rhs): nothing left to reduce
                alpha[j] = done[j] ? 0.0 : rz[j] / pq[j];
            }
#pragma unroll
            for (int a = 0; a < VPT; ++a) {
                const int v = gt + a * GT;
                if (v < V) {
#pragma unroll
                    for (int j = 0; j < SB; ++j) {
                        x[a][j] += alpha[j] * p[v * SB + j];
                        r[v * SB + j] -= alpha[j] * q[a][j];
                    }
                }
            }
            group_bar(bar_id, GT);
            double z[VPT][SB];
            precond(z);
            double t2[2 * SB];
#pragma unroll
            for (int j = 0; j < 2 * SB; ++j) t2[j] = 0.0;
#pragma unroll
            for (int a = 0; a < VPT; ++a) {
                const int v = gt + a * GT;
                if (v < V) {
#pragma unroll
                    for (int j = 0; j < SB; ++j) {
                        const double rv = r[v * SB + j];
                        t2[j] += rv * rv;
                        t2[SB + j] += rv * z[a][j];
                    }
                }
            }
            group_sum<GT, 2 * SB>(t2, red, flip, bar_id);
            double bet[SB];
            all_done = true;
#pragma unroll
            for (int j = 0; j < SB; ++j) {
                if (!done[j]) {
                    its[j] = it;
                    rrj[j] = t2[j];
                    if (t2[j] <= tol2[j]) done[j] = true;
                }
                bet[j] = done[j] ? 0.0 : t2[SB + j] / rz[j];
                if (!done[j]) rz[j] = t2[SB + j];
                all_done = all_done && done[j];
            }
            if (all_done) break;
#pragma unroll
            for (int a = 0; a < VPT; ++a) {
                const int v = gt + a * GT;
                if (v < V) {
#pragma unroll
                    for (int j = 0; j < SB; ++j)
                        if (!done[j]) p[v * SB + j] = z[a][j] + bet[j] * p[v * SB + j];
                }
            }
            group_bar(bar_id, GT);
        }
        // ---- write u_G and the per-system stats
#pragma unroll
        for (int a = 0; a < VPT; ++a) {
            const int v = gt + a * GT;
            if (v < V) {
#pragma unroll
                for (int j = 0; j < SB; ++j)
                    if (j < ns) uG[ug_index(s0 + j, v, l, L, V, csl)] = x[a][j] * sup[j];
            }
        }
        if (gt == 0) {
#pragma unroll
            for (int j = 0; j < SB; ++j) {
                if (j < ns) {
                    iters[(s0 + j) * L + l] = its[j];
                    relres[(s0 + j) * L + l] = gg[j] > 0.0 ? sqrt(rrj[j] / gg[j]) : 0.0;
                }
            }
        }
        group_bar(bar_id, GT);  // r/p are rewritten by the next batch's gather
    }
}

size_t vec_bytes(const DevGraph& g, int SB, int NG) { return sizeof(double) * 2 * (size_t)g.V * SB * NG; }
size_t staged_bytes(const DevGraph& g) {
    return sizeof(double) * (size_t)table_stride(g.V, g.ell_w) + sizeof(int) * 2 * (size_t)g.ell_w * g.V;
}

template <int GT, int SB, int VPT, int W>
bool launch_t(const DevGraph& g, const DevPlan& p, int64_t n_samples, const PcgParams& prm, const double* rhs,
              double* uG, int32_t* iters, double* relres, cudaStream_t st) {
    constexpr int NG = PCG_THREADS / GT;
    if (g.ell_w != W || g.V > GT * VPT) return false;
    const size_t vb = vec_bytes(g, SB, NG);
    if (vb > SMEM_LIMIT) return false;
    const bool staged = vb + staged_bytes(g) <= SMEM_LIMIT;
    const size_t smem = staged ? vb + staged_bytes(g) : vb;
    // chunks of samples per CTA: the CTAs run in waves over (resident CTAs per SM) x 148 slots and
    // a wave lasts about one CTA's batches, so pick the CTA count per node minimising
    // waves x (batches per group); ties go to fewer CTAs
    const int64_t batches = (n_samples + SB - 1) / SB;
    const int64_t maxg = (batches + NG - 1) / NG;
    auto* kern = staged ? pcg_kernel<GT, SB, VPT, W, true> : pcg_kernel<GT, SB, VPT, W, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PCG_THREADS, smem);
    const int64_t slots = (int64_t)(g.n_sm > 0 ? g.n_sm : 148) * (per_sm > 0 ? per_sm : 1);
    int64_t groups = 1, best = -1;
    for (int64_t gc = 1; gc <= maxg; gc *= 2) {
        const int64_t per_group = (batches + gc * NG - 1) / (gc * NG);
        const int64_t cost = ((p.L * gc + slots - 1) / slots) * per_group;
        if (best < 0 || cost < best) {
            best = cost;
            groups = gc;
        }
    }
    const int32_t spc = (int32_t)(((batches + groups - 1) / groups) * SB);
    groups = (n_samples + spc - 1) / spc;
    const dim3 grid(p.L, (unsigned)groups);
    const int32_t csl = sample_tile_log2(n_samples);
    if (staged) {
        cudaFuncSetAttribute(pcg_kernel<GT, SB, VPT, W, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        pcg_kernel<GT, SB, VPT, W, true><<<grid, PCG_THREADS, smem, st>>>(g, p.L, p.ops, prm, n_samples, spc, csl, rhs,
                                                                        uG, iters, relres);
    } else {
        cudaFuncSetAttribute(pcg_kernel<GT, SB, VPT, W, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        pcg_kernel<GT, SB, VPT, W, false><<<grid, PCG_THREADS, smem, st>>>(g, p.L, p.ops, prm, n_samples, spc, csl, rhs,
                                                                         uG, iters, relres);
    }
    return true;
}


template <int W>
bool launch_w(const DevGraph& g, const DevPlan& p, int64_t n_samples, const PcgParams& prm, const double* rhs,
              double* uG, int32_t* iters, double* relres, cudaStream_t st) {
    if (launch_t<128, 1, 8, W>(g, p, n_samples, prm, rhs, uG, iters, relres, st)) return true;   // V <= 1024
    if (launch_t<256, 1, 8, W>(g, p, n_samples, prm, rhs, uG, iters, relres, st)) return true;   // V <= 2048
    return launch_t<512, 1, 8, W>(g, p, n_samples, prm, rhs, uG, iters, relres, st);            // V <= 4096
}

// K4a: condensed right-hand side g_v = W_v + sum_j (c_L/h_e) w_{code_j(v)} (P233-239)
// for every (node, sample), from the sample-tiled end values into rhs [tile][l][cs][v].
// CTA per (tile, l, block of 32 vertices): phase 1 reads the incident end-value rows with the
// sample index fastest (coalesced), phase 2 transposes through shared memory and writes
// vertex-contiguous rows of rhs (coalesced), adding W_v read vertex-contiguous as well.
constexpr int ASM_VB = 32;

__global__ void __launch_bounds__(256) assemble_rhs_kernel(DevGraph g, int32_t L, const double* __restrict__ ops,
                                                           int64_t S, int32_t csl, const double* __restrict__ Wn,
                                                           const double* __restrict__ ends, double* __restrict__ rhs) {
    __shared__ double acc[ASM_VB][33];
    __shared__ double gks[32][ASM_VB];  // c_L/h_e of incidence slot j of the block's vertices (0: padding)
    __shared__ int codes[32][ASM_VB];   // incidence code 2e+end of slot j (0 for padding: a valid row)
    const int V = g.V, E = g.E;
    const int cs = 1 << csl;
    const int vblocks = (V + ASM_VB - 1) / ASM_VB;
    const int64_t tiles = (S + cs - 1) >> csl;
    const int64_t stride = ops_stride(g);
    // incidence slots per vertex handled through the staged arrays; hubs (CSR mode, > 32 slots)
    // read their remaining slots from global memory
    const int Wd = g.csr ? 32 : g.ell_w;
    // work unit = (node l, vertex block): the incidence codes and coefficients are staged once
    // and reused for every sample tile
    for (int64_t b = blockIdx.x; b < (int64_t)L * vblocks; b += gridDim.x) {
        const int vb = (int)(b % vblocks);
        const int l = (int)(b / vblocks);
        const double* GK = ops + l * stride + 3 * (int64_t)V + 2 * ops_nslots(g);
        for (int x = threadIdx.x; x < Wd * ASM_VB; x += blockDim.x) {
            const int j = x / ASM_VB, vl = x % ASM_VB;
            const int v = vb * ASM_VB + vl;
            const bool ok = v < V && j < g.inc_ptr[v + 1] - g.inc_ptr[v];
            const int64_t k = ok ? ops_slot(g, v, j) : 0;
            codes[j][vl] = ok ? ops_code(g, k) : 0;
            gks[j][vl] = ok ? GK[k] : 0.0;
        }
        __syncthreads();
      for (int64_t tile = 0; tile < tiles; ++tile) {
        const int64_t tl = tile * L + l;
        const double* slab = ends + ((tl * 2 * E) << csl);
        for (int x = threadIdx.x; x < ASM_VB * cs; x += blockDim.x) {
            const int vl = x >> csl, si = x & (cs - 1);
            double a = 0.0;
            for (int j = 0; j < Wd; ++j) a = fma(gks[j][vl], slab[((int64_t)codes[j][vl] << csl) + si], a);
            const int v = vb * ASM_VB + vl;
            if (g.csr && v < V) {
                const int dg = g.inc_ptr[v + 1] - g.inc_ptr[v];
                for (int j = Wd; j < dg; ++j) {
                    const int64_t k = ops_slot(g, v, j);
                    a = fma(GK[k], slab[((int64_t)ops_code(g, k) << csl) + si], a);
                }
            }
            acc[vl][si] = a;
        }
        __syncthreads();
        for (int x = threadIdx.x; x < ASM_VB * cs; x += blockDim.x) {
            const int si = x / ASM_VB, vl = x % ASM_VB;
            const int v = vb * ASM_VB + vl;
            const int64_t s = (tile << csl) + si;
            if (v < V) {
                // W_v enters once: only the owning part adds it (edge-partitioned graphs, dist.cu)
                const bool own = g.vowned == nullptr || g.vowned[v];
                const double wv = own ? Wn[(s < S ? s : S - 1) * g.N + g.NI + v] : 0.0;
                rhs[((tl << csl) + si) * (int64_t)V + v] = wv + acc[vl][si];
            }
        }
        __syncthreads();
      }
    }
}

}  // namespace

int32_t pcg_max_vertices() { return 8 * PCG_THREADS; }

size_t pcg_smem_bytes(const DevGraph& g) { return vec_bytes(g, 1, 1); }

size_t pcg_table_doubles(const DevGraph& g) { return (size_t)ops_stride(g); }

bool pcg_shared_ok(const DevGraph& g) {
    return !g.csr && g.V <= pcg_max_vertices() && g.ell_w <= 32 && vec_bytes(g, 1, 1) <= SMEM_LIMIT;
}

bool pcg_supported(const DevGraph& g) {
    return true;  // larger vertex sets and hubs take the global-memory variant (pcg_global.cu)
}

void launch_pcg_tables(const DevGraph& g, const DevPlan& p, cudaStream_t st) {
    const int64_t n = (int64_t)p.L * g.V;
    int blocks = (int)((n + 255) / 256);
    if (blocks > g.n_sm * 8) blocks = g.n_sm * 8;
    pcg_tables_kernel<<<blocks, 256, 0, st>>>(g, p.L, p.cI, p.cL, p.kappa * p.kappa, p.mass, reinterpret_cast<const double4*>(p.sig), p.ops);
}

void launch_assemble_rhs(const DevGraph& g, const DevPlan& p, int64_t n_samples, const double* W, const double* ends,
                         double* rhs, cudaStream_t st) {
    const int32_t csl = sample_tile_log2(n_samples);
    const int64_t work = (int64_t)p.L * ((g.V + ASM_VB - 1) / ASM_VB);
    // one CTA per work unit (the hardware scheduler balances the tail): config 3 K4a 0.415 ->
    // 0.395 ms (ncu) against a grid-stride cap of 8 CTAs per SM (4: 0.60 ms, 16: 0.41 ms)
    const int blocks = (int)(work < INT32_MAX ? work : INT32_MAX);
    assemble_rhs_kernel<<<blocks, 256, 0, st>>>(g, p.L, p.ops, n_samples, csl, W, ends, rhs);
}

constexpr int64_t PCG_FUSE_MAX_S = 8;

cudaError_t launch_pcg(const DevGraph& g, const DevPlan& p, int64_t n_samples, const PcgParams& prm, const double* W,
                       const double* ends, double* rhs, double* uG, int32_t* iters, double* relres, void* gws,
                       cudaStream_t st, bool need_rhs, int64_t* launches) {
    const int64_t cs = (int64_t)1 << sample_tile_log2(n_samples);
    // up to one sample octet the warp-per-system kernel (V <= 1024, W <= 8) assembles its rhs itself
    // (K4a fused, from the end values; rhs written only for the exit checks): one launch and one
    // DRAM round trip less for the latency-bound single-sample calls (config 2 K4a + K4 0.065 ->
    // 0.054 ms).  For more samples the fill stalls the CTA (one per SM, shared-memory bound) on
    // DRAM once per octet, which the separate, coalesced K4a does not: config 3 K4a + K4 1.97 ms
    // against 2.48 / 2.78 ms fused (sample-fastest / vertex-per-thread fills).
    if (!prm.global && n_samples <= PCG_FUSE_MAX_S &&
        launch_pcg_warp(g, p, n_samples, prm, W, ends, need_rhs ? rhs : nullptr, uG, iters, relres, st)) {
        if (launches) *launches += 1;
        return cudaGetLastError();
    }
    // K4a + K4 (the global-memory variant launches once per sample tile)
    if (launches) *launches += 1 + (prm.global ? (n_samples + cs - 1) / cs : 1);
    launch_assemble_rhs(g, p, n_samples, W, ends, rhs, st);
    if (prm.global) return launch_pcg_global(g, p, n_samples, prm, rhs, uG, iters, relres, gws, st);
    if (launch_pcg_warp(g, p, n_samples, prm, W, nullptr, rhs, uG, iters, relres, st)) return cudaGetLastError();
    switch (g.ell_w) {
        case 4: launch_w<4>(g, p, n_samples, prm, rhs, uG, iters, relres, st); break;
        case 8: launch_w<8>(g, p, n_samples, prm, rhs, uG, iters, relres, st); break;
        case 16: launch_w<16>(g, p, n_samples, prm, rhs, uG, iters, relres, st); break;
        default: launch_w<32>(g, p, n_samples, prm, rhs, uG, iters, relres, st); break;
    }
    return cudaGetLastError();
}

namespace {
// True residual of every vertex system at exit (SURVEY §8c Q10, P296 "J ~ 0"): per (node l,
// sample s) ||g - S u_G||_2^2 and ||g||_2^2 with the plan's operator tables (the Dirichlet step
// of P247-258 applied to the PCG's answer).  One block per (l, sample), threads over vertices,
// fixed-order reduction.
__global__ void true_residual_kernel(DevGraph g, int32_t L, const double* __restrict__ ops, int64_t S, int32_t csl,
                                     const double* __restrict__ rhs, const double* __restrict__ uG,
                                     double* __restrict__ out /* [S][L] relative residual */) {
    __shared__ double red[2][8];
    const int l = blockIdx.x % L;
    const int64_t s = blockIdx.x / L;
    const int V = g.V;
    const int64_t ns = ops_nslots(g);
    const double* tab = ops + l * ops_stride(g);
    double rr = 0.0, gg = 0.0;
    for (int v = threadIdx.x; v < V; v += blockDim.x) {
        const double x = uG[ug_index(s, v, l, L, V, csl)];
        double sx = tab[v] * x;
        const int dg = g.inc_ptr[v + 1] - g.inc_ptr[v];
        for (int j = 0; j < dg; ++j) {
            const int64_t k = ops_slot(g, v, j);
            sx = fma(tab[3 * (int64_t)V + k], uG[ug_index(s, ops_other(g, k), l, L, V, csl)], sx);
        }
        const double gv = rhs[rhs_index(s, l, v, L, V, csl)];
        rr = fma(gv - sx, gv - sx, rr);
        gg = fma(gv, gv, gg);
    }
    (void)ns;
    for (int o = 16; o > 0; o >>= 1) {
        rr += __shfl_xor_sync(0xffffffffu, rr, o);
        gg += __shfl_xor_sync(0xffffffffu, gg, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = rr;
        red[1][threadIdx.x >> 5] = gg;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            a += red[0][w];
            b += red[1][w];
        }
        out[s * L + l] = b > 0.0 ? sqrt(a / b) : 0.0;
    }
}

// count of non-finite entries of u (S x N), one partial per block, summed by the host
__global__ void nonfinite_kernel(const double* __restrict__ u, int64_t n, unsigned long long* __restrict__ count) {
    unsigned int c = 0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        c += isfinite(u[t]) ? 0u : 1u;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, (unsigned long long)c);
}
}  // namespace

void launch_true_residual(const DevGraph& g, const DevPlan& p, int64_t n_samples, const double* rhs, const double* uG,
                          double* out, cudaStream_t st) {
    true_residual_kernel<<<(unsigned)(p.L * n_samples), 256, 0, st>>>(g, p.L, p.ops, n_samples,
                                                                       sample_tile_log2(n_samples), rhs, uG, out);
}

void launch_nonfinite(const double* u, int64_t n, unsigned long long* count, cudaStream_t st) {
    cudaMemsetAsync(count, 0, sizeof(unsigned long long), st);
    int64_t blocks = (n + 255) / 256;
    if (blocks > (int64_t)device_sms() * 16) blocks = (int64_t)device_sms() * 16;
    if (blocks < 1) blocks = 1;
    nonfinite_kernel<<<(unsigned)blocks, 256, 0, st>>>(u, n, count);
}

}  // namespace grf
