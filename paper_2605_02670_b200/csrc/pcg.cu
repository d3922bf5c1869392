// K4: batched matrix-free PCG on the vertex Schur systems  (PAPER.md P111-118, P241-298).
//
//     S^{(l)} u_G = g,   S^{(l)} = sum_e R_e^T S^{(l,e)} R_e        (P113-116, P244 [eq:goal_func_1])
//
// Dirichlet step (P247-258): y = S p evaluated edge-locally; with the exact 2x2 local
// Schur blocks of K2 this is q_v = sum_{(e,end) at v} (s_d p_v + s_o p_other).
// Neumann step (P260-298): z = D^{-1} (sum_e R_e^T S_e^{-1} R_e) D^{-1} r, i.e.
//     r~ = r / d (eq:distribute_dv), delta = S_e^{-1} r~ per edge, z_v = (1/d_v) sum delta
// (eq:induced_displacements); D_vv = d_v = incident edge ends.
// A loop edge has other == v, so both its ends add to v (sum of all 4 entries, Q18).
// Stopping rule: ||r_k||_2 <= rtol ||g||_2, x_0 = 0.
//
// Mapping: one CTA per (node l, sample s) system; the vertex vectors x, r, z, p, q live in
// shared memory (V <= pcg_max_vertices); dot products are warp-shuffle + smem block
// reductions; every system iterates to its own convergence inside the kernel (no host
// round trip).  g is gathered from K3's end values ends[((s*E + e)*2 + end)*L + l] and
// u_G written to uG[(s*V + v)*L + l]; CTAs with consecutive l (the fastest grid index)
// share the L2 sectors of these node-minor layouts.
#include "grf_internal.h"

#include <cub/block/block_reduce.cuh>

namespace grf {
namespace {

constexpr int PCG_THREADS = 256;

struct Sum2 {
    __device__ __forceinline__ double2 operator()(const double2& a, const double2& b) const {
        return make_double2(a.x + b.x, a.y + b.y);
    }
};

__global__ void __launch_bounds__(PCG_THREADS) pcg_kernel(DevGraph g, int32_t L, const double* __restrict__ cLt,
                                                          const double4* __restrict__ sig, PcgParams prm,
                                                          const double* __restrict__ W, const double* __restrict__ ends,
                                                          double* __restrict__ uG, int32_t* __restrict__ iters,
                                                          double* __restrict__ relres) {
    using BR1 = cub::BlockReduce<double, PCG_THREADS>;
    using BR2 = cub::BlockReduce<double2, PCG_THREADS>;
    __shared__ union {
        typename BR1::TempStorage r1;
        typename BR2::TempStorage r2;
    } tmp;
    __shared__ double bcast[2];
    extern __shared__ double sm[];
    const int V = g.V;
    double* x = sm;
    double* r = x + V;
    double* z = r + V;
    double* p = z + V;
    double* q = p + V;

    const int l = blockIdx.x;
    const int64_t s = blockIdx.y;
    const double4* sg = sig + (int64_t)l * g.E;
    double* ucol = uG + (s * V) * (int64_t)L + l;
    const double* ecol = ends + (s * g.E) * 2 * (int64_t)L + l;
    const double cL = cLt[l];

    auto reduce1 = [&](double v) -> double {
        double t = BR1(tmp.r1).Sum(v);
        if (threadIdx.x == 0) bcast[0] = t;
        __syncthreads();
        t = bcast[0];
        __syncthreads();
        return t;
    };
    auto reduce2 = [&](double a, double b) -> double2 {
        double2 t = BR2(tmp.r2).Reduce(make_double2(a, b), Sum2());
        if (threadIdx.x == 0) {
            bcast[0] = t.x;
            bcast[1] = t.y;
        }
        __syncthreads();
        t = make_double2(bcast[0], bcast[1]);
        __syncthreads();
        return t;
    };
    auto precond = [&]() {  // z = M^{-1} r
        for (int v = threadIdx.x; v < V; v += blockDim.x) {
            const int k0 = g.inc_ptr[v], k1 = g.inc_ptr[v + 1];
            double zv;
            if (prm.precond == 0) {          // Neumann-Neumann (P298)
                const double idv = g.inv_deg[v];
                const double rv = r[v] * idv;
                double acc = 0.0;
                for (int k = k0; k < k1; ++k) {
                    const double4 c = sg[g.inc[k] >> 1];
                    const int o = g.inc_other[k];
                    acc += c.z * rv + c.w * (r[o] * g.inv_deg[o]);
                }
                zv = idv * acc;
            } else if (prm.precond == 1) {   // Jacobi on diag(S)
                double dg = 0.0;
                for (int k = k0; k < k1; ++k) {
                    const double4 c = sg[g.inc[k] >> 1];
                    dg += c.x + (g.inc_other[k] == v ? c.y : 0.0);
                }
                zv = r[v] / dg;
            } else {
                zv = r[v];
            }
            z[v] = zv;
        }
    };

    // condensed rhs g_v = W_v + sum_{(e,end) at v} (c_L/h_e) w_end   (P233-239)
    double part = 0.0;
    for (int v = threadIdx.x; v < V; v += blockDim.x) {
        double gv = W[s * g.N + g.NI + v];
        for (int k = g.inc_ptr[v]; k < g.inc_ptr[v + 1]; ++k) {
            const int code = g.inc[k];
            gv += (cL / g.h[code >> 1]) * ecol[(int64_t)code * L];
        }
        r[v] = gv;
        x[v] = 0.0;
        part += gv * gv;
    }
    const double gg = reduce1(part);  // (syncs: r complete)
    int it = 0;
    double rr = gg;
    if (gg > 0.0) {
        precond();
        __syncthreads();
        part = 0.0;
        for (int v = threadIdx.x; v < V; v += blockDim.x) {
            p[v] = z[v];
            part += r[v] * z[v];
        }
        double rz = reduce1(part);
        const double tol2 = prm.rtol * prm.rtol * gg;
        while (it < prm.max_iter) {
            ++it;
            // q = S p  (Dirichlet step, matrix free)
            part = 0.0;
            for (int v = threadIdx.x; v < V; v += blockDim.x) {
                const int k0 = g.inc_ptr[v], k1 = g.inc_ptr[v + 1];
                const double pv = p[v];
                double acc = 0.0;
                for (int k = k0; k < k1; ++k) {
                    const double4 c = sg[g.inc[k] >> 1];
                    acc += c.x * pv + c.y * p[g.inc_other[k]];
                }
                q[v] = acc;
                part += pv * acc;
            }
            const double pq = reduce1(part);
            const double alpha = rz / pq;
            for (int v = threadIdx.x; v < V; v += blockDim.x) {
                x[v] += alpha * p[v];
                r[v] -= alpha * q[v];
            }
            __syncthreads();
            precond();
            double pr = 0.0, pz = 0.0;
            for (int v = threadIdx.x; v < V; v += blockDim.x) {
                pr += r[v] * r[v];
                pz += r[v] * z[v];
            }
            const double2 t = reduce2(pr, pz);
            rr = t.x;
            if (rr <= tol2) break;
            const double bet = t.y / rz;
            rz = t.y;
            for (int v = threadIdx.x; v < V; v += blockDim.x) p[v] = z[v] + bet * p[v];
            __syncthreads();
        }
    }
    for (int v = threadIdx.x; v < V; v += blockDim.x) ucol[(int64_t)v * L] = x[v];
    if (threadIdx.x == 0) {
        iters[s * L + l] = it;
        relres[s * L + l] = gg > 0.0 ? sqrt(rr / gg) : 0.0;
    }
}

}  // namespace

int32_t pcg_max_vertices() { return 5000; }

size_t pcg_smem_bytes(const DevGraph& g) { return sizeof(double) * 5 * (size_t)g.V; }

void launch_pcg(const DevGraph& g, const DevPlan& p, int64_t n_samples, const PcgParams& prm, const double* W,
                const double* ends, double* uG, int32_t* iters, double* relres, cudaStream_t st) {
    const size_t smem = pcg_smem_bytes(g);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(pcg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set = true;
    }
    dim3 grid(p.L, (unsigned)n_samples);
    pcg_kernel<<<grid, PCG_THREADS, smem, st>>>(g, p.L, p.cL, reinterpret_cast<const double4*>(p.sig), prm, W, ends,
                                                uG, iters, relres);
}

}  // namespace grf
