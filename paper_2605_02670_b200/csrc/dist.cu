// Edge-partitioned NN-PCG ("the largest graph additionally
// edge-partitions, with a vertex-halo exchange and an allreduce for the PCG dot products").
//
// The edges are split into parts; a part holds its edges' interiors and every vertex they
// touch (interface vertices are shared).  The vertex Schur operator is the sum of the
// parts' edge contributions (PAPER.md P242-244: S = sum_e R_e^T S_e R_e), and so is the NN
// preconditioner (P298) with the GLOBAL degrees d_v.  The PCG keeps x, r, p, z, q
// assembled (equal on every part that holds a vertex):
//   - an operator application gives a part's partial sums at its vertices; the halo step
//     sums the partial values of the interface vertices over all parts (pack into a
//     [n_interface][L][cs] buffer, sum over parts -- in this process or by an NCCL
//     allreduce across ranks -- unpack);
//   - a dot product sums over the vertices a part OWNS (each vertex has one owner), then
//     over parts.
// Vectors are [L][V_part][cs] (node, vertex, sample tile), as in pcg_global.cu.  Dot
// products use per-(node, vertex block) partials reduced in fixed order, and the cross-part
// sums run in fixed part order, so the in-process mode is deterministic.
#include "grf_internal.h"

namespace grf {
namespace dist {
namespace {

constexpr int BT = 256;


// r = rhs (partial sums at interface vertices), x = 0, p = 0
template <int CS>
__global__ void init_kernel(DevGraph g, int32_t L, int64_t S, int32_t csl, int64_t tile, const double* __restrict__ rhs,
                            double* __restrict__ x, double* __restrict__ r, double* __restrict__ p) {
    const int V = g.V;
    const int64_t n = (int64_t)L * V;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int l = (int)(t / V), v = (int)(t % V);
#pragma unroll
        for (int s = 0; s < CS; ++s) {
            const int64_t sg = (tile << csl) + s;
            r[t * CS + s] = sg < S ? rhs[rhs_index(sg, l, v, L, V, csl)] : 0.0;
            x[t * CS + s] = 0.0;
            p[t * CS + s] = 0.0;
        }
    }
}

// z = M_part r: this part's edge contributions of the NN (or Jacobi / identity) preconditioner
template <int CS>
__global__ void precond_kernel(DevGraph g, int32_t L, const double* __restrict__ ops, int32_t precond,
                               const double* __restrict__ r, double* __restrict__ z) {
    const int V = g.V;
    const int64_t ns = ops_nslots(g);
    const int64_t n = (int64_t)L * V;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int l = (int)(t / V), v = (int)(t % V);
        const double* tab = ops + l * ops_stride(g);
        double zv[CS];
        if (precond == 0) {
            const double dm = tab[V + v];
#pragma unroll
            for (int s = 0; s < CS; ++s) zv[s] = dm * r[t * CS + s];
            const int dg = g.inc_ptr[v + 1] - g.inc_ptr[v];
            for (int j = 0; j < dg; ++j) {
                const int64_t k = ops_slot(g, v, j);
                const double c = tab[3 * (int64_t)V + ns + k];
                const double* ro = r + ((int64_t)l * V + ops_other(g, k)) * CS;
#pragma unroll
                for (int s = 0; s < CS; ++s) zv[s] = fma(c, ro[s], zv[s]);
            }
        } else {
            const double d = precond == 1 ? tab[2 * V + v] : 1.0;
#pragma unroll
            for (int s = 0; s < CS; ++s) zv[s] = d * r[t * CS + s];
        }
#pragma unroll
        for (int s = 0; s < CS; ++s) z[t * CS + s] = zv[s];
    }
}

// p' = z + beta p (own vertex), q = S_part p' (neighbour p' formed on the fly)
template <int CS>
__global__ void spmv_kernel(DevGraph g, int32_t L, const double* __restrict__ ops, const double* __restrict__ beta,
                            const double* __restrict__ z, const double* __restrict__ po, double* __restrict__ pn,
                            double* __restrict__ q) {
    const int V = g.V;
    const int64_t ns = ops_nslots(g);
    const int64_t n = (int64_t)L * V;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int l = (int)(t / V), v = (int)(t % V);
        const double* tab = ops + l * ops_stride(g);
        double bt[CS], pv[CS], qv[CS];
        const double ds = tab[v];
#pragma unroll
        for (int s = 0; s < CS; ++s) {
            bt[s] = beta[l * CS + s];
            pv[s] = fma(bt[s], po[t * CS + s], z[t * CS + s]);
            qv[s] = ds * pv[s];
        }
        const int dg = g.inc_ptr[v + 1] - g.inc_ptr[v];
        for (int j = 0; j < dg; ++j) {
            const int64_t k = ops_slot(g, v, j);
            const double c = tab[3 * (int64_t)V + k];
            const int64_t ob = ((int64_t)l * V + ops_other(g, k)) * CS;
#pragma unroll
            for (int s = 0; s < CS; ++s) qv[s] = fma(c, fma(bt[s], po[ob + s], z[ob + s]), qv[s]);
        }
#pragma unroll
        for (int s = 0; s < CS; ++s) {
            pn[t * CS + s] = pv[s];
            q[t * CS + s] = qv[s];
        }
    }
}

// x += alpha p', r' = r - alpha q, z = M_part r' (neighbour r' formed on the fly)
template <int CS>
__global__ void update_kernel(DevGraph g, int32_t L, const double* __restrict__ ops, int32_t precond,
                              const double* __restrict__ alpha, const double* __restrict__ q,
                              const double* __restrict__ pn, const double* __restrict__ ro, double* __restrict__ rn,
                              double* __restrict__ x, double* __restrict__ z) {
    const int V = g.V;
    const int64_t ns = ops_nslots(g);
    const int64_t n = (int64_t)L * V;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int l = (int)(t / V), v = (int)(t % V);
        const double* tab = ops + l * ops_stride(g);
        double al[CS], rv[CS], zv[CS];
#pragma unroll
        for (int s = 0; s < CS; ++s) {
            al[s] = alpha[l * CS + s];
            rv[s] = fma(-al[s], q[t * CS + s], ro[t * CS + s]);
            x[t * CS + s] = fma(al[s], pn[t * CS + s], x[t * CS + s]);
        }
        if (precond == 0) {
            const double dm = tab[V + v];
#pragma unroll
            for (int s = 0; s < CS; ++s) zv[s] = dm * rv[s];
            const int dg = g.inc_ptr[v + 1] - g.inc_ptr[v];
            for (int j = 0; j < dg; ++j) {
                const int64_t k = ops_slot(g, v, j);
                const double c = tab[3 * (int64_t)V + ns + k];
                const int64_t ob = ((int64_t)l * V + ops_other(g, k)) * CS;
#pragma unroll
                for (int s = 0; s < CS; ++s) zv[s] = fma(c, fma(-al[s], q[ob + s], ro[ob + s]), zv[s]);
            }
        } else {
            const double d = precond == 1 ? tab[2 * V + v] : 1.0;
#pragma unroll
            for (int s = 0; s < CS; ++s) zv[s] = d * rv[s];
        }
#pragma unroll
        for (int s = 0; s < CS; ++s) {
            rn[t * CS + s] = rv[s];
            z[t * CS + s] = zv[s];
        }
    }
}

// block partials of sum_{owned v} a_v b_v (K pairs) per (node, sample): part[k][l][vb][s]
template <int CS, int K>
__global__ void __launch_bounds__(BT) dot_kernel(DevGraph g, int32_t L, const double* __restrict__ a0,
                                                 const double* __restrict__ b0, const double* __restrict__ a1,
                                                 const double* __restrict__ b1, double* __restrict__ part) {
    __shared__ double red[BT / 32][K * CS];
    const int V = g.V;
    const int nvb = (V + BT - 1) / BT;
    const int l = blockIdx.x / nvb, vb = blockIdx.x % nvb;
    const int v = vb * BT + threadIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool own = v < V && (g.vowned == nullptr || g.vowned[v]);
    const int64_t t = ((int64_t)l * V + v) * CS;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const double* a = k ? a1 : a0;
        const double* b = k ? b1 : b0;
#pragma unroll
        for (int s = 0; s < CS; ++s) {
            double w = own ? a[t + s] * b[t + s] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
            if (lane == 0) red[warp][k * CS + s] = w;
        }
    }
    __syncthreads();
    if (threadIdx.x < K * CS) {
        double w = 0.0;
        for (int q = 0; q < BT / 32; ++q) w += red[q][threadIdx.x];
        const int k = threadIdx.x / CS, s = threadIdx.x % CS;
        part[(((int64_t)k * L + l) * nvb + vb) * CS + s] = w;
    }
}

// out[k][l][s] = sum over vertex blocks (fixed order)
__global__ void dot_reduce_kernel(int32_t K, int32_t L, int32_t nvb, int32_t cs, const double* __restrict__ part,
                                  double* __restrict__ out) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)K * L * cs) return;
    const int s = (int)(t % cs);
    const int64_t kl = t / cs;
    double w = 0.0;
    for (int b = 0; b < nvb; ++b) w += part[(kl * nvb + b) * cs + s];
    out[t] = w;
}

// halo: buf[iface(v)][l][s] = X[l][v][s] for the part's interface vertices (buf pre-zeroed)
template <int CS>
__global__ void pack_kernel(DevGraph g, int32_t L, const double* __restrict__ X, double* __restrict__ buf) {
    const int V = g.V;
    const int64_t n = (int64_t)L * V;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int l = (int)(t / V), v = (int)(t % V);
        const int64_t f = g.viface[v];
        if (f < 0) continue;
#pragma unroll
        for (int s = 0; s < CS; ++s) buf[(f * L + l) * CS + s] = X[t * CS + s];
    }
}

template <int CS>
__global__ void unpack_kernel(DevGraph g, int32_t L, const double* __restrict__ buf, double* __restrict__ X) {
    const int V = g.V;
    const int64_t n = (int64_t)L * V;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int l = (int)(t / V), v = (int)(t % V);
        const int64_t f = g.viface[v];
        if (f < 0) continue;
#pragma unroll
        for (int s = 0; s < CS; ++s) X[t * CS + s] = buf[(f * L + l) * CS + s];
    }
}

// neighbour halo (p2p): send[j][l][s] = X[l][idx[j]][s] for the shared vertices of every neighbour
template <int CS>
__global__ void halo_pack_kernel(int32_t V, int32_t L, int64_t n, const int32_t* __restrict__ idx,
                                 const double* __restrict__ X, double* __restrict__ send) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * L; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / L;
        const int l = (int)(t % L);
        const double* src = X + ((int64_t)l * V + idx[j]) * CS;
#pragma unroll
        for (int s = 0; s < CS; ++s) send[t * CS + s] = src[s];
    }
}

// X[l][v][s] = sum over the parts touching interface vertex v, in ascending part order, of their
// values: own (src = -1) or received (src = slot of recv); every part evaluates the same sum
template <int CS>
__global__ void halo_combine_kernel(int32_t V, int32_t L, int32_t nif, const int32_t* __restrict__ vert,
                                    const int32_t* __restrict__ ptr, const int32_t* __restrict__ src,
                                    const double* __restrict__ recv, double* __restrict__ X) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)nif * L;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(t / L), l = (int)(t % L);
        double* x = X + ((int64_t)l * V + vert[i]) * CS;
        double acc[CS];
        bool first = true;
        for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
            const double* y = src[k] < 0 ? x : recv + ((int64_t)src[k] * L + l) * CS;
#pragma unroll
            for (int s = 0; s < CS; ++s) acc[s] = first ? y[s] : acc[s] + y[s];
            first = false;
        }
#pragma unroll
        for (int s = 0; s < CS; ++s) x[s] = acc[s];
    }
}

// out = sum_p in[p] (fixed part order)
__global__ void sum_parts_kernel(int32_t P, double* const* __restrict__ in, int64_t n, double* __restrict__ out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        double w = 0.0;
        for (int p = 0; p < P; ++p) w += in[p][t];
        out[t] = w;
    }
}

// scalar state of the L x cs systems (shared by every part)
__global__ void scal_init_kernel(int32_t n, int32_t cs, int64_t S, int64_t tile, int32_t csl,
                                 const double* __restrict__ dots /* [2][n]: r.r, r.z */, double* gg, double* rr,
                                 double* rz, double* beta, int32_t* done, int32_t* its, int32_t* active) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int64_t sg = (tile << csl) + t % cs;
    gg[t] = rr[t] = dots[t];
    rz[t] = dots[n + t];
    beta[t] = 0.0;
    its[t] = 0;
    done[t] = !(dots[t] > 0.0) || sg >= S;
    if (!done[t]) atomicAdd(active, 1);
}

__global__ void scal_alpha_kernel(int32_t n, const double* __restrict__ pq, const double* __restrict__ rz,
                                  int32_t* __restrict__ done, double* __restrict__ alpha, int32_t* active) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    if (!done[t] && !(pq[t] > 0.0)) {  // p = 0 (underflowed rhs): nothing left to reduce
        done[t] = 1;
        atomicSub(active, 1);
    }
    alpha[t] = done[t] ? 0.0 : rz[t] / pq[t];
}

__global__ void scal_beta_kernel(int32_t n, double tol2, const double* __restrict__ dots /* [2][n] */,
                                 const double* __restrict__ gg, double* rr, double* rz, double* beta, int32_t* done,
                                 int32_t* its, int32_t* active) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    if (done[t]) {
        beta[t] = 0.0;
        return;
    }
    its[t] += 1;
    rr[t] = dots[t];
    if (dots[t] <= tol2 * gg[t]) {
        done[t] = 1;
        beta[t] = 0.0;
        atomicSub(active, 1);
    } else {
        beta[t] = dots[n + t] / rz[t];
    }
    rz[t] = dots[n + t];
}

// u_G of the tile and the per-system statistics
template <int CS>
__global__ void finish_kernel(DevGraph g, int32_t L, int64_t S, int32_t csl, int64_t tile, const double* __restrict__ x,
                              const double* __restrict__ gg, const double* __restrict__ rr,
                              const int32_t* __restrict__ its, double* __restrict__ uG, int32_t* __restrict__ iters,
                              double* __restrict__ relres) {
    const int V = g.V;
    const int64_t n = (int64_t)L * V;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int l = (int)(t / V), v = (int)(t % V);
#pragma unroll
        for (int s = 0; s < CS; ++s) {
            const int64_t sg = (tile << csl) + s;
            if (sg >= S) continue;
            uG[ug_index(sg, v, l, L, V, csl)] = x[t * CS + s];
            if (v == 0) {
                const int sy = l * CS + s;
                iters[sg * L + l] = its[sy];
                relres[sg * L + l] = gg[sy] > 0.0 ? sqrt(rr[sy] / gg[sy]) : 0.0;
            }
        }
    }
}

int grid_for(int64_t n) {
    int64_t b = (n + BT - 1) / BT;
    const int64_t cap = (int64_t)device_sms() * 16;
    return (int)(b < cap ? (b < 1 ? 1 : b) : cap);
}

}  // namespace

#define GRF_CS_SWITCH(cs, CALL) \
    switch (cs) {               \
        case 1: {               \
            constexpr int C = 1; \
            CALL;               \
            break;              \
        }                       \
        case 16: {              \
            constexpr int C = 16; \
            CALL;               \
            break;              \
        }                       \
        default: {              \
            constexpr int C = 32; \
            CALL;               \
            break;              \
        }                       \
    }

void init(const DevGraph& g, int32_t L, int64_t S, int32_t csl, int64_t tile, const double* rhs, const Vecs& v,
          cudaStream_t st) {
    const int grid = grid_for((int64_t)L * g.V);
    GRF_CS_SWITCH(1 << csl, (init_kernel<C><<<grid, BT, 0, st>>>(g, L, S, csl, tile, rhs, v.x, v.r0, v.p0)));
}

void precond(const DevGraph& g, const DevPlan& p, int32_t pc, int32_t cs, const double* r, double* z, cudaStream_t st) {
    const int grid = grid_for((int64_t)p.L * g.V);
    GRF_CS_SWITCH(cs, (precond_kernel<C><<<grid, BT, 0, st>>>(g, p.L, p.ops, pc, r, z)));
}

void spmv(const DevGraph& g, const DevPlan& p, int32_t cs, const double* beta, const double* z, const double* po,
          double* pn, double* q, cudaStream_t st) {
    const int grid = grid_for((int64_t)p.L * g.V);
    GRF_CS_SWITCH(cs, (spmv_kernel<C><<<grid, BT, 0, st>>>(g, p.L, p.ops, beta, z, po, pn, q)));
}

void update(const DevGraph& g, const DevPlan& p, int32_t pc, int32_t cs, const double* alpha, const double* q,
            const double* pn, const double* ro, double* rn, double* x, double* z, cudaStream_t st) {
    const int grid = grid_for((int64_t)p.L * g.V);
    GRF_CS_SWITCH(cs, (update_kernel<C><<<grid, BT, 0, st>>>(g, p.L, p.ops, pc, alpha, q, pn, ro, rn, x, z)));
}

void dots(const DevGraph& g, int32_t L, int32_t cs, int K, const double* a0, const double* b0, const double* a1,
          const double* b1, double* part, double* out, cudaStream_t st) {
    const int nvb = (g.V + BT - 1) / BT;
    if (K == 1) {
        GRF_CS_SWITCH(cs, (dot_kernel<C, 1><<<L * nvb, BT, 0, st>>>(g, L, a0, b0, a1, b1, part)));
    } else {
        GRF_CS_SWITCH(cs, (dot_kernel<C, 2><<<L * nvb, BT, 0, st>>>(g, L, a0, b0, a1, b1, part)));
    }
    const int64_t n = (int64_t)K * L * cs;
    dot_reduce_kernel<<<(unsigned)((n + BT - 1) / BT), BT, 0, st>>>(K, L, nvb, cs, part, out);
}

void pack(const DevGraph& g, int32_t L, int32_t cs, const double* X, double* buf, cudaStream_t st) {
    const int grid = grid_for((int64_t)L * g.V);
    GRF_CS_SWITCH(cs, (pack_kernel<C><<<grid, BT, 0, st>>>(g, L, X, buf)));
}

void unpack(const DevGraph& g, int32_t L, int32_t cs, const double* buf, double* X, cudaStream_t st) {
    const int grid = grid_for((int64_t)L * g.V);
    GRF_CS_SWITCH(cs, (unpack_kernel<C><<<grid, BT, 0, st>>>(g, L, buf, X)));
}

void halo_pack(const DevGraph& g, int32_t L, int32_t cs, int64_t n, const int32_t* idx, const double* X, double* send,
               cudaStream_t st) {
    if (n == 0) return;
    const int grid = grid_for(n * L);
    GRF_CS_SWITCH(cs, (halo_pack_kernel<C><<<grid, BT, 0, st>>>(g.V, L, n, idx, X, send)));
}

void halo_combine(const DevGraph& g, int32_t L, int32_t cs, int32_t nif, const int32_t* vert, const int32_t* ptr,
                  const int32_t* src, const double* recv, double* X, cudaStream_t st) {
    if (nif == 0) return;
    const int grid = grid_for((int64_t)nif * L);
    GRF_CS_SWITCH(cs, (halo_combine_kernel<C><<<grid, BT, 0, st>>>(g.V, L, nif, vert, ptr, src, recv, X)));
}

void sum_parts(int32_t P, double* const* in_dev, int64_t n, double* out, cudaStream_t st) {
    sum_parts_kernel<<<grid_for(n), BT, 0, st>>>(P, in_dev, n, out);
}

void scal_init(int32_t n, int32_t cs, int64_t S, int64_t tile, int32_t csl, const double* dots, const Scal& sc,
               cudaStream_t st) {
    scal_init_kernel<<<(n + BT - 1) / BT, BT, 0, st>>>(n, cs, S, tile, csl, dots, sc.gg, sc.rr, sc.rz, sc.beta,
                                                       sc.done, sc.its, sc.active);
}

void scal_alpha(int32_t n, const double* pq, const Scal& sc, cudaStream_t st) {
    scal_alpha_kernel<<<(n + BT - 1) / BT, BT, 0, st>>>(n, pq, sc.rz, sc.done, sc.alpha, sc.active);
}

void scal_beta(int32_t n, double tol2, const double* dots, const Scal& sc, cudaStream_t st) {
    scal_beta_kernel<<<(n + BT - 1) / BT, BT, 0, st>>>(n, tol2, dots, sc.gg, sc.rr, sc.rz, sc.beta, sc.done, sc.its,
                                                       sc.active);
}

void finish(const DevGraph& g, int32_t L, int64_t S, int32_t csl, int64_t tile, const double* x, const Scal& sc,
            double* uG, int32_t* iters, double* relres, cudaStream_t st) {
    const int grid = grid_for((int64_t)L * g.V);
    GRF_CS_SWITCH(1 << csl,
                  (finish_kernel<C><<<grid, BT, 0, st>>>(g, L, S, csl, tile, x, sc.gg, sc.rr, sc.its, uG, iters, relres)));
}

int32_t dot_blocks(const DevGraph& g) { return (g.V + BT - 1) / BT; }

}  // namespace dist
}  // namespace grf
