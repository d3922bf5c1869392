// Nested-mesh transfer for the strong-error study (§4.1, P335; SPEC S119-127,
// S256-264): the fine mesh of a graph refines the coarse one edge by
// edge (fine n_e = r_e x coarse n_e).  P is the hat-function interpolation of coarse nodal
// values at the fine nodes; the noise is projected down by P^T.  Both are gathers (no
// atomics), one thread per (sample, output DOF); the sums run in a fixed order.
#include <algorithm>

#include "grf_internal.h"

namespace grf {
namespace {

// coarse node c (0..n_c) of edge e -> coarse DOF
__device__ __forceinline__ int64_t cnode(const DevGraph& g, int e, int c, int nc) {
    if (c == 0) return g.NI + g.eu[e];
    if (c == nc) return g.NI + g.ev[e];
    return g.off[e] + c - 1;
}
__device__ __forceinline__ int64_t fnode(const DevGraph& g, int e, int j, int nf) {
    if (j == 0) return g.NI + g.eu[e];
    if (j == nf) return g.NI + g.ev[e];
    return g.off[e] + j - 1;
}

// u_f = P u_c.  Fine interior node j of edge e: c = j / r, q = j % r ->
// (1 - q/r) u_c[c] + (q/r) u_c[c+1]; vertices copy.
__global__ void prolong_kernel(DevGraph gc, DevGraph gf, const int32_t* __restrict__ fedge, int64_t S,
                               const double* __restrict__ uc, double* __restrict__ uf) {
    const int64_t Nf = gf.N;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < S * Nf; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = t / Nf, i = t - s * Nf;
        const double* u = uc + s * gc.N;
        double val;
        if (i >= gf.NI) {
            val = u[gc.NI + (i - gf.NI)];
        } else {
            const int e = fedge[i];
            const int nf = gf.m[e] + 1, nc = gc.m[e] + 1, r = nf / nc;
            const int j = (int)(i - gf.off[e]) + 1;
            const int c = j / r, q = j - c * r;
            const double w = (double)q / (double)r;
            val = (1.0 - w) * u[cnode(gc, e, c, nc)];
            if (q) val += w * u[cnode(gc, e, c + 1, nc)];
        }
        uf[s * Nf + i] = val;
    }
}

// W_c = P^T W_f.  Coarse interior node c of edge e: fine nodes j in ((c-1) r, (c+1) r) with
// weight 1 - |j - c r| / r.  Vertex v: W_f[v] + for every incident edge end the fine nodes
// q = 1..r-1 from that end with weight 1 - q/r (incidence CSR order: ascending edge, u end first).
__global__ void project_kernel(DevGraph gc, DevGraph gf, const int32_t* __restrict__ cedge, int64_t S,
                               const double* __restrict__ wf, double* __restrict__ wc) {
    const int64_t Nc = gc.N;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < S * Nc; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = t / Nc, i = t - s * Nc;
        const double* w = wf + s * gf.N;
        double acc;
        if (i >= gc.NI) {
            const int v = (int)(i - gc.NI);
            acc = w[gf.NI + v];
            for (int k = gc.inc_ptr[v]; k < gc.inc_ptr[v + 1]; ++k) {
                const int code = gc.inc[k];
                const int e = code >> 1, end = code & 1;
                const int nf = gf.m[e] + 1, nc = gc.m[e] + 1, r = nf / nc;
                for (int q = 1; q < r; ++q) {
                    const int j = end ? nf - q : q;
                    acc += (1.0 - (double)q / (double)r) * w[fnode(gf, e, j, nf)];
                }
            }
        } else {
            const int e = cedge[i];
            const int nf = gf.m[e] + 1, nc = gc.m[e] + 1, r = nf / nc;
            const int c = (int)(i - gc.off[e]) + 1;
            acc = w[fnode(gf, e, c * r, nf)];
            for (int q = 1; q < r; ++q) {
                const double wt = 1.0 - (double)q / (double)r;
                acc += wt * w[fnode(gf, e, c * r - q, nf)];
                acc += wt * w[fnode(gf, e, c * r + q, nf)];
            }
        }
        wc[s * Nc + i] = acc;
    }
}

// out[s] = sum_i M_ii (a_si - b_si)^2: per-block partials in fixed order, then a fixed-order sum
__global__ void mnorm_partial_kernel(int64_t N, const double* __restrict__ m2 /* M_L diagonal */, const double* __restrict__ a,
                                     const double* __restrict__ b, double* __restrict__ part, int nblk) {
    __shared__ double red[8];
    const int64_t s = blockIdx.y;
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)nblk * blockDim.x) {
        const double d = a[s * N + i] - b[s * N + i];
        acc = fma(m2[i] * d, d, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        part[s * nblk + blockIdx.x] = t;
    }
}

__global__ void mnorm_final_kernel(int64_t S, int nblk, const double* __restrict__ part, double* __restrict__ out) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= S) return;
    double t = 0.0;
    for (int b = 0; b < nblk; ++b) t += part[s * nblk + b];
    out[s] = t;
}

// y += x (fixed order per element: used for the rank-ordered reduce of node-shard partial sums)
__global__ void add_kernel(double* __restrict__ y, const double* __restrict__ x, int64_t n) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        y[t] += x[t];
}

}  // namespace

void launch_add(double* y, const double* x, int64_t n, cudaStream_t st) {
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)device_sms() * 16);
    add_kernel<<<blocks, 256, 0, st>>>(y, x, n);
}

void launch_prolong(const DevGraph& gc, const DevGraph& gf, const int32_t* fedge, int64_t S, const double* uc,
                    double* uf, cudaStream_t st) {
    const int64_t n = S * gf.N;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)device_sms() * 32);
    prolong_kernel<<<blocks, 256, 0, st>>>(gc, gf, fedge, S, uc, uf);
}

void launch_project(const DevGraph& gc, const DevGraph& gf, const int32_t* cedge, int64_t S, const double* wf,
                    double* wc, cudaStream_t st) {
    const int64_t n = S * gc.N;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)device_sms() * 32);
    project_kernel<<<blocks, 256, 0, st>>>(gc, gf, cedge, S, wf, wc);
}

void launch_mnorm_sq_diff(const DevGraph& g, int64_t S, const double* a, const double* b, double* part, double* out,
                          cudaStream_t st) {
    const int nblk = MNORM_PARTS;
    mnorm_partial_kernel<<<dim3(nblk, (unsigned)S), 256, 0, st>>>(g.N, g.ml, a, b, part, nblk);
    mnorm_final_kernel<<<(unsigned)((S + 127) / 128), 128, 0, st>>>(S, nblk, part, out);
}

}  // namespace grf
