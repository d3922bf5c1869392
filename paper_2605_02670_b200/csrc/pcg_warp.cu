// K4 warp-per-system variant of the batched NN-PCG (pcg.cu has the operator definitions,
// the table layout and the thread-group variant for larger vertex sets).
#include <cstdlib>

#include "grf_internal.h"

namespace grf {
namespace {

constexpr size_t SMEM_LIMIT = 227 * 1024;
// per node l: [DS (V) | DM (V) | DJ (V) | OS (W*V) | OM (W*V) | GK (W*V)], slot-major [j][v] (pcg.cu)
__host__ __device__ inline int64_t table_stride(int V, int W) { return 3 * (int64_t)V + 3 * (int64_t)W * V; }

// ---------------------------------------------------------------------------------------
// Warp-group-per-system variant (V <= 1024).  CTA = node l x one octet of consecutive samples
// per pass (the CTA walks `octs` octets); a group of WPS warps solves one (l, s) system: r and p
// in shared memory (neighbour access of the two operators), x, q = S p and z = M^{-1} r in
// registers (VPL vertices v = 32 (WPS k + wi) + lane per lane of group warp wi), dot products by
// 5-level xor shuffles then a fixed-order sum over the group's warps through shared memory,
// group barriers (bar.sync, one id per system) between the phases -- no block barriers after the
// optional staging of node l's operator tables and ELL neighbour indices.  WPS = 1 is the
// warp-per-system form (__syncwarp only); WPS = 2 halves the registers per thread, so twice the
// warps are resident for the same shared memory (latency hiding of the neighbour loads).
constexpr int WARP_NW = 8;  // systems per CTA (an octet)
// shared-memory stride of one system's r, p: 2V + 1 doubles (odd), so the octet's 8 values of a
// vertex lie in 8 different banks when u_G is written out sample-fastest (an even stride put
// them all in one bank: an 8-way conflict, 6 % of the kernel's shared-memory wavefronts)
__host__ __device__ inline int sys_stride(int V) { return 2 * V + 1; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int VPL, int W, bool STAGE, int WPS, bool FUSE>
__global__ void __launch_bounds__(WARP_NW * WPS * 32) pcg_warp_kernel(DevGraph g, int32_t L, const double* __restrict__ ops,
                                                                PcgParams prm, int64_t S, int32_t octs, int32_t csl,
                                                                const double* __restrict__ Wn, const double* __restrict__ ends,
                                                                double* __restrict__ rhs_out, double* __restrict__ uG,
                                                                int32_t* __restrict__ iters, double* __restrict__ relres) {
    extern __shared__ double sm[];
    const int V = g.V;
    const int l = blockIdx.x;
    constexpr int NT = WARP_NW * WPS * 32;
    const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) / WPS, wi = (threadIdx.x >> 5) % WPS;
    __shared__ double xch[WARP_NW][4][WPS];  // group dot-product exchange: [system][slot][warp]
    // barrier over the system's warp group (id 1 + system: id 0 is __syncthreads)
    auto gsync = [&]() {
        if (WPS == 1)
            __syncwarp();
        else
            asm volatile("bar.sync %0, %1;" ::"r"(1 + warp), "r"(WPS * 32) : "memory");
    };
    // fixed-order group sum of a warp-reduced value (every warp of the group gets the same total)
    auto gsum = [&](double v, int slot) {
        if (WPS == 1) return v;
        if (lane == 0) xch[warp][slot][wi] = v;
        gsync();
        double t = xch[warp][slot][0];
#pragma unroll
        for (int q = 1; q < WPS; ++q) t += xch[warp][slot][q];
        return t;
    };
    const int64_t stride = table_stride(V, W);
    const double* tab = ops + l * stride;
    const double* DS = tab;
    const double* DM = DS + V;
    const double* DJ = DM + V;
    const double* OS = DJ + V;
    const double* OM = OS + (size_t)W * V;
    const double* GK = OM + (size_t)W * V;  // c_L/h_e per incidence slot (K4a's coefficients, fused below)
    const int* eo = g.ell_other;
    double* r = sm + (size_t)warp * sys_stride(V);
    double* p = r + V;
    // packed staging (W = 4): per vertex the 4 neighbour indices as one ushort4 (V <= 1024) and
    // the 4 slot coefficients of each operator as two double2: a vertex's operator row is one
    // LDS.64 + two LDS.128
    constexpr bool PACK = STAGE && W == 4;
    const ushort4* nb4 = nullptr;
    const double2 *os01 = nullptr, *os23 = nullptr, *om01 = nullptr, *om23 = nullptr;
    if (STAGE) {  // DS, DM, OS, OM and the neighbour indices of node l, once per CTA
        double* st = sm + (size_t)((WARP_NW * sys_stride(V) + 1) & ~1);  // 16-byte aligned
        if (PACK) {
            double* sD = st;                                          // DS [V], DM [V]
            double2* sO = reinterpret_cast<double2*>(st + 2 * V);     // OS01, OS23, OM01, OM23: [V] each
            ushort4* sN = reinterpret_cast<ushort4*>(sO + 4 * V);     // neighbours [V]
            for (int i = threadIdx.x; i < 2 * V; i += NT) sD[i] = tab[i];
            for (int v = threadIdx.x; v < V; v += NT) {
                const double* oS = OS + v;
                const double* oM = OM + v;
                sO[v] = make_double2(oS[0], oS[V]);
                sO[V + v] = make_double2(oS[2 * V], oS[3 * V]);
                sO[2 * V + v] = make_double2(oM[0], oM[V]);
                sO[3 * V + v] = make_double2(oM[2 * V], oM[3 * V]);
                sN[v] = make_ushort4((unsigned short)eo[v], (unsigned short)eo[V + v], (unsigned short)eo[2 * V + v],
                                     (unsigned short)eo[3 * V + v]);
            }
            __syncthreads();
            DS = sD;
            DM = sD + V;
            os01 = sO;
            os23 = sO + V;
            om01 = sO + 2 * V;
            om23 = sO + 3 * V;
            nb4 = sN;
        } else {
            int* so = reinterpret_cast<int*>(st + (size_t)(2 + 2 * W) * V);
            for (int i = threadIdx.x; i < 2 * V; i += NT) st[i] = tab[i];                      // DS, DM
            for (int i = threadIdx.x; i < 2 * W * V; i += NT) st[2 * V + i] = tab[3 * V + i];  // OS, OM
            for (int i = threadIdx.x; i < W * V; i += NT) so[i] = eo[i];
            __syncthreads();
            DS = st;
            DM = st + V;
            OS = st + 2 * V;
            OM = OS + (size_t)W * V;
            eo = so;
        }
    }
    // y = D x + sum_j O_j x_{o_j} for this lane's vertices (x in shared memory), with the lane
    // partials of the dot products that read the same x_v fused in (same per-lane order as a
    // separate pass): MODE 1: d1 += x.y (p.q); MODE 2: d1 += x.x, d2 += x.y (r.r, r.z)
    auto apply = [&](const double* D, const double* O, const double2* O01, const double2* O23, const double* xs,
                     double (&y)[VPL], int mode, double& d1, double& d2) {
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
            const int v = lane + 32 * (WPS * k + wi);
            if (v < V) {
                const double xv = xs[v];
                double a = D[v] * xv;
                if (PACK) {
                    const ushort4 nb = nb4[v];
                    const double2 c01 = O01[v], c23 = O23[v];
                    a = fma(c01.x, xs[nb.x], a);
                    a = fma(c01.y, xs[nb.y], a);
                    a = fma(c23.x, xs[nb.z], a);
                    a = fma(c23.y, xs[nb.w], a);
                } else {
#pragma unroll
                    for (int j = 0; j < W; ++j) a = fma(O[j * V + v], xs[eo[j * V + v]], a);
                }
                y[k] = a;
                if (mode == 1) d1 = fma(xv, a, d1);
                if (mode == 2) {
                    d1 = fma(xv, xv, d1);
                    d2 = fma(xv, a, d2);
                }
            }
        }
    };
    auto precond = [&](double (&z)[VPL], int mode, double& d1, double& d2) {
        if (prm.precond == 0) {
            apply(DM, OM, om01, om23, r, z, mode, d1, d2);
        } else {
#pragma unroll
            for (int k = 0; k < VPL; ++k) {
                const int v = lane + 32 * (WPS * k + wi);
                if (v < V) {
                    const double rv = r[v];
                    z[k] = (prm.precond == 1 ? DJ[v] : 1.0) * rv;
                    if (mode == 2) {
                        d1 = fma(rv, rv, d1);
                        d2 = fma(rv, z[k], d2);
                    }
                }
            }
        }
    };

    for (int oc = 0; oc < octs; ++oc) {
        const int64_t s0 = ((int64_t)blockIdx.y * octs + oc) * WARP_NW;
        if (s0 >= S) break;  // block-uniform
        // K4a fused: condensed rhs g_v = W_v + sum_j (c_L/h_e) w_{code_j(v)} (P233-239)
        // of the octet's 8 systems, assembled by the whole CTA straight from K3's end values into
        // each system's r: the 8 samples of a (vertex, slot) are one 64-byte run of `ends` (sample
        // fastest), so 8 consecutive threads take the 8 samples of one vertex; slot order and
        // arithmetic are K4a's (padding slots: code 0, coefficient 0), so g is bitwise K4a's.
        // rhs_out (only when the caller asked for the exit checks) keeps g for the true residual.
        // ends == nullptr: K4a ran separately and rhs_out is its assembled rhs, read per system.
        // a thread per vertex, all 8 samples: its W incidence codes and coefficients, then every
        // end-value run of the vertex (8 samples = 64 bytes = 4 x 16-byte loads per slot) issued
        // before the first use -- one dependent DRAM round trip per vertex instead of one per value
        const bool full = csl >= 3 && s0 + WARP_NW <= S;  // block-uniform: 8 samples in one tile
        for (int v = threadIdx.x; FUSE && v < V; v += NT) {
            int code[W];
            double gk[W];
#pragma unroll
            for (int j = 0; j < W; ++j) {
                code[j] = g.ell_code[j * V + v];
                gk[j] = GK[j * V + v];
            }
            const bool own = g.vowned == nullptr || g.vowned[v];
            double acc[WARP_NW];
            if (full) {
#pragma unroll
                for (int w = 0; w < WARP_NW; ++w) acc[w] = 0.0;
                constexpr int JC = W < 4 ? W : 4;  // slots whose runs are in flight together (registers)
#pragma unroll
                for (int j0 = 0; j0 < W; j0 += JC) {
                    double2 ev[JC][WARP_NW / 2];
#pragma unroll
                    for (int j = 0; j < JC; ++j) {
                        const double2* run =
                            reinterpret_cast<const double2*>(ends + ends_index(s0, l, code[j0 + j], L, g.E, csl));
#pragma unroll
                        for (int q = 0; q < WARP_NW / 2; ++q) ev[j][q] = run[q];
                    }
#pragma unroll
                    for (int j = 0; j < JC; ++j) {
#pragma unroll
                        for (int q = 0; q < WARP_NW / 2; ++q) {
                            acc[2 * q] = fma(gk[j0 + j], ev[j][q].x, acc[2 * q]);
                            acc[2 * q + 1] = fma(gk[j0 + j], ev[j][q].y, acc[2 * q + 1]);
                        }
                    }
                }
            } else {
#pragma unroll
                for (int w = 0; w < WARP_NW; ++w) {
                    acc[w] = 0.0;
                    if (s0 + w < S) {
#pragma unroll
                        for (int j = 0; j < W; ++j)
                            acc[w] = fma(gk[j], ends[ends_index(s0 + w, l, code[j], L, g.E, csl)], acc[w]);
                    }
                }
            }
#pragma unroll
            for (int w = 0; w < WARP_NW; ++w) {
                const int64_t s = s0 + w;
                if (s < S) {
                    const double gv = (own ? Wn[s * g.N + g.NI + v] : 0.0) + acc[w];
                    sm[(size_t)w * sys_stride(V) + v] = gv;
                    if (rhs_out) rhs_out[rhs_index(s, l, v, L, V, csl)] = gv;
                }
            }
        }
        if (FUSE) __syncthreads();  // the octet's r complete
        const int64_t s = s0 + warp;
        if (s < S) {  // warp-uniform; no block barriers inside
            double x[VPL], t[VPL];  // t holds q = S p, then z = M^{-1} r (disjoint lifetimes)
            // condensed rhs g_v = W_v + sum_j (c_L/h_e) w_{code_j(v)} (P233-239); x_0 = 0, r = g
            // a rhs whose squared norm is near the fp64 range limits (e.g. a unit rhs deep inside a long
            // edge at a mass-dominated node decays to ~1e-300) is solved for g / 2^e with 2^e ~ max|g|:
            // power-of-two scaling is exact (every PCG quantity scales exactly, alpha and beta are
            // unchanged) and keeps the dot products away from underflow
            double gg = 0.0;
            const double* gs = FUSE ? nullptr : rhs_out + rhs_index(s, l, 0, L, V, csl);  // K4a rhs
    #pragma unroll
            for (int k = 0; k < VPL; ++k) {
                const int v = lane + 32 * (WPS * k + wi);
                x[k] = 0.0;
                if (v < V) {
                    double gv;
                    if (FUSE) {
                        gv = r[v];
                    } else {
                        gv = gs[v];
                        r[v] = gv;
                    }
                    gg = fma(gv, gv, gg);
                }
            }
            gg = gsum(warp_sum(gg), 0);
            double sup = 1.0;
            if (gg > 0.0 && (gg < 0x1p-900 || gg > 0x1p900)) {  // rare: rescale by a power of two (exact)
                double gmax = 0.0;
    #pragma unroll
                for (int k = 0; k < VPL; ++k) {
                    const int v = lane + 32 * (WPS * k + wi);
                    if (v < V) gmax = fmax(gmax, fabs(r[v]));
                }
    #pragma unroll
                for (int o = 16; o > 0; o >>= 1) gmax = fmax(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
                if (WPS > 1) {
                    if (lane == 0) xch[warp][1][wi] = gmax;
                    gsync();
#pragma unroll
                    for (int q = 0; q < WPS; ++q) gmax = fmax(gmax, xch[warp][1][q]);
                }
                int e = 0;
                frexp(gmax, &e);
                e = e < -1000 ? -1000 : (e > 1000 ? 1000 : e);
                const double sdown = ldexp(1.0, -e);
                sup = ldexp(1.0, e);
                gg = 0.0;
    #pragma unroll
                for (int k = 0; k < VPL; ++k) {
                    const int v = lane + 32 * (WPS * k + wi);
                    if (v < V) {
                        const double gv = r[v] * sdown;
                        r[v] = gv;
                        gg = fma(gv, gv, gg);
                    }
                }
                gg = gsum(warp_sum(gg), 2);
            }
            gsync();  // r complete
            double d0a = 0.0, d0b = 0.0;
            precond(t, 0, d0a, d0b);
            double rz = 0.0;
    #pragma unroll
            for (int k = 0; k < VPL; ++k) {
                const int v = lane + 32 * (WPS * k + wi);
                if (v < V) {
                    p[v] = t[k];
                    rz = fma(r[v], t[k], rz);
                }
            }
            rz = gsum(warp_sum(rz), 3);
            gsync();  // p complete
            const double tol2 = prm.rtol * prm.rtol * gg;
            bool done = !(gg > 0.0);
            double rr = gg;
            int it = 0;
            while (!done && it < prm.max_iter) {
                ++it;
                double pq = 0.0, unused = 0.0;
                apply(DS, OS, os01, os23, p, t, 1, pq, unused);  // Dirichlet step (P247-258): t = q, pq = p.q
                pq = gsum(warp_sum(pq), 0);
                if (!(pq > 0.0)) break;  // p = 0 (e.g. an underflowed rhs): nothing left to reduce
                const double alpha = rz / pq;
    #pragma unroll
                for (int k = 0; k < VPL; ++k) {
                    const int v = lane + 32 * (WPS * k + wi);
                    if (v < V) {
                        x[k] = fma(alpha, p[v], x[k]);
                        r[v] = fma(-alpha, t[k], r[v]);
                    }
                }
                gsync();  // r complete
                double t_rr = 0.0, t_rz = 0.0;
                precond(t, 2, t_rr, t_rz);  // Neumann step (P260-298): t = z, with r.r and r.z
                t_rr = warp_sum(t_rr);
                t_rz = warp_sum(t_rz);
                if (WPS > 1) {  // both totals through one exchange (slots 1, 2)
                    if (lane == 0) {
                        xch[warp][1][wi] = t_rr;
                        xch[warp][2][wi] = t_rz;
                    }
                    gsync();
                    t_rr = xch[warp][1][0];
                    t_rz = xch[warp][2][0];
#pragma unroll
                    for (int q = 1; q < WPS; ++q) {
                        t_rr += xch[warp][1][q];
                        t_rz += xch[warp][2][q];
                    }
                }
                rr = t_rr;
                if (t_rr <= tol2) break;
                const double beta = t_rz / rz;
                rz = t_rz;
    #pragma unroll
                for (int k = 0; k < VPL; ++k) {
                    const int v = lane + 32 * (WPS * k + wi);
                    if (v < V) p[v] = fma(beta, p[v], t[k]);
                }
                gsync();  // p complete
            }
            gsync();
    #pragma unroll
            for (int k = 0; k < VPL; ++k) {  // u_G of this system parked in r (free now)
                const int v = lane + 32 * (WPS * k + wi);
                if (v < V) r[v] = x[k] * sup;
            }
            if (lane == 0 && wi == 0) {
                iters[s * L + l] = it;
                relres[s * L + l] = gg > 0.0 ? sqrt(rr / gg) : 0.0;
            }
        }
        __syncthreads();
        // the octet's 8 samples are consecutive slots of one sample tile: write u_G [tile][v][l][cs]
        // as 64-byte runs (vertex-major, sample fastest) instead of 8-byte scatters
        for (int i = threadIdx.x; i < V * WARP_NW; i += NT) {
            const int v = i / WARP_NW, w = i % WARP_NW;
            if (s0 + w < S) uG[ug_index(s0 + w, v, l, L, V, csl)] = sm[(size_t)w * sys_stride(V) + v];
        }
        __syncthreads();  // r / p are rewritten by the next octet
    }
}

size_t warp_smem_bytes(const DevGraph& g, int W, bool stage) {
    size_t b = sizeof(double) * (size_t)((WARP_NW * sys_stride(g.V) + 1) & ~1);
    if (stage) b += sizeof(double) * (size_t)(2 + 2 * W) * g.V + sizeof(int) * (size_t)W * g.V;
    return b;
}

template <int VPL, int W, int WPS>
bool launch_warp_t(const DevGraph& g, const DevPlan& p, int64_t n_samples, const PcgParams& prm, const double* Wn,
                   const double* ends, double* rhs, double* uG, int32_t* iters, double* relres, cudaStream_t st) {
    constexpr int NT = WARP_NW * WPS * 32;
    const bool stage = warp_smem_bytes(g, W, true) <= SMEM_LIMIT;
    const size_t smem = warp_smem_bytes(g, W, stage);
    if (smem > SMEM_LIMIT) return false;
    const int64_t n_oct = (n_samples + WARP_NW - 1) / WARP_NW;
    // octets per CTA: the CTAs run in waves of (resident CTAs per SM) x 148 and a wave lasts about
    // `octs` octet solves, so pick the power of two minimising waves x octs (the partial last wave
    // included); ties go to the larger octs (fewer table stagings).  Config 3: 2 (23 waves).
    // FUSE (template, no per-octet branch in the K4a-separate form): ends != nullptr
    auto* kern = ends ? (stage ? pcg_warp_kernel<VPL, W, true, WPS, true> : pcg_warp_kernel<VPL, W, false, WPS, true>)
                      : (stage ? pcg_warp_kernel<VPL, W, true, WPS, false> : pcg_warp_kernel<VPL, W, false, WPS, false>);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem);
    const int64_t slots = (int64_t)g.n_sm * (per_sm > 0 ? per_sm : 1);
    int64_t octs = 1, best = -1;
    for (int64_t o = 1; o <= n_oct; o *= 2) {
        const int64_t ctas = p.L * ((n_oct + o - 1) / o);
        const int64_t cost = ((ctas + slots - 1) / slots) * o;
        if (best < 0 || cost <= best) {
            best = cost;
            octs = o;
        }
    }
    const dim3 grid(p.L, (unsigned)((n_oct + octs - 1) / octs));
    const int32_t csl = sample_tile_log2(n_samples);
    kern<<<grid, NT, smem, st>>>(g, p.L, p.ops, prm, n_samples, (int32_t)octs, csl, Wn, ends, rhs, uG, iters, relres);
    return true;
}

template <int W>
bool launch_warp(const DevGraph& g, const DevPlan& p, int64_t n_samples, const PcgParams& prm, const double* Wn,
                 const double* ends, double* rhs, double* uG, int32_t* iters, double* relres, cudaStream_t st) {
    const int vpl = (g.V + 31) / 32;
    // warps per system: 2 once a lane holds 16+ vertices (the register file, not the shared memory,
    // bounds the resident systems there); design study override: env GRF_PCG_WPS
    static const int wps_env = [] {
        const char* e = getenv("GRF_PCG_WPS");
        return e ? atoi(e) : 0;
    }();
    const int wps = wps_env > 0 ? wps_env : (vpl > 8 ? 2 : 1);
#define GRF_PW(N)                                                                                      \
    if (vpl <= N) {                                                                                    \
        if (wps >= 4 && N >= 4) return launch_warp_t<(N >= 4 ? N / 4 : 1), W, 4>(g, p, n_samples, prm, Wn, ends, rhs, uG, iters, relres, st); \
        if (wps >= 2 && N >= 2) return launch_warp_t<(N >= 2 ? N / 2 : 1), W, 2>(g, p, n_samples, prm, Wn, ends, rhs, uG, iters, relres, st); \
        return launch_warp_t<N, W, 1>(g, p, n_samples, prm, Wn, ends, rhs, uG, iters, relres, st);               \
    }
    GRF_PW(1) GRF_PW(2) GRF_PW(4) GRF_PW(8) GRF_PW(16) GRF_PW(32)
#undef GRF_PW
    return false;
}

}  // namespace

bool launch_pcg_warp(const DevGraph& g, const DevPlan& p, int64_t n_samples, const PcgParams& prm, const double* Wn,
                     const double* ends, double* rhs, double* uG, int32_t* iters, double* relres, cudaStream_t st) {
    if (g.V > 32 * 32) return false;
    if (g.ell_w == 4) return launch_warp<4>(g, p, n_samples, prm, Wn, ends, rhs, uG, iters, relres, st);
    if (g.ell_w == 8) return launch_warp<8>(g, p, n_samples, prm, Wn, ends, rhs, uG, iters, relres, st);
    return false;
}

}  // namespace grf
