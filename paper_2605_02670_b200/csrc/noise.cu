// K1: lumped-mass white noise W = M_L^{1/2} z  (PAPER.md P99-109 [eq:wh_def], P150).
//
// Canonical stream:
//   key = (lo32(seed+s), hi32(seed+s)), counter = (lo32(i), hi32(i), 0, 0)
//   (x0..x3) = Philox4x32-10, u1 = ((x0<<21 | x1>>11) + 1) 2^-53, u2 = (x2<<21 | x3>>11) 2^-53
//   z = sqrt(-2 ln(u1)) cos(2 pi u2) with the FIXED ln / cos operation sequences below,
//   W_i = sqrt(M_L,ii) z.
// Bit-exactness with the CPU oracle needs every operation correctly rounded and
// un-fused: this TU is compiled with --fmad=false AND uses the explicit
// __d*_rn intrinsics (never contracted).
//
// Layout: W[s * N + i] (sample-major, the grf_sample output layout).  One thread
// per (s, i), grid-stride; the write is a plain coalesced store -- the kernel is
// bound by the fp64 polynomial work (~70 ops + 1 division per draw), not HBM.
#include "grf_internal.h"

namespace grf {
namespace {

__device__ __forceinline__ uint4 philox_round(uint4 c, uint2 k) {
    const unsigned int M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const unsigned int hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    const unsigned int hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    return make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
}

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        c = philox_round(c, k);
        if (r < 9) {
            k.x += 0x9E3779B9u;
            k.y += 0xBB67AE85u;
        }
    }
    return c;
}

// ln x for x in (0, 1]: x = m 2^e, m in [sqrt(1/2), sqrt(2)); s = (m-1)/(m+1);
// ln m = 2 s sum_{j=0}^{12} s^{2j}/(2j+1) (Horner, constants 1.0/(2j+1)).
__device__ __forceinline__ double ln_fixed(double x) {
    const double LN2 = 0.6931471805599453;
    const double SQRT_HALF = 0.7071067811865476;
    // frexp for the normal x this sees (u1 >= 2^-53): the exponent field and the mantissa with
    // exponent -1, exactly frexp's (m in [1/2, 1)) without its zero / subnormal / inf checks
    const unsigned long long xb = (unsigned long long)__double_as_longlong(x);
    int e = (int)((xb >> 52) & 0x7ffu) - 1022;
    double m = __longlong_as_double((long long)((xb & 0x800fffffffffffffull) | 0x3fe0000000000000ull));
    if (m < SQRT_HALF) {
        m = __dmul_rn(m, 2.0);
        e -= 1;
    }
    const double f = __dsub_rn(m, 1.0);
    const double s = __ddiv_rn(f, __dadd_rn(m, 1.0));
    const double s2 = __dmul_rn(s, s);
    double p = 1.0 / 25.0;
#pragma unroll
    for (int j = 11; j >= 0; --j) p = __dadd_rn(1.0 / (double)(2 * j + 1), __dmul_rn(s2, p));
    const double t = __dmul_rn(s, p);
    return __dadd_rn(__dmul_rn((double)e, LN2), __dadd_rn(t, t));
}

// cos(2 pi u), u in [0,1) a multiple of 2^-53: t = 4u, q = floor(t + 1/2), f = t - q (exact),
// theta = f pi/2 in [-pi/4, pi/4]; cos/sin by Taylor (10 Horner steps, constants 1.0/(n(n-1))).
// Horner constants of the two series, k[odd][j - 1] = 1/((2j+1) 2j) (sine) or 1/(2j (2j-1)) (cosine),
// as a per-CTA shared table: a lane reads its quadrant's constant with one load instead of
// materialising both 64-bit immediates and selecting (the same constant values, so the same bits)
__device__ __forceinline__ double cos2pi_fixed(double u, const double (*ktab)[10]) {
    const double HALF_PI = 1.5707963267948966;
    const double t = __dmul_rn(4.0, u);
    const double q = floor(__dadd_rn(t, 0.5));
    const double f = __dsub_rn(t, q);
    const double th = __dmul_rn(f, HALF_PI);
    const double th2 = __dmul_rn(th, th);
    // only the polynomial the quadrant needs is evaluated (the same operations as that branch of
    // the two-polynomial definition): odd quadrants take the sine series, even ones the cosine
    const int qi = ((int)q) & 3;
    const bool odd = qi & 1;
    double p = 1.0;
    const double* kq = ktab[odd ? 1 : 0];
#pragma unroll
    for (int j = 10; j >= 1; --j) {
        const double k = kq[j - 1];
        p = __dsub_rn(1.0, __dmul_rn(__dmul_rn(th2, k), p));
    }
    const double v = odd ? __dmul_rn(th, p) : p;
    return (qi == 1 || qi == 2) ? -v : v;
}

__global__ void __launch_bounds__(256) noise_kernel(const double* __restrict__ sqrt_ml,
                                                    const int64_t* __restrict__ dof_gid, int64_t N,
                                                    int64_t total, uint64_t seed, double* __restrict__ W) {
    __shared__ double ktab[2][10];
    if (threadIdx.x < 20) {
        const int odd = threadIdx.x / 10, j = threadIdx.x % 10 + 1;
        ktab[odd][j - 1] = odd ? 1.0 / (double)((2 * j + 1) * (2 * j)) : 1.0 / (double)((2 * j) * (2 * j - 1));
    }
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t s = t / N, i = t - s * N;  // (sample, dof) of t, advanced without a 64-bit division
    const int64_t ds = stride / N, di = stride - ds * N;
    for (; t < total; t += stride) {
        const uint64_t key = seed + (uint64_t)s;
        const int64_t ig = dof_gid ? dof_gid[i] : i;  // counter = GLOBAL DOF index (edge-partitioned parts)
        const uint4 x = philox4x32_10(make_uint4((unsigned)ig, (unsigned)((uint64_t)ig >> 32), 0u, 0u),
                                      make_uint2((unsigned)key, (unsigned)(key >> 32)));
        const uint64_t A = ((uint64_t)x.x << 21) | (uint64_t)(x.y >> 11);
        const uint64_t B = ((uint64_t)x.z << 21) | (uint64_t)(x.w >> 11);
        const double u1 = __dmul_rn((double)(A + 1ull), 0x1.0p-53);
        const double u2 = __dmul_rn((double)B, 0x1.0p-53);
        const double r = __dsqrt_rn(__dmul_rn(-2.0, ln_fixed(u1)));
        const double z = __dmul_rn(r, cos2pi_fixed(u2, ktab));
        W[t] = sqrt_ml ? __dmul_rn(sqrt_ml[i], z) : z;  // sqrt_ml == nullptr: the raw normals xi
        s += ds;
        i += di;
        if (i >= N) {
            i -= N;
            ++s;
        }
    }
}

// Consistent mass (P129-136, P148-150): W = R xi with R the natural-order Cholesky factor of M,
// R = [[L_II, 0], [M_GI L_II^{-T}, L_S]]: L_II is block-diagonal over the edges (the Cholesky
// factor of each interior chain tridiag(h/6, 2h/3, h/6): diagonal Ld, sub-diagonal Lo, per
// table class), L_S the Cholesky factor of the vertex Schur complement M_GG - M_GI M_II^{-1} M_IG.
// Thread per (sample, edge): y = L_II^{-T} xi_I by back substitution (its end values feed the
// edge's two vertices through M_GI = h/6), then W_I = L_II xi_I in place.
__global__ void cnoise_edge_kernel(DevGraph g, const double* __restrict__ Ld, const double* __restrict__ Lo,
                                   int64_t S, double* __restrict__ W, double* __restrict__ evec) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= S * g.E) return;
    const int64_t s = t / g.E;
    const int e = (int)(t - s * g.E);
    const int m = g.m[e];
    const int64_t tb = g.toff[e];
    double* w = W + s * g.N + g.off[e];
    double y1 = 0.0, ym = 0.0;
    if (m > 0) {
        double y = w[m - 1] / Ld[tb + m - 1];  // y_m
        ym = y;
        for (int i = m - 2; i >= 0; --i) y = (w[i] - Lo[tb + i + 1] * y) / Ld[tb + i];
        y1 = y;
        double prev = 0.0;
        for (int i = 0; i < m; ++i) {
            const double xi = w[i];
            w[i] = Ld[tb + i] * xi + (i ? Lo[tb + i] * prev : 0.0);
            prev = xi;
        }
    }
    const double c = g.h[e] / 6.0;
    evec[s * 2 * g.E + 2 * e] = c * y1;      // to vertex edge_u (end 0)
    evec[s * 2 * g.E + 2 * e + 1] = c * ym;  // to vertex edge_v (end 1)
}

// W_G = L_S xi_G + sum over the vertex's incidences (CSR order) of the edge terms; thread per (s, v)
__global__ void cnoise_vertex_kernel(DevGraph g, const double* __restrict__ Ls, int64_t S, const double* __restrict__ W,
                                     const double* __restrict__ evec, double* __restrict__ out) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= S * g.V) return;
    const int64_t s = t / g.V;
    const int v = (int)(t - s * g.V);
    const double* xi = W + s * g.N + g.NI;
    const double* row = Ls + (int64_t)v * g.V;
    double acc = 0.0;
    for (int k = 0; k <= v; ++k) acc = fma(row[k], xi[k], acc);
    for (int q = g.inc_ptr[v]; q < g.inc_ptr[v + 1]; ++q) acc += evec[s * 2 * g.E + g.inc[q]];
    out[t] = acc;
}

}  // namespace

void launch_noise(const DevGraph& g, uint64_t seed, int64_t n_samples, double* W, cudaStream_t st) {
    const int64_t total = n_samples * g.N;
    if (total == 0) return;
    int64_t blocks = (total + 255) / 256;
    const int64_t cap = (int64_t)g.n_sm * 16;
    if (blocks > cap) blocks = cap;
    noise_kernel<<<(unsigned)blocks, 256, 0, st>>>(g.sqrt_ml, g.dof_gid, g.N, total, seed, W);
}

void launch_noise_consistent(const DevGraph& g, const double* Ld, const double* Lo, const double* Ls, uint64_t seed,
                             int64_t S, double* W, double* evec, double* vtmp, cudaStream_t st) {
    const int64_t total = S * g.N;
    int64_t blocks = (total + 255) / 256;
    if (blocks > (int64_t)g.n_sm * 64) blocks = (int64_t)g.n_sm * 64;
    noise_kernel<<<(unsigned)blocks, 256, 0, st>>>(nullptr, g.dof_gid, g.N, total, seed, W);
    cnoise_edge_kernel<<<(unsigned)((S * g.E + 127) / 128), 128, 0, st>>>(g, Ld, Lo, S, W, evec);
    cnoise_vertex_kernel<<<(unsigned)((S * g.V + 127) / 128), 128, 0, st>>>(g, Ls, S, W, evec, vtmp);
    cudaMemcpy2DAsync(W + g.NI, g.N * sizeof(double), vtmp, g.V * sizeof(double), g.V * sizeof(double), S,
                      cudaMemcpyDeviceToDevice, st);
}

}  // namespace grf
