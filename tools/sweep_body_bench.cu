// Ceiling of the condense / recover step bodies alone (no staging, barriers or items): the
// same register tile (TL = 7 nodes x TS = 4 samples, two chains) iterating over a shared-memory
// block of coefficients and noise, 8 warps per SM.  PF: the next step's coefficients and noise
// are loaded into registers one step ahead.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

constexpr int TL = 7, TS = 4, NP = TL / 2, IB = 8, RN = 32 * TL, CS = 32;

template <bool REC, bool PF, bool NK = false>
__global__ void __launch_bounds__(256) body(double* out, int steps) {
    __shared__ double cmu[IB * RN], cga[IB * RN], wb[IB * 2 * CS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ll = REC ? lane % 4 : lane % 8, sl = REC ? lane / 4 : lane / 8;
    const int lt = REC ? (warp * 4 + ll) : ((warp % 4) * 8 + ll);
    const int st0 = REC ? sl * TS : ((warp / 4) * 4 + sl) * TS;
    for (int i = tid; i < IB * RN; i += 256) { cmu[i] = 0.01 * (i % 7); cga[i] = 0.02 * (i % 5); }
    for (int i = tid; i < IB * 2 * CS; i += 256) wb[i] = 0.001 * i;
    __syncthreads();
    double Y[TL][TS], Z[TL][TS];
    for (int n = 0; n < TL; ++n) for (int j = 0; j < TS; ++j) Y[n][j] = Z[n][j] = 0.0;
    double accL = 0.0, accR = 0.0;
    double2 m2n[NP], g2n[NP];
    double mon = 0, gon = 0, wln[TS], wrn[TS];
    auto ld = [&](int st) {
        const int tt = st & (IB - 1);
#pragma unroll
        for (int q = 0; q < TS / 2; ++q) {
            const double2 a = *reinterpret_cast<const double2*>(wb + (tt * 2 + 0) * CS + st0 + 2 * q);
            const double2 c = *reinterpret_cast<const double2*>(wb + (tt * 2 + 1) * CS + st0 + 2 * q);
            wln[2 * q] = a.x; wln[2 * q + 1] = a.y; wrn[2 * q] = c.x; wrn[2 * q + 1] = c.y;
        }
        const double* rmu = cmu + tt * RN;
        const double* rga = cga + tt * RN;
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            m2n[q] = *reinterpret_cast<const double2*>(rmu + 2 * lt + 64 * q);
            if (REC) g2n[q] = *reinterpret_cast<const double2*>(rga + 2 * lt + 64 * q);
        }
        mon = rmu[64 * NP + lt];
        if (REC) gon = rga[64 * NP + lt];
    };
    if (PF) ld(0);
    for (int st = 0; st < steps; ++st) {
        if (!PF) ld(st);
        double2 m2[NP], g2[NP];
        double mo = mon, go = gon, wl[TS], wr[TS];
#pragma unroll
        for (int q = 0; q < NP; ++q) { m2[q] = m2n[q]; g2[q] = g2n[q]; }
#pragma unroll
        for (int j = 0; j < TS; ++j) { wl[j] = wln[j]; wr[j] = wrn[j]; }
        if (PF) ld(st + 1);
        double aL[TS] = {0, 0, 0, 0}, aR[TS] = {0, 0, 0, 0};
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            if (REC && NK) {
#pragma unroll
                for (int j = 0; j < TS; ++j) {
                    Y[2 * q][j] = fma(-m2[q].x, Y[2 * q][j], wl[j]);
                    aL[j] = fma(g2[q].x, Y[2 * q][j], aL[j]);
                    Z[2 * q][j] = fma(-m2[q].x, Z[2 * q][j], wr[j]);
                    aR[j] = fma(g2[q].x, Z[2 * q][j], aR[j]);
                    Y[2 * q + 1][j] = fma(-m2[q].y, Y[2 * q + 1][j], wl[j]);
                    aL[j] = fma(g2[q].y, Y[2 * q + 1][j], aL[j]);
                    Z[2 * q + 1][j] = fma(-m2[q].y, Z[2 * q + 1][j], wr[j]);
                    aR[j] = fma(g2[q].y, Z[2 * q + 1][j], aR[j]);
                }
            } else if (REC) {
                const double k0 = g2[q].x * m2[q].x, k1 = g2[q].y * m2[q].y;
#pragma unroll
                for (int j = 0; j < TS; ++j) {
                    aL[j] = fma(-k0, Y[2 * q][j], aL[j]);
                    Y[2 * q][j] = fma(-m2[q].x, Y[2 * q][j], wl[j]);
                    Z[2 * q][j] = fma(-m2[q].x, Z[2 * q][j], wr[j]);
                    aR[j] = fma(g2[q].x, Z[2 * q][j], aR[j]);
                    aL[j] = fma(-k1, Y[2 * q + 1][j], aL[j]);
                    Y[2 * q + 1][j] = fma(-m2[q].y, Y[2 * q + 1][j], wl[j]);
                    Z[2 * q + 1][j] = fma(-m2[q].y, Z[2 * q + 1][j], wr[j]);
                    aR[j] = fma(g2[q].y, Z[2 * q + 1][j], aR[j]);
                }
            } else {
#pragma unroll
                for (int j = 0; j < TS; ++j) {
                    Y[2 * q][j] = fma(-m2[q].x, Y[2 * q][j], wl[j]);
                    Z[2 * q][j] = fma(-m2[q].x, Z[2 * q][j], wr[j]);
                    Y[2 * q + 1][j] = fma(-m2[q].y, Y[2 * q + 1][j], wl[j]);
                    Z[2 * q + 1][j] = fma(-m2[q].y, Z[2 * q + 1][j], wr[j]);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < TS; ++j) {
            if (REC && !NK) aL[j] = fma(-go * mo, Y[TL - 1][j], aL[j]);
            Y[TL - 1][j] = fma(-mo, Y[TL - 1][j], wl[j]);
            if (REC && NK) aL[j] = fma(go, Y[TL - 1][j], aL[j]);
            Z[TL - 1][j] = fma(-mo, Z[TL - 1][j], wr[j]);
            if (REC) aR[j] = fma(go, Z[TL - 1][j], aR[j]);
        }
        if (REC) {  // the select-free reduce-scatter (2 levels) as in sweep_impl.cuh
            aL[0] += __shfl_xor_sync(0xffffffffu, aL[2], 1);
            aL[1] += __shfl_xor_sync(0xffffffffu, aL[3], 1);
            aR[0] += __shfl_xor_sync(0xffffffffu, aR[2], 1);
            aR[1] += __shfl_xor_sync(0xffffffffu, aR[3], 1);
            aL[0] += __shfl_xor_sync(0xffffffffu, aL[1], 2);
            aR[0] += __shfl_xor_sync(0xffffffffu, aR[1], 2);
            accL += aL[0];
            accR += aR[0];
        }
    }
    double s = accL + accR;
    for (int n = 0; n < TL; ++n) for (int j = 0; j < TS; ++j) s += Y[n][j] + Z[n][j];
    if (s == 1234.5) out[tid] = s;
}

template <bool REC, bool PF, bool NK = false>
void run(double* d, const char* name) {
    const int steps = 20000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0;
    for (int it = 0; it < 2; ++it) {
        cudaEventRecord(a);
        body<REC, PF, NK><<<148, 256>>>(d, steps);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
    }
    const double fma_per_step = REC ? (4.0 * TL * TS + TL) : 2.0 * TL * TS;
    const double fmas = 148.0 * 256 * steps * fma_per_step;
    printf("%-12s body: %.3f ms, %.2f TFMA/s = %.1f%% of 16.78 measured\n", name, ms, fmas / ms / 1e9,
           100.0 * fmas / ms / 1e9 / 16.78);
}

int main() {
    double* d;
    cudaMalloc(&d, 1 << 16);
    run<false, false>(d, "condense");
    run<false, true>(d, "condense-pf");
    run<true, false>(d, "recover");
    run<true, true>(d, "recover-pf");
    run<true, false, true>(d, "recover-nk");
    return 0;
}
