// Microbenchmark of the warp-autonomous recover step body (design study for sweep v2): one warp
// owns ALL nodes of a round (LW l-lanes x TL nodes) for WS = (32/LW) x TS samples, accumulates
// the per-step sums over l by a select-free shuffle reduce-scatter (side flip + sample-slot
// permutation) and writes them straight into a per-warp output tile (first visit store, second
// visit add, __syncwarp per step) -- no cross-warp partials, folds or block barriers.
// Steady state only: coefficients / noise from a fixed shared-memory block.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o body2_bench body2_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int IB = 8;

template <int TL, int TS, int LW, int NW, bool PIPE>
__global__ void __launch_bounds__(NW * 32, 1) body(double* out, int steps, int M) {
    constexpr int SW = 32 / LW, WS = SW * TS, CS = NW * WS, RN = LW * TL, NP = TL / 2;
    constexpr bool ODD = TL & 1;
    constexpr int LB = LW == 32 ? 5 : (LW == 16 ? 4 : 3);  // l-lane bits
    extern __shared__ double sm[];
    double* cmu = sm;                    // [IB][RN]
    double* cga = cmu + IB * RN;         // [IB][RN]
    double* wb = cga + IB * RN;          // [IB][2 side][2 copy][CS]
    double* otile = wb + IB * 4 * CS;    // [CS][M]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ll = lane % LW, sl = lane / LW;
    for (int i = tid; i < IB * RN; i += NW * 32) { cmu[i] = 0.01 * (i % 7); cga[i] = 0.02 * (i % 5); }
    for (int i = tid; i < IB * 4 * CS; i += NW * 32) wb[i] = 0.001 * i;
    __syncthreads();
    // lane roles: side flip = top l-lane bit, sample permutation from the next two
    const int side = (ll >> (LB - 1)) & 1;
    const int perm = (((ll >> (LB - 2)) & 1) << 1) | ((ll >> (LB - 3)) & 1);
    const bool writer = (ll & ((1 << (LB - 3)) - 1)) == 0;
    const int s0 = warp * WS + sl * TS;  // first sample of this lane (within the CTA's CS)
    double Y[TL][TS], Z[TL][TS];
#pragma unroll
    for (int n = 0; n < TL; ++n)
#pragma unroll
        for (int j = 0; j < TS; ++j) Y[n][j] = Z[n][j] = 0.0;
    double* myrow = otile + (s0 + perm) * M;  // slot 0 after the reduction: sample s0 + perm
    double pA[TS], pB[TS];
#pragma unroll
    for (int j = 0; j < TS; ++j) pA[j] = pB[j] = 0.0;
    int t = 0;
    auto reduce_write = [&](double (&xA)[TS], double (&xB)[TS], int tw) {
#pragma unroll
        for (int j = 0; j < TS; ++j) xA[j] += __shfl_xor_sync(0xffffffffu, xB[j], LW / 2);
        xA[0] += __shfl_xor_sync(0xffffffffu, xA[2], LW / 4);
        xA[1] += __shfl_xor_sync(0xffffffffu, xA[3], LW / 4);
        xA[0] += __shfl_xor_sync(0xffffffffu, xA[1], LW / 8);
#pragma unroll
        for (int o = LW / 16; o >= 1; o >>= 1) xA[0] += __shfl_xor_sync(0xffffffffu, xA[0], o);
        if (writer) myrow[side * CS * M + tw] = xA[0];  // separate L / R tiles: one writer lane each
    };
    for (int st = 0; st < steps; ++st) {
        const int tt = st & (IB - 1);
        const double* rmu = cmu + tt * RN;
        const double* rga = cga + tt * RN;
        double wl[TS], wr[TS];
        {
            const int cp = perm & 1, px = perm >> 1;
#pragma unroll
            for (int q = 0; q < TS / 2; ++q) {
                const int o = s0 + 2 * (q ^ px);
                const double2 a = *reinterpret_cast<const double2*>(wb + ((tt * 2 + side) * 2 + cp) * CS + o);
                const double2 c = *reinterpret_cast<const double2*>(wb + ((tt * 2 + (side ^ 1)) * 2 + cp) * CS + o);
                wl[2 * q] = a.x; wl[2 * q + 1] = a.y; wr[2 * q] = c.x; wr[2 * q + 1] = c.y;
            }
        }
        double aA[TS], aB[TS];
#pragma unroll
        for (int j = 0; j < TS; ++j) aA[j] = aB[j] = 0.0;
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const double2 m2 = *reinterpret_cast<const double2*>(rmu + 2 * ll + 2 * LW * q);
            const double2 g2 = *reinterpret_cast<const double2*>(rga + 2 * ll + 2 * LW * q);
#pragma unroll
            for (int j = 0; j < TS; ++j) {
                Y[2 * q][j] = fma(-m2.x, Y[2 * q][j], wl[j]);
                aA[j] = fma(g2.x, Y[2 * q][j], aA[j]);
                Z[2 * q][j] = fma(-m2.x, Z[2 * q][j], wr[j]);
                aB[j] = fma(g2.x, Z[2 * q][j], aB[j]);
                Y[2 * q + 1][j] = fma(-m2.y, Y[2 * q + 1][j], wl[j]);
                aA[j] = fma(g2.y, Y[2 * q + 1][j], aA[j]);
                Z[2 * q + 1][j] = fma(-m2.y, Z[2 * q + 1][j], wr[j]);
                aB[j] = fma(g2.y, Z[2 * q + 1][j], aB[j]);
            }
        }
        if (ODD) {
            const double mu = rmu[2 * LW * NP + ll], gg = rga[2 * LW * NP + ll];
#pragma unroll
            for (int j = 0; j < TS; ++j) {
                Y[TL - 1][j] = fma(-mu, Y[TL - 1][j], wl[j]);
                aA[j] = fma(gg, Y[TL - 1][j], aA[j]);
                Z[TL - 1][j] = fma(-mu, Z[TL - 1][j], wr[j]);
                aB[j] = fma(gg, Z[TL - 1][j], aB[j]);
            }
        }
        if (PIPE) {
            reduce_write(pA, pB, t == 0 ? M - 1 : t - 1);
#pragma unroll
            for (int j = 0; j < TS; ++j) { pA[j] = aA[j]; pB[j] = aB[j]; }
            if (++t == M) t = 0;
            continue;
        }
        // reduce-scatter over the LW l-lanes: flip level, two halving levels, full levels
#pragma unroll
        for (int j = 0; j < TS; ++j) aA[j] += __shfl_xor_sync(0xffffffffu, aB[j], LW / 2);
        aA[0] += __shfl_xor_sync(0xffffffffu, aA[2], LW / 4);
        aA[1] += __shfl_xor_sync(0xffffffffu, aA[3], LW / 4);
        aA[0] += __shfl_xor_sync(0xffffffffu, aA[1], LW / 8);
#pragma unroll
        for (int o = LW / 16; o >= 1; o >>= 1) aA[0] += __shfl_xor_sync(0xffffffffu, aA[0], o);
        const int pos = side ? (M - 1 - t) : t;
        if (writer) {
            double* d = myrow + pos;
            *d = (2 * t < M) ? aA[0] : *d + aA[0];
        }
        __syncwarp();
        if (++t == M) t = 0;
    }
    double s = 0.0;
    for (int n = 0; n < TL; ++n) for (int j = 0; j < TS; ++j) s += Y[n][j] + Z[n][j];
    if (s == 1234.5) out[tid] = s + otile[tid];
}

template <int TL, int TS, int LW, int NW, bool PIPE = false>
void run(double* d, const char* name) {
    constexpr int SW = 32 / LW, CS = NW * SW * TS, RN = LW * TL;
    const int M = 149;
    const int steps = 20000;
    const size_t smem = sizeof(double) * (2 * IB * RN + IB * 4 * CS + (size_t)CS * M * 2);
    cudaFuncSetAttribute(body<TL, TS, LW, NW, PIPE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, body<TL, TS, LW, NW, PIPE>, NW * 32, smem);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, body<TL, TS, LW, NW, PIPE>);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0;
    for (int it = 0; it < 2; ++it) {
        cudaEventRecord(a);
        body<TL, TS, LW, NW, PIPE><<<148 * per_sm, NW * 32, smem>>>(d, steps, M);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
    }
    cudaError_t e = cudaGetLastError();
    const double fmas = 148.0 * per_sm * NW * 32 * steps * (4.0 * TL * TS);
    printf("%-28s regs %3d  CTAs/SM %d  warps/SM %2d: %.3f ms, %.2f TFMA/s = %.1f%% of 16.78 measured %s\n", name,
           fa.numRegs, per_sm, per_sm * NW, ms, fmas / ms / 1e9, 100.0 * fmas / ms / 1e9 / 16.78,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    double* d;
    cudaMalloc(&d, 1 << 20);
    run<7, 4, 32, 8, true>(d, "PIPE LW32 TL7 TS4 8w");
    run<7, 4, 16, 8, true>(d, "PIPE LW16 TL7 TS4 8w");
    run<7, 4, 8, 8, true>(d, "PIPE LW8 TL7 TS4 8w");
    run<4, 4, 32, 8, true>(d, "PIPE LW32 TL4 TS4 8w");
    run<4, 4, 16, 8, true>(d, "PIPE LW16 TL4 TS4 8w");
    run<8, 4, 16, 8, true>(d, "PIPE LW16 TL8 TS4 8w");
    run<6, 4, 32, 8, true>(d, "PIPE LW32 TL6 TS4 8w");
    run<7, 4, 32, 8>(d, "LW32 TL7 TS4 8w");
    run<7, 4, 16, 8>(d, "LW16 TL7 TS4 8w");
    run<7, 4, 8, 8>(d, "LW8  TL7 TS4 8w");
    run<4, 4, 32, 8>(d, "LW32 TL4 TS4 8w (x2/SM?)");
    run<4, 4, 16, 8>(d, "LW16 TL4 TS4 8w (x2/SM?)");
    run<4, 4, 16, 4>(d, "LW16 TL4 TS4 4w");
    run<5, 4, 16, 8>(d, "LW16 TL5 TS4 8w");
    run<6, 4, 16, 8>(d, "LW16 TL6 TS4 8w");
    run<8, 4, 16, 8>(d, "LW16 TL8 TS4 8w");
    run<6, 4, 32, 8>(d, "LW32 TL6 TS4 8w");
    return 0;
}
