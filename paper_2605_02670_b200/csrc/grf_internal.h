// Internal declarations shared by the host orchestration (grf_api.cpp) and the
// CUDA kernels (*.cu).  Not part of the ABI: see include/grf.h.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace grf {

// Device view of a graph + mesh (grf_graph_create).  All arrays device-resident.
struct DevGraph {
    int32_t V = 0, E = 0;
    int64_t N = 0, NI = 0;            // all DOFs / interior DOFs
    int32_t max_m = 0;                // max interior count over edges
    const int32_t* eu = nullptr;      // [E] edge_u
    const int32_t* ev = nullptr;      // [E] edge_v
    const int32_t* m = nullptr;       // [E] interior nodes n_e - 1
    const int64_t* off = nullptr;     // [E] first interior DOF
    const double* h = nullptr;        // [E] h_e
    const int32_t* inc_ptr = nullptr; // [V+1] vertex -> incidence list
    const int32_t* inc = nullptr;     // [2E] code 2*e + end (end 0 = edge_u side, 1 = edge_v side)
    const int32_t* inc_other = nullptr; // [2E] the other endpoint of that edge
    const double* inv_deg = nullptr;  // [V] 1 / d_v, d_v = incident edge ends (P261)
    const int32_t* owner = nullptr;   // [V] incidence code that writes the vertex value in recovery
    const double* sqrt_ml = nullptr;  // [N] sqrt of the lumped mass diagonal
};

// Device per-plan tables (one (kappa, beta, k, node range)).
struct DevPlan {
    int32_t L = 0;                    // nodes in this plan's range
    double kappa = 0.0;
    const double* cI = nullptr;       // [L]
    const double* cL = nullptr;       // [L]
    double* invd = nullptr;           // [NI * L]: 1/d'_i of A_II^{(l,e)}, layout [(off_e + i) * L + l]
    double* sig = nullptr;            // [L * E * 4]: (s_d, s_o, p_d, p_o) local Schur + its inverse
};

struct PcgParams {
    double rtol = 1e-13;
    int32_t max_iter = 0;
    int32_t precond = 0;
};

// K1  noise (noise.cu): W[s*N + i] = sqrt(M_L,ii) z(seed + s, i)
void launch_noise(const DevGraph& g, uint64_t seed, int64_t n_samples, double* W, cudaStream_t st);
// K2  per-(node, edge) Thomas pivots + local Schur blocks (edge_setup.cu)
void launch_edge_setup(const DevGraph& g, DevPlan& p, cudaStream_t st);
// K3  condensed vertex rhs g[(s*V + v)*L + l] (condense.cu)
void launch_condense(const DevGraph& g, const DevPlan& p, int64_t n_samples, const double* W,
                     double* gu, cudaStream_t st);
// K4  batched NN-PCG on the vertex Schur systems, in place g -> u_Gamma (pcg.cu)
void launch_pcg(const DevGraph& g, const DevPlan& p, int64_t n_samples, const PcgParams& prm,
                double* gu, int32_t* iters, double* relres, cudaStream_t st);
// K5  Thomas recovery + accumulation over nodes, W -> u in place (recover.cu)
cudaError_t launch_recover(const DevGraph& g, const DevPlan& p, int64_t n_samples, double* Wu,
                           const double* gu, cudaStream_t st);

size_t pcg_smem_bytes(const DevGraph& g);
int32_t pcg_max_vertices();
int32_t recover_max_interior();
int32_t max_nodes_per_block();

}  // namespace grf
