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
    int32_t n_sm = 148;               // multiprocessors of the graph's device (persistent grids)
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
    const double* sqrt_ml = nullptr;  // [N] sqrt of the lumped mass diagonal (noise scaling)
    const double* ml = nullptr;       // [N] lumped mass diagonal of this mesh
    const int32_t* dof_edge = nullptr; // [NI] edge of each interior DOF
    const int32_t* edge_order = nullptr; // [E] edges by descending interior length (work-queue order)
    // breadth-first vertex positions for the global-memory PCG (pcg_global.cu): its vectors and
    // tables are stored in this order so that a vertex's neighbours sit close by (L2 reuse)
    const int32_t* vorder = nullptr;  // [V] position -> vertex
    const int32_t* gp_ptr = nullptr;  // [V+1] incidence list of the vertex at each position
    const int32_t* gp_other = nullptr; // [2E] position of the other endpoint
    const int32_t* gp_code = nullptr; // [2E] incidence code 2e+end
    // Thomas tables depend on an edge only through (m_e, h_e): edges with identical meshes share
    // one set of table rows (config 5: all 3848 edges share one).
    int64_t NT = 0;                   // table rows (sum of m_e over distinct (m_e, h_e))
    const int64_t* toff = nullptr;    // [E] first table row of the edge's (m_e, h_e) class
    const int32_t* tab_rep = nullptr; // [E] 1 for the edge that writes its class's rows
    // edge-partitioned graphs (grf_graph_create_part; all null for a whole graph):
    const int64_t* dof_gid = nullptr; // [N] global DOF index (noise counter) of each local DOF
    const uint8_t* vowned = nullptr;  // [V] 1: this part owns the vertex (rhs W_v, dot products)
    const int64_t* viface = nullptr;  // [V] interface id (vertex shared with other parts) or -1
    int32_t max_deg = 0;              // max vertex degree (incident edge ends)
    int32_t csr = 0;                  // 1: operator tables in CSR incidence order (a vertex has > 32 edge ends)
    int32_t ell_w = 0;                // ELL width = max_deg rounded up to 4/8/16/32 (0 in CSR mode)
    const int32_t* ell_other = nullptr; // [ell_w][V] other endpoint of incidence slot j of v (v if padding)
    const int32_t* ell_code = nullptr;  // [ell_w][V] incidence code 2e+end of slot j (0 if padding)
    const int32_t* ell_valid = nullptr; // [ell_w][V] 1 for a real incidence, 0 for padding
};

// Per-node PCG operator tables (pcg_tables_kernel): [DS (V) | DM (V) | DJ (V) | OS | OM | GK],
// the three slot arrays indexed by an incidence slot k of vertex v: ELL mode k = j * V + v
// (j < ell_w, padding slots point at v with zero coefficients), CSR mode k = inc_ptr[v] + j.
// Slots j < deg(v) = inc_ptr[v+1] - inc_ptr[v] are the real incidences in both modes.
__host__ __device__ inline int64_t ops_nslots(const DevGraph& g) {
    return g.csr ? 2 * (int64_t)g.E : (int64_t)g.ell_w * g.V;
}
__host__ __device__ inline int64_t ops_stride(const DevGraph& g) { return 3 * (int64_t)g.V + 3 * ops_nslots(g); }
__device__ __forceinline__ int64_t ops_slot(const DevGraph& g, int v, int j) {
    return g.csr ? (int64_t)g.inc_ptr[v] + j : (int64_t)j * g.V + v;
}
__device__ __forceinline__ int ops_other(const DevGraph& g, int64_t k) { return g.csr ? g.inc_other[k] : g.ell_other[k]; }
__device__ __forceinline__ int ops_code(const DevGraph& g, int64_t k) { return g.csr ? g.inc[k] : g.ell_code[k]; }

// Device per-plan tables (one (kappa, beta, k, node range)).
struct DevPlan {
    int32_t L = 0;                    // nodes in this plan's range
    double kappa = 0.0;
    int32_t mass = 0;                 // 0 lumped (P137-145), 1 consistent (P129-136) mass in the operator
    const double* cI = nullptr;       // [L]
    const double* cL = nullptr;       // [Lp] (zero for l >= L)
    int32_t Lp = 0;                   // padded node row of the Thomas tables (sweep_impl.cuh tiling)
    int32_t TL = 0;                   // nodes per thread of the sweep kernels
    int32_t rounds = 0;               // node rounds: Lp = rounds * 32 * TL
    double* mu = nullptr;             // [NT * Lp] Thomas multipliers  b/d'_{t-1}, layout [(toff_e + t) * Lp + l]
    double* gam = nullptr;            // [NT * Lp] diag of A_II^{-1}: 1/(d'_t + d'_{m+1-t} - a); 0 for l >= L
    double* sig = nullptr;            // [L * E * 4]: (s_d, s_o, p_d, p_o) local Schur + its inverse
    double* ops = nullptr;            // per-node tables of S and M^{-1} (pcg.cu, ops_stride)
    double* ops_pos = nullptr;        // [L * (3V + 4E)]: the same in breadth-first positions (pcg_global.cu)
};

struct PcgParams {
    double rtol = 1e-13;
    int32_t max_iter = 0;
    int32_t precond = 0;
    int32_t global = 0;  // 1: use the global-memory K4 kernel (pcg_global.cu)
};

// Sample-tiled layouts of the per-call intermediates (shared by K3, K4, K5): samples are
// grouped in tiles of cs = sample_tile(S) (the sweep kernels' samples per item, a power of
// two), and within a tile the sample index is the fastest dimension, so a sweep item
// (edge, sample tile) writes / reads contiguous runs and a PCG CTA (node, sample octet)
// reads 64-byte runs.
//   ends  (K3 -> K4): end values w^{(l,s)}_{code}, code = 2 e + end   [tile][l][code][cs]
//   uG    (K4 -> K5): vertex solution u_G^{(l,s)}(v)                   [tile][v][l][cs]
__host__ __device__ inline int64_t ends_index(int64_t s, int32_t l, int32_t code, int32_t L, int32_t E, int32_t cs_log2) {
    return ((((s >> cs_log2) * L + l) * (int64_t)(2 * E) + code) << cs_log2) + (s & ((1 << cs_log2) - 1));
}
__host__ __device__ inline int64_t ug_index(int64_t s, int32_t v, int32_t l, int32_t L, int32_t V, int32_t cs_log2) {
    return ((((s >> cs_log2) * V + v) * (int64_t)L + l) << cs_log2) + (s & ((1 << cs_log2) - 1));
}
//   rhs   (K4a -> K4): condensed right-hand side g^{(l,s)}(v)        [tile][l][cs][v]
__host__ __device__ inline int64_t rhs_index(int64_t s, int32_t l, int32_t v, int32_t L, int32_t V, int32_t cs_log2) {
    return (((((s >> cs_log2) * L + l) << cs_log2) + (s & ((1 << cs_log2) - 1))) * (int64_t)V) + v;
}
// SM count of the current device (queried once per device, cached): grid caps of the
// grid-stride kernels (sweep.cu)
int device_sms();
// fixed split of grf_mnorm_sq_diff's reduction (a partition of the DOFs, not an SM count: the same
// summation order on every device)
constexpr int MNORM_PARTS = 148;
// log2 of the sample tile for S samples (sweep.cu)
int32_t sample_tile_log2(int64_t S);

// K1  noise (noise.cu): W[s*N + i] = sqrt(M_L,ii) z(seed + s, i)
void launch_noise(const DevGraph& g, uint64_t seed, int64_t n_samples, double* W, cudaStream_t st);
// K1' consistent-mass noise W = R xi (noise.cu); evec [S][2E], vtmp [S][V] scratch
void launch_noise_consistent(const DevGraph& g, const double* Ld, const double* Lo, const double* Ls, uint64_t seed,
                             int64_t S, double* W, double* evec, double* vtmp, cudaStream_t st);
// K2  per-(node, edge) Thomas pivots + local Schur blocks (edge_setup.cu)
void launch_edge_setup(const DevGraph& g, DevPlan& p, cudaStream_t st);
// K3  Thomas end values per (sample, edge, end, node) (sweep.cu): ends[((s*E + e)*2 + end)*L + l]
// (items = (edge, sample tile), handed out longest edge first through the device counter)
cudaError_t launch_condense(const DevGraph& g, const DevPlan& p, int64_t n_samples, const double* W,
                            double* ends, int32_t* counter, cudaStream_t st);
// K4  batched NN-PCG on the vertex Schur systems (pcg.cu): g from (W, ends), u_G -> uG[(s*V + v)*L + l]
// (K4a first assembles g = W_G + sum (c_L/h_e) w_end from the end values into rhs; the warp
// kernel does that itself and writes rhs only if need_rhs, i.e. for the exit checks)
// (gws: workspace of the global-memory variant, pcg_global_ws_bytes; used when V > 4096)
cudaError_t launch_pcg(const DevGraph& g, const DevPlan& p, int64_t n_samples, const PcgParams& prm, const double* W,
                       const double* ends, double* rhs, double* uG, int32_t* iters, double* relres, void* gws,
                       cudaStream_t st, bool need_rhs = true, int64_t* launches = nullptr);
// K4a condensed rhs (pcg.cu): rhs [tile][l][cs][v] from W and the end values
void launch_assemble_rhs(const DevGraph& g, const DevPlan& p, int64_t n_samples, const double* W, const double* ends,
                         double* rhs, cudaStream_t st);
// exit checks (pcg.cu), run when the caller asks for statistics: the true relative residual
// ||g - S u_G|| / ||g|| of every vertex system (out [S][L]) and the count of non-finite outputs
void launch_true_residual(const DevGraph& g, const DevPlan& p, int64_t n_samples, const double* rhs, const double* uG,
                          double* out, cudaStream_t st);
void launch_nonfinite(const double* u, int64_t n, unsigned long long* count, cudaStream_t st);
// K4 global-memory variant (pcg_global.cu) and its workspace
bool pcg_shared_ok(const DevGraph& g);
void launch_pcg_tables_pos(const DevGraph& g, const DevPlan& p, cudaStream_t st);
cudaError_t launch_pcg_global(const DevGraph& g, const DevPlan& p, int64_t n_samples, const PcgParams& prm,
                              const double* rhs, double* uG, int32_t* iters, double* relres, void* ws,
                              cudaStream_t st);
size_t pcg_global_ws_bytes(const DevGraph& g, int32_t L, int64_t n_samples);
// K5  Thomas recovery + accumulation over nodes (sweep.cu): u[s*N + dof] from W and u_G
cudaError_t launch_recover(const DevGraph& g, const DevPlan& p, int64_t n_samples, const double* W, double* u,
                           const double* uG, int32_t* counter, cudaStream_t st);
// true when K5 + K5b write every output value exactly once by plain stores (no read-modify-write
// of u: every edge fits the recovery's shared-memory output tile), so u may be page-locked host
// memory mapped into the device (grf_sample_host's last chunk)
bool recover_out_write_only(const DevGraph& g, const DevPlan& p, int64_t n_samples);
// K5b vertex values u_v = sum_l u_G^{(l)}(v) (sweep.cu)
cudaError_t launch_vertex_sum(const DevGraph& g, const DevPlan& p, int64_t n_samples, const double* uG, double* u,
                              cudaStream_t st);
// node tiling of the Thomas tables for L nodes: Lp = rounds * 32 * TL (sweep.cu)
void plan_tiling(int32_t L, int32_t* Lp, int32_t* tl, int32_t* rounds);

// K4 warp-per-system variant (pcg_warp.cu); false if the graph is outside its range
// with K4a fused (ends != nullptr): g from W and the end values, written to rhs when rhs is not
// null; ends == nullptr: g read from rhs (K4a's output)
bool launch_pcg_warp(const DevGraph& g, const DevPlan& p, int64_t n_samples, const PcgParams& prm, const double* W,
                     const double* ends, double* rhs, double* uG, int32_t* iters, double* relres, cudaStream_t st);

// Edge-partitioned NN-PCG stages (dist.cu); vectors [L][V][cs] per part
namespace dist {
struct Vecs {
    double *x, *r0, *r1, *p0, *p1, *q, *z;
};
struct Scal {  // [L * cs] per system, shared by all parts of the problem
    double *alpha, *beta, *rz, *gg, *rr;
    int32_t *done, *its, *active;  // active: [1] count of unconverged systems
};
void init(const DevGraph& g, int32_t L, int64_t S, int32_t csl, int64_t tile, const double* rhs, const Vecs& v,
          cudaStream_t st);
void precond(const DevGraph& g, const DevPlan& p, int32_t pc, int32_t cs, const double* r, double* z, cudaStream_t st);
void spmv(const DevGraph& g, const DevPlan& p, int32_t cs, const double* beta, const double* z, const double* po,
          double* pn, double* q, cudaStream_t st);
void update(const DevGraph& g, const DevPlan& p, int32_t pc, int32_t cs, const double* alpha, const double* q,
            const double* pn, const double* ro, double* rn, double* x, double* z, cudaStream_t st);
void dots(const DevGraph& g, int32_t L, int32_t cs, int K, const double* a0, const double* b0, const double* a1,
          const double* b1, double* part, double* out, cudaStream_t st);
void pack(const DevGraph& g, int32_t L, int32_t cs, const double* X, double* buf, cudaStream_t st);
void unpack(const DevGraph& g, int32_t L, int32_t cs, const double* buf, double* X, cudaStream_t st);
void sum_parts(int32_t P, double* const* in_dev, int64_t n, double* out, cudaStream_t st);
// neighbour halo: pack the shared vertices per neighbour, combine own + received in part order
void halo_pack(const DevGraph& g, int32_t L, int32_t cs, int64_t n, const int32_t* idx, const double* X, double* send,
               cudaStream_t st);
void halo_combine(const DevGraph& g, int32_t L, int32_t cs, int32_t nif, const int32_t* vert, const int32_t* ptr,
                  const int32_t* src, const double* recv, double* X, cudaStream_t st);
void scal_init(int32_t n, int32_t cs, int64_t S, int64_t tile, int32_t csl, const double* dots, const Scal& sc,
               cudaStream_t st);
void scal_alpha(int32_t n, const double* pq, const Scal& sc, cudaStream_t st);
void scal_beta(int32_t n, double tol2, const double* dots, const Scal& sc, cudaStream_t st);
void finish(const DevGraph& g, int32_t L, int64_t S, int32_t csl, int64_t tile, const double* x, const Scal& sc,
            double* uG, int32_t* iters, double* relres, cudaStream_t st);
int32_t dot_blocks(const DevGraph& g);
}  // namespace dist

// y += x (refine.cu)
void launch_add(double* y, const double* x, int64_t n, cudaStream_t st);
// nested-mesh transfer for the strong-error study (refine.cu)
void launch_prolong(const DevGraph& gc, const DevGraph& gf, const int32_t* fedge, int64_t S, const double* uc,
                    double* uf, cudaStream_t st);
void launch_project(const DevGraph& gc, const DevGraph& gf, const int32_t* cedge, int64_t S, const double* wf,
                    double* wc, cudaStream_t st);
void launch_mnorm_sq_diff(const DevGraph& g, int64_t S, const double* a, const double* b, double* part, double* out,
                          cudaStream_t st);

// K2b per-node CSR operator tables for K4 (pcg.cu)
void launch_pcg_tables(const DevGraph& g, const DevPlan& p, cudaStream_t st);
size_t pcg_table_doubles(const DevGraph& g);
bool pcg_supported(const DevGraph& g);

size_t pcg_smem_bytes(const DevGraph& g);
int32_t pcg_max_vertices();

}  // namespace grf
