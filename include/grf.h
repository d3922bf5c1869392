/*
 * grf.h -- C ABI of the B200-native fractional-SPDE Gaussian-random-field sampler
 * on metric graphs (arxiv 2605.02670, Kovacs / Molnar / Szaraz).  Implementation:
 * libgrf.so (paper_2605_02670_b200/csrc, CUDA sm_100a, fp64).
 *
 * What one grf_sample call computes (PAPER.md = "P<line>"):
 *
 *     u_s = sum_{l=-K^-}^{K^+} (c_I^{(l)} M_L + c_L^{(l)} (kappa^2 M_L + G))^{-1} W_s,
 *     W_s = M_L^{1/2} z_s,                                  s = 0 .. n_samples-1
 *
 *   P1 FEM on the metric graph with mesh size h (P122-123), lumped mass M_L
 *   (P106-109, P137-145), stiffness G (P152-160), sinc-quadrature coefficients
 *   c_I, c_L and limits K^-, K^+ (P60-67 [eq:coefficients], P335), kappa^2 M_L in
 *   the operator per SURVEY §8c Q3.  Each node's system is solved by
 *   Neumann-Neumann domain decomposition (P162-311): per-edge Thomas condensation
 *   to the vertex Schur complement, matrix-free NN-preconditioned CG on it, and a
 *   Thomas interior recovery; the node solutions are summed (P313-324).  The sum
 *   over l equals (2k sin(pi beta)/pi) sum_l e^{2 beta y_l} (M + e^{2 y_l} K)^{-1} W
 *   (the north_star weights) exactly.
 *
 * DOF order (SPEC.md S97; P150): interior nodes of edge 0 by ascending local x,
 * then edge 1, ..., then the vertices 0..V-1.  Edge e = (edge_u[e], edge_v[e]) has
 * local x = 0 at edge_u and x = length[e] at edge_v.
 *
 * Noise stream: sample j of a call with
 * base seed sigma uses Philox4x32-10 key (lo32(sigma+j), hi32(sigma+j)) and for
 * DOF i the counter (lo32(i), hi32(i), 0, 0); Box-Muller with the fixed ln / cos
 * operation sequences of DESIGN.md; W_i = sqrt(M_L,ii) z_i.  Hence
 * grf_sample(seed=s0, n=1) reproduces sample s0 of grf_sample(seed=0, n > s0) -- and, the flip
 * side, calls with base seeds sigma and sigma + 1 share all but one sample (shifted by one):
 * independent calls must use base seeds at least n_samples apart (the chunked host path and the
 * sample-sharded path rely on the shift to draw sample ranges).
 *
 * Conventions for every call:
 *   - status codes, never exceptions / aborts across the ABI; grf_last_error()
 *     returns a thread-local message for the last failing call on this thread;
 *   - "device" pointers are CUDA device (or managed) memory on the current device,
 *     "host" pointers are host memory; arrays are C-contiguous;
 *   - the caller owns every buffer it passes; the library copies host inputs;
 *   - stream arguments are cudaStream_t passed as void* (NULL = legacy default
 *     stream); device work is enqueued asynchronously on that stream unless a
 *     call says it synchronises.
 *   - thread safety: distinct graph handles are independent; calls on one
 *     handle must be externally serialised (the plan cache is mutated).
 */
#ifndef GRF_H_
#define GRF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GRF_ABI_VERSION 1

typedef enum grf_status {
    GRF_OK = 0,
    GRF_EINVAL = 1,        /* invalid argument (message says which) */
    GRF_ENOMEM = 2,        /* allocation failed / workspace too small */
    GRF_ECUDA = 3,         /* CUDA runtime error (message carries cudaGetErrorString) */
    GRF_ENCCL = 4,         /* NCCL error */
    GRF_ENOCONV = 5,       /* some (node, sample) PCG missed rtol in max_iter; output still written */
    GRF_EUNSUPPORTED = 6   /* configuration outside what this build's kernels handle */
} grf_status;

/* Thread-local text of the last error on this thread ("" if none). */
const char* grf_last_error(void);
/* Build string, e.g. "grf 1 sm_100a". */
const char* grf_version(void);

/* Device-memory allocator used for the graph handle's persistent device data
 * (mesh arrays, cached per-plan tables).  alloc returns NULL on failure.
 * Pass NULL to grf_graph_create to use cudaMalloc / cudaFree. */
typedef struct grf_allocator {
    void* (*alloc)(size_t bytes, void* ctx, void* stream);
    void (*free)(void* ptr, size_t bytes, void* ctx, void* stream);
    void* ctx;
} grf_allocator;

typedef struct grf_graph grf_graph;
typedef struct grf_comm grf_comm;

/* Create a metric graph + its P1 mesh (P122-123: n_e = ceil(l_e/h) in fp64,
 * h_e = l_e/n_e).  Host arrays of length n_edges, copied.  Self-loops and
 * multi-edges are accepted.  GRF_EINVAL when: n_vertices < 1,
 * n_edges < 1, an endpoint is out of range, a length is <= 0 or not finite, h <= 0
 * or not finite, or a vertex has no incident edge (zero lumped mass).
 * Device data is allocated through `alloc` (NULL: cudaMalloc) on the current
 * device and uploaded synchronously.  *out receives the handle. */
grf_status grf_graph_create(int64_t n_vertices, int64_t n_edges, const int64_t* edge_u,
                            const int64_t* edge_v, const double* length, double h,
                            const grf_allocator* alloc, grf_graph** out);
/* ---- edge-partitioned graphs (the largest graph, config 4) ------------
 * The edges of a whole graph are split into parts; a part is the subgraph of its edges with
 * every vertex they touch.  Vertices touched by several parts are interface vertices.
 *
 * grf_partition_edges (host only, deterministic): edge_part[e] in [0, n_parts) for every edge
 * (host array of length E).  With vertex coordinates xy (host [V][2], nullable) the edges are
 * split by recursive coordinate bisection of their midpoints weighted by their DOF weight n_e
 * (SURVEY §8e); without, the breadth-first edge order is cut into runs of equal DOF weight.
 * info (host int64[4], nullable): interface vertices, max / min part DOF weight, empty parts.
 *
 * grf_graph_create_part: part `part` of that partition as a graph handle, everything it needs
 * from the whole graph derived inside the library from (whole, edge_part): its edges (ascending
 * global id) and vertices (ascending global id, local ids 0..V_part-1; edge orientation as in
 * the whole graph), the global DOF index of every local DOF (noise counters),
 * the whole graph's lumped vertex masses (P137-145) and degrees d_v (P261), vertex ownership
 * (the lowest part touching it adds W_v and counts it in dot products) and the interface
 * numbering and halo neighbour lists.  The part's device data uses `alloc` (NULL: the whole
 * graph's allocator).  EINVAL for a part id or edge_part entry out of range, or an empty part.
 * grf_graph_part_dofs: global DOF index of each local DOF (host int64[N_part]; the identity
 * for a whole graph). */
grf_status grf_partition_edges(const grf_graph* whole, int32_t n_parts, const double* xy, int32_t* edge_part,
                               int64_t* info);
grf_status grf_graph_create_part(const grf_graph* whole, const int32_t* edge_part, int32_t n_parts, int32_t part,
                                 const grf_allocator* alloc, grf_graph** out);
grf_status grf_graph_part_dofs(const grf_graph* g, int64_t* gid);

/* Frees the handle and everything it allocated (synchronises the device first). */
void grf_graph_destroy(grf_graph* g);

/* N (all DOFs) and the number of edge-interior DOFs N_I = N - |V|. */
grf_status grf_graph_num_dofs(const grf_graph* g, int64_t* n_dofs, int64_t* n_interior);
/* Per-edge mesh layout into caller host arrays of length E (any may be NULL):
 * n_el[e] = n_e, h_e[e], offset[e] = global index of the first interior DOF. */
grf_status grf_graph_edge_layout(const grf_graph* g, int64_t* n_el, double* h_e, int64_t* offset);
/* Lumped mass diagonal (P137-145) into a host array of length N; vertex sums in
 * ascending edge id, edge_u end before edge_v end. */
grf_status grf_graph_lumped_mass(const grf_graph* g, double* ml_host);

/* Sinc-quadrature plan (P335, P60-65): K^- = ceil(pi^2/(4 k^2 beta)),
 * K^+ = ceil(pi^2/(4 k^2 (1-beta))), L = K^- + K^+ + 1 nodes l = -K^-..K^+.
 * c_I / c_L: optional host arrays of length L.  GRF_EINVAL unless 1/4 < beta < 1, k > 0. */
grf_status grf_plan_info(double beta, double k, int64_t* k_minus, int64_t* k_plus,
                         double* c_I, double* c_L);

enum { GRF_PRECOND_NN = 0, GRF_PRECOND_JACOBI = 1, GRF_PRECOND_NONE = 2 };
enum { GRF_PCG_AUTO = 0, GRF_PCG_SHARED = 1, GRF_PCG_GLOBAL = 2 };
enum { GRF_MASS_LUMPED = 0, GRF_MASS_CONSISTENT = 1 };

typedef struct grf_options {
    double rtol;          /* PCG stop: ||r||_2 <= rtol ||g||_2 (recursive residual), default 1e-13 */
    int32_t max_iter;     /* default |V| + 10 */
    int32_t precond;      /* GRF_PRECOND_*, default NN (P260-298) */
    int64_t node_begin;   /* sum only over quadrature nodes [node_begin, node_end) of 0..L-1 */
    int64_t node_end;     /* (node sharding across GPUs); default 0 and -1 = all L nodes */
    int32_t pcg_variant;  /* GRF_PCG_*: which K4 kernel family solves the vertex systems;
                             AUTO picks the shared-memory kernels when the vertex vectors fit
                             on chip (V <= 4096) and the global-memory kernel otherwise */
    int32_t mass;         /* GRF_MASS_*: LUMPED (default, the paper's method, P106-109) or
                             CONSISTENT (the paper's comparison baseline, P129-136: consistent M in
                             the operator, noise W = R xi with R the natural-order Cholesky factor
                             of M, P148-150; V <= 8192, not for edge-partitioned parts) */
    int64_t node_stride;  /* nodes node_begin, node_begin + node_stride, ... < node_end (round-robin
                             node shards); default 1 (0 is read as 1) */
} grf_options;
void grf_options_default(grf_options* opt);

typedef struct grf_stats {
    int64_t n_nodes;           /* nodes summed by this call */
    int64_t k_minus, k_plus;
    int64_t n_systems;         /* (node, sample) vertex systems solved */
    int64_t n_unconverged;     /* systems that hit max_iter */
    int32_t iter_min, iter_max;
    double iter_mean;
    double worst_rel_residual; /* max over systems of the final recursive ||r||_2/||g||_2 (the stop test) */
    int64_t gpu_launches;      /* kernels this call launched (without the checks below) */
    /* exit checks (computed because stats were requested; not in gpu_launches):
     * the TRUE relative residual ||g - S u_G||_2 / ||g||_2 of every vertex system (the Dirichlet
     * operator applied to the answer; -1 where not computed: edge-partitioned),
     * the count of non-finite entries of the output (GRF_ENOCONV when > 0), and the device time
     * of the phases in ms: [noise, edge setup (plan build, 0 when cached), condense, PCG, recover] */
    double worst_true_rel_residual;
    int64_t n_nonfinite;
    double phase_ms[5];
} grf_stats;

/* Workspace bytes grf_sample / grf_apply need for these arguments. */
grf_status grf_workspace_size(const grf_graph* g, double kappa, double beta, double k,
                              int64_t n_samples, const grf_options* opt, size_t* bytes);

/* White noise only: W_out[j*N + i] = W_i of sample j (device, n_samples x N). */
grf_status grf_noise(grf_graph* g, uint64_t seed, int64_t n_samples, double* W_out, void* stream);
/* The same for either mass mode (GRF_MASS_*): CONSISTENT gives W = R xi, M = R R^T (natural-order
 * Cholesky, the same standard normals xi as the lumped stream); synchronises. */
grf_status grf_noise_mass(grf_graph* g, uint64_t seed, int64_t n_samples, int32_t mass, double* W_out,
                          void* stream);

/* GRF samples (see top of file).  u_out: device array n_samples x N, written.
 * workspace: device, >= grf_workspace_size bytes (NULL/0 -> allocated and freed
 * internally through the graph's allocator).  EINVAL unless kappa > 0,
 * 1/4 < beta < 1, k > 0, n_samples >= 1.  The first call for a new
 * (kappa, beta, k, node range) builds the per-(node, edge) plan tables (cached
 * in the handle).  stats (nullable) is filled after synchronising the stream;
 * GRF_ENOCONV is reported only when stats != NULL (it needs the sync).
 * With stats == NULL the call is fully asynchronous. */
grf_status grf_sample(grf_graph* g, double kappa, double beta, double k, uint64_t seed,
                      int64_t n_samples, const grf_options* opt, double* u_out,
                      void* workspace, size_t ws_bytes, void* stream, grf_stats* stats);

/* Same as grf_sample with HOST output u_host (n_samples x N): device staging,
 * device->host copy and a stream synchronisation happen inside the call.  For n_samples >= 64
 * the samples are computed in chunks -- B = max(64, ~n/6) samples each, then a tail of two
 * 32-sample chunks (256 samples: 64 64 64 32 32), every chunk >= 17 samples -- whose
 * device->host copies overlap the following chunks' computation on an internal stream (three
 * device staging buffers, one shared workspace); the field is bitwise the one-call field (chunk
 * c uses seed + its first sample index, the noise stream's per-sample key, and the same kernel
 * variants).  Page-locked u_host lets the copies run asynchronously; when it is also mapped into
 * the device (cudaHostAlloc / pinned memory under unified addressing) and the call has one or two
 * chunks, the last chunk's kernels write their result straight into u_host over PCIe (no staging,
 * no copy after them) -- unless an edge is too long for the recovery's output tile, whose values
 * are accumulated in u by read-modify-write and so stay on the device.  ENOMEM if the staging
 * buffers or the workspace cannot be allocated. */
grf_status grf_sample_host(grf_graph* g, double kappa, double beta, double k, uint64_t seed,
                           int64_t n_samples, const grf_options* opt, double* u_host,
                           void* stream, grf_stats* stats);

/* Apply sum_l (A^{(l)})^{-1} to caller right-hand sides (no noise): rhs and
 * u_out are distinct device arrays n_rhs x N (EINVAL if they alias). */
grf_status grf_apply(grf_graph* g, double kappa, double beta, double k, int64_t n_rhs,
                     const double* rhs, const grf_options* opt, double* u_out,
                     void* workspace, size_t ws_bytes, void* stream, grf_stats* stats);

/* Edge-partitioned grf_sample.  Same field as grf_sample on the whole graph:
 * every part draws its DOFs' noise with the global counters, condenses its own edges,
 * and the vertex Schur systems S^{(l)} = sum_e R_e^T S_e R_e (P242-244) are solved by an
 * NN-PCG whose vectors stay assembled: each operator application (Dirichlet step, NN step
 * with global degrees, P247-298) is followed by a halo sum of the interface vertices over
 * all parts, and each dot product sums the owned vertices over all parts.
 *   comm == NULL: all n_parts parts live in this process (sums on the device, fixed order);
 *   comm != NULL: this rank passes its single part; halo and dot sums are NCCL allreduces.
 * u_out[q]: device n_samples x N_q field on part q's local DOFs (interior of its edges,
 * then its vertices).  Synchronises the stream (convergence is checked every iteration).
 * GRF_ENOCONV is reported only when stats != NULL. */
grf_status grf_sample_edgepart(grf_graph* const* parts, int32_t n_parts, struct grf_comm* comm,
                               double kappa, double beta, double k, uint64_t seed, int64_t n_samples,
                               const grf_options* opt, double* const* u_out, void* stream,
                               grf_stats* stats);

/* ---- nested meshes (strong-error study, §4.1 P335; SPEC S119-127, S256-264) ----
 * `coarse` and `fine` are meshes of the same graph (equal vertex/edge lists and lengths) with
 * every fine n_e an integer multiple of the coarse n_e; EINVAL otherwise.  Device arrays are
 * n x N_coarse / n x N_fine (DOF order of each graph), asynchronous on `stream`.
 *   grf_prolong:       u_fine = P u_coarse, P = hat-function interpolation of coarse nodal
 *                      values at the fine nodes (the "upsample" of P335)
 *   grf_project_noise: W_coarse = P^T W_fine ("project the noise generated on the overkill
 *                      mesh down", P335)
 *   grf_mnorm_sq_diff: out[s] = (a_s - b_s)^T M_L (a_s - b_s) on g's mesh (device out[n]; the
 *                      squared L2(Gamma) error of P335 with the lumped mass); synchronises. */
grf_status grf_prolong(const grf_graph* coarse, const grf_graph* fine, int64_t n, const double* u_coarse,
                       double* u_fine, void* stream);
grf_status grf_project_noise(const grf_graph* fine, const grf_graph* coarse, int64_t n, const double* W_fine,
                             double* W_coarse, void* stream);
grf_status grf_mnorm_sq_diff(grf_graph* g, int64_t n, const double* a, const double* b, double* out,
                             void* stream);

/* Stage entry point (tests, diagnostics): the local Schur blocks
 * S^{(l,e)} = [[s_d, s_o], [s_o, s_d]] (P204-213 [eq:local_reduced_schur]) for the
 * nodes of opt's range, into host array sigma[(l*E + e)*2 + {0,1}].  Synchronises. */
grf_status grf_edge_schur(grf_graph* g, double kappa, double beta, double k,
                          const grf_options* opt, double* sigma_host);

/* ---- kernel timing (bench / diagnostics) ------------------------------------------
 * With profiling enabled the library brackets every kernel it launches with CUDA events
 * recorded on the launching stream (no synchronisation).  grf_profile_read synchronises
 * those events, returns per-kernel totals since the last read and clears them:
 * ms[k] / launches[k] for k = GRF_K_NOISE .. GRF_K_RECOVER (host arrays of length
 * GRF_K_COUNT, either may be NULL). */
enum { GRF_K_NOISE = 0, GRF_K_EDGE_SETUP = 1, GRF_K_CONDENSE = 2, GRF_K_PCG = 3, GRF_K_RECOVER = 4, GRF_K_COUNT = 5 };
grf_status grf_profile_enable(grf_graph* g, int enable);
grf_status grf_profile_read(grf_graph* g, double* ms, int64_t* launches);

/* ---- multi-GPU (one process per GPU, NCCL over NVLink/NVSwitch) ---------------
 * grf_comm_get_unique_id on rank 0, broadcast the 128 bytes with any process
 * group, then grf_comm_init on every rank (binds the current device). */
grf_status grf_comm_get_unique_id(void* id128);
grf_status grf_comm_init(const void* id128, int rank, int nranks, grf_comm** out);
void grf_comm_destroy(grf_comm* c);

/* Sample-then-node sharding (policy BY_SAMPLE_THEN_NODE) of one grf_sample call
 * over the communicator's ranks: P_s = min(world, n_samples) contiguous sample ranges, and the
 * P_l = world / P_s ranks sharing a range split the quadrature nodes ROUND-ROBIN (shard li takes
 * nodes li, li + P_l, li + 2 P_l, ...: the PCG cost varies strongly with l, P162-165, so strided
 * shards balance it).  Their partial sums (P313-324) meet on the range's root through a binomial
 * tree of NCCL send/recv pairs (fixed pairing: the same addition order on every call).
 * grf_dist_shard (host only) fills out[6] = {sample_begin, sample_end, node_begin, node_end,
 * root_rank, flags}, flags = active | is_root << 1 | P_l << 2; the shard's nodes are node_begin,
 * node_begin + P_l, ... < node_end.  grf_sample_dist writes range_out[6] likewise and, on an
 * active rank, u_out (device, n_local x N, n_local = sample_end - sample_begin): the full field of
 * the range on its root, scratch elsewhere.  Inactive ranks (world > P_s P_l) touch no output.
 * EVERY rank of the communicator must call grf_sample_dist with the same arguments: after its
 * local work each rank joins one status allreduce when P_l > 1, so a local failure on any rank
 * makes every rank return an error (GRF_ENCCL "a peer rank ... failed" on the others) instead
 * of blocking in the exchange.  opt's node range must be left at its default.  Synchronises the
 * stream when P_l > 1; pure sample shards (P_l = 1) exchange nothing and stay asynchronous.  (The EDGE_PARTITION policy is grf_sample_edgepart.) */
grf_status grf_dist_shard(int32_t world, int32_t rank, int64_t n_samples, int64_t n_nodes, int64_t* out);
grf_status grf_sample_dist(grf_graph* g, grf_comm* comm, double kappa, double beta, double k, uint64_t seed,
                           int64_t n_samples, const grf_options* opt, double* u_out, int64_t* range_out,
                           void* stream, grf_stats* stats);

/* Sum-reduce a device fp64 buffer of `count` elements to `root` over NCCL on
 * `stream` (the l-shard reduction of partial quadrature sums). */
grf_status grf_reduce_sum(grf_comm* c, const double* send, double* recv, int64_t count,
                          int root, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GRF_H_ */
