// C-ABI implementation (include/grf.h): graph/mesh setup on the host (PAPER.md P122-160),
// quadrature plan (P60-67, P335), plan cache, workspace carving and the per-call launch
// sequence K1 noise -> K3 condense -> K4 PCG -> K5 recover (K2 on a plan-cache miss).
#include "grf.h"

#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <list>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "grf_internal.h"

namespace {

thread_local std::string g_err;

grf_status fail(grf_status st, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

#define CUDA_TRY(expr)                                                                          \
    do {                                                                                        \
        cudaError_t e_ = (expr);                                                                \
        if (e_ != cudaSuccess) return fail(GRF_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
    } while (0)

struct Alloc {
    grf_allocator a{};
    bool custom = false;
    void* get(size_t bytes, cudaStream_t st) {
        if (bytes == 0) bytes = 8;
        if (custom) return a.alloc(bytes, a.ctx, st);
        void* p = nullptr;
        if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
        return p;
    }
    void put(void* p, size_t bytes, cudaStream_t st) {
        if (!p) return;
        if (bytes == 0) bytes = 8;
        if (custom)
            a.free(p, bytes, a.ctx, st);
        else
            cudaFree(p);
    }
};

struct Block {
    void* p;
    size_t bytes;
};

struct PlanKey {
    double kappa, beta, k;
    int64_t nb, ne, stride;  // nodes nb, nb + stride, ... < ne of 0..L-1
    int64_t mass;            // GRF_MASS_*
    bool operator==(const PlanKey& o) const {
        return std::memcmp(this, &o, sizeof(PlanKey)) == 0;
    }
};

// What a part of an edge partition needs from the whole graph (grf_graph_create_part derives it)
struct PartSpec {
    int32_t part = 0, n_parts = 1;
    int64_t global_n_interior = 0;
    std::vector<int64_t> vertex_gid, edge_goff, vertex_iface;
    std::vector<double> vertex_mass;    // whole-graph lumped vertex mass (P137-145)
    std::vector<int32_t> vertex_degree; // whole-graph incident edge ends (d_v of the NN step, P261)
    std::vector<uint8_t> vertex_owned;  // 1 on exactly one part per vertex (the lowest touching it)
    int64_t n_interface = 0;
    // halo neighbours: every other part sharing a vertex with this one, ascending, with the local
    // ids of the shared vertices in ascending global id (both sides list them in the same order)
    std::vector<int32_t> nbr_part;
    std::vector<std::vector<int32_t>> nbr_verts;
};

struct Plan {
    PlanKey key{};
    int64_t Km = 0, Kp = 0;
    grf::DevPlan dev;
    std::vector<Block> blocks;
};

}  // namespace

struct grf_graph {
    int device = 0;
    Alloc alloc;
    int64_t V = 0, E = 0, N = 0, NI = 0;
    double h = 0.0;
    std::vector<int64_t> eu, ev, n_el, off;
    std::vector<double> len, he, ml;
    grf::DevGraph dev;
    std::vector<Block> blocks;  // graph-lifetime device allocations
    std::list<std::unique_ptr<Plan>> plans;  // most recent first
    bool partitioned = false;                // created by grf_graph_create_part
    int32_t part = 0, n_parts = 1;           // this part's index in its partition
    std::vector<int64_t> dof_gid;            // part: global DOF index of every local DOF
    std::vector<int32_t> nbr_part;           // part: halo neighbours (PartSpec)
    std::vector<std::vector<int32_t>> nbr_verts;
    // consistent-mass noise factor (NEXT-3), built on first use: chain Cholesky factors per
    // Thomas-table class (Ld, Lo) and the dense Cholesky factor of the vertex Schur complement
    const double *cLd = nullptr, *cLo = nullptr, *cLs = nullptr;
    int64_t n_iface = 0;                     // interface vertices of the whole partition
    // kernel timing (grf_profile_enable / grf_profile_read)
    bool prof = false;
    struct Rec {
        int kind;
        cudaEvent_t a, b;
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    cudaEvent_t new_event() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e = nullptr;
        cudaEventCreate(&e);
        return e;
    }
    // run `launch` (enqueues one kernel on st), bracketed by events when profiling
    template <class F>
    cudaError_t timed(int kind, cudaStream_t st, F&& launch) {
        // NVTX range per phase (header-only NVTX v3: a no-op unless a tool such as nsys is attached)
        static const char* const names[GRF_K_COUNT] = {"grf:noise", "grf:edge_setup", "grf:condense", "grf:pcg",
                                                       "grf:recover"};
        struct Range {
            explicit Range(const char* n) { nvtxRangePushA(n); }
            ~Range() { nvtxRangePop(); }
        } range(kind >= 0 && kind < GRF_K_COUNT ? names[kind] : "grf");
        if (!prof) {
            launch();
            return cudaGetLastError();
        }
        Rec r{kind, new_event(), new_event()};
        cudaEventRecord(r.a, st);
        launch();
        cudaError_t e = cudaGetLastError();
        cudaEventRecord(r.b, st);
        recs.push_back(r);
        return e;
    }

    template <class T>
    T* upload(const std::vector<T>& v, grf_status* st) {
        const size_t bytes = v.size() * sizeof(T);
        void* p = alloc.get(bytes, nullptr);
        if (!p) {
            *st = fail(GRF_ENOMEM, "device allocation of %zu bytes failed", bytes);
            return nullptr;
        }
        blocks.push_back({p, bytes});
        if (bytes && cudaMemcpy(p, v.data(), bytes, cudaMemcpyHostToDevice) != cudaSuccess) {
            *st = fail(GRF_ECUDA, "upload failed");
            return nullptr;
        }
        return static_cast<T*>(p);
    }
};

namespace {

grf_status plan_limits(double beta, double k, int64_t* Km, int64_t* Kp) {
    if (!(beta > 0.25 && beta < 1.0)) return fail(GRF_EINVAL, "beta must lie in (1/4, 1), got %g", beta);
    if (!(k > 0.0) || !std::isfinite(k)) return fail(GRF_EINVAL, "k must be positive, got %g", k);
    const double a = std::ceil((M_PI * M_PI) / (4.0 * k * k * beta));
    const double b = std::ceil((M_PI * M_PI) / (4.0 * k * k * (1.0 - beta)));
    if (!(a < 1e7 && b < 1e7)) return fail(GRF_EINVAL, "quadrature too large (k too small)");
    *Km = (int64_t)a;
    *Kp = (int64_t)b;
    return GRF_OK;
}

// c_const = pi / (2 k sin(pi beta)); c_I = c_const e^{-2 beta y_l}; c_L = c_I e^{2 y_l}; y_l = l k  (P61-65)
// for the nodes t = lo, lo + stride, ... < hi of 0..L-1 (l = t - K^-)
void plan_coefficients(double beta, double k, int64_t Km, int64_t lo, int64_t hi, int64_t stride, double* cI,
                       double* cL) {
    const double c_const = M_PI / (2.0 * k * std::sin(M_PI * beta));
    int64_t q = 0;
    for (int64_t t = lo; t < hi; t += stride, ++q) {
        const double y = (double)(t - Km) * k;
        const double ci = c_const * std::exp(-2.0 * beta * y);
        cI[q] = ci;
        cL[q] = ci * std::exp(2.0 * y);
    }
}

// nodes of opt's range: [node_begin, node_end) with stride node_stride (0 or 1: contiguous)
grf_status resolve_range(const grf_options* opt, int64_t L, int64_t* nb, int64_t* ne, int64_t* stride) {
    int64_t b = 0, e = L, d = 1;
    if (opt) {
        b = opt->node_begin;
        e = opt->node_end < 0 ? L : opt->node_end;
        d = opt->node_stride > 1 ? opt->node_stride : 1;
        if (opt->node_stride < 0) return fail(GRF_EINVAL, "node_stride must be >= 0");
    }
    if (b < 0 || e > L || b >= e) return fail(GRF_EINVAL, "node range [%lld, %lld) invalid for L=%lld",
                                              (long long)b, (long long)e, (long long)L);
    *nb = b;
    *ne = e;
    *stride = d;
    return GRF_OK;
}
int64_t range_count(int64_t nb, int64_t ne, int64_t stride) { return (ne - nb + stride - 1) / stride; }

grf_status check_params(const grf_graph* g, double kappa, double beta, double k, int64_t n) {
    if (!g) return fail(GRF_EINVAL, "graph is NULL");
    if (!(kappa > 0.0) || !std::isfinite(kappa)) return fail(GRF_EINVAL, "kappa must be positive, got %g", kappa);
    int64_t a, b;
    grf_status st = plan_limits(beta, k, &a, &b);
    if (st) return st;
    if (n < 1) return fail(GRF_EINVAL, "n_samples must be >= 1");
    if (n > 65535) return fail(GRF_EUNSUPPORTED, "n_samples > 65535 per call; split the call");
    return GRF_OK;
}

grf_status get_plan(grf_graph* g, double kappa, double beta, double k, const grf_options* opt, cudaStream_t st,
                    Plan** out) {
    int64_t Km, Kp;
    grf_status s = plan_limits(beta, k, &Km, &Kp);
    if (s) return s;
    const int64_t Lfull = Km + Kp + 1;
    int64_t nb, ne, nd;
    s = resolve_range(opt, Lfull, &nb, &ne, &nd);
    if (s) return s;
    PlanKey key{kappa, beta, k, nb, ne, nd, (int64_t)(opt ? opt->mass : GRF_MASS_LUMPED)};
    for (auto it = g->plans.begin(); it != g->plans.end(); ++it) {
        if ((*it)->key == key) {
            g->plans.splice(g->plans.begin(), g->plans, it);
            *out = g->plans.front().get();
            return GRF_OK;
        }
    }
    const int64_t L = range_count(nb, ne, nd);
    int32_t Lp = 0, TL = 0, rounds = 0;
    grf::plan_tiling((int32_t)L, &Lp, &TL, &rounds);
    auto p = std::make_unique<Plan>();
    p->key = key;
    p->Km = Km;
    p->Kp = Kp;
    std::vector<double> cI(L), cL(Lp, 0.0);  // c_L zero padded to the table row Lp
    plan_coefficients(beta, k, Km, nb, ne, nd, cI.data(), cL.data());
    auto grab = [&](size_t bytes) -> void* {
        void* q = g->alloc.get(bytes, st);
        if (q) p->blocks.push_back({q, bytes});
        return q;
    };
    double* dcI = (double*)grab(L * sizeof(double));
    double* dcL = (double*)grab(Lp * sizeof(double));
    const size_t tab = (size_t)std::max<int64_t>(g->dev.NT, 1) * Lp * sizeof(double);
    double* mu = (double*)grab(tab);
    double* gam = (double*)grab(tab);
    double* sig = (double*)grab((size_t)L * g->E * 4 * sizeof(double));
    double* ops = (double*)grab((size_t)L * grf::pcg_table_doubles(g->dev) * sizeof(double));
    double* ops_pos = (double*)grab((size_t)L * (3 * (size_t)g->dev.V + 4 * (size_t)g->dev.E) * sizeof(double));
    if (!dcI || !dcL || !mu || !gam || !sig || !ops || !ops_pos) {
        for (auto& b : p->blocks) g->alloc.put(b.p, b.bytes, st);
        return fail(GRF_ENOMEM, "plan tables (%.1f MB) could not be allocated",
                    (double)(2 * tab + (size_t)L * g->E * 32) / 1e6);
    }
    CUDA_TRY(cudaMemcpyAsync(dcI, cI.data(), L * sizeof(double), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(dcL, cL.data(), Lp * sizeof(double), cudaMemcpyHostToDevice, st));
    p->dev.L = (int32_t)L;
    p->dev.Lp = Lp;
    p->dev.TL = TL;
    p->dev.rounds = rounds;
    p->dev.kappa = kappa;
    p->dev.mass = (int32_t)key.mass;
    p->dev.cI = dcI;
    p->dev.cL = dcL;
    p->dev.mu = mu;
    p->dev.gam = gam;
    p->dev.sig = sig;
    p->dev.ops = ops;
    p->dev.ops_pos = ops_pos;
    CUDA_TRY(g->timed(GRF_K_EDGE_SETUP, st, [&] {
        grf::launch_edge_setup(g->dev, p->dev, st);
        grf::launch_pcg_tables(g->dev, p->dev, st);
        grf::launch_pcg_tables_pos(g->dev, p->dev, st);
    }));
    CUDA_TRY(cudaStreamSynchronize(st));  // host vectors cI/cL die at return
    // keep at most 4 plans
    while (g->plans.size() >= 4) {
        CUDA_TRY(cudaStreamSynchronize(st));
        for (auto& b : g->plans.back()->blocks) g->alloc.put(b.p, b.bytes, st);
        g->plans.pop_back();
    }
    g->plans.push_front(std::move(p));
    *out = g->plans.front().get();
    return GRF_OK;
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct WsLayout {
    size_t w = 0, cnoise = 0, ends = 0, rhs = 0, ug = 0, gws = 0, iters = 0, relres = 0, truer = 0, counter = 0,
           total = 0;
};

// with_noise: grf_sample keeps the white noise W (S x N) in the workspace
// K4 kernel family for these options (grf_options.pcg_variant)
bool use_global_pcg(const grf_graph* g, const grf_options* opt) {
    const int32_t v = opt ? opt->pcg_variant : GRF_PCG_AUTO;
    if (g->dev.csr) return true;  // hub vertices: only the global-memory kernel reads CSR tables
    return v == GRF_PCG_GLOBAL || (v == GRF_PCG_AUTO && !grf::pcg_shared_ok(g->dev));
}

WsLayout ws_layout(const grf_graph* g, int64_t L, int64_t S, bool with_noise, bool global_pcg, bool consistent) {
    WsLayout w;
    size_t o = 0;
    w.w = o;
    if (with_noise) o += align_up((size_t)S * g->N * sizeof(double));
    w.cnoise = o;  // consistent noise scratch: [S][2E] edge terms + [S][V] vertex values
    if (with_noise && consistent) o += align_up((size_t)S * (2 * g->E + g->V) * sizeof(double));
    // ends / uG are sample-tiled (grf_internal.h): sized for whole tiles
    const int64_t cs = (int64_t)1 << grf::sample_tile_log2(S);
    const int64_t Sp = (S + cs - 1) / cs * cs;
    w.ends = o;
    o += align_up((size_t)Sp * g->E * 2 * L * sizeof(double));
    w.rhs = o;
    o += align_up((size_t)Sp * g->V * L * sizeof(double));
    w.ug = o;
    o += align_up((size_t)Sp * g->V * L * sizeof(double));
    w.gws = o;
    if (global_pcg) o += align_up(grf::pcg_global_ws_bytes(g->dev, (int32_t)L, S));
    w.iters = o;
    o += align_up((size_t)S * L * sizeof(int32_t));
    w.relres = o;
    o += align_up((size_t)S * L * sizeof(double));
    w.truer = o;  // exit checks: true relative residuals [S][L], then the non-finite count
    o += align_up((size_t)S * L * sizeof(double) + sizeof(unsigned long long));
    w.counter = o;
    o += align_up(2 * sizeof(int32_t));
    w.total = o;
    return w;
}

grf_status check_kernel_limits(const grf_graph* g) {
    if (!grf::pcg_supported(g->dev))
        return fail(GRF_EUNSUPPORTED, "PCG operator tables unavailable for this graph");
    return GRF_OK;
}

// NEXT-3: the natural-order Cholesky factor of the consistent mass matrix (P148-150, SPEC S241),
// in the block form R = [[L_II, 0], [M_GI L_II^{-T}, L_S]] (noise.cu):
//   L_II: per interior chain tridiag(h/6, 2h/3, h/6): Ld_0 = sqrt(2h/3), Lo_t = (h/6)/Ld_{t-1},
//         Ld_t = sqrt(2h/3 - Lo_t^2) -- one set per Thomas-table class;
//   L_S:  dense Cholesky of S_M = M_GG - M_GI M_II^{-1} M_IG, assembled from each edge's 2x2 block
//         (the local Schur formula of edge_setup.cu with a = 2h/3, b = h/6, share = h/3).
// Dense on the host (O(V^3 / 3)), so limited to V <= 8192.
grf_status ensure_consistent_factor(grf_graph* g) {
    if (g->cLs) return GRF_OK;
    if (g->V > 8192) return fail(GRF_EUNSUPPORTED, "consistent-mass noise: %lld vertices (dense vertex Cholesky "
                                 "handles <= 8192)", (long long)g->V);
    if (g->partitioned) return fail(GRF_EUNSUPPORTED, "consistent-mass noise on an edge-partitioned part");
    const int64_t V = g->V, E = g->E, NT = std::max<int64_t>(g->dev.NT, 1);
    std::vector<double> Ld(NT, 0.0), Lo(NT, 0.0), S((size_t)V * V, 0.0);
    std::vector<int64_t> toff(E);
    CUDA_TRY(cudaMemcpy(toff.data(), g->dev.toff, E * sizeof(int64_t), cudaMemcpyDeviceToHost));
    std::vector<int32_t> rep(E);
    CUDA_TRY(cudaMemcpy(rep.data(), g->dev.tab_rep, E * sizeof(int32_t), cudaMemcpyDeviceToHost));
    for (int64_t e = 0; e < E; ++e) {
        const double h = g->he[e];
        const int64_t m = g->n_el[e] - 1;
        const double a = 2.0 * h / 3.0, b = h / 6.0, share = h / 3.0;
        if (rep[e]) {
            for (int64_t t = 0; t < m; ++t) {
                const double lo = t ? b / Ld[toff[e] + t - 1] : 0.0;
                Lo[toff[e] + t] = lo;
                Ld[toff[e] + t] = std::sqrt(a - lo * lo);
            }
        }
        double sd = share, so = b;
        if (m > 0) {
            double inv = 0.0, prod = 1.0;
            for (int64_t t = 0; t < m; ++t) {
                const double mu = b * inv;
                inv = 1.0 / (a - mu * b);
                if (t > 0) prod *= -mu;
            }
            sd = share - b * b * inv;
            so = -b * b * (prod * inv);
        }
        const int64_t u = g->eu[e], v = g->ev[e];
        S[u * V + u] += sd;
        S[v * V + v] += sd;
        S[u * V + v] += so;
        S[v * V + u] += so;
    }
    for (int64_t j = 0; j < V; ++j) {  // dense Cholesky, lower triangle, row-major
        double d = S[j * V + j];
        for (int64_t q = 0; q < j; ++q) d -= S[j * V + q] * S[j * V + q];
        if (!(d > 0.0)) return fail(GRF_EINVAL, "consistent mass Schur complement not positive definite");
        const double ljj = std::sqrt(d);
        S[j * V + j] = ljj;
        for (int64_t i = j + 1; i < V; ++i) {
            double x = S[i * V + j];
            for (int64_t q = 0; q < j; ++q) x -= S[i * V + q] * S[j * V + q];
            S[i * V + j] = x / ljj;
        }
        for (int64_t q = j + 1; q < V; ++q) S[j * V + q] = 0.0;
    }
    grf_status st = GRF_OK;
    g->cLd = g->upload(Ld, &st);
    if (!st) g->cLo = g->upload(Lo, &st);
    if (!st) g->cLs = g->upload(S, &st);
    return st;
}

// Shared tail of grf_sample / grf_apply: u (holding W on entry) -> u.
// W (S x N, device) -> u (S x N, device).  When W is null the noise for `seed` is first
// generated into the workspace (grf_sample); otherwise W is the caller's rhs (grf_apply).
grf_status solve(grf_graph* g, Plan* p, int64_t S, const grf_options* opt, const double* W, uint64_t seed,
                 double* u, void* ws, size_t ws_bytes, cudaStream_t st, grf_stats* stats) {
    const int64_t L = p->dev.L;
    const bool gen = (W == nullptr);
    const bool consistent = p->dev.mass == GRF_MASS_CONSISTENT;
    if (gen && consistent) {
        grf_status cs = ensure_consistent_factor(g);
        if (cs) return cs;
    }
    WsLayout w = ws_layout(g, L, S, gen, use_global_pcg(g, opt), consistent);
    void* own = nullptr;
    if (!ws) {
        own = g->alloc.get(w.total, st);
        if (!own) return fail(GRF_ENOMEM, "workspace of %zu bytes could not be allocated", w.total);
        ws = own;
    } else if (ws_bytes < w.total) {
        return fail(GRF_ENOMEM, "workspace too small: %zu < %zu bytes", ws_bytes, w.total);
    }
    char* base = static_cast<char*>(ws);
    // with statistics: device time of the phases (events on the stream) and the exit checks
    cudaEvent_t ph[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    if (stats)
        for (auto& e : ph) cudaEventCreate(&e);
    auto mark = [&](int i) {
        if (ph[i]) cudaEventRecord(ph[i], st);
    };
    mark(0);
    // kernels this call launches: [noise] condense, K4 (+ assemble, see launch_pcg), recover, vertex sum
    int64_t launches = 3;
    if (gen) {
        double* Wd = reinterpret_cast<double*>(base + w.w);
        cudaError_t ne = g->timed(GRF_K_NOISE, st, [&] {
            if (consistent) {
                double* ev = reinterpret_cast<double*>(base + w.cnoise);
                grf::launch_noise_consistent(g->dev, g->cLd, g->cLo, g->cLs, seed, S, Wd, ev, ev + S * 2 * g->E, st);
            } else {
                grf::launch_noise(g->dev, seed, S, Wd, st);
            }
        });
        if (ne != cudaSuccess) {
            if (own) g->alloc.put(own, w.total, st);
            return fail(GRF_ECUDA, "noise launch: %s", cudaGetErrorString(ne));
        }
        W = Wd;
        launches += 1;
    }
    mark(1);
    double* ends = reinterpret_cast<double*>(base + w.ends);
    double* uG = reinterpret_cast<double*>(base + w.ug);
    double* rhs = reinterpret_cast<double*>(base + w.rhs);
    void* gws = base + w.gws;
    int32_t* iters = reinterpret_cast<int32_t*>(base + w.iters);
    double* relres = reinterpret_cast<double*>(base + w.relres);
    int32_t* counters = reinterpret_cast<int32_t*>(base + w.counter);
    grf::PcgParams prm;
    prm.rtol = opt ? opt->rtol : 1e-13;
    prm.max_iter = (opt && opt->max_iter > 0) ? opt->max_iter : (int32_t)(g->V + 10);
    prm.precond = opt ? opt->precond : GRF_PRECOND_NN;
    prm.global = use_global_pcg(g, opt) ? 1 : 0;
    grf_status rc = GRF_OK;
    cudaError_t le = cudaSuccess;
    cudaError_t ce = g->timed(GRF_K_CONDENSE, st, [&] {
        le = grf::launch_condense(g->dev, p->dev, S, W, ends, counters, st);
    });
    if (ce == cudaSuccess) ce = le;
    mark(2);
    if (ce == cudaSuccess)
        ce = g->timed(GRF_K_PCG, st, [&] {
            le = grf::launch_pcg(g->dev, p->dev, S, prm, W, ends, rhs, uG, iters, relres, gws, st, stats != nullptr,
                                 &launches);
        });
    if (ce == cudaSuccess) ce = le;
    mark(3);
    if (ce == cudaSuccess)
        ce = g->timed(GRF_K_RECOVER, st, [&] {
            le = grf::launch_recover(g->dev, p->dev, S, W, u, uG, counters + 1, st);
            if (le == cudaSuccess) le = grf::launch_vertex_sum(g->dev, p->dev, S, uG, u, st);
        });
    if (ce == cudaSuccess) ce = le;
    mark(4);
    double* truer = reinterpret_cast<double*>(base + w.truer);
    unsigned long long* nonfin = reinterpret_cast<unsigned long long*>(truer + S * L);
    if (ce == cudaSuccess && stats) {  // exit checks: true residuals, non-finite outputs
        grf::launch_true_residual(g->dev, p->dev, S, rhs, uG, truer, st);
        grf::launch_nonfinite(u, S * g->N, nonfin, st);
        ce = cudaGetLastError();
    }
    if (ce != cudaSuccess) rc = fail(GRF_ECUDA, "kernel launch failed: %s", cudaGetErrorString(ce));
    if (rc == GRF_OK && stats) {
        std::vector<int32_t> it(S * L);
        std::vector<double> rr(S * L), tr(S * L);
        unsigned long long nf = 0;
        ce = cudaMemcpyAsync(it.data(), iters, it.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st);
        if (ce == cudaSuccess)
            ce = cudaMemcpyAsync(rr.data(), relres, rr.size() * sizeof(double), cudaMemcpyDeviceToHost, st);
        if (ce == cudaSuccess)
            ce = cudaMemcpyAsync(tr.data(), truer, tr.size() * sizeof(double), cudaMemcpyDeviceToHost, st);
        if (ce == cudaSuccess) ce = cudaMemcpyAsync(&nf, nonfin, sizeof(nf), cudaMemcpyDeviceToHost, st);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
        if (ce != cudaSuccess) {
            rc = fail(GRF_ECUDA, "stats readback: %s", cudaGetErrorString(ce));
        } else {
            std::memset(stats, 0, sizeof(*stats));
            stats->n_nodes = L;
            stats->k_minus = p->Km;
            stats->k_plus = p->Kp;
            stats->n_systems = S * L;
            stats->iter_min = it.empty() ? 0 : *std::min_element(it.begin(), it.end());
            stats->iter_max = it.empty() ? 0 : *std::max_element(it.begin(), it.end());
            double sum = 0.0, worst = 0.0;
            int64_t bad = 0;
            for (size_t i = 0; i < it.size(); ++i) {
                sum += it[i];
                worst = std::max(worst, rr[i]);
                if (!(rr[i] <= prm.rtol)) ++bad;
            }
            stats->iter_mean = it.empty() ? 0.0 : sum / it.size();
            stats->worst_rel_residual = worst;
            stats->n_unconverged = bad;
            stats->gpu_launches = launches;
            stats->worst_true_rel_residual = tr.empty() ? 0.0 : *std::max_element(tr.begin(), tr.end());
            stats->n_nonfinite = (int64_t)nf;
            const int slot[4] = {0, 2, 3, 4};  // noise, condense, pcg, recover (edge setup: grf_sample)
            for (int i = 0; i < 4; ++i) {
                float ms = 0.f;
                if (cudaEventElapsedTime(&ms, ph[i], ph[i + 1]) == cudaSuccess) stats->phase_ms[slot[i]] = ms;
            }
            if (bad) rc = fail(GRF_ENOCONV, "%lld of %lld PCG systems missed rtol %g (worst %g)", (long long)bad,
                               (long long)(S * L), prm.rtol, worst);
            else if (nf) rc = fail(GRF_ENOCONV, "%llu non-finite output values", nf);
        }
    }
    for (auto e : ph)
        if (e) cudaEventDestroy(e);
    if (own) {
        cudaStreamSynchronize(st);
        g->alloc.put(own, w.total, st);
    }
    return rc;
}

}  // namespace

extern "C" {

const char* grf_last_error(void) { return g_err.c_str(); }
const char* grf_version(void) { return "grf 1 sm_100a fp64"; }

void grf_options_default(grf_options* opt) {
    if (!opt) return;
    opt->rtol = 1e-13;
    opt->max_iter = 0;
    opt->precond = GRF_PRECOND_NN;
    opt->node_begin = 0;
    opt->node_end = -1;
    opt->node_stride = 1;
    opt->pcg_variant = GRF_PCG_AUTO;
    opt->mass = GRF_MASS_LUMPED;
}

}  // extern "C"

namespace {
grf_status create_impl(int64_t n_vertices, int64_t n_edges, const int64_t* edge_u, const int64_t* edge_v,
                       const double* length, double h, const PartSpec* part, const grf_allocator* alloc,
                       grf_graph** out) {
    if (!out) return fail(GRF_EINVAL, "out is NULL");
    *out = nullptr;
    if (n_vertices < 1) return fail(GRF_EINVAL, "n_vertices must be >= 1");
    if (n_edges < 1) return fail(GRF_EINVAL, "n_edges must be >= 1");
    if (n_vertices > (1LL << 30) || n_edges > (1LL << 29)) return fail(GRF_EUNSUPPORTED, "graph too large");
    if (!edge_u || !edge_v || !length) return fail(GRF_EINVAL, "edge arrays must not be NULL");
    if (!(h > 0.0) || !std::isfinite(h)) return fail(GRF_EINVAL, "h must be positive and finite, got %g", h);
    if (alloc && (!alloc->alloc || !alloc->free)) return fail(GRF_EINVAL, "allocator callbacks must be non-NULL");
    auto g = std::make_unique<grf_graph>();
    if (alloc) {
        g->alloc.a = *alloc;
        g->alloc.custom = true;
    }
    cudaGetDevice(&g->device);
    const int64_t V = n_vertices, E = n_edges;
    g->V = V;
    g->E = E;
    g->h = h;
    g->eu.assign(edge_u, edge_u + E);
    g->ev.assign(edge_v, edge_v + E);
    g->len.assign(length, length + E);
    std::vector<int64_t> deg(V, 0);
    for (int64_t e = 0; e < E; ++e) {
        if (g->eu[e] < 0 || g->eu[e] >= V || g->ev[e] < 0 || g->ev[e] >= V)
            return fail(GRF_EINVAL, "edge %lld has an endpoint out of range", (long long)e);
        if (!(g->len[e] > 0.0) || !std::isfinite(g->len[e]))
            return fail(GRF_EINVAL, "edge %lld has non-positive or non-finite length", (long long)e);
        deg[g->eu[e]]++;
        deg[g->ev[e]]++;
    }
    for (int64_t v = 0; v < V; ++v)
        if (deg[v] == 0) return fail(GRF_EINVAL, "vertex %lld is isolated (zero lumped mass)", (long long)v);
    // Phase 1 mesh (P123): n_e = ceil(l_e / h), h_e = l_e / n_e
    g->n_el.resize(E);
    g->he.resize(E);
    g->off.resize(E);
    int64_t NI = 0;
    int32_t max_m = 0;
    std::vector<int32_t> mm(E);
    for (int64_t e = 0; e < E; ++e) {
        const double q = std::ceil(g->len[e] / h);
        if (!(q < 1e9)) return fail(GRF_EUNSUPPORTED, "edge %lld needs %g elements", (long long)e, q);
        int64_t n = std::max<int64_t>(1, (int64_t)q);
        g->n_el[e] = n;
        g->he[e] = g->len[e] / (double)n;
        g->off[e] = NI;
        mm[e] = (int32_t)(n - 1);
        max_m = std::max(max_m, mm[e]);
        NI += n - 1;
    }
    g->NI = NI;
    g->N = NI + V;
    // Thomas-table classes: edges with the same (m_e, bits of h_e) share table rows
    std::vector<int64_t> toff(E);
    std::vector<int32_t> tab_rep(E, 0);
    int64_t NT = 0;
    {
        std::map<std::pair<int32_t, uint64_t>, int64_t> cls;
        for (int64_t e = 0; e < E; ++e) {
            uint64_t hb;
            std::memcpy(&hb, &g->he[e], sizeof(hb));
            auto it = cls.find({mm[e], hb});
            if (it == cls.end()) {
                cls[{mm[e], hb}] = NT;
                toff[e] = NT;
                tab_rep[e] = 1;
                NT += mm[e];
            } else {
                toff[e] = it->second;
            }
        }
    }
    // lumped mass (P137-145): interior h_e/2 + h_e/2; vertices sum h_e/2 in ascending edge, u end then v end
    g->ml.assign(g->N, 0.0);
    for (int64_t e = 0; e < E; ++e) {
        const double half = g->he[e] / 2;
        for (int64_t i = 0; i < g->n_el[e] - 1; ++i) g->ml[g->off[e] + i] = half + half;
    }
    for (int64_t e = 0; e < E; ++e) {
        const double half = g->he[e] / 2;
        g->ml[NI + g->eu[e]] += half;
        g->ml[NI + g->ev[e]] += half;
    }
    std::vector<double> sq(g->N);
    for (int64_t i = 0; i < g->N; ++i) sq[i] = std::sqrt(g->ml[i]);
    // edge-partitioned part: the noise of a vertex uses its WHOLE-graph lumped mass and its
    // global DOF index as the Philox counter, so every part draws the same W_v
    std::vector<int64_t> dof_gid;
    std::vector<uint8_t> vowned;
    std::vector<int64_t> viface;
    if (part) {
        dof_gid.resize(g->N);
        for (int64_t e = 0; e < E; ++e)
            for (int64_t i = 0; i < g->n_el[e] - 1; ++i) dof_gid[g->off[e] + i] = part->edge_goff[e] + i;
        vowned.resize(V);
        viface.resize(V);
        for (int64_t v = 0; v < V; ++v) {
            dof_gid[NI + v] = part->global_n_interior + part->vertex_gid[v];
            sq[NI + v] = std::sqrt(part->vertex_mass[v]);
            vowned[v] = part->vertex_owned[v] ? 1 : 0;
            viface[v] = part->vertex_iface[v];
        }
        g->n_iface = part->n_interface;
        g->part = part->part;
        g->n_parts = part->n_parts;
        g->nbr_part = part->nbr_part;
        g->nbr_verts = part->nbr_verts;
        g->dof_gid = dof_gid;
    }
    // incidence CSR in (edge, end) order, owner = first incidence, 1/d_v
    std::vector<int32_t> ptr(V + 1, 0), inc(2 * E), other(2 * E), owner(V, -1);
    for (int64_t v = 0; v < V; ++v) ptr[v + 1] = ptr[v] + (int32_t)deg[v];
    std::vector<int32_t> fill(ptr.begin(), ptr.end() - 1);
    for (int64_t e = 0; e < E; ++e) {
        const int64_t a = g->eu[e], b = g->ev[e];
        inc[fill[a]] = (int32_t)(2 * e);
        other[fill[a]++] = (int32_t)b;
        inc[fill[b]] = (int32_t)(2 * e + 1);
        other[fill[b]++] = (int32_t)a;
    }
    // ELL (padded) copy of the incidence lists for the PCG kernels
    int32_t max_deg = 0;
    for (int64_t v = 0; v < V; ++v) max_deg = std::max<int32_t>(max_deg, (int32_t)deg[v]);
    const bool csr = max_deg > 32;  // hubs (e.g. Barabasi-Albert graphs): CSR operator tables, no ELL copy
    int32_t ell_w = 4;
    while (ell_w < max_deg) ell_w *= 2;
    if (csr) ell_w = 0;
    std::vector<int32_t> ell_other((size_t)ell_w * V), ell_code((size_t)ell_w * V, 0), ell_valid((size_t)ell_w * V, 0);
    for (int64_t v = 0; v < V && !csr; ++v) {
        for (int32_t j = 0; j < ell_w; ++j) ell_other[(size_t)j * V + v] = (int32_t)v;
        for (int32_t k = ptr[v]; k < ptr[v + 1]; ++k) {
            const int32_t j = k - ptr[v];
            ell_other[(size_t)j * V + v] = other[k];
            ell_code[(size_t)j * V + v] = inc[k];
            ell_valid[(size_t)j * V + v] = 1;
        }
    }
    std::vector<double> inv_deg(V);
    for (int64_t v = 0; v < V; ++v) {
        owner[v] = inc[ptr[v]];
        inv_deg[v] = 1.0 / (double)(part ? part->vertex_degree[v] : deg[v]);  // GLOBAL d_v (P261)
    }
    // breadth-first vertex positions (each component from its lowest-numbered vertex) and the
    // incidence lists in that order, for the global-memory PCG
    std::vector<int32_t> vorder, vpos(V, -1), gp_ptr(V + 1, 0), gp_other(std::max<int64_t>(2 * E, 1)),
        gp_code(std::max<int64_t>(2 * E, 1));
    vorder.reserve(V);
    for (int64_t r = 0; r < V; ++r) {
        if (vpos[r] >= 0) continue;
        size_t head = vorder.size();
        vpos[r] = (int32_t)vorder.size();
        vorder.push_back((int32_t)r);
        while (head < vorder.size()) {
            const int32_t v = vorder[head++];
            for (int32_t k = ptr[v]; k < ptr[v + 1]; ++k) {
                const int32_t o = other[k];
                if (vpos[o] < 0) {
                    vpos[o] = (int32_t)vorder.size();
                    vorder.push_back(o);
                }
            }
        }
    }
    for (int64_t q = 0; q < V; ++q) {
        const int32_t v = vorder[q];
        gp_ptr[q + 1] = gp_ptr[q] + (ptr[v + 1] - ptr[v]);
        for (int32_t k = ptr[v]; k < ptr[v + 1]; ++k) {
            gp_other[gp_ptr[q] + (k - ptr[v])] = vpos[other[k]];
            gp_code[gp_ptr[q] + (k - ptr[v])] = inc[k];
        }
    }
    std::vector<int32_t> order(E);
    for (int64_t e = 0; e < E; ++e) order[e] = (int32_t)e;
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return mm[a] > mm[b]; });
    std::vector<int32_t> eu32(E), ev32(E);
    for (int64_t e = 0; e < E; ++e) {
        eu32[e] = (int32_t)g->eu[e];
        ev32[e] = (int32_t)g->ev[e];
    }
    grf_status st = GRF_OK;
    grf::DevGraph& d = g->dev;
    {
        int nsm = 0;
        if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, g->device) == cudaSuccess && nsm > 0)
            d.n_sm = nsm;
    }
    d.V = (int32_t)V;
    d.E = (int32_t)E;
    d.N = g->N;
    d.NI = NI;
    d.max_m = max_m;
    d.NT = NT;
    d.eu = g->upload(eu32, &st);
    if (!st) d.toff = g->upload(toff, &st);
    if (!st) d.tab_rep = g->upload(tab_rep, &st);
    if (!st) d.ev = g->upload(ev32, &st);
    if (!st) d.m = g->upload(mm, &st);
    if (!st) d.off = g->upload(g->off, &st);
    if (!st) d.h = g->upload(g->he, &st);
    if (!st) d.inc_ptr = g->upload(ptr, &st);
    if (!st) d.inc = g->upload(inc, &st);
    if (!st) d.inc_other = g->upload(other, &st);
    if (!st) d.inv_deg = g->upload(inv_deg, &st);
    if (!st) d.vorder = g->upload(vorder, &st);
    if (!st) d.gp_ptr = g->upload(gp_ptr, &st);
    if (!st) d.gp_other = g->upload(gp_other, &st);
    if (!st) d.gp_code = g->upload(gp_code, &st);
    if (!st) d.owner = g->upload(owner, &st);
    if (!st) d.sqrt_ml = g->upload(sq, &st);
    if (!st) d.ml = g->upload(g->ml, &st);
    {
        std::vector<int32_t> dof_edge(std::max<int64_t>(NI, 1), 0);
        for (int64_t e = 0; e < E; ++e)
            for (int64_t t = 0; t < g->n_el[e] - 1; ++t) dof_edge[g->off[e] + t] = (int32_t)e;
        if (!st) d.dof_edge = g->upload(dof_edge, &st);
    }
    if (!st) d.edge_order = g->upload(order, &st);
    d.max_deg = max_deg;
    d.ell_w = ell_w;
    d.csr = csr ? 1 : 0;
    if (!csr) {
        if (!st) d.ell_other = g->upload(ell_other, &st);
        if (!st) d.ell_code = g->upload(ell_code, &st);
        if (!st) d.ell_valid = g->upload(ell_valid, &st);
    }
    if (part) {
        if (!st) d.dof_gid = g->upload(dof_gid, &st);
        if (!st) d.vowned = g->upload(vowned, &st);
        if (!st) d.viface = g->upload(viface, &st);
        g->partitioned = true;
    }
    if (st) {
        grf_graph_destroy(g.release());
        return st;
    }
    *out = g.release();
    return GRF_OK;
}

}  // namespace

extern "C" {

grf_status grf_graph_create(int64_t n_vertices, int64_t n_edges, const int64_t* edge_u, const int64_t* edge_v,
                            const double* length, double h, const grf_allocator* alloc, grf_graph** out) {
    return create_impl(n_vertices, n_edges, edge_u, edge_v, length, h, nullptr, alloc, out);
}

grf_status grf_graph_create_part(const grf_graph* whole, const int32_t* edge_part, int32_t n_parts, int32_t part,
                                 const grf_allocator* alloc, grf_graph** out) {
    if (out) *out = nullptr;
    if (!whole || !edge_part || !out) return fail(GRF_EINVAL, "NULL argument");
    if (whole->partitioned) return fail(GRF_EINVAL, "the whole graph is itself a part");
    if (n_parts < 1 || part < 0 || part >= n_parts) return fail(GRF_EINVAL, "part %d of %d invalid", part, n_parts);
    const int64_t V = whole->V, E = whole->E;
    // parts touching each vertex (ascending, distinct)
    std::vector<std::vector<int32_t>> touch(V);
    auto add = [&](int64_t v, int32_t q) {
        auto& t = touch[v];
        auto it = std::lower_bound(t.begin(), t.end(), q);
        if (it == t.end() || *it != q) t.insert(it, q);
    };
    for (int64_t e = 0; e < E; ++e) {
        const int32_t q = edge_part[e];
        if (q < 0 || q >= n_parts) return fail(GRF_EINVAL, "edge_part[%lld] = %d out of range", (long long)e, q);
        add(whole->eu[e], q);
        add(whole->ev[e], q);
    }
    PartSpec ps;
    ps.part = part;
    ps.n_parts = n_parts;
    ps.global_n_interior = whole->NI;
    std::vector<int64_t> iface_id(V, -1);
    for (int64_t v = 0; v < V; ++v)
        if (touch[v].size() > 1) iface_id[v] = ps.n_interface++;
    // local edges (ascending global id) and vertices (ascending global id)
    std::vector<int64_t> edges, loc(V, -1);
    for (int64_t e = 0; e < E; ++e)
        if (edge_part[e] == part) edges.push_back(e);
    if (edges.empty()) return fail(GRF_EINVAL, "part %d has no edges", part);
    for (int64_t e : edges) loc[whole->eu[e]] = loc[whole->ev[e]] = 0;
    int64_t nv = 0;
    for (int64_t v = 0; v < V; ++v)
        if (loc[v] == 0) {
            loc[v] = nv++;
            ps.vertex_gid.push_back(v);
        }
    std::vector<int64_t> leu, lev;
    std::vector<double> llen;
    std::vector<int32_t> deg(V, 0);
    for (int64_t e = 0; e < E; ++e) {
        deg[whole->eu[e]]++;
        deg[whole->ev[e]]++;
    }
    for (int64_t e : edges) {
        leu.push_back(loc[whole->eu[e]]);
        lev.push_back(loc[whole->ev[e]]);
        llen.push_back(whole->len[e]);
        ps.edge_goff.push_back(whole->off[e]);
    }
    std::map<int32_t, std::vector<int32_t>> nb;
    for (int64_t i = 0; i < nv; ++i) {
        const int64_t v = ps.vertex_gid[i];
        ps.vertex_mass.push_back(whole->ml[whole->NI + v]);  // the whole graph's vertex mass (noise, P150)
        ps.vertex_degree.push_back(deg[v]);
        ps.vertex_owned.push_back(touch[v].front() == part ? 1 : 0);
        ps.vertex_iface.push_back(iface_id[v]);
        for (int32_t r : touch[v])
            if (r != part) nb[r].push_back((int32_t)i);
    }
    for (auto& kv : nb) {
        ps.nbr_part.push_back(kv.first);
        ps.nbr_verts.push_back(kv.second);
    }
    return create_impl(nv, (int64_t)edges.size(), leu.data(), lev.data(), llen.data(), whole->h, &ps,
                       alloc ? alloc : (whole->alloc.custom ? &whole->alloc.a : nullptr), out);
}

grf_status grf_partition_edges(const grf_graph* g, int32_t n_parts, const double* xy, int32_t* edge_part,
                               int64_t* info) {
    if (!g || !edge_part) return fail(GRF_EINVAL, "NULL argument");
    if (g->partitioned) return fail(GRF_EINVAL, "partition the whole graph, not a part");
    const int64_t E = g->E, V = g->V;
    if (n_parts < 1 || n_parts > E) return fail(GRF_EINVAL, "n_parts must lie in [1, E]");
    // DOF weight of an edge: its n_e elements (m_e interior DOFs + one for its end vertices, P123)
    std::vector<double> w(E);
    for (int64_t e = 0; e < E; ++e) w[e] = (double)g->n_el[e];
    // cut `ids` (in order) into consecutive runs for parts [p0, p0 + np) at equal weight fractions
    auto cut_runs = [&](const std::vector<int64_t>& ids, int32_t p0, int32_t np) {
        double tot = 0.0;
        for (int64_t e : ids) tot += w[e];
        double acc = 0.0;
        int32_t q = 0;
        for (size_t i = 0; i < ids.size(); ++i) {
            // the edge goes to the part whose weight interval holds its weight midpoint
            const double mid = acc + 0.5 * w[ids[i]];
            while (q + 1 < np && mid >= tot * (q + 1) / np) ++q;
            edge_part[ids[i]] = p0 + q;
            acc += w[ids[i]];
        }
    };
    if (xy) {
        // recursive coordinate bisection of the edge midpoints, weighted by n_e:
        // split the longer extent at the weight fraction of the two halves' part counts
        std::vector<double> mx(E), my(E);
        for (int64_t e = 0; e < E; ++e) {
            mx[e] = 0.5 * (xy[2 * g->eu[e]] + xy[2 * g->ev[e]]);
            my[e] = 0.5 * (xy[2 * g->eu[e] + 1] + xy[2 * g->ev[e] + 1]);
        }
        std::vector<int64_t> all(E);
        for (int64_t e = 0; e < E; ++e) all[e] = e;
        std::vector<std::tuple<std::vector<int64_t>, int32_t, int32_t>> work;
        work.emplace_back(std::move(all), 0, n_parts);
        while (!work.empty()) {
            auto [ids, p0, np] = std::move(work.back());
            work.pop_back();
            if (np == 1) {
                for (int64_t e : ids) edge_part[e] = p0;
                continue;
            }
            double x0 = 1e300, x1 = -1e300, y0 = 1e300, y1 = -1e300;
            for (int64_t e : ids) {
                x0 = std::min(x0, mx[e]);
                x1 = std::max(x1, mx[e]);
                y0 = std::min(y0, my[e]);
                y1 = std::max(y1, my[e]);
            }
            const std::vector<double>& c = (x1 - x0 >= y1 - y0) ? mx : my;
            std::stable_sort(ids.begin(), ids.end(), [&](int64_t a, int64_t b) { return c[a] < c[b]; });
            const int32_t nl = np / 2;
            double tot = 0.0;
            for (int64_t e : ids) tot += w[e];
            double acc = 0.0;
            size_t k = 0;
            while (k < ids.size() && acc + 0.5 * w[ids[k]] < tot * nl / np) acc += w[ids[k++]];
            k = std::max<size_t>(1, std::min(k, ids.size() - 1));
            std::vector<int64_t> left(ids.begin(), ids.begin() + k), right(ids.begin() + k, ids.end());
            work.emplace_back(std::move(left), p0, nl);
            work.emplace_back(std::move(right), p0 + nl, np - nl);
        }
    } else {
        // breadth-first edge order (an edge takes the visit rank of its earlier-visited end; each
        // component from its lowest vertex), cut into runs of equal DOF weight
        std::vector<std::vector<int64_t>> adj(V);
        for (int64_t e = 0; e < E; ++e) {
            adj[g->eu[e]].push_back(g->ev[e]);
            adj[g->ev[e]].push_back(g->eu[e]);
        }
        std::vector<int64_t> rank(V, -1), queue;
        int64_t nxt = 0;
        for (int64_t r = 0; r < V; ++r) {
            if (rank[r] >= 0) continue;
            rank[r] = nxt++;
            queue.assign(1, r);
            for (size_t i = 0; i < queue.size(); ++i)
                for (int64_t b : adj[queue[i]])
                    if (rank[b] < 0) {
                        rank[b] = nxt++;
                        queue.push_back(b);
                    }
        }
        std::vector<int64_t> ids(E);
        for (int64_t e = 0; e < E; ++e) ids[e] = e;
        std::stable_sort(ids.begin(), ids.end(), [&](int64_t a, int64_t b) {
            return std::min(rank[g->eu[a]], rank[g->ev[a]]) < std::min(rank[g->eu[b]], rank[g->ev[b]]);
        });
        cut_runs(ids, 0, n_parts);
    }
    if (info) {  // [0] interface vertices, [1] max part weight, [2] min part weight, [3] parts that got no edge
        std::vector<int32_t> first(V, -1);
        std::vector<uint8_t> multi(V, 0);
        std::vector<double> pw(n_parts, 0.0);
        for (int64_t e = 0; e < E; ++e) {
            pw[edge_part[e]] += w[e];
            for (int64_t v : {g->eu[e], g->ev[e]}) {
                if (first[v] < 0) first[v] = edge_part[e];
                else if (first[v] != edge_part[e]) multi[v] = 1;
            }
        }
        int64_t ni = 0, empty_parts = 0;
        for (int64_t v = 0; v < V; ++v) ni += multi[v];
        for (double x : pw) empty_parts += x == 0.0;
        info[0] = ni;
        info[1] = (int64_t)*std::max_element(pw.begin(), pw.end());
        info[2] = (int64_t)*std::min_element(pw.begin(), pw.end());
        info[3] = empty_parts;
    }
    return GRF_OK;
}

grf_status grf_graph_part_dofs(const grf_graph* g, int64_t* gid) {
    if (!g || !gid) return fail(GRF_EINVAL, "NULL argument");
    if (!g->partitioned) {
        for (int64_t i = 0; i < g->N; ++i) gid[i] = i;
        return GRF_OK;
    }
    std::copy(g->dof_gid.begin(), g->dof_gid.end(), gid);
    return GRF_OK;
}

void grf_graph_destroy(grf_graph* g) {
    if (!g) return;
    cudaDeviceSynchronize();
    for (auto& p : g->plans)
        for (auto& b : p->blocks) g->alloc.put(b.p, b.bytes, nullptr);
    for (auto& b : g->blocks) g->alloc.put(b.p, b.bytes, nullptr);
    for (auto& r : g->recs) {
        g->pool.push_back(r.a);
        g->pool.push_back(r.b);
    }
    for (auto e : g->pool) cudaEventDestroy(e);
    delete g;
}

grf_status grf_graph_num_dofs(const grf_graph* g, int64_t* n_dofs, int64_t* n_interior) {
    if (!g) return fail(GRF_EINVAL, "graph is NULL");
    if (n_dofs) *n_dofs = g->N;
    if (n_interior) *n_interior = g->NI;
    return GRF_OK;
}

grf_status grf_graph_edge_layout(const grf_graph* g, int64_t* n_el, double* h_e, int64_t* offset) {
    if (!g) return fail(GRF_EINVAL, "graph is NULL");
    if (n_el) std::copy(g->n_el.begin(), g->n_el.end(), n_el);
    if (h_e) std::copy(g->he.begin(), g->he.end(), h_e);
    if (offset) std::copy(g->off.begin(), g->off.end(), offset);
    return GRF_OK;
}

grf_status grf_graph_lumped_mass(const grf_graph* g, double* ml_host) {
    if (!g || !ml_host) return fail(GRF_EINVAL, "NULL argument");
    std::copy(g->ml.begin(), g->ml.end(), ml_host);
    return GRF_OK;
}

grf_status grf_plan_info(double beta, double k, int64_t* k_minus, int64_t* k_plus, double* c_I, double* c_L) {
    int64_t Km, Kp;
    grf_status st = plan_limits(beta, k, &Km, &Kp);
    if (st) return st;
    if (k_minus) *k_minus = Km;
    if (k_plus) *k_plus = Kp;
    if (c_I || c_L) {
        const int64_t L = Km + Kp + 1;
        std::vector<double> a(L), b(L);
        plan_coefficients(beta, k, Km, 0, L, 1, a.data(), b.data());
        if (c_I) std::copy(a.begin(), a.end(), c_I);
        if (c_L) std::copy(b.begin(), b.end(), c_L);
    }
    return GRF_OK;
}

grf_status grf_workspace_size(const grf_graph* g, double kappa, double beta, double k, int64_t n_samples,
                              const grf_options* opt, size_t* bytes) {
    grf_status st = check_params(g, kappa, beta, k, n_samples);
    if (st) return st;
    if (!bytes) return fail(GRF_EINVAL, "bytes is NULL");
    int64_t Km, Kp, nb, ne, nd;
    plan_limits(beta, k, &Km, &Kp);
    st = resolve_range(opt, Km + Kp + 1, &nb, &ne, &nd);
    if (st) return st;
    *bytes = ws_layout(g, range_count(nb, ne, nd), n_samples, true, use_global_pcg(g, opt),
                       opt && opt->mass == GRF_MASS_CONSISTENT).total;
    return GRF_OK;
}

grf_status grf_noise(grf_graph* g, uint64_t seed, int64_t n_samples, double* W_out, void* stream) {
    if (!g || !W_out) return fail(GRF_EINVAL, "NULL argument");
    if (n_samples < 1) return fail(GRF_EINVAL, "n_samples must be >= 1");
    CUDA_TRY(g->timed(GRF_K_NOISE, (cudaStream_t)stream,
                      [&] { grf::launch_noise(g->dev, seed, n_samples, W_out, (cudaStream_t)stream); }));
    return GRF_OK;
}

grf_status grf_noise_mass(grf_graph* g, uint64_t seed, int64_t n_samples, int32_t mass, double* W_out,
                          void* stream) {
    if (mass == GRF_MASS_LUMPED) return grf_noise(g, seed, n_samples, W_out, stream);
    if (!g || !W_out || n_samples < 1 || mass != GRF_MASS_CONSISTENT) return fail(GRF_EINVAL, "bad arguments");
    grf_status s = ensure_consistent_factor(g);
    if (s) return s;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t bytes = sizeof(double) * (size_t)n_samples * (2 * g->E + g->V);
    double* ev = (double*)g->alloc.get(bytes, st);
    if (!ev) return fail(GRF_ENOMEM, "consistent noise scratch");
    grf::launch_noise_consistent(g->dev, g->cLd, g->cLo, g->cLs, seed, n_samples, W_out, ev,
                                 ev + n_samples * 2 * g->E, st);
    cudaError_t e = cudaStreamSynchronize(st);
    g->alloc.put(ev, bytes, st);
    if (e != cudaSuccess) return fail(GRF_ECUDA, "consistent noise: %s", cudaGetErrorString(e));
    return GRF_OK;
}

grf_status grf_sample(grf_graph* g, double kappa, double beta, double k, uint64_t seed, int64_t n_samples,
                      const grf_options* opt, double* u_out, void* workspace, size_t ws_bytes, void* stream,
                      grf_stats* stats) {
    grf_status st = check_params(g, kappa, beta, k, n_samples);
    if (st) return st;
    if (!u_out) return fail(GRF_EINVAL, "u_out is NULL");
    st = check_kernel_limits(g);
    if (st) return st;
    cudaStream_t s = (cudaStream_t)stream;
    Plan* p = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    st = get_plan(g, kappa, beta, k, opt, s, &p);  // synchronises when it builds the tables (K2)
    const double setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (st) return st;
    st = solve(g, p, n_samples, opt, nullptr, seed, u_out, workspace, ws_bytes, s, stats);
    if (stats) stats->phase_ms[1] = setup_ms;
    return st;
}

grf_status grf_apply(grf_graph* g, double kappa, double beta, double k, int64_t n_rhs, const double* rhs,
                     const grf_options* opt, double* u_out, void* workspace, size_t ws_bytes, void* stream,
                     grf_stats* stats) {
    grf_status st = check_params(g, kappa, beta, k, n_rhs);
    if (st) return st;
    if (!u_out || !rhs) return fail(GRF_EINVAL, "NULL argument");
    st = check_kernel_limits(g);
    if (st) return st;
    cudaStream_t s = (cudaStream_t)stream;
    Plan* p = nullptr;
    st = get_plan(g, kappa, beta, k, opt, s, &p);
    if (st) return st;
    if (rhs == u_out) return fail(GRF_EINVAL, "grf_apply: rhs and u_out must not alias");
    return solve(g, p, n_rhs, opt, rhs, 0, u_out, workspace, ws_bytes, s, stats);
}

grf_status grf_sample_host(grf_graph* g, double kappa, double beta, double k, uint64_t seed, int64_t n_samples,
                           const grf_options* opt, double* u_host, void* stream, grf_stats* stats) {
    grf_status st = check_params(g, kappa, beta, k, n_samples);
    if (st) return st;
    if (!u_host) return fail(GRF_EINVAL, "u_host is NULL");
    cudaStream_t s = (cudaStream_t)stream;
    // Sample chunks, chunk c's device->host copy running on a second stream while chunk c+1 is
    // computed (three device staging buffers in turn).  The copy of the LAST chunk cannot be
    // hidden, and a chunk of fewer samples runs the kernels less efficiently, so the call is cut
    // into chunks of B = max(64, ~n/6) samples followed by a tail of two 32-sample chunks (every
    // chunk >= 17 samples: the same kernel variants as the whole call, so the field is bitwise the
    // one-call field; per-sample arithmetic does not depend on the chunking).  Config 3 (256
    // samples): 64, 64, 64, 32, 32.  Chunk c draws samples [c0, c0 + n_c) with seed + c0, so its
    // noise is that of the same samples in one call (key = seed + sample index, noise.cu).
    std::vector<int64_t> sizes;
    if (n_samples < 64) {
        sizes.push_back(n_samples);
    } else {
        const int64_t B = std::max<int64_t>(64, ((n_samples / 6 + 31) / 32) * 32);
        int64_t rem = n_samples;
        while (rem > B + 64) {
            sizes.push_back(B);
            rem -= B;
        }
        if (rem - 64 >= 32) {
            sizes.push_back(rem - 64);
            sizes.push_back(32);
            sizes.push_back(32);
        } else if (rem - 32 >= 32) {
            sizes.push_back(rem - 32);
            sizes.push_back(32);
        } else {
            sizes.push_back(rem);
        }
    }
    {  // design study: env GRF_HOST_CHUNKS = comma-separated chunk sizes summing to n_samples
        const char* e = getenv("GRF_HOST_CHUNKS");
        if (e && *e) {
            std::vector<int64_t> v;
            int64_t sum = 0;
            for (const char* q = e; *q;) {
                char* end = nullptr;
                const long long x = strtoll(q, &end, 10);
                if (end == q || x <= 0) break;
                v.push_back(x);
                sum += x;
                q = *end == ',' ? end + 1 : end;
                if (*end != ',') break;
            }
            if (sum == n_samples) sizes = v;
        }
    }
    const int64_t n_chunks = (int64_t)sizes.size();
    const int64_t max_chunk = *std::max_element(sizes.begin(), sizes.end());
    const size_t cbytes = (size_t)max_chunk * g->N * sizeof(double);
    // The last chunk writes straight into u_host when that is page-locked memory mapped into the
    // device (cudaHostAlloc / torch pin_memory under unified addressing) and its recovery writes
    // every output value exactly once by plain stores: its kernels then stream the result over
    // PCIe while they run, instead of a device->host copy after them (the copy nothing can hide).
    // Only for calls of one or two chunks: with more, the copy of the chunk before still holds the
    // link while the last chunk's kernels store over it (measured: config 5, two chunks, 24.6 ->
    // 20.6 ms; config 4, one chunk, 605 -> 554 ms; config 3, five chunks, 12.37 -> 12.49 ms).
    // Design-study switch: env GRF_HOST_ZC (0 off, 2 for any chunk count).
    double* u_mapped = nullptr;
    {
        static const int zc_env = [] {
            const char* e = getenv("GRF_HOST_ZC");
            return e ? atoi(e) : 1;
        }();
        cudaPointerAttributes pa{};
        if (zc_env && (n_chunks <= 2 || zc_env == 2) && cudaPointerGetAttributes(&pa, u_host) == cudaSuccess &&
            pa.type == cudaMemoryTypeHost &&
            pa.devicePointer != nullptr) {
            Plan* pl = nullptr;
            if (get_plan(g, kappa, beta, k, opt, s, &pl) == GRF_OK &&
                grf::recover_out_write_only(g->dev, pl->dev, sizes.back()))
                u_mapped = static_cast<double*>(pa.devicePointer);
        }
        cudaGetLastError();  // clear the (non-sticky) error a pointer query may leave behind
    }
    const int64_t n_copied = n_chunks - (u_mapped ? 1 : 0);  // chunks that go through staging
    // one workspace for every chunk (stream-ordered reuse): a call that allocates its own
    // workspace synchronises before returning it, which would stall the host between chunks
    size_t wbytes = 0;
    st = grf_workspace_size(g, kappa, beta, k, max_chunk, opt, &wbytes);
    if (st) return st;
    // NB staging buffers: a chunk never waits for the copy-out of the chunk before last
    constexpr int NB = 3;
    const int nbuf = (int)std::min<int64_t>(NB, n_copied);
    void* du[NB] = {nullptr, nullptr, nullptr};
    bool ok = true;
    for (int b = 0; b < nbuf; ++b) ok = ok && (du[b] = g->alloc.get(cbytes, s)) != nullptr;
    void* wsp = ok ? g->alloc.get(wbytes, s) : nullptr;
    if (!ok || !wsp) {
        for (int b = 0; b < nbuf; ++b)
            if (du[b]) g->alloc.put(du[b], cbytes, s);
        if (wsp) g->alloc.put(wsp, wbytes, s);
        return fail(GRF_ENOMEM, "staging buffers of %d x %zu bytes + a %zu-byte workspace could not be allocated",
                    nbuf, cbytes, wbytes);
    }
    cudaStream_t cs = nullptr;
    cudaEvent_t done[NB] = {nullptr, nullptr, nullptr}, copied[NB] = {nullptr, nullptr, nullptr};
    cudaError_t ce = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    for (int b = 0; b < nbuf && ce == cudaSuccess; ++b) {
        ce = cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming);
        if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&copied[b], cudaEventDisableTiming);
    }
    grf_stats tot{};
    double iter_sum = 0.0;
    bool enoconv = false;
    if (ce != cudaSuccess) st = fail(GRF_ECUDA, "copy stream / events: %s", cudaGetErrorString(ce));
    int64_t c0 = 0;
    for (int64_t c = 0; c < n_chunks && st == GRF_OK; c0 += sizes[c], ++c) {
        const bool direct = u_mapped != nullptr && c == n_chunks - 1;  // written in place, no copy
        const int b = direct ? 0 : (int)(c % nbuf);
        const int64_t nc = sizes[c];
        if (!direct && c >= nbuf) cudaStreamWaitEvent(s, copied[b], 0);  // staging buffer b has been copied out
        grf_stats cst{};
        grf_status sc = grf_sample(g, kappa, beta, k, seed + (uint64_t)c0, nc, opt,
                                   direct ? u_mapped + c0 * g->N : (double*)du[b], wsp, wbytes, s,
                                   stats ? &cst : nullptr);
        if (sc == GRF_ENOCONV) {
            enoconv = true;
        } else if (sc != GRF_OK) {
            st = sc;
            break;
        }
        if (!direct) {
            ce = cudaEventRecord(done[b], s);
            if (ce == cudaSuccess) ce = cudaStreamWaitEvent(cs, done[b], 0);
            if (ce == cudaSuccess)
                ce = cudaMemcpyAsync(u_host + c0 * g->N, du[b], (size_t)nc * g->N * sizeof(double),
                                     cudaMemcpyDeviceToHost, cs);
            if (ce == cudaSuccess) ce = cudaEventRecord(copied[b], cs);
        }
        if (ce != cudaSuccess) st = fail(GRF_ECUDA, "device->host copy: %s", cudaGetErrorString(ce));
        if (stats) {
            if (c == 0) {
                tot = cst;
            } else {
                tot.n_systems += cst.n_systems;
                tot.n_unconverged += cst.n_unconverged;
                tot.iter_min = std::min(tot.iter_min, cst.iter_min);
                tot.iter_max = std::max(tot.iter_max, cst.iter_max);
                tot.worst_rel_residual = std::max(tot.worst_rel_residual, cst.worst_rel_residual);
                tot.gpu_launches += cst.gpu_launches;
                tot.worst_true_rel_residual = std::max(tot.worst_true_rel_residual, cst.worst_true_rel_residual);
                tot.n_nonfinite += cst.n_nonfinite;
                for (int i = 0; i < 5; ++i) tot.phase_ms[i] += cst.phase_ms[i];
            }
            iter_sum += cst.iter_mean * (double)cst.n_systems;
        }
    }
    if (cs) {
        ce = cudaStreamSynchronize(cs);
        if (ce != cudaSuccess && st == GRF_OK) st = fail(GRF_ECUDA, "device->host copy: %s", cudaGetErrorString(ce));
    }
    cudaStreamSynchronize(s);
    for (int b = 0; b < nbuf; ++b) {
        if (done[b]) cudaEventDestroy(done[b]);
        if (copied[b]) cudaEventDestroy(copied[b]);
        if (du[b]) g->alloc.put(du[b], cbytes, s);
    }
    g->alloc.put(wsp, wbytes, s);
    if (cs) cudaStreamDestroy(cs);
    if (stats && st == GRF_OK) {
        tot.iter_mean = tot.n_systems > 0 ? iter_sum / (double)tot.n_systems : 0.0;
        *stats = tot;
    }
    if (st == GRF_OK && enoconv) return GRF_ENOCONV;
    return st;
}

grf_status grf_edge_schur(grf_graph* g, double kappa, double beta, double k, const grf_options* opt,
                          double* sigma_host) {
    grf_status st = check_params(g, kappa, beta, k, 1);
    if (st) return st;
    if (!sigma_host) return fail(GRF_EINVAL, "sigma_host is NULL");
    Plan* p = nullptr;
    st = get_plan(g, kappa, beta, k, opt, nullptr, &p);
    if (st) return st;
    const int64_t n = (int64_t)p->dev.L * g->E;
    std::vector<double> buf(n * 4);
    CUDA_TRY(cudaMemcpy(buf.data(), p->dev.sig, n * 4 * sizeof(double), cudaMemcpyDeviceToHost));
    for (int64_t t = 0; t < n; ++t) {
        sigma_host[2 * t] = buf[4 * t];
        sigma_host[2 * t + 1] = buf[4 * t + 1];
    }
    return GRF_OK;
}

grf_status grf_profile_enable(grf_graph* g, int enable) {
    if (!g) return fail(GRF_EINVAL, "graph is NULL");
    g->prof = enable != 0;
    return GRF_OK;
}

grf_status grf_profile_read(grf_graph* g, double* ms, int64_t* launches) {
    if (!g) return fail(GRF_EINVAL, "graph is NULL");
    double acc[GRF_K_COUNT] = {0};
    int64_t cnt[GRF_K_COUNT] = {0};
    grf_status rc = GRF_OK;
    for (auto& r : g->recs) {
        float t = 0.f;
        cudaError_t e = cudaEventSynchronize(r.b);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&t, r.a, r.b);
        if (e != cudaSuccess && rc == GRF_OK) rc = fail(GRF_ECUDA, "event timing: %s", cudaGetErrorString(e));
        acc[r.kind] += t;
        cnt[r.kind] += 1;
        g->pool.push_back(r.a);
        g->pool.push_back(r.b);
    }
    g->recs.clear();
    for (int k = 0; k < GRF_K_COUNT; ++k) {
        if (ms) ms[k] = acc[k];
        if (launches) launches[k] = cnt[k];
    }
    return rc;
}

// ---------------------------------------------------------------- NCCL (dlopen'ed)
typedef int (*nccl_get_id_fn)(void*);
typedef int (*nccl_init_fn)(void**, int, const void*, int);  // ncclComm_t*, nranks, ncclUniqueId (by value 128B), rank
typedef int (*nccl_reduce_fn)(const void*, void*, size_t, int, int, int, void*, cudaStream_t);
typedef int (*nccl_destroy_fn)(void*);
typedef const char* (*nccl_err_fn)(int);

}  // extern "C"

namespace {
struct NcclApi {
    void* h = nullptr;
    nccl_get_id_fn get_id = nullptr;
    void* init = nullptr;
    nccl_reduce_fn reduce = nullptr;
    nccl_destroy_fn destroy = nullptr;
    nccl_err_fn err = nullptr;
    bool load() {
        if (h) return true;
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* n : names) {
            h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) return false;
        get_id = (nccl_get_id_fn)dlsym(h, "ncclGetUniqueId");
        init = dlsym(h, "ncclCommInitRank");
        reduce = (nccl_reduce_fn)dlsym(h, "ncclReduce");
        destroy = (nccl_destroy_fn)dlsym(h, "ncclCommDestroy");
        err = (nccl_err_fn)dlsym(h, "ncclGetErrorString");
        return get_id && init && reduce && destroy;
    }
};
NcclApi g_nccl;
struct UniqueId {
    char internal[128];
};
typedef int (*nccl_init_real_fn)(void**, int, UniqueId, int);
}  // namespace

struct grf_comm {
    void* comm = nullptr;
    int rank = 0, nranks = 1;
};

extern "C" {

grf_status grf_comm_get_unique_id(void* id128) {
    if (!id128) return fail(GRF_EINVAL, "id is NULL");
    if (!g_nccl.load()) return fail(GRF_ENCCL, "libnccl.so.2 could not be loaded");
    int r = g_nccl.get_id(id128);
    if (r) return fail(GRF_ENCCL, "ncclGetUniqueId: %s", g_nccl.err ? g_nccl.err(r) : "error");
    return GRF_OK;
}

grf_status grf_comm_init(const void* id128, int rank, int nranks, grf_comm** out) {
    if (!id128 || !out || nranks < 1 || rank < 0 || rank >= nranks) return fail(GRF_EINVAL, "bad comm arguments");
    if (!g_nccl.load()) return fail(GRF_ENCCL, "libnccl.so.2 could not be loaded");
    UniqueId uid;
    std::memcpy(uid.internal, id128, 128);
    auto c = std::make_unique<grf_comm>();
    int r = ((nccl_init_real_fn)g_nccl.init)(&c->comm, nranks, uid, rank);
    if (r) return fail(GRF_ENCCL, "ncclCommInitRank: %s", g_nccl.err ? g_nccl.err(r) : "error");
    c->rank = rank;
    c->nranks = nranks;
    *out = c.release();
    return GRF_OK;
}

void grf_comm_destroy(grf_comm* c) {
    if (!c) return;
    if (c->comm && g_nccl.destroy) g_nccl.destroy(c->comm);
    delete c;
}

grf_status grf_reduce_sum(grf_comm* c, const double* send, double* recv, int64_t count, int root, void* stream) {
    if (!c || !send || count < 0 || root < 0 || root >= c->nranks) return fail(GRF_EINVAL, "bad reduce arguments");
    // ncclDouble = 8, ncclSum = 0
    int r = g_nccl.reduce(send, recv, (size_t)count, 8, 0, root, c->comm, (cudaStream_t)stream);
    if (r) return fail(GRF_ENCCL, "ncclReduce: %s", g_nccl.err ? g_nccl.err(r) : "error");
    return GRF_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- edge-partitioned sampling
namespace {
typedef int (*nccl_allreduce_fn)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_p2p_fn)(void*, size_t, int, int, void*, cudaStream_t);  // ncclSend / ncclRecv
typedef int (*nccl_group_fn)();

// sum of a device fp64 buffer over the ranks (in place); ncclDouble = 8, ncclSum = 0
grf_status allreduce_sum(grf_comm* c, double* buf, int64_t n, cudaStream_t st) {
    static nccl_allreduce_fn fn = nullptr;
    if (!fn) fn = (nccl_allreduce_fn)dlsym(g_nccl.h, "ncclAllReduce");
    if (!fn) return fail(GRF_ENCCL, "ncclAllReduce not found");
    int r = fn(buf, buf, (size_t)n, 8, 0, c->comm, st);
    if (r) return fail(GRF_ENCCL, "ncclAllReduce: %s", g_nccl.err ? g_nccl.err(r) : "error");
    return GRF_OK;
}

// per-part device state of one grf_sample_edgepart call
struct PartRun {
    grf_graph* g = nullptr;
    Plan* plan = nullptr;
    std::vector<Block> mem;
    double *W = nullptr, *ends = nullptr, *rhs = nullptr, *uG = nullptr, *relres = nullptr;
    int32_t* iters = nullptr;
    int32_t* counters = nullptr;
    grf::dist::Vecs v{};
    double *dpart = nullptr, *dots = nullptr;
    // neighbour halo: send / recv [n_shared][L][cs] (segments per neighbour, in grf_graph::nbr_part
    // order), the local vertex of every send slot, and per local interface vertex the ordered
    // sources of its sum (-1: own value, else a recv slot)
    std::vector<int64_t> seg;  // [n_nbr + 1] slot offsets of the neighbour segments
    double *send = nullptr, *recv = nullptr;
    int32_t *pidx = nullptr, *cvert = nullptr, *cptr = nullptr, *csrc = nullptr;
    int32_t n_if = 0;
    void* get(size_t bytes, cudaStream_t st) {
        void* p = g->alloc.get(bytes, st);
        if (p) mem.push_back({p, bytes});
        return p;
    }
    template <class T>
    T* put_vec(const std::vector<T>& h, cudaStream_t st) {
        T* d = (T*)get(std::max<size_t>(h.size(), 1) * sizeof(T), st);
        if (d && !h.empty()) cudaMemcpyAsync(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st);
        return d;
    }
    void release(cudaStream_t st) {
        cudaStreamSynchronize(st);
        for (auto& b : mem) g->alloc.put(b.p, b.bytes, st);
        mem.clear();
    }
};

// halo tables of one part from its neighbour lists (grf_graph_create_part): the sum at a shared
// vertex runs over the parts touching it in ascending part order, own value at its own place
void halo_tables(const grf_graph* g, std::vector<int64_t>& seg, std::vector<int32_t>& pidx, std::vector<int32_t>& cvert,
                 std::vector<int32_t>& cptr, std::vector<int32_t>& csrc) {
    const size_t nn = g->nbr_part.size();
    seg.assign(nn + 1, 0);
    for (size_t k = 0; k < nn; ++k) seg[k + 1] = seg[k] + (int64_t)g->nbr_verts[k].size();
    pidx.clear();
    std::map<int32_t, std::vector<std::pair<int32_t, int32_t>>> src;  // local vertex -> (part, recv slot)
    for (size_t k = 0; k < nn; ++k)
        for (size_t i = 0; i < g->nbr_verts[k].size(); ++i) {
            const int32_t v = g->nbr_verts[k][i];
            pidx.push_back(v);
            src[v].push_back({g->nbr_part[k], (int32_t)(seg[k] + i)});
        }
    cvert.clear();
    cptr.assign(1, 0);
    csrc.clear();
    for (auto& kv : src) {
        auto list = kv.second;
        list.push_back({g->part, -1});
        std::sort(list.begin(), list.end());
        cvert.push_back(kv.first);
        for (auto& ps : list) csrc.push_back(ps.second);
        cptr.push_back((int32_t)csrc.size());
    }
}
}  // namespace

extern "C" grf_status grf_sample_edgepart(grf_graph* const* parts, int32_t n_parts, grf_comm* comm, double kappa,
                                          double beta, double k, uint64_t seed, int64_t n_samples,
                                          const grf_options* opt, double* const* u_out, void* stream,
                                          grf_stats* stats) {
    if (!parts || n_parts < 1 || !u_out) return fail(GRF_EINVAL, "grf_sample_edgepart: NULL argument or no parts");
    if (comm && n_parts != 1) return fail(GRF_EINVAL, "with a communicator each rank passes exactly one part");
    if (opt && opt->mass != GRF_MASS_LUMPED)
        return fail(GRF_EUNSUPPORTED, "edge-partitioned sampling uses the lumped mass (the paper's method)");
    cudaStream_t st = (cudaStream_t)stream;
    const int32_t P = comm ? comm->nranks : n_parts;  // parts of the partition
    for (int32_t q = 0; q < n_parts; ++q) {
        grf_status s = check_params(parts[q], kappa, beta, k, n_samples);
        if (s) return s;
        if (!u_out[q]) return fail(GRF_EINVAL, "u_out[%d] is NULL", q);
        const bool part_ok = parts[q]->partitioned ? parts[q]->n_parts == P : P == 1;
        if (!part_ok) return fail(GRF_EINVAL, "part %d does not belong to a partition into %d parts", q, P);
        if (!comm && parts[q]->partitioned && parts[q]->part != q)
            return fail(GRF_EINVAL, "parts must be passed in part order (got part %d at %d)", parts[q]->part, q);
        if (comm && parts[q]->partitioned && parts[q]->part != comm->rank)
            return fail(GRF_EINVAL, "rank %d must pass part %d", comm->rank, comm->rank);
        s = check_kernel_limits(parts[q]);
        if (s) return s;
    }
    const int32_t csl = grf::sample_tile_log2(n_samples);
    const int32_t cs = 1 << csl;
    const int64_t tiles = (n_samples + cs - 1) / cs;
    const int64_t Sp = tiles * cs;
    std::vector<PartRun> R(n_parts);
    grf_status rc = GRF_OK;
    auto cleanup = [&]() {
        for (auto& r : R) r.release(st);
    };
    int32_t L = 0;
    int64_t V_sum = 0;
    for (int32_t q = 0; q < n_parts && !rc; ++q) {
        PartRun& r = R[q];
        r.g = parts[q];
        rc = get_plan(r.g, kappa, beta, k, opt, st, &r.plan);
        if (rc) break;
        L = r.plan->dev.L;
        const int64_t N = r.g->N, V = r.g->V, E = r.g->E;
        V_sum += V;
        const size_t vec = sizeof(double) * (size_t)L * V * cs;
        r.W = (double*)r.get(sizeof(double) * n_samples * N, st);
        r.ends = (double*)r.get(sizeof(double) * Sp * E * 2 * L, st);
        r.rhs = (double*)r.get(sizeof(double) * Sp * V * L, st);
        r.uG = (double*)r.get(sizeof(double) * Sp * V * L, st);
        r.iters = (int32_t*)r.get(sizeof(int32_t) * n_samples * L, st);
        r.relres = (double*)r.get(sizeof(double) * n_samples * L, st);
        r.counters = (int32_t*)r.get(2 * sizeof(int32_t), st);
        double** vv[7] = {&r.v.x, &r.v.r0, &r.v.r1, &r.v.p0, &r.v.p1, &r.v.q, &r.v.z};
        for (auto p : vv) *p = (double*)r.get(vec, st);
        r.dpart = (double*)r.get(sizeof(double) * 2 * L * grf::dist::dot_blocks(r.g->dev) * cs, st);
        r.dots = (double*)r.get(sizeof(double) * 2 * L * cs, st);
        std::vector<int32_t> pidx, cvert, cptr, csrc;
        halo_tables(r.g, r.seg, pidx, cvert, cptr, csrc);
        const int64_t ns = r.seg.back();
        r.n_if = (int32_t)cvert.size();
        r.send = (double*)r.get(sizeof(double) * std::max<int64_t>(ns, 1) * L * cs, st);
        r.recv = (double*)r.get(sizeof(double) * std::max<int64_t>(ns, 1) * L * cs, st);
        r.pidx = r.put_vec(pidx, st);
        r.cvert = r.put_vec(cvert, st);
        r.cptr = r.put_vec(cptr, st);
        r.csrc = r.put_vec(csrc, st);
        for (auto& b : r.mem)
            if (!b.p) rc = fail(GRF_ENOMEM, "edge-partitioned workspace could not be allocated");
        if (!r.W || !r.ends || !r.rhs || !r.uG || !r.iters || !r.relres || !r.counters || !r.v.x || !r.v.r0 ||
            !r.v.r1 || !r.v.p0 || !r.v.p1 || !r.v.q || !r.v.z || !r.dpart || !r.dots || !r.send || !r.recv ||
            !r.pidx || !r.cvert || !r.cptr || !r.csrc)
            rc = fail(GRF_ENOMEM, "edge-partitioned workspace could not be allocated");
    }
    // shared (all-part) state: summed dots and the system scalars, on part 0's allocator
    PartRun& R0 = R[0];
    const int32_t nsys = L * cs;
    double* dsum = nullptr;
    double** ptrs = nullptr;
    int32_t* flag_host = nullptr;  // pinned: the device's count of unconverged systems, polled
    grf::dist::Scal sc{};
    if (!rc) {
        dsum = (double*)R0.get(sizeof(double) * 2 * nsys, st);
        ptrs = (double**)R0.get(sizeof(double*) * n_parts, st);
        double** sd[5] = {&sc.alpha, &sc.beta, &sc.rz, &sc.gg, &sc.rr};
        for (auto p : sd) *p = (double*)R0.get(sizeof(double) * nsys, st);
        sc.done = (int32_t*)R0.get(sizeof(int32_t) * nsys, st);
        sc.its = (int32_t*)R0.get(sizeof(int32_t) * nsys, st);
        sc.active = (int32_t*)R0.get(sizeof(int32_t), st);
        if (cudaHostAlloc((void**)&flag_host, 2 * sizeof(int32_t), cudaHostAllocDefault) != cudaSuccess) flag_host = nullptr;
        if (!dsum || !ptrs || !sc.alpha || !sc.beta || !sc.rz || !sc.gg || !sc.rr || !sc.done || !sc.its ||
            !sc.active || !flag_host)
            rc = fail(GRF_ENOMEM, "edge-partitioned workspace could not be allocated");
    }
    cudaEvent_t polled[2] = {nullptr, nullptr};
    for (auto& e : polled)
        if (!rc && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
            rc = fail(GRF_ECUDA, "event creation failed");
    auto finish_all = [&]() {
        cleanup();
        for (auto e : polled)
            if (e) cudaEventDestroy(e);
        if (flag_host) cudaFreeHost(flag_host);
    };
    if (rc) {
        finish_all();
        return rc;
    }
    {  // device array of the parts' dot buffers for the in-process sums
        std::vector<double*> hp(n_parts);
        for (int32_t q = 0; q < n_parts; ++q) hp[q] = R[q].dots;
        cudaMemcpyAsync(ptrs, hp.data(), sizeof(double*) * hp.size(), cudaMemcpyHostToDevice, st);
        cudaStreamSynchronize(st);  // the host vector dies here
    }
    const int32_t pc = opt ? opt->precond : GRF_PRECOND_NN;
    const double rtol = opt ? opt->rtol : 1e-13;
    const int32_t max_iter = (opt && opt->max_iter > 0) ? opt->max_iter : (int32_t)(V_sum + 10);
    static nccl_p2p_fn nsend = nullptr, nrecv = nullptr;
    static nccl_group_fn gstart = nullptr, gend = nullptr;
    if (comm && !nsend) {
        nsend = (nccl_p2p_fn)dlsym(g_nccl.h, "ncclSend");
        nrecv = (nccl_p2p_fn)dlsym(g_nccl.h, "ncclRecv");
        gstart = (nccl_group_fn)dlsym(g_nccl.h, "ncclGroupStart");
        gend = (nccl_group_fn)dlsym(g_nccl.h, "ncclGroupEnd");
    }
    if (comm && (!nsend || !nrecv || !gstart || !gend)) {
        finish_all();
        return fail(GRF_ENCCL, "ncclSend/ncclRecv/ncclGroup* not found");
    }

    // halo of vector X (per part): every shared vertex gets the sum of the parts' values, in part
    // order.  Each part packs the shared vertices per neighbour; the segments travel to the
    // neighbours (NCCL send/recv pairs across ranks, device copies between in-process parts);
    // each part then combines its own and the received values.
    auto halo = [&](auto getX) -> grf_status {
        for (auto& r : R) grf::dist::halo_pack(r.g->dev, L, cs, r.seg.back(), r.pidx, getX(r), r.send, st);
        const size_t row = sizeof(double) * (size_t)L * cs;
        if (comm) {
            PartRun& r = R0;
            if (!r.g->nbr_part.empty()) {
                int e = gstart();
                for (size_t kk = 0; kk < r.g->nbr_part.size() && !e; ++kk) {
                    const size_t cnt = (size_t)(r.seg[kk + 1] - r.seg[kk]) * L * cs;
                    e = nsend(r.send + r.seg[kk] * L * cs, cnt, 8, r.g->nbr_part[kk], comm->comm, st);
                    if (!e) e = nrecv(r.recv + r.seg[kk] * L * cs, cnt, 8, r.g->nbr_part[kk], comm->comm, st);
                }
                int e2 = gend();
                if (e || e2) return fail(GRF_ENCCL, "halo send/recv: %s", g_nccl.err ? g_nccl.err(e ? e : e2) : "error");
            }
        } else {
            for (int32_t q = 0; q < n_parts; ++q) {
                const grf_graph* gq = R[q].g;
                for (size_t kk = 0; kk < gq->nbr_part.size(); ++kk) {  // q's segment for r -> r's segment for q
                    const int32_t rr = gq->nbr_part[kk];
                    const grf_graph* gr = R[rr].g;
                    const size_t back = std::find(gr->nbr_part.begin(), gr->nbr_part.end(), q) - gr->nbr_part.begin();
                    CUDA_TRY(cudaMemcpyAsync(R[rr].recv + R[rr].seg[back] * L * cs, R[q].send + R[q].seg[kk] * L * cs,
                                             (size_t)(R[q].seg[kk + 1] - R[q].seg[kk]) * row, cudaMemcpyDeviceToDevice,
                                             st));
                }
            }
        }
        for (auto& r : R)
            grf::dist::halo_combine(r.g->dev, L, cs, r.n_if, r.cvert, r.cptr, r.csrc, r.recv, getX(r), st);
        return GRF_OK;
    };
    // dot products (owned vertices) summed over parts into dsum [K][nsys]
    auto dotsum = [&](int K, auto a0, auto b0, auto a1, auto b1) -> grf_status {
        for (int32_t q = 0; q < n_parts; ++q)
            grf::dist::dots(R[q].g->dev, L, cs, K, a0(R[q]), b0(R[q]), a1(R[q]), b1(R[q]), R[q].dpart, R[q].dots, st);
        if (comm) {
            grf_status s = allreduce_sum(comm, R0.dots, (int64_t)K * nsys, st);
            if (s) return s;
            CUDA_TRY(cudaMemcpyAsync(dsum, R0.dots, sizeof(double) * K * nsys, cudaMemcpyDeviceToDevice, st));
        } else {
            grf::dist::sum_parts(n_parts, ptrs, (int64_t)K * nsys, dsum, st);
        }
        return GRF_OK;
    };

    // kernels launched (per-call count for grf_stats) and the profiling brackets (grf_profile_*)
    int64_t nlaunch = 0;
    grf_graph* gp = R0.g;  // the bracket events go to the first part's profile
    cudaEvent_t pcg_a = nullptr;
    // stage 1 (per part, no communication): noise, condensation, partial condensed rhs
    for (auto& r : R) {
        CUDA_TRY(gp->timed(GRF_K_NOISE, st, [&] { grf::launch_noise(r.g->dev, seed, n_samples, r.W, st); }));
        cudaError_t le = cudaSuccess;
        CUDA_TRY(gp->timed(GRF_K_CONDENSE, st, [&] {
            le = grf::launch_condense(r.g->dev, r.plan->dev, n_samples, r.W, r.ends, r.counters, st);
        }));
        CUDA_TRY(le);
        grf::launch_assemble_rhs(r.g->dev, r.plan->dev, n_samples, r.W, r.ends, r.rhs, st);
        nlaunch += 3;
    }
    if (gp->prof) {  // the whole distributed PCG (every tile, halos and collectives) as one record
        pcg_a = gp->new_event();
        cudaEventRecord(pcg_a, st);
    }
    // stage 2: distributed NN-PCG per sample tile.  The iterations are enqueued without host
    // round trips: every POLL iterations the device's count of unconverged systems is copied to
    // pinned memory and the copy of the PREVIOUS chunk is inspected, so the host never waits for
    // the GPU to drain; iterations enqueued after convergence do no work (converged systems have
    // alpha = beta = 0 and every system is masked once the count reaches 0).
    constexpr int32_t POLL = 8;
    for (int64_t tile = 0; tile < tiles && !rc; ++tile) {
        for (auto& r : R) grf::dist::init(r.g->dev, L, n_samples, csl, tile, r.rhs, r.v, st);
        rc = halo([](PartRun& r) { return r.v.r0; });  // g = W_G + sum over ALL parts' edges
        if (rc) break;
        for (auto& r : R) grf::dist::precond(r.g->dev, r.plan->dev, pc, cs, r.v.r0, r.v.z, st);
        rc = halo([](PartRun& r) { return r.v.z; });
        if (rc) break;
        rc = dotsum(2, [](PartRun& r) { return (const double*)r.v.r0; }, [](PartRun& r) { return (const double*)r.v.r0; },
                    [](PartRun& r) { return (const double*)r.v.r0; }, [](PartRun& r) { return (const double*)r.v.z; });
        if (rc) break;
        CUDA_TRY(cudaMemsetAsync(sc.active, 0, sizeof(int32_t), st));
        grf::dist::scal_init(nsys, cs, n_samples, tile, csl, dsum, sc, st);
        bool flip = false;  // which of the double-buffered p / r is current
        int64_t chunk = 0;
        int64_t ran = 0;  // iterations enqueued
        for (int32_t it = 0; it < max_iter; ++it) {
            ran = it + 1;
            for (auto& r : R) {
                double* po = flip ? r.v.p1 : r.v.p0;
                double* pn = flip ? r.v.p0 : r.v.p1;
                grf::dist::spmv(r.g->dev, r.plan->dev, cs, sc.beta, r.v.z, po, pn, r.v.q, st);
            }
            rc = halo([](PartRun& r) { return r.v.q; });
            if (rc) break;
            rc = dotsum(1, [&](PartRun& r) { return (const double*)(flip ? r.v.p0 : r.v.p1); },
                        [](PartRun& r) { return (const double*)r.v.q; }, [](PartRun&) { return (const double*)nullptr; },
                        [](PartRun&) { return (const double*)nullptr; });
            if (rc) break;
            grf::dist::scal_alpha(nsys, dsum, sc, st);
            for (auto& r : R) {
                double* pn = flip ? r.v.p0 : r.v.p1;
                double* ro = flip ? r.v.r1 : r.v.r0;
                double* rn = flip ? r.v.r0 : r.v.r1;
                grf::dist::update(r.g->dev, r.plan->dev, pc, cs, sc.alpha, r.v.q, pn, ro, rn, r.v.x, r.v.z, st);
            }
            rc = halo([](PartRun& r) { return r.v.z; });
            if (rc) break;
            rc = dotsum(2, [&](PartRun& r) { return (const double*)(flip ? r.v.r0 : r.v.r1); },
                        [&](PartRun& r) { return (const double*)(flip ? r.v.r0 : r.v.r1); },
                        [&](PartRun& r) { return (const double*)(flip ? r.v.r0 : r.v.r1); },
                        [](PartRun& r) { return (const double*)r.v.z; });
            if (rc) break;
            grf::dist::scal_beta(nsys, rtol * rtol, dsum, sc, st);
            flip = !flip;
            if ((it + 1) % POLL == 0) {
                const int slot = (int)(chunk & 1);
                if (chunk >= 1) {  // the previous chunk's count: the GPU is a chunk ahead of this check
                    CUDA_TRY(cudaEventSynchronize(polled[slot ^ 1]));
                    if (flag_host[slot ^ 1] == 0) break;
                }
                CUDA_TRY(cudaMemcpyAsync(&flag_host[slot], sc.active, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
                CUDA_TRY(cudaEventRecord(polled[slot], st));
                ++chunk;
            }
        }
        if (rc) break;
        for (auto& r : R) grf::dist::finish(r.g->dev, L, n_samples, csl, tile, r.v.x, sc, r.uG, r.iters, r.relres, st);
        // per iteration and part: spmv, update, 2 x (halo pack + combine), 3 dot kernels x 2, plus 2 scalars
        nlaunch += ran * (n_parts * 12 + 2) + n_parts * 9 + 2;
    }
    if (pcg_a) {
        cudaEvent_t pcg_b = gp->new_event();
        cudaEventRecord(pcg_b, st);
        gp->recs.push_back({GRF_K_PCG, pcg_a, pcg_b});
    }
    // stage 3 (per part): recovery of the interiors and the vertex values
    for (int32_t q = 0; q < n_parts && !rc; ++q) {
        PartRun& r = R[q];
        cudaError_t e = cudaSuccess;
        cudaError_t te = gp->timed(GRF_K_RECOVER, st, [&] {
            e = grf::launch_recover(r.g->dev, r.plan->dev, n_samples, r.W, u_out[q], r.uG, r.counters + 1, st);
            if (e == cudaSuccess) e = grf::launch_vertex_sum(r.g->dev, r.plan->dev, n_samples, r.uG, u_out[q], st);
        });
        if (e == cudaSuccess) e = te;
        nlaunch += 2;
        if (e != cudaSuccess) rc = fail(GRF_ECUDA, "edge-partitioned recovery: %s", cudaGetErrorString(e));
    }
    if (!rc) {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) rc = fail(GRF_ECUDA, "edge-partitioned launch: %s", cudaGetErrorString(e));
    }
    if (!rc && stats) {
        std::vector<int32_t> its((size_t)n_samples * L);
        std::vector<double> rr((size_t)n_samples * L);
        CUDA_TRY(cudaMemcpyAsync(its.data(), R0.iters, its.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(rr.data(), R0.relres, rr.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        std::memset(stats, 0, sizeof(*stats));
        stats->n_nodes = L;
        stats->k_minus = R0.plan->Km;
        stats->k_plus = R0.plan->Kp;
        stats->n_systems = n_samples * L;
        stats->iter_min = *std::min_element(its.begin(), its.end());
        stats->iter_max = *std::max_element(its.begin(), its.end());
        double sum = 0.0, worst = 0.0;
        int64_t bad = 0;
        for (size_t i = 0; i < its.size(); ++i) {
            sum += its[i];
            worst = std::max(worst, rr[i]);
            if (!(rr[i] <= rtol)) ++bad;
        }
        stats->iter_mean = sum / its.size();
        stats->worst_rel_residual = worst;
        stats->n_unconverged = bad;
        stats->gpu_launches = nlaunch;
        stats->worst_true_rel_residual = -1.0;  // not computed for edge-partitioned solves
        if (bad) rc = fail(GRF_ENOCONV, "%lld PCG systems missed rtol %g", (long long)bad, rtol);
    }
    finish_all();
    return rc;
}

// ---------------------------------------------------------------- nested-mesh transfer (strong-error study)
namespace {
grf_status check_nested(const grf_graph* c, const grf_graph* f) {
    if (!c || !f) return fail(GRF_EINVAL, "graph is NULL");
    if (c->V != f->V || c->E != f->E || c->partitioned || f->partitioned)
        return fail(GRF_EINVAL, "meshes of different (or partitioned) graphs");
    for (int64_t e = 0; e < c->E; ++e) {
        if (c->eu[e] != f->eu[e] || c->ev[e] != f->ev[e] || std::memcmp(&c->len[e], &f->len[e], sizeof(double)))
            return fail(GRF_EINVAL, "edge %lld differs between the two graphs", (long long)e);
        if (f->n_el[e] % c->n_el[e])
            return fail(GRF_EINVAL, "edge %lld: fine n_e = %lld is not a multiple of coarse n_e = %lld (not nested)",
                        (long long)e, (long long)f->n_el[e], (long long)c->n_el[e]);
    }
    return GRF_OK;
}
}  // namespace

extern "C" grf_status grf_prolong(const grf_graph* coarse, const grf_graph* fine, int64_t n, const double* u_coarse,
                                  double* u_fine, void* stream) {
    grf_status s = check_nested(coarse, fine);
    if (s) return s;
    if (n < 1 || !u_coarse || !u_fine) return fail(GRF_EINVAL, "bad prolongation arguments");
    grf::launch_prolong(coarse->dev, fine->dev, fine->dev.dof_edge, n, u_coarse, u_fine, (cudaStream_t)stream);
    CUDA_TRY(cudaGetLastError());
    return GRF_OK;
}

extern "C" grf_status grf_project_noise(const grf_graph* fine, const grf_graph* coarse, int64_t n, const double* W_fine,
                                        double* W_coarse, void* stream) {
    grf_status s = check_nested(coarse, fine);
    if (s) return s;
    if (n < 1 || !W_fine || !W_coarse) return fail(GRF_EINVAL, "bad projection arguments");
    grf::launch_project(coarse->dev, fine->dev, coarse->dev.dof_edge, n, W_fine, W_coarse, (cudaStream_t)stream);
    CUDA_TRY(cudaGetLastError());
    return GRF_OK;
}

extern "C" grf_status grf_mnorm_sq_diff(grf_graph* g, int64_t n, const double* a, const double* b, double* out,
                                        void* stream) {
    if (!g || n < 1 || !a || !b || !out) return fail(GRF_EINVAL, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t bytes = sizeof(double) * (size_t)n * grf::MNORM_PARTS;
    void* part = g->alloc.get(bytes, st);
    if (!part) return fail(GRF_ENOMEM, "partial buffer");
    grf::launch_mnorm_sq_diff(g->dev, n, a, b, (double*)part, out, st);
    cudaError_t e = cudaStreamSynchronize(st);
    g->alloc.put(part, bytes, st);
    if (e != cudaSuccess) return fail(GRF_ECUDA, "mnorm: %s", cudaGetErrorString(e));
    return GRF_OK;
}

// ---------------------------------------------------------------- sample-then-node sharded sampling
namespace {
int64_t split_lo(int64_t n, int64_t parts, int64_t i) {
    const int64_t base = n / parts, extra = n % parts;
    return i * base + std::min(i, extra);
}
}  // namespace

extern "C" grf_status grf_dist_shard(int32_t world, int32_t rank, int64_t n_samples, int64_t n_nodes, int64_t* out) {
    if (!out || world < 1 || rank < 0 || rank >= world || n_samples < 1 || n_nodes < 1)
        return fail(GRF_EINVAL, "bad shard arguments");
    const int64_t ps = std::min<int64_t>(world, n_samples);
    const int64_t pl = std::max<int64_t>(1, std::min<int64_t>(world / ps, n_nodes));
    const bool active = rank < ps * pl;
    const int64_t gi = active ? rank / pl : 0, li = active ? rank % pl : 0;
    out[0] = active ? split_lo(n_samples, ps, gi) : 0;
    out[1] = active ? split_lo(n_samples, ps, gi + 1) : 0;
    out[2] = active ? li : 0;             // round-robin node shard: nodes li, li + P_l, ... < n_nodes
    out[3] = active ? n_nodes : 0;
    out[4] = gi * pl;                       // root rank of the sample range
    out[5] = (active ? 1 : 0) | ((active && li == 0) ? 2 : 0) | (pl << 2);  // active, is_root, P_l (= node stride)
    return GRF_OK;
}

namespace {
// max of an int32 over all ranks of the communicator (every rank must call it)
grf_status allreduce_max_i32(grf_comm* c, int32_t* dev_buf, int32_t* host_val, cudaStream_t st) {
    static nccl_allreduce_fn fn = nullptr;
    if (!fn) fn = (nccl_allreduce_fn)dlsym(g_nccl.h, "ncclAllReduce");
    if (!fn) return fail(GRF_ENCCL, "ncclAllReduce not found");
    CUDA_TRY(cudaMemcpyAsync(dev_buf, host_val, sizeof(int32_t), cudaMemcpyHostToDevice, st));
    int r = fn(dev_buf, dev_buf, 1, 2 /* ncclInt32 */, 2 /* ncclMax */, c->comm, st);
    if (r) return fail(GRF_ENCCL, "ncclAllReduce: %s", g_nccl.err ? g_nccl.err(r) : "error");
    CUDA_TRY(cudaMemcpyAsync(host_val, dev_buf, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return GRF_OK;
}
}  // namespace

extern "C" grf_status grf_sample_dist(grf_graph* g, grf_comm* comm, double kappa, double beta, double k,
                                      uint64_t seed, int64_t n_samples, const grf_options* opt, double* u_out,
                                      int64_t* range_out, void* stream, grf_stats* stats) {
    // With node shards (P_l > 1) every rank of the communicator -- active or not -- takes part in
    // one status agreement (an int32 max allreduce) after its local work, so that a rank whose
    // local call failed cannot leave its peers blocked in the partial-sum exchange: on any failure
    // every rank returns (GRF_ENCCL "a peer failed" on the others) before a single partial is
    // sent.  Pure sample shards (P_l = 1) exchange nothing and stay asynchronous.
    if (!g || !comm || !range_out) return fail(GRF_EINVAL, "NULL argument");
    grf_status st = check_params(g, kappa, beta, k, n_samples);
    if (st) return st;  // identical arguments on every rank: every rank fails here alike
    int64_t Km, Kp;
    st = plan_limits(beta, k, &Km, &Kp);
    if (st) return st;
    int64_t L = Km + Kp + 1;
    if (opt && (opt->node_begin != 0 || opt->node_end >= 0 || opt->node_stride > 1))
        return fail(GRF_EINVAL, "grf_sample_dist shards the whole node range; leave the node range default");
    int64_t sh[6];
    st = grf_dist_shard(comm->nranks, comm->rank, n_samples, L, sh);
    if (st) return st;
    for (int i = 0; i < 6; ++i) range_out[i] = sh[i];
    const bool active = sh[5] & 1;
    const int64_t pl = sh[5] >> 2;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t s0 = sh[0], ns = sh[1] - sh[0];
    grf_status local = GRF_OK;
    if (active) {
        if (!u_out) {
            local = fail(GRF_EINVAL, "u_out is NULL");
        } else {
            grf_options o;
            grf_options_default(&o);
            if (opt) o = *opt;
            o.node_begin = sh[2];
            o.node_end = sh[3];
            o.node_stride = pl;
            local = grf_sample(g, kappa, beta, k, seed + (uint64_t)s0, ns, &o, u_out, nullptr, 0, s, stats);
        }
    }
    const std::string local_msg = g_err;
    if (pl > 1) {  // only node shards exchange data; P_l is the same on every rank
        int32_t* flag = (int32_t*)g->alloc.get(sizeof(int32_t), s);
        if (!flag) return fail(GRF_ENOMEM, "status buffer");  // (a peer then blocks: allocation of 8 B failed)
        int32_t worst = (local == GRF_OK || local == GRF_ENOCONV) ? 0 : 1;
        grf_status ar = allreduce_max_i32(comm, flag, &worst, s);
        g->alloc.put(flag, sizeof(int32_t), s);
        if (ar) return ar;
        if (local != GRF_OK && local != GRF_ENOCONV) return fail(local, "%s", local_msg.c_str());
        if (worst) return fail(GRF_ENCCL, "grf_sample_dist: a peer rank's local sampling failed");
    } else if (local != GRF_OK && local != GRF_ENOCONV) {
        return local;
    }
    if (active && pl > 1) {
        // the P_l node shards of this sample range: a binomial tree over the range's ranks (fixed
        // pairing, so the partial sums are added in the same order on every call): in round d
        // (d = 1, 2, 4, ...) shard li with li % 2d == d sends its running sum to li - d, which adds it
        static nccl_p2p_fn send = nullptr, recv = nullptr;
        if (!send) {
            send = (nccl_p2p_fn)dlsym(g_nccl.h, "ncclSend");
            recv = (nccl_p2p_fn)dlsym(g_nccl.h, "ncclRecv");
        }
        if (!send || !recv) return fail(GRF_ENCCL, "ncclSend/ncclRecv not found");
        const size_t count = (size_t)ns * g->N;
        const int64_t root = sh[4], li = comm->rank - root;
        double* tmp = nullptr;
        grf_status rc = GRF_OK;
        for (int64_t d = 1; d < pl && rc == GRF_OK; d <<= 1) {
            if (li % (2 * d) == d) {
                int e = send(u_out, count, 8, (int)(root + li - d), comm->comm, s);
                if (e) rc = fail(GRF_ENCCL, "ncclSend: %s", g_nccl.err ? g_nccl.err(e) : "error");
                break;  // this shard's sum has been handed on
            }
            if (li % (2 * d) == 0 && li + d < pl) {
                if (!tmp) tmp = (double*)g->alloc.get(count * sizeof(double), s);
                if (!tmp) {
                    rc = fail(GRF_ENOMEM, "reduce buffer of %zu bytes", count * sizeof(double));
                    break;
                }
                int e = recv(tmp, count, 8, (int)(root + li + d), comm->comm, s);
                if (e) {
                    rc = fail(GRF_ENCCL, "ncclRecv: %s", g_nccl.err ? g_nccl.err(e) : "error");
                    break;
                }
                grf::launch_add(u_out, tmp, (int64_t)count, s);
            }
        }
        if (tmp) {
            cudaStreamSynchronize(s);
            g->alloc.put(tmp, count * sizeof(double), s);
        }
        if (rc) return rc;
    }
    CUDA_TRY(cudaGetLastError());
    return local;
}
