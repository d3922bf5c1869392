"""Strong-error refinement study on the GPU (§4.1, P332-335).

For nested meshes h = 2^-j of one graph: draw the noise on the overkill mesh, solve there
(grf_apply), project the noise down (grf_project_noise, P^T), solve on each coarse mesh,
upsample (grf_prolong, P) and take the squared L2(Gamma) error with the overkill lumped mass
(grf_mnorm_sq_diff); err(h) = mean over realizations (P335).  Every array step runs in the
library's kernels; the rate fit ln err = c + r ln h on the handful of (h, err) pairs is host
arithmetic.  Theory (P334, Bolin et al.): err ~ h^(2(2 beta - 1/2)) for the mean square, i.e.
the RMS error decays at rate 2 beta - 1/2.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, load
from .grf import Graph, _stream_ptr, _torch


def project_noise(fine: Graph, coarse: Graph, W_fine):
    torch = _torch()
    n = W_fine.shape[0]
    out = torch.empty((n, coarse.n_dofs), dtype=torch.float64, device=W_fine.device)
    check(load().grf_project_noise(fine._h, coarse._h, n, C.c_void_p(W_fine.data_ptr()), C.c_void_p(out.data_ptr()),
                                   C.c_void_p(_stream_ptr(None))))
    return out


def prolong(coarse: Graph, fine: Graph, u_coarse):
    torch = _torch()
    n = u_coarse.shape[0]
    out = torch.empty((n, fine.n_dofs), dtype=torch.float64, device=u_coarse.device)
    check(load().grf_prolong(coarse._h, fine._h, n, C.c_void_p(u_coarse.data_ptr()), C.c_void_p(out.data_ptr()),
                             C.c_void_p(_stream_ptr(None))))
    return out


def mnorm_sq_diff(g: Graph, a, b):
    torch = _torch()
    n = a.shape[0]
    out = torch.empty(n, dtype=torch.float64, device=a.device)
    check(load().grf_mnorm_sq_diff(g._h, n, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()),
                                   C.c_void_p(out.data_ptr()), C.c_void_p(_stream_ptr(None))))
    return out


def fit_rate(h, err):
    x, y = np.log(np.asarray(h, float)), np.log(np.asarray(err, float))
    r = ((x - x.mean()) * (y - y.mean())).sum() / ((x - x.mean()) ** 2).sum()
    return float(r), float(y.mean() - r * x.mean())


def strong_error(graph, levels, ok_level, kappa, beta, k, seed=0, n_samples=64, batch=64, **opts):
    """Per coarse level: h, mean squared error, RMS error; plus the fitted rates."""
    torch = _torch()
    Gf = Graph.from_metric_graph(graph, 2.0 ** -ok_level)
    coarse = [Graph.from_metric_graph(graph, 2.0 ** -j) for j in levels]
    sq = {j: [] for j in levels}
    for s0 in range(0, n_samples, batch):
        nb = min(batch, n_samples - s0)
        Wf = Gf.noise(seed + s0, nb)
        u_ok = Gf.apply(kappa, beta, k, Wf, **opts)
        for j, Gc in zip(levels, coarse):
            uc = Gc.apply(kappa, beta, k, project_noise(Gf, Gc, Wf), **opts)
            sq[j].append(mnorm_sq_diff(Gf, u_ok, prolong(Gc, Gf, uc)).cpu().numpy())
            del uc
        del Wf, u_ok
        torch.cuda.empty_cache()
    h = [2.0 ** -j for j in levels]
    ms = [float(np.concatenate(sq[j]).mean()) for j in levels]
    rate_ms, _ = fit_rate(h, ms)
    return {"levels": list(levels), "ok_level": ok_level, "h": h, "mean_sq_err": ms,
            "rms_err": [float(np.sqrt(m)) for m in ms], "rate_mean_sq": rate_ms, "rate_rms": rate_ms / 2,
            "theory_rate_rms": 2 * beta - 0.5, "n_samples": n_samples, "per_sample_sq": {j: np.concatenate(sq[j]) for j in levels}}


def covariance(g: Graph, kappa, beta, k, batch=4096, **opts):
    """Covariance matrix C = B M_L B of the discrete field u = B W, Cov(W) = M_L (P99-109),
    B = sum_l (A^{(l)})^{-1} (symmetric): B is applied to the identity columns with batched
    grf_apply (the sampler's own kernels); the dense products are cuBLAS GEMMs (torch)."""
    torch = _torch()
    N = g.n_dofs
    dev = f"cuda:{g.device}"
    B = torch.empty((N, N), dtype=torch.float64, device=dev)
    for c0 in range(0, N, batch):
        nb = min(batch, N - c0)
        E = torch.zeros((nb, N), dtype=torch.float64, device=dev)
        E[torch.arange(nb), torch.arange(c0, c0 + nb)] = 1.0
        g.apply(kappa, beta, k, E, out=B[c0:c0 + nb], **opts)
    M = torch.from_numpy(g.lumped_mass()).to(dev)
    return B @ (M[:, None] * B)


def covariance_error(graph, levels, ok_level, kappa, beta, k, **opts):
    """L2(Gamma x Gamma) covariance errors ||C_ok - P C_h P^T||, the norm with the overkill lumped
    mass on both factors (P337-338; overkill h = 2^-8), and the
    fitted rate (theory min(4 beta - 1/2, 2))."""
    torch = _torch()
    Gf = Graph.from_metric_graph(graph, 2.0 ** -ok_level)
    Cok = covariance(Gf, kappa, beta, k, **opts)
    Mf = torch.from_numpy(Gf.lumped_mass()).to(Cok.device)
    errs = []
    for j in levels:
        Gc = Graph.from_metric_graph(graph, 2.0 ** -j)
        Cc = covariance(Gc, kappa, beta, k, **opts)
        Nc = Gc.n_dofs
        Pt = prolong(Gc, Gf, torch.eye(Nc, dtype=torch.float64, device=Cok.device))  # row i = P e_i -> P^T
        D = Cok - Pt.T @ Cc @ Pt
        errs.append(float(torch.sqrt(((Mf[:, None] * D * D) * Mf[None, :]).sum()).item()))
    h = [2.0 ** -j for j in levels]
    r, _ = fit_rate(h, errs)
    return {"levels": list(levels), "ok_level": ok_level, "h": h, "cov_err": errs, "rate": r,
            "theory_rate": min(4 * beta - 0.5, 2.0)}
