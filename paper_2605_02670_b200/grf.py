"""Thin Python binding of libgrf.so (include/grf.h) -- argument marshalling only.

PyTorch provides device memory (its caching allocator is handed to the library
as the grf_allocator), streams and process groups; every step of the sampler runs
in the library's CUDA kernels.  Names follow the C ABI:

    g = Graph(n_vertices, edge_u, edge_v, length, h)            # grf_graph_create
    u = g.sample(kappa, beta, k, seed=0, n_samples=1)            # grf_sample  -> cuda fp64 [S, N]
    W = g.noise(seed, n_samples)                                 # grf_noise
    x = g.apply(kappa, beta, k, rhs)                             # grf_apply
    S = g.edge_schur(kappa, beta, k)                             # grf_edge_schur (stage check)
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Tuple

import numpy as np

from ._lib import (ALLOC_FN, FREE_FN, GRF_ENOCONV, GRF_OK, GrfError, check, grf_allocator, grf_options,
                   grf_stats, load)

PRECOND = {"nn": 0, "neumann-neumann": 0, "jacobi": 1, "none": 2}


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2605_02670_b200 needs a CUDA device (B200); there is no CPU fallback")
    return torch


def _stream_ptr(stream) -> Optional[int]:
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def plan_info(beta: float, k: float):
    """(K^-, K^+, c_I[L], c_L[L]) of the sinc plan (P60-67, P335), via grf_plan_info."""
    lib = load()
    km, kp = C.c_int64(), C.c_int64()
    check(lib.grf_plan_info(beta, k, C.byref(km), C.byref(kp), None, None))
    L = km.value + kp.value + 1
    cI = np.empty(L)
    cL = np.empty(L)
    check(lib.grf_plan_info(beta, k, C.byref(km), C.byref(kp), cI.ctypes.data_as(C.POINTER(C.c_double)),
                            cL.ctypes.data_as(C.POINTER(C.c_double))))
    return km.value, kp.value, cI, cL


PCG_VARIANT = {"auto": 0, "shared": 1, "global": 2}


MASS = {"lumped": 0, "consistent": 1}


def make_options(rtol=1e-13, max_iter=0, precond="nn", node_range=None, pcg="auto", mass="lumped",
                 node_stride=1) -> grf_options:
    o = grf_options()
    load().grf_options_default(C.byref(o))
    o.rtol = rtol
    o.max_iter = max_iter
    o.precond = PRECOND[precond] if isinstance(precond, str) else int(precond)
    if node_range is not None:
        o.node_begin, o.node_end = int(node_range[0]), int(node_range[1])
    o.node_stride = int(node_stride)
    o.pcg_variant = PCG_VARIANT[pcg] if isinstance(pcg, str) else int(pcg)
    o.mass = MASS[mass] if isinstance(mass, str) else int(mass)
    return o


class Graph:
    """A metric graph + its P1 mesh, resident on the current CUDA device."""

    def __init__(self, n_vertices, edge_u, edge_v, length, h, use_torch_allocator: bool = True, _part=None):
        torch = _torch()
        lib = load()
        self._lib = lib
        self.device = torch.cuda.current_device()
        self.h = float(h)
        self._alloc = None
        if use_torch_allocator:
            dev = self.device

            def _a(nbytes, ctx, stream):
                try:
                    return torch.cuda.caching_allocator_alloc(int(nbytes), dev, int(stream or 0) or None)
                except Exception:
                    return None

            cad = torch.cuda.caching_allocator_delete  # bound now: module globals may be gone at exit

            def _f(ptr, nbytes, ctx, stream):
                try:
                    cad(int(ptr))
                except Exception:  # interpreter shutdown: the process is releasing the device anyway
                    pass

            self._cb = (ALLOC_FN(_a), FREE_FN(_f))
            self._alloc = grf_allocator(self._cb[0], self._cb[1], None)
        h_ = C.c_void_p()
        pi64 = C.POINTER(C.c_int64)
        alloc = C.byref(self._alloc) if self._alloc is not None else None
        self.part = None
        if _part is None:
            eu = np.ascontiguousarray(edge_u, dtype=np.int64)
            ev = np.ascontiguousarray(edge_v, dtype=np.int64)
            ln = np.ascontiguousarray(length, dtype=np.float64)
            self.n_vertices = int(n_vertices)
            self.n_edges = int(len(eu))
            check(lib.grf_graph_create(self.n_vertices, self.n_edges, eu.ctypes.data_as(pi64),
                                       ev.ctypes.data_as(pi64), ln.ctypes.data_as(C.POINTER(C.c_double)), self.h,
                                       alloc, C.byref(h_)))
        else:  # part q of an edge partition of a whole graph: grf_graph_create_part
            whole, edge_part, n_parts, q = _part
            ep = np.ascontiguousarray(edge_part, dtype=np.int32)
            if ep.shape != (whole.n_edges,):
                raise ValueError("edge_part needs one entry per edge of the whole graph")
            check(lib.grf_graph_create_part(whole._h, ep.ctypes.data_as(C.POINTER(C.c_int32)), int(n_parts), int(q),
                                            alloc, C.byref(h_)))
            self.part = (int(q), int(n_parts))
            self._whole = whole  # the part borrows nothing, but keep creation order for teardown
        self._h = h_
        n, ni = C.c_int64(), C.c_int64()
        check(lib.grf_graph_num_dofs(self._h, C.byref(n), C.byref(ni)))
        self.n_dofs = n.value
        self.n_interior = ni.value
        if _part is not None:
            self.n_edges = int(np.count_nonzero(ep == q))
            self.n_vertices = self.n_dofs - self.n_interior

    @classmethod
    def from_metric_graph(cls, g, h, **kw):
        return cls(g.n_vertices, g.edge_u, g.edge_v, g.length, h, **kw)

    @classmethod
    def part_of(cls, whole: "Graph", edge_part, n_parts: int, q: int, **kw):
        """Part q of an edge partition of `whole` (grf_graph_create_part: the library derives the
        local mesh, global DOF ids, whole-graph vertex masses / degrees, ownership and halo lists)."""
        return cls(0, None, None, None, whole.h, _part=(whole, edge_part, n_parts, q), **kw)

    def partition(self, n_parts: int, xy=None):
        """grf_partition_edges: (edge_part [E] int32, info dict).  xy: vertex coordinates [V, 2] for
        recursive coordinate bisection, else breadth-first runs of equal DOF weight."""
        ep = np.empty(self.n_edges, dtype=np.int32)
        info = np.zeros(4, dtype=np.int64)
        pxy = None
        if xy is not None:
            xy = np.ascontiguousarray(xy, dtype=np.float64)
            pxy = xy.ctypes.data_as(C.POINTER(C.c_double))
        check(self._lib.grf_partition_edges(self._h, int(n_parts), pxy, ep.ctypes.data_as(C.POINTER(C.c_int32)),
                                            info.ctypes.data_as(C.POINTER(C.c_int64))))
        return ep, {"n_interface": int(info[0]), "max_part_weight": int(info[1]), "min_part_weight": int(info[2]),
                    "empty_parts": int(info[3])}

    def part_dofs(self) -> np.ndarray:
        """Global DOF index of every local DOF (grf_graph_part_dofs; the identity for a whole graph)."""
        out = np.empty(self.n_dofs, dtype=np.int64)
        check(self._lib.grf_graph_part_dofs(self._h, out.ctypes.data_as(C.POINTER(C.c_int64))))
        return out

    # ------------------------------------------------------------------ queries
    def edge_layout(self):
        n_el = np.empty(self.n_edges, dtype=np.int64)
        he = np.empty(self.n_edges)
        off = np.empty(self.n_edges, dtype=np.int64)
        check(self._lib.grf_graph_edge_layout(self._h, n_el.ctypes.data_as(C.POINTER(C.c_int64)),
                                              he.ctypes.data_as(C.POINTER(C.c_double)),
                                              off.ctypes.data_as(C.POINTER(C.c_int64))))
        return n_el, he, off

    def lumped_mass(self):
        ml = np.empty(self.n_dofs)
        check(self._lib.grf_graph_lumped_mass(self._h, ml.ctypes.data_as(C.POINTER(C.c_double))))
        return ml

    def workspace_size(self, kappa, beta, k, n_samples, **opts) -> int:
        o = make_options(**opts)
        b = C.c_size_t()
        check(self._lib.grf_workspace_size(self._h, kappa, beta, k, n_samples, C.byref(o), C.byref(b)))
        return b.value

    # ------------------------------------------------------------------ compute
    def noise(self, seed: int, n_samples: int, out=None, stream=None, mass="lumped"):
        """grf_noise (lumped, sqrt(M_L) xi) or grf_noise_mass (mass="consistent": R xi, M = R R^T)."""
        torch = _torch()
        if out is None:
            out = torch.empty((n_samples, self.n_dofs), dtype=torch.float64, device=f"cuda:{self.device}")
        self._check_out(out, n_samples)
        if mass == "lumped":
            check(self._lib.grf_noise(self._h, C.c_uint64(seed & (2 ** 64 - 1)), n_samples,
                                      C.c_void_p(out.data_ptr()), C.c_void_p(_stream_ptr(stream))))
        else:
            check(self._lib.grf_noise_mass(self._h, C.c_uint64(seed & (2 ** 64 - 1)), n_samples, MASS[mass],
                                           C.c_void_p(out.data_ptr()), C.c_void_p(_stream_ptr(stream))))
        return out

    def _check_out(self, out, n):
        torch = _torch()
        if out.dtype != torch.float64 or not out.is_cuda or not out.is_contiguous() or out.numel() != n * self.n_dofs:
            raise ValueError(f"out must be a contiguous cuda float64 tensor with {n}x{self.n_dofs} elements")

    def sample(self, kappa, beta, k, seed=0, n_samples=1, out=None, workspace=None, stream=None,
               return_stats=False, strict=True, **opts):
        """GRF samples u [n_samples, N] (cuda fp64).  opts: rtol, max_iter, precond, node_range,
        pcg ("auto" | "shared" | "global": the K4 kernel family)."""
        torch = _torch()
        o = make_options(**opts)
        if out is None:
            out = torch.empty((n_samples, self.n_dofs), dtype=torch.float64, device=f"cuda:{self.device}")
        self._check_out(out, n_samples)
        ws_ptr, ws_bytes = self._workspace(workspace, kappa, beta, k, n_samples, o)
        st = grf_stats() if return_stats else None
        rc = self._lib.grf_sample(self._h, kappa, beta, k, C.c_uint64(seed & (2 ** 64 - 1)), n_samples, C.byref(o),
                                  C.c_void_p(out.data_ptr()), ws_ptr, ws_bytes, C.c_void_p(_stream_ptr(stream)),
                                  C.byref(st) if st is not None else None)
        self._keep = workspace
        if rc == GRF_ENOCONV and not strict:
            pass
        else:
            check(rc)
        return (out, st.as_dict()) if return_stats else out

    def sample_host(self, kappa, beta, k, seed=0, n_samples=1, stream=None, return_stats=False, **opts):
        """grf_sample_host: the e2e call -- device staging + D2H copy + sync inside."""
        o = make_options(**opts)
        out = np.empty((n_samples, self.n_dofs))
        st = grf_stats() if return_stats else None
        check(self._lib.grf_sample_host(self._h, kappa, beta, k, C.c_uint64(seed & (2 ** 64 - 1)), n_samples,
                                        C.byref(o), C.c_void_p(out.ctypes.data), C.c_void_p(_stream_ptr(stream)),
                                        C.byref(st) if st is not None else None))
        return (out, st.as_dict()) if return_stats else out

    def sample_into_host(self, kappa, beta, k, seed, n_samples, host_out, stream=None, **opts):
        """grf_sample_host into a caller (e.g. pinned) host buffer; returns host_out."""
        torch = _torch()
        if (host_out.is_cuda or host_out.dtype != torch.float64 or not host_out.is_contiguous()
                or host_out.numel() != n_samples * self.n_dofs):
            raise ValueError(f"host_out must be a contiguous CPU float64 tensor with {n_samples}x{self.n_dofs} "
                             "elements (pinned memory lets the copies overlap)")
        o = make_options(**opts)
        check(self._lib.grf_sample_host(self._h, kappa, beta, k, C.c_uint64(seed & (2 ** 64 - 1)), n_samples,
                                        C.byref(o), C.c_void_p(host_out.data_ptr()), C.c_void_p(_stream_ptr(stream)),
                                        None))
        return host_out

    def apply(self, kappa, beta, k, rhs, out=None, workspace=None, stream=None, return_stats=False, **opts):
        torch = _torch()
        o = make_options(**opts)
        rhs = rhs.contiguous()
        n = rhs.shape[0] if rhs.dim() == 2 else 1
        if out is None:
            out = torch.empty((n, self.n_dofs), dtype=torch.float64, device=rhs.device)
        self._check_out(rhs, n)
        self._check_out(out, n)
        ws_ptr, ws_bytes = self._workspace(workspace, kappa, beta, k, n, o)
        st = grf_stats() if return_stats else None
        check(self._lib.grf_apply(self._h, kappa, beta, k, n, C.c_void_p(rhs.data_ptr()), C.byref(o),
                                  C.c_void_p(out.data_ptr()), ws_ptr, ws_bytes, C.c_void_p(_stream_ptr(stream)),
                                  C.byref(st) if st is not None else None))
        self._keep = workspace
        return (out, st.as_dict()) if return_stats else out

    def edge_schur(self, kappa, beta, k, **opts):
        """Local Schur blocks (s_d, s_o) per (node, edge): numpy [L, E, 2] (grf_edge_schur)."""
        o = make_options(**opts)
        km, kp, _, _ = plan_info(beta, k)
        L = km + kp + 1
        nb = o.node_begin
        ne = L if o.node_end < 0 else o.node_end
        nd = max(1, o.node_stride)
        buf = np.empty(((ne - nb + nd - 1) // nd, self.n_edges, 2))
        check(self._lib.grf_edge_schur(self._h, kappa, beta, k, C.byref(o), buf.ctypes.data_as(C.POINTER(C.c_double))))
        return buf

    def _workspace(self, workspace, kappa, beta, k, n, o):
        torch = _torch()
        b = C.c_size_t()
        check(self._lib.grf_workspace_size(self._h, kappa, beta, k, n, C.byref(o), C.byref(b)))
        if workspace is None:
            workspace = torch.empty(b.value, dtype=torch.uint8, device=f"cuda:{self.device}")
            self._ws_tmp = workspace
        if workspace.numel() * workspace.element_size() < b.value:
            raise ValueError(f"workspace needs {b.value} bytes")
        return C.c_void_p(workspace.data_ptr()), C.c_size_t(workspace.numel() * workspace.element_size())

    def profile(self, enable: bool = True):
        """Bracket every kernel launch with CUDA events (grf_profile_enable)."""
        check(self._lib.grf_profile_enable(self._h, 1 if enable else 0))

    def profile_read(self):
        """{kernel: (total_ms, launches)} since the last read (synchronises the recorded events)."""
        from ._lib import KERNEL_NAMES
        ms = np.zeros(len(KERNEL_NAMES))
        n = np.zeros(len(KERNEL_NAMES), dtype=np.int64)
        check(self._lib.grf_profile_read(self._h, ms.ctypes.data_as(C.POINTER(C.c_double)),
                                         n.ctypes.data_as(C.POINTER(C.c_int64))))
        return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(KERNEL_NAMES)}

    def close(self):
        if getattr(self, "_h", None):
            self._lib.grf_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def version() -> str:
    return load().grf_version().decode()


def sample_edgepart(graphs, kappa, beta, k, seed=0, n_samples=1, comm=None, stream=None, return_stats=False,
                    **opts):
    """grf_sample_edgepart: the field on every part's local DOFs (list of cuda fp64 [S, N_q]).

    graphs: the parts (Graph.from_part) held by this process -- all of them (comm=None, the
    halo / dot sums run on the device in fixed order) or this rank's one part with an NCCL
    communicator (comm: an object with a ``handle`` attribute from grf_comm_init)."""
    torch = _torch()
    lib = load()
    o = make_options(**opts)
    outs = [torch.empty((n_samples, g.n_dofs), dtype=torch.float64, device=f"cuda:{g.device}") for g in graphs]
    hs = (C.c_void_p * len(graphs))(*[g._h.value for g in graphs])
    us = (C.c_void_p * len(graphs))(*[u.data_ptr() for u in outs])
    st = grf_stats() if return_stats else None
    check(lib.grf_sample_edgepart(hs, len(graphs), comm.handle if comm is not None else None, kappa, beta, k,
                                  C.c_uint64(seed & (2 ** 64 - 1)), n_samples, C.byref(o), us,
                                  C.c_void_p(_stream_ptr(stream)), C.byref(st) if st is not None else None))
    return (outs, st.as_dict()) if return_stats else outs


class Comm:
    """grf_comm: an NCCL communicator of the library for one rank (one process per GPU).

    The 128-byte NCCL unique id is made on rank 0 and broadcast with a torch.distributed
    process group (any backend); the library then talks NCCL directly on its streams."""

    def __init__(self, group=None):
        import torch.distributed as dist
        _torch()
        lib = load()
        self._lib = lib
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        uid = (C.c_char * 128)()
        if self.rank == 0:
            check(lib.grf_comm_get_unique_id(uid))
        box = [bytes(uid.raw) if self.rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=group)
        uid = (C.c_char * 128).from_buffer_copy(box[0])
        h = C.c_void_p()
        check(lib.grf_comm_init(uid, self.rank, self.world, C.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            self._lib.grf_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dist_shard(world: int, rank: int, n_samples: int, n_nodes: int):
    """grf_dist_shard: (sample_range, node_range, root, active, is_root, ranks_per_range)."""
    out = (C.c_int64 * 6)()
    check(load().grf_dist_shard(world, rank, n_samples, n_nodes, out))
    f = out[5]
    return (out[0], out[1]), (out[2], out[3]), out[4], bool(f & 1), bool(f & 2), f >> 2


def sample_dist(graph: "Graph", comm: "Comm", kappa, beta, k, seed=0, n_samples=1, stream=None, out=None,
                return_stats=False, **opts):
    """grf_sample_dist (sample-then-node sharding in the library, NCCL reduce of node shards):
    returns (u or None, sample_range, is_root[, stats]); u is the rank's [n_local, N] result (the
    full field of its sample range on the range's root).  Every rank of the communicator calls it."""
    torch = _torch()
    o = make_options(**opts)
    km, kp, _, _ = plan_info(beta, k)
    (s0, s1), _, _, active, is_root, _ = dist_shard(comm.world, comm.rank, n_samples, km + kp + 1)
    u = None
    if active:
        u = out if out is not None else torch.empty((s1 - s0, graph.n_dofs), dtype=torch.float64,
                                                    device=f"cuda:{graph.device}")
        graph._check_out(u, s1 - s0)
    rng = (C.c_int64 * 6)()
    st = grf_stats() if return_stats else None
    rc = load().grf_sample_dist(graph._h, comm.handle, kappa, beta, k, C.c_uint64(seed & (2 ** 64 - 1)), n_samples,
                                C.byref(o), C.c_void_p(u.data_ptr() if u is not None else 0), rng,
                                C.c_void_p(_stream_ptr(stream)), C.byref(st) if st is not None else None)
    check(rc)
    res = (u if active else None, (s0, s1) if active else (0, 0), bool(is_root and active))
    return res + (st.as_dict(),) if return_stats else res
