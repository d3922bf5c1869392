"""ctypes loader for libgrf.so (the C ABI of include/grf.h).

The product path has no fallback: if the library is missing or fails to load this
module raises, and every call into it goes through the CUDA kernels.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GRF_LIB") or os.path.join(HERE, "lib", "libgrf.so")  # GRF_LIB: experiments only

GRF_OK, GRF_EINVAL, GRF_ENOMEM, GRF_ECUDA, GRF_ENCCL, GRF_ENOCONV, GRF_EUNSUPPORTED = range(7)
STATUS_NAMES = {0: "GRF_OK", 1: "GRF_EINVAL", 2: "GRF_ENOMEM", 3: "GRF_ECUDA", 4: "GRF_ENCCL",
                5: "GRF_ENOCONV", 6: "GRF_EUNSUPPORTED"}

ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)


class grf_allocator(C.Structure):
    _fields_ = [("alloc", ALLOC_FN), ("free", FREE_FN), ("ctx", C.c_void_p)]


class grf_options(C.Structure):
    _fields_ = [("rtol", C.c_double), ("max_iter", C.c_int32), ("precond", C.c_int32),
                ("node_begin", C.c_int64), ("node_end", C.c_int64), ("pcg_variant", C.c_int32),
                ("mass", C.c_int32), ("node_stride", C.c_int64)]


class grf_stats(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("k_minus", C.c_int64), ("k_plus", C.c_int64),
                ("n_systems", C.c_int64), ("n_unconverged", C.c_int64), ("iter_min", C.c_int32),
                ("iter_max", C.c_int32), ("iter_mean", C.c_double), ("worst_rel_residual", C.c_double),
                ("gpu_launches", C.c_int64), ("worst_true_rel_residual", C.c_double), ("n_nonfinite", C.c_int64),
                ("phase_ms", C.c_double * 5)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["phase_ms"] = dict(zip(("noise", "edge_setup", "condense", "pcg", "recover"), list(self.phase_ms)))
        return d


EXPORTS = [
    "grf_last_error", "grf_version", "grf_options_default", "grf_graph_create", "grf_graph_destroy",
    "grf_graph_num_dofs", "grf_graph_edge_layout", "grf_graph_lumped_mass", "grf_plan_info",
    "grf_workspace_size", "grf_noise", "grf_sample", "grf_sample_host", "grf_apply", "grf_edge_schur",
    "grf_comm_get_unique_id", "grf_comm_init", "grf_comm_destroy", "grf_reduce_sum",
    "grf_profile_enable", "grf_profile_read", "grf_graph_create_part", "grf_sample_edgepart",
    "grf_prolong", "grf_project_noise", "grf_mnorm_sq_diff", "grf_noise_mass", "grf_dist_shard",
    "grf_sample_dist", "grf_partition_edges", "grf_graph_part_dofs",
]
KERNEL_NAMES = ["noise", "edge_setup", "condense", "pcg", "recover"]

_lib = None


class GrfError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2605_02670_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, I64, D, U64, SZ = C.c_void_p, C.c_int64, C.c_double, C.c_uint64, C.c_size_t
    pi64 = C.POINTER(C.c_int64)
    pd = C.POINTER(C.c_double)
    sig = {
        "grf_last_error": (C.c_char_p, []),
        "grf_version": (C.c_char_p, []),
        "grf_options_default": (None, [C.POINTER(grf_options)]),
        "grf_graph_create": (C.c_int, [I64, I64, pi64, pi64, pd, D, C.POINTER(grf_allocator), C.POINTER(P)]),
        "grf_graph_destroy": (None, [P]),
        "grf_graph_num_dofs": (C.c_int, [P, pi64, pi64]),
        "grf_graph_edge_layout": (C.c_int, [P, pi64, pd, pi64]),
        "grf_graph_lumped_mass": (C.c_int, [P, pd]),
        "grf_plan_info": (C.c_int, [D, D, pi64, pi64, pd, pd]),
        "grf_workspace_size": (C.c_int, [P, D, D, D, I64, C.POINTER(grf_options), C.POINTER(SZ)]),
        "grf_noise": (C.c_int, [P, U64, I64, P, P]),
        "grf_sample": (C.c_int, [P, D, D, D, U64, I64, C.POINTER(grf_options), P, P, SZ, P, C.POINTER(grf_stats)]),
        "grf_sample_host": (C.c_int, [P, D, D, D, U64, I64, C.POINTER(grf_options), P, P, C.POINTER(grf_stats)]),
        "grf_apply": (C.c_int, [P, D, D, D, I64, P, C.POINTER(grf_options), P, P, SZ, P, C.POINTER(grf_stats)]),
        "grf_edge_schur": (C.c_int, [P, D, D, D, C.POINTER(grf_options), pd]),
        "grf_comm_get_unique_id": (C.c_int, [P]),
        "grf_comm_init": (C.c_int, [P, C.c_int, C.c_int, C.POINTER(P)]),
        "grf_comm_destroy": (None, [P]),
        "grf_reduce_sum": (C.c_int, [P, P, P, I64, C.c_int, P]),
        "grf_profile_enable": (C.c_int, [P, C.c_int]),
        "grf_graph_create_part": (C.c_int, [P, C.POINTER(C.c_int32), C.c_int32, C.c_int32,
                                            C.POINTER(grf_allocator), C.POINTER(P)]),
        "grf_partition_edges": (C.c_int, [P, C.c_int32, pd, C.POINTER(C.c_int32), pi64]),
        "grf_graph_part_dofs": (C.c_int, [P, pi64]),
        "grf_prolong": (C.c_int, [P, P, I64, P, P, P]),
        "grf_noise_mass": (C.c_int, [P, U64, I64, C.c_int32, P, P]),
        "grf_dist_shard": (C.c_int, [C.c_int32, C.c_int32, I64, I64, pi64]),
        "grf_sample_dist": (C.c_int, [P, P, D, D, D, U64, I64, C.POINTER(grf_options), P, pi64, P,
                                      C.POINTER(grf_stats)]),
        "grf_project_noise": (C.c_int, [P, P, I64, P, P, P]),
        "grf_mnorm_sq_diff": (C.c_int, [P, I64, P, P, P, P]),
        "grf_sample_edgepart": (C.c_int, [C.POINTER(P), C.c_int32, P, D, D, D, U64, I64, C.POINTER(grf_options),
                                          C.POINTER(P), P, C.POINTER(grf_stats)]),
        "grf_profile_read": (C.c_int, [P, pd, pi64]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(status: int) -> int:
    if status not in (GRF_OK,):
        raise GrfError(status, load().grf_last_error().decode())
    return status
