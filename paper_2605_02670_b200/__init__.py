"""B200-native fractional-SPDE Gaussian random fields on metric graphs (arxiv 2605.02670).

The hot path (noise -> Thomas condensation -> vertex NN-PCG -> Thomas recovery ->
quadrature sum) lives in libgrf.so (csrc/, CUDA sm_100a); this package is its thin
ctypes binding.  See include/grf.h and DESIGN.md.
"""
from .grf import Comm, Graph, make_options, plan_info, sample_edgepart, version  # noqa: F401
from ._lib import GrfError, LIB_PATH, EXPORTS, load  # noqa: F401
