"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This package holds NONE of the method's arithmetic (no mesh, no FEM, no
quadrature, no noise): it only builds metric graphs (vertex count, edge
endpoint lists, edge lengths) from fixed seeds, plus the text file format of
SPEC.md S79.  Both the CPU oracle (`oracle/`) and the CUDA path
(`paper_2605_02670_b200`) consume its output; neither side imports the other.
"""
from .graphs import (  # noqa: F401
    MetricGraph,
    tadpole,
    lattice,
    star_of_lattices,
    rgg_knn,
    barabasi_albert,
    single_edge,
    path_graph,
    triangle_pendant,
    load_graph,
    save_graph,
    config_graph,
    CONFIGS,
)
