"""Seeded synthetic inputs shared by the oracle tests and the GPU harness.

Holds no arithmetic of the method (SURVEY.md §8(d) input recipe only)."""
from .graphs import (CONFIGS, config_graph, edges_to_csr, largest_component, grid2d, grid3d, rgg,
                     sbm, chung_lu, path_graph, cycle_graph, star_graph, complete_graph, random_tree,
                     erdos_renyi, n_edges, random_csr)
from .layout import init_layout, uniform_layout, clustered_layout, random_state

__all__ = [
    "CONFIGS", "config_graph", "edges_to_csr", "largest_component", "grid2d", "grid3d", "rgg", "sbm",
    "chung_lu", "path_graph", "cycle_graph", "star_graph", "complete_graph", "random_tree",
    "erdos_renyi", "n_edges", "random_csr", "init_layout", "uniform_layout", "clustered_layout", "random_state",
]
