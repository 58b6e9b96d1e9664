"""B200-native enhanced discrete PSO solve path (arXiv 1706.04399).

Drop-in for the reference's DPSO solve call (``inspectour.solver``):
``DiscreteSwarmSolver``, ``SolveReport``, ``solve_matrix``; plus the device
versions of the helpers the reference's baselines and tests use.
"""
from .solver import DiscreteSwarmSolver, SolveReport, solve_matrix
from .islands import IslandSolver
from .kernels import (best_exchange_batch, nearest_neighbor_tour,
                      nearest_neighbor_two_opt, tour_cost_batch)
from .graph import (TourGraph, build_cost_matrix, build_graph,
                    load_cost_matrix, load_cost_matrix_device,
                    save_cost_matrix, shortest_path, tour_legs)

__version__ = "0.1.0"

__all__ = [
    "DiscreteSwarmSolver", "SolveReport", "solve_matrix", "IslandSolver",
    "best_exchange_batch", "nearest_neighbor_tour",
    "nearest_neighbor_two_opt", "tour_cost_batch",
    "TourGraph", "build_cost_matrix", "build_graph",
    "load_cost_matrix", "load_cost_matrix_device", "save_cost_matrix",
    "shortest_path", "tour_legs",
]
