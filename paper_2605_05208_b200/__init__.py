"""B200-native (sm_100a) batched local search of MDFIHA-ETGA (arxiv 2605.05208).

Drop-in for the reference package `mdroute`'s local-search path:

    batch.SolutionCache / evaluate_candidates / leader_and_followers
    moves.enumerate_candidates
    localsearch.local_search (+ local_search_population, the batched form)

Everything on that path runs in hand-written CUDA kernels for sm_100a behind
the C-ABI of include/mdr_sm100.h (libmdr_sm100.so); there is no CPU fallback.
"""
from .model import INF, Instance, Node, Route, Solution, Variant
from .evaluation import LAMBDA_MAX, LAMBDA_MIN, PenaltyState, ScalingConstants, adapt_penalties
from .neighborhood import NeighborConfig, NeighborLists, build as build_neighbors, build_device as build_neighbors_device
from .moves import (ALL_OPS, MODE_ARRIVE, MODE_BOTH, MODE_DEPART, CandidateSet, Move, Op, RoutePlan,
                    SolutionIndex, enumerate_candidates, move_plan)
from .batch import DeltaArrays, SolutionCache, evaluate_candidates, leader_and_followers
from .localsearch import (DeviceSearch, SearchConfig, apply_moves, enabled_operators, evaluate_batch,
                          local_search, local_search_population, select_moves)
from .genetic import InsertionOperator, initial_solution, initial_solutions, repair_insert, repair_population
from .formats import ParseError, parse_instance, read_solution, write_solution
from .engine import RunStats, SolverConfig, run, run_batched, run_islands
from .evaluation import EvalBreakdown, RouteAttr, evaluate
from .feasibility import FeasibilityReport, check_feasible, minimal_duration, simulate_route

__all__ = [
    "INF", "Instance", "Node", "Route", "Solution", "Variant", "LAMBDA_MAX", "LAMBDA_MIN", "PenaltyState",
    "ScalingConstants", "adapt_penalties", "NeighborConfig", "NeighborLists", "build_neighbors", "build_neighbors_device", "ALL_OPS",
    "MODE_ARRIVE", "MODE_BOTH", "MODE_DEPART", "CandidateSet", "Move", "Op", "RoutePlan", "SolutionIndex",
    "enumerate_candidates", "move_plan", "DeltaArrays", "SolutionCache", "evaluate_candidates",
    "leader_and_followers", "DeviceSearch", "SearchConfig", "apply_moves", "enabled_operators",
    "evaluate_batch", "local_search", "local_search_population", "select_moves",
    "InsertionOperator", "initial_solution", "initial_solutions", "repair_insert", "repair_population",
    "ParseError", "parse_instance", "read_solution", "write_solution",
    "RunStats", "SolverConfig", "run", "run_batched", "run_islands",
    "EvalBreakdown", "RouteAttr", "evaluate", "FeasibilityReport", "check_feasible", "minimal_duration",
    "simulate_route",
]
