"""B200-native ORCA steering step (arXiv 2008.11578) behind the reference's
public simulation API. See DESIGN.md / INTEGRATION.md.

Importing the package does not touch the GPU; the first call into
`engine` / `lp` loads liborca_b200.so and fails loudly if it (or a CUDA device)
is missing -- there is no CPU fallback.
"""

from .types import (AgentClass, ClassParams, FrameLog, FrameMetrics, ResponsibilityMatrix,
                    RunResult, RunSummary, ScenarioConfig, SimState)
from .engine import Simulation, desired_velocity, init_state, problem_seed, run, step
from .scenario import (Region, ScenarioError, build_agents, load_scenario, read_trajectories,
                       scenario_from_dict, write_metrics_summary, write_trajectories)
from .crossings import crossing_config, four_way_dict, two_way_dict
from .lp import (HalfPlaneConstraint, LpBatch, LpProblem, LpResult, LpStatus, shuffle_order,
                 solve_batch, solve_closest_point, solve_least_penetration, solve_range)
from .orca import AgentState, VoExit, build_orca_halfplane, compute_vo_exit, gather_constraints
from .grid import UniformGrid, query_neighbors, rebuild
from .scenario import sample_spawns
from .benchmark import BenchReport, BenchRow, run_bench, write_bench_report

__all__ = ["AgentClass", "ClassParams", "FrameMetrics", "ResponsibilityMatrix",
           "ScenarioConfig", "SimState", "Simulation", "desired_velocity", "init_state",
           "problem_seed", "run", "step", "FrameLog", "RunResult", "RunSummary", "HalfPlaneConstraint", "LpBatch", "LpProblem", "LpResult",
           "LpStatus", "shuffle_order", "solve_batch", "solve_closest_point", "solve_range",
           "Region", "ScenarioError", "build_agents", "load_scenario", "read_trajectories",
           "scenario_from_dict", "write_metrics_summary", "write_trajectories", "crossing_config",
           "four_way_dict", "two_way_dict", "solve_least_penetration", "AgentState", "VoExit",
           "build_orca_halfplane", "compute_vo_exit", "gather_constraints", "UniformGrid", "query_neighbors",
           "rebuild", "sample_spawns", "BenchReport", "BenchRow", "run_bench", "write_bench_report"]
