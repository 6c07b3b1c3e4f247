"""Shared helpers for the parity tests (test infrastructure)."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2008_11578_b200.types import (AgentClass, ResponsibilityMatrix,  # noqa: E402
                                         ScenarioConfig, SimState)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name)) as z:
        return {k: z[k] for k in z.files}


def state_from_frame_fixture(g):
    """(SimState, ScenarioConfig) from a tests/golden/frame_*.npz fixture."""
    f64 = lambda a: np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
    st = SimState(frame=int(g["frame"]), time=float(g["frame"]) * float(g["dt"]),
                  ids=g["ids"].astype(np.int64), positions=f64(g["positions"]),
                  velocities=f64(g["velocities"]), radii=f64(g["radii"]),
                  pref_speeds=f64(g["pref_speeds"]), max_speeds=f64(g["max_speeds"]),
                  goals=f64(g["goals"]), goal_tols=f64(g["goal_tols"]),
                  class_codes=g["class_codes"].astype(np.int64))
    fm = g["fmat"]
    P, V = AgentClass.PEDESTRIAN, AgentClass.VEHICLE
    resp = ResponsibilityMatrix({(P, P): fm[0, 0], (P, V): fm[0, 1], (V, P): fm[1, 0],
                                 (V, V): fm[1, 1]})
    cfg = ScenarioConfig(responsibility=resp, dt=float(g["dt"]), tau=float(g["tau"]),
                         neighbor_radius=float(g["neighbor_radius"]),
                         max_neighbors=int(g["max_neighbors"]),
                         avoidance_margin=float(g["avoidance_margin"]))
    return st, cfg


FRAME_FIXTURES = ["frame_mixed_512.npz", "frame_dense_720.npz", "frame_odd_360.npz",
                  "frame_sparse_210.npz"]
LP_FIXTURES = ["lp_batch_feasible.npz", "lp_batch_mixed.npz", "lp_batch_infeasible.npz",
               "lp_batch_small_k.npz"]
