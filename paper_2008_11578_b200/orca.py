"""Object-level ORCA operators of the reference (pkg/src/orcasim/orca.py), evaluated on
the device through the single-op taps of the C ABI:

    AgentState, VoExit                              orca.py:48-73, 133-142
    compute_vo_exit(rel_position, rel_velocity, combined_radius, tau, dt)      orca.py:145-165
    build_orca_halfplane(self_agent, other, f, tau, dt)                        orca.py:168-181
    gather_constraints(self_agent, neighbors, matrix, tau, dt)                 orca.py:184-196

Same names, argument meaning and error text. The arithmetic of the exit vector is
`vo_exit<double>` in csrc/orca_math.cuh (orca_vo_exit_batch); these wrappers are for
inspection and tests -- the step itself builds its half-planes inside k_solve*.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._lib import ORCA_F64, check, load, ptr
from .lp import HalfPlaneConstraint
from .types import AgentClass, ResponsibilityMatrix

__all__ = ["AgentState", "VoExit", "compute_vo_exit", "build_orca_halfplane", "gather_constraints",
           "vo_exit_batch"]


@dataclass
class AgentState:
    """Snapshot of one simulated entity (orca.py:48-73)."""

    id: int
    position: np.ndarray
    velocity: np.ndarray
    radius: float
    pref_speed: float
    max_speed: float
    goal: np.ndarray
    agent_class: AgentClass = AgentClass.PEDESTRIAN

    def __post_init__(self):
        for name in ("position", "velocity", "goal"):
            setattr(self, name, np.asarray(getattr(self, name), dtype=float))
        for name in ("radius", "pref_speed", "max_speed"):
            setattr(self, name, float(getattr(self, name)))
        self.agent_class = AgentClass(self.agent_class)
        if self.radius <= 0:
            raise ValueError(f"agent {self.id}: radius must be positive")
        if not 0 < self.pref_speed <= self.max_speed:
            raise ValueError(f"agent {self.id}: need 0 < pref_speed <= max_speed, "
                             f"got {self.pref_speed}/{self.max_speed}")


@dataclass
class VoExit:
    """Shortest displacement from the relative velocity to the velocity-obstacle boundary
    (`u`) and the outward unit normal there (orca.py:133-142)."""

    u: np.ndarray
    normal: np.ndarray

    def __post_init__(self):
        self.u = np.asarray(self.u, dtype=float)
        self.normal = np.asarray(self.normal, dtype=float)


def vo_exit_batch(cases, device: int = 0) -> np.ndarray:
    """cases float64[m, 7] = (rpx, rpy, rvx, rvy, combined_radius, tau, dt) -> float64[m, 5] =
    (ux, uy, nx, ny, ok), evaluated on the device in FP64 (_kernels.py:343-419)."""
    cases = np.ascontiguousarray(cases, dtype=np.float64).reshape(-1, 7)
    out = np.empty((cases.shape[0], 5))
    check(load().orca_vo_exit_batch(device, ORCA_F64, cases.shape[0], ptr(cases), ptr(out)))
    return out


def _checked_case(rel_position, rel_velocity, combined_radius, tau, dt):
    rp = np.asarray(rel_position, dtype=float).reshape(2)
    rv = np.asarray(rel_velocity, dtype=float).reshape(2)
    if not (np.all(np.isfinite(rp)) and np.all(np.isfinite(rv))):
        raise ValueError("non-finite relative position or velocity")
    combined_radius, tau, dt = float(combined_radius), float(tau), float(dt)
    if combined_radius <= 0 or tau <= 0 or dt <= 0:
        raise ValueError("combined_radius, tau and dt must all be positive")
    return [rp[0], rp[1], rv[0], rv[1], combined_radius, tau, dt]


def compute_vo_exit(rel_position, rel_velocity, combined_radius: float, tau: float, dt: float,
                    *, device: int = 0) -> VoExit:
    """Exit vector of the truncated-cone velocity obstacle with lookahead tau; overlapping
    agents use the dt-horizon disc instead (orca.py:145-165)."""
    out = vo_exit_batch([_checked_case(rel_position, rel_velocity, combined_radius, tau, dt)], device)[0]
    if out[4] == 0.0:
        raise ValueError("coincident agent centers: exit direction is undefined")
    return VoExit(out[0:2].copy(), out[2:4].copy())


def _halfplane_inputs(self_agent, other, f, tau, dt):
    if self_agent.id == other.id:
        raise ValueError(f"agent {self_agent.id}: cannot avoid itself")
    f = float(f)
    if not 0.0 <= f <= 1.0:
        raise ValueError(f"responsibility fraction {f} outside [0, 1]")
    return f, _checked_case(other.position - self_agent.position, self_agent.velocity - other.velocity,
                            self_agent.radius + other.radius, tau, dt)


def build_orca_halfplane(self_agent, other, f: float, tau: float, dt: float, *,
                         device: int = 0) -> HalfPlaneConstraint:
    """Half-plane of velocities that keeps self clear of `other` for time tau, taking
    fraction f of the avoidance (orca.py:168-181)."""
    f, case = _halfplane_inputs(self_agent, other, f, tau, dt)
    out = vo_exit_batch([case], device)[0]
    if out[4] == 0.0:
        raise ValueError("coincident agent centers: exit direction is undefined")
    return HalfPlaneConstraint(point=self_agent.velocity + f * out[0:2], normal=out[2:4].copy())


def gather_constraints(self_agent, neighbors, matrix: ResponsibilityMatrix, tau: float, dt: float, *,
                       device: int = 0) -> list:
    """One constraint per neighbour, order-aligned with the neighbour list (orca.py:184-196);
    all exits are evaluated in one device call."""
    fs, cases = [], []
    for other in neighbors:
        try:
            f, case = _halfplane_inputs(self_agent, other, matrix.get(self_agent.agent_class, other.agent_class),
                                        tau, dt)
        except ValueError as exc:
            raise ValueError(f"neighbor {other.id}: {exc}") from exc
        fs.append(f)
        cases.append(case)
    if not cases:
        return []
    out = vo_exit_batch(cases, device)
    for other, row in zip(neighbors, out):
        if row[4] == 0.0:
            raise ValueError(f"neighbor {other.id}: coincident agent centers: exit direction is undefined")
    return [HalfPlaneConstraint(point=self_agent.velocity + f * row[0:2], normal=row[2:4].copy())
            for f, row in zip(fs, out)]
