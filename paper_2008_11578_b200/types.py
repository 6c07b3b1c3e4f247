"""Host-side mirror of the reference's public types for the steering step.

Same names, fields, defaults and error behaviour as the reference so callers
can switch imports (reference file:line, paths under pkg/src/orcasim/):

    AgentClass            orca.py:31-45
    ResponsibilityMatrix  orca.py:76-129   (default(): PP .5, VV .5, PV 1, VP 0)
    ClassParams           scenario.py:64-68
    ScenarioConfig        scenario.py:79-114 (hot-path fields only; the YAML
                          schema / spawn regions are out of scope)
    SimState              engine.py:55-87
    FrameMetrics          engine.py:46-52

Objects of the reference's own classes are accepted everywhere these are
(attribute access only).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import IntEnum

import math

import numpy as np

__all__ = ["AgentClass", "ResponsibilityMatrix", "ClassParams", "ScenarioConfig",
           "SimState", "FrameMetrics", "FrameLog", "RunSummary", "RunResult", "DEFAULTS",
           "DEFAULT_CLASS_PARAMS"]


class AgentClass(IntEnum):
    PEDESTRIAN = 0
    VEHICLE = 1

    @property
    def label(self) -> str:
        return self.name.lower()

    @classmethod
    def from_label(cls, label: str) -> "AgentClass":
        try:
            return cls[label.strip().upper()]
        except KeyError:
            raise ValueError(f"unknown agent class {label!r}") from None


# scenario.py:43-56
DEFAULT_CLASS_PARAMS = {
    AgentClass.PEDESTRIAN: (0.25, 1.4, 2.0),
    AgentClass.VEHICLE: (1.0, 3.0, 5.0),
}

DEFAULTS = {
    "dt": 0.1,
    "tau": 2.0,
    "neighbor_radius": 15.0,
    "max_neighbors": 16,
    "clearance_time": 0.5,
    "avoidance_margin": 0.1,
    "seed": 0,
}


@dataclass
class ResponsibilityMatrix:
    """Avoidance fractions f[(A, B)]: the share of the exit displacement an
    agent of class A applies when avoiding class B (orca.py:76-129)."""

    f: dict = field(default_factory=dict)

    def __post_init__(self):
        clean = {}
        for (a, b), value in self.f.items():
            value = float(value)
            if not 0.0 <= value <= 1.0:
                raise ValueError(f"responsibility f[{a},{b}] = {value} outside [0, 1]")
            clean[(AgentClass(a), AgentClass(b))] = value
        self.f = clean

    @classmethod
    def default(cls) -> "ResponsibilityMatrix":
        P, V = AgentClass.PEDESTRIAN, AgentClass.VEHICLE
        return cls({(P, P): 0.5, (V, V): 0.5, (P, V): 1.0, (V, P): 0.0})

    def get(self, a, b) -> float:
        try:
            return self.f[(AgentClass(a), AgentClass(b))]
        except KeyError:
            raise KeyError(f"responsibility matrix has no entry for ({a}, {b})") from None

    def guarantee_holds(self, a, b) -> bool:
        return self.get(a, b) + self.get(b, a) >= 1.0

    def unguaranteed_pairs(self) -> list:
        """Unordered class pairs (low, high) whose two fractions sum below 1, in the order
        the matrix first lists them (orca.py:110-121). Pairs with one direction missing
        are not reported."""
        visited, below = set(), []
        for a, b in self.f:
            pair = (min(a, b), max(a, b))
            if (b, a) in self.f and pair not in visited:
                visited.add(pair)
                if not self.guarantee_holds(a, b):
                    below.append(pair)
        return below

    def as_array(self) -> np.ndarray:
        n = max(int(c) for c in AgentClass) + 1
        arr = np.zeros((n, n), dtype=np.float64)
        for (a, b), value in self.f.items():
            arr[int(a), int(b)] = value
        return arr


@dataclass
class ClassParams:
    radius: float
    pref_speed: float
    max_speed: float


def _default_class_params():
    return {c: ClassParams(*p) for c, p in DEFAULT_CLASS_PARAMS.items()}


@dataclass
class ScenarioConfig:
    """The fields of scenario.ScenarioConfig the per-frame step reads
    (scenario.py:79-99). `regions` is kept for signature compatibility; spawn
    sampling itself is outside the accelerated path."""

    regions: list = field(default_factory=list)
    class_params: dict = field(default_factory=_default_class_params)
    responsibility: ResponsibilityMatrix = field(default_factory=ResponsibilityMatrix.default)
    dt: float = DEFAULTS["dt"]
    tau: float = DEFAULTS["tau"]
    neighbor_radius: float = DEFAULTS["neighbor_radius"]
    max_neighbors: int = DEFAULTS["max_neighbors"]
    goal_tolerance: float | None = None
    clearance_time: float = DEFAULTS["clearance_time"]
    avoidance_margin: float = DEFAULTS["avoidance_margin"]
    seed: int = DEFAULTS["seed"]
    max_frames: int | None = None
    warnings: list = field(default_factory=list)

    def goal_tolerance_for(self, agent_class) -> float:
        if self.goal_tolerance is not None:
            return self.goal_tolerance
        return self.class_params[AgentClass(agent_class)].radius

    def frame_guard(self) -> int:
        """max_frames, defaulting to a generous multiple of the straight-line crossing
        time over the scenario extent (scenario.py:101-114). Regions are objects with
        .spawn / .goal rectangles (x0, y0, x1, y1) and .agent_class."""
        if self.max_frames is not None:
            return self.max_frames
        rects = [r.spawn for r in self.regions] + [r.goal for r in self.regions]
        if not rects:
            return 1
        xs = [r[0] for r in rects] + [r[2] for r in rects]
        ys = [r[1] for r in rects] + [r[3] for r in rects]
        diag = math.hypot(max(xs) - min(xs), max(ys) - min(ys))
        used = {AgentClass(r.agent_class) for r in self.regions}
        min_pref = min(self.class_params[c].pref_speed for c in used)
        return max(1, int(100.0 * (diag / min_pref) / self.dt))


@dataclass
class FrameMetrics:
    frame: int
    wall_ms: float
    min_separation: float
    collision_count: int
    active_agents: int


@dataclass
class SimState:
    """Simulation state after `frame` completed steps (time = frame * dt);
    field-for-field the reference's engine.SimState (engine.py:55-87)."""

    frame: int
    time: float
    ids: np.ndarray
    positions: np.ndarray
    velocities: np.ndarray
    radii: np.ndarray
    pref_speeds: np.ndarray
    max_speeds: np.ndarray
    goals: np.ndarray
    goal_tols: np.ndarray
    class_codes: np.ndarray
    rng_state: object = None
    lp_fallbacks: int = 0

    @property
    def active_count(self) -> int:
        return int(self.ids.shape[0])

    @property
    def agents(self) -> list:
        """One orca.AgentState per row, in storage order (engine.py:80-87)."""
        from .orca import AgentState
        return [AgentState(id=int(self.ids[i]), position=self.positions[i].copy(),
                           velocity=self.velocities[i].copy(), radius=float(self.radii[i]),
                           pref_speed=float(self.pref_speeds[i]), max_speed=float(self.max_speeds[i]),
                           goal=self.goals[i].copy(), agent_class=AgentClass(int(self.class_codes[i])))
                for i in range(self.active_count)]


@dataclass(eq=False)
class FrameLog:
    """Positions and velocities of every agent active during one frame
    (scenario.py:117-140): post-step values, arrivals of that frame included."""

    frame: int
    time: float
    ids: np.ndarray
    classes: np.ndarray
    positions: np.ndarray
    velocities: np.ndarray
    radii: np.ndarray

    def __eq__(self, other):
        if not isinstance(other, FrameLog):
            return NotImplemented
        return (self.frame == other.frame and self.time == other.time
                and all(np.array_equal(getattr(self, k), getattr(other, k))
                        for k in ("ids", "classes", "positions", "velocities", "radii")))


@dataclass
class RunSummary:
    """engine.py:90-102"""

    total_collisions: int
    min_separation: float
    mean_frame_ms: float
    p95_frame_ms: float
    agents: int
    seed: int
    frames: int
    terminated: bool
    arrived: int
    total_fallbacks: int
    mean_travel_time: dict


@dataclass
class RunResult:
    """engine.py:105-111"""

    frame_logs: list
    frame_metrics: list
    summary: RunSummary
    agent_records: list = field(default_factory=list)
    final_state: SimState | None = None
