"""Scenario documents, seeded spawn sampling and the trajectory / metrics files: the
callers and data formats on either side of the steering step.

Mirrors pkg/src/orcasim/scenario.py of the reference -- same names, argument meaning,
error type and messages -- so a script written against `orcasim.scenario` runs on this
package unchanged:

    ScenarioError, Region                      scenario.py:60-77
    scenario_from_dict / load_scenario         scenario.py:170-322
    sample_spawns / sample_goal_points /
    build_agents                               scenario.py:328-428
    write_trajectories / read_trajectories /
    write_metrics_summary / atomic_write_text  scenario.py:434-519

Host-side setup and I/O, once per run: none of it is on the per-frame path. Two things are
contracts rather than conveniences and are pinned by tests/golden/scenario_*.json:
the spawn sampler consumes the seeded `numpy.random.default_rng(seed)` stream exactly as the
reference does (two doubles per attempt, regions in order, spawns then goals), so the same
scenario spawns the same crowd bit for bit; and the CSV grammar (column order, `repr`
floats, CRLF rows) is byte-identical, so trajectory files hash equal across the two
implementations when the step runs in f64 mode.
"""

from __future__ import annotations

import math
import os
import tempfile
from dataclasses import dataclass

import numpy as np

from ._lib import ORCA_MAX_NEIGHBORS

from .types import (DEFAULT_CLASS_PARAMS, DEFAULTS, AgentClass, ClassParams, FrameLog,
                    ResponsibilityMatrix, ScenarioConfig)

__all__ = ["ScenarioError", "Region", "Agent", "scenario_from_dict", "load_scenario", "sample_spawns",
           "sample_goal_points", "build_agents", "spawn_arrays", "write_trajectories",
           "read_trajectories", "write_metrics_summary", "atomic_write_text", "FORMAT_VERSION",
           "TRAJECTORY_COLUMNS", "METRICS_COLUMNS"]

FORMAT_VERSION = 1
TRAJECTORY_COLUMNS = ["frame", "time", "agent_id", "class", "x", "y", "vx", "vy", "radius"]
METRICS_COLUMNS = ["total_collisions", "min_separation", "mean_frame_ms", "p95_frame_ms", "agents", "seed"]
SPAWN_ATTEMPTS_PER_POINT = 2000          # scenario.py:58
HEX_PACKING = 0.9069                     # scenario.py:352-354


class ScenarioError(ValueError):
    """Scenario validation failure; the message names the offending field."""


@dataclass
class Region:
    spawn: tuple
    goal: tuple
    agent_class: AgentClass
    count: int


@dataclass
class Agent:
    """What orcasim.orca.AgentState carries (orca.py:48-73): one spawned agent."""
    id: int
    position: np.ndarray
    velocity: np.ndarray
    radius: float
    pref_speed: float
    max_speed: float
    goal: np.ndarray
    agent_class: AgentClass


# ---------------------------------------------------------------------------
# schema (scenario.py:144-311)
# ---------------------------------------------------------------------------

def _is_num(v) -> bool:
    return isinstance(v, (int, float)) and not isinstance(v, bool)


def _is_int(v) -> bool:
    return isinstance(v, int) and not isinstance(v, bool)


def _number(mapping, key, where, positive=True, allow_none=False):
    v = mapping.get(key)
    if v is None and allow_none:
        return None
    if not _is_num(v):
        raise ScenarioError(f"{where}.{key}: expected a number, got {v!r}")
    v = float(v)
    if not math.isfinite(v):
        raise ScenarioError(f"{where}.{key}: must be finite")
    if positive and v <= 0:
        raise ScenarioError(f"{where}.{key}: must be positive, got {v}")
    return v


def _rect(v, where):
    if not isinstance(v, (list, tuple)) or len(v) != 4 or not all(_is_num(c) for c in v):
        raise ScenarioError(f"{where}: expected [x0, y0, x1, y1]")
    r = tuple(float(c) for c in v)
    if not all(math.isfinite(c) for c in r):
        raise ScenarioError(f"{where}: coordinates must be finite")
    if r[0] >= r[2] or r[1] >= r[3]:
        raise ScenarioError(f"{where}: rectangle is degenerate (need x0 < x1 and y0 < y1)")
    return r


def _agent_class(name, where) -> AgentClass:
    if isinstance(name, AgentClass):
        return name
    if not isinstance(name, str):
        raise ScenarioError(f"{where}: expected an agent class name, got {name!r}")
    try:
        return AgentClass.from_label(name)
    except ValueError:
        valid = ", ".join(c.label for c in AgentClass)
        raise ScenarioError(f"{where}: unknown agent class {name!r} (valid: {valid})") from None


def _only(mapping, allowed, where):
    for key in mapping:
        if key not in allowed:
            raise ScenarioError(f"{where}.{key}: unknown field")


_TOP_LEVEL = ("format_version", "seed", "dt", "tau", "neighbor_radius", "max_neighbors", "goal_tolerance",
              "clearance_time", "avoidance_margin", "max_frames", "classes", "responsibility", "regions")


def _responsibility(raw, used, source):
    if raw is None:
        matrix = ResponsibilityMatrix.default()
    else:
        if not isinstance(raw, dict):
            raise ScenarioError(f"{source}.responsibility: expected a mapping like 'pedestrian|vehicle: 1.0'")
        entries = {}
        for key, value in raw.items():
            where = f"{source}.responsibility.{key}"
            if not isinstance(key, str) or key.count("|") != 1:
                raise ScenarioError(f"{where}: key must look like 'classA|classB'")
            left, right = key.split("|")
            pair = (_agent_class(left, where), _agent_class(right, where))
            if not _is_num(value):
                raise ScenarioError(f"{where}: expected a number in [0, 1]")
            if not 0.0 <= float(value) <= 1.0:
                raise ScenarioError(f"{where}: fraction {float(value)} outside [0, 1]")
            entries[pair] = float(value)
        matrix = ResponsibilityMatrix(entries)
    for a in used:
        for b in used:
            if (a, b) not in matrix.f:
                raise ScenarioError(f"{source}.responsibility: missing entry {a.label}|{b.label} "
                                    "for a class used by the regions")
    warnings = [f"responsibility sum f[{a.label}|{b.label}] + f[{b.label}|{a.label}] "
                f"= {matrix.get(a, b) + matrix.get(b, a):g} < 1: "
                "collision-free motion is not guaranteed for this pair"
                for a, b in matrix.unguaranteed_pairs() if a in used and b in used]
    return matrix, warnings


def scenario_from_dict(data: dict, source: str = "<dict>") -> ScenarioConfig:
    """Validate a scenario mapping and fill defaults (scenario.py:170-259). Raises
    ScenarioError naming field and location; a responsibility pair summing below 1 is a
    warning on the returned config, not an error."""
    if not isinstance(data, dict):
        raise ScenarioError(f"{source}: scenario document must be a mapping")
    version = data.get("format_version", FORMAT_VERSION)
    if version != FORMAT_VERSION:
        raise ScenarioError(f"{source}.format_version: unsupported version {version!r}")
    _only(data, _TOP_LEVEL, source)

    def opt(key, positive=True):
        return _number(data, key, source, positive=positive) if key in data else DEFAULTS[key]

    dt, tau, neighbor_radius = opt("dt"), opt("tau"), opt("neighbor_radius")
    clearance_time = opt("clearance_time", positive=False)
    if clearance_time is not None and clearance_time < 0:
        raise ScenarioError(f"{source}.clearance_time: must be >= 0")
    goal_tolerance = _number(data, "goal_tolerance", source, allow_none=True)
    avoidance_margin = opt("avoidance_margin", positive=False)
    if avoidance_margin < 0:
        raise ScenarioError(f"{source}.avoidance_margin: must be >= 0")
    max_neighbors = data.get("max_neighbors", DEFAULTS["max_neighbors"])
    if not _is_int(max_neighbors) or max_neighbors < 0:
        raise ScenarioError(f"{source}.max_neighbors: expected an integer >= 0")
    if max_neighbors > ORCA_MAX_NEIGHBORS:
        # the reference accepts any count; the device keeps an agent's list in registers
        raise ScenarioError(f"{source}.max_neighbors: {max_neighbors} exceeds the {ORCA_MAX_NEIGHBORS} "
                            "neighbours per agent this GPU build supports")
    seed = data.get("seed", DEFAULTS["seed"])
    if not _is_int(seed):
        raise ScenarioError(f"{source}.seed: expected an integer")
    max_frames = data.get("max_frames")
    if max_frames is not None and (not _is_int(max_frames) or max_frames < 1):
        raise ScenarioError(f"{source}.max_frames: expected an integer >= 1 or null")

    class_params = {c: ClassParams(*DEFAULT_CLASS_PARAMS[c]) for c in AgentClass}
    for name, raw in (data.get("classes") or {}).items():
        cls = _agent_class(name, f"{source}.classes")
        where = f"{source}.classes.{name}"
        if not isinstance(raw, dict):
            raise ScenarioError(f"{where}: expected a mapping")
        cur = class_params[cls]
        vals = [_number(raw, k, where) if k in raw else getattr(cur, k)
                for k in ("radius", "pref_speed", "max_speed")]
        _only(raw, ("radius", "pref_speed", "max_speed"), where)
        if vals[1] > vals[2]:
            raise ScenarioError(f"{where}: pref_speed {vals[1]} exceeds max_speed {vals[2]}")
        class_params[cls] = ClassParams(*vals)

    raw_regions = data.get("regions")
    if not isinstance(raw_regions, list):
        raise ScenarioError(f"{source}.regions: expected a list of regions")
    regions = []
    for i, raw in enumerate(raw_regions):
        where = f"{source}.regions[{i}]"
        if not isinstance(raw, dict):
            raise ScenarioError(f"{where}: expected a mapping")
        _only(raw, ("spawn", "goal", "agent_class", "count"), where)
        spawn = _rect(raw.get("spawn"), f"{where}.spawn")
        goal = _rect(raw.get("goal"), f"{where}.goal")
        cls = _agent_class(raw.get("agent_class", "pedestrian"), f"{where}.agent_class")
        count = raw.get("count")
        if not _is_int(count) or count < 0:
            raise ScenarioError(f"{where}.count: expected an integer >= 0")
        regions.append(Region(spawn, goal, cls, count))

    used = sorted({r.agent_class for r in regions}) or [AgentClass.PEDESTRIAN]
    matrix, warnings = _responsibility(data.get("responsibility"), used, source)
    return ScenarioConfig(regions=regions, class_params=class_params, responsibility=matrix, dt=dt, tau=tau,
                          neighbor_radius=neighbor_radius, max_neighbors=max_neighbors,
                          goal_tolerance=goal_tolerance, clearance_time=clearance_time,
                          avoidance_margin=avoidance_margin, seed=seed, max_frames=max_frames,
                          warnings=warnings)


def load_scenario(path) -> ScenarioConfig:
    """Parse and validate a scenario YAML file (scenario.py:314-322)."""
    import yaml
    with open(path, "r", encoding="utf-8") as f:
        try:
            data = yaml.safe_load(f)
        except yaml.YAMLError as exc:
            raise ScenarioError(f"{path}: parse error: {exc}") from exc
    return scenario_from_dict(data, source=str(path))


# ---------------------------------------------------------------------------
# spawn sampling (scenario.py:328-428)
# ---------------------------------------------------------------------------

class _Placed:
    """Accepted points of one region, bucketed by cells of edge `min_dist` so that an
    acceptance test looks at 3x3 buckets only."""

    def __init__(self, count: int, cell: float):
        self.xy = np.empty((count, 2), dtype=np.float64)
        self.n = 0
        self.cell = cell
        self.buckets: dict = {}

    def key(self, x, y):
        return int(math.floor(x / self.cell)), int(math.floor(y / self.cell))

    def clear_of(self, x, y, min_d2) -> bool:
        kx, ky = self.key(x, y)
        near = []
        for gx in (kx - 1, kx, kx + 1):
            for gy in (ky - 1, ky, ky + 1):
                near.extend(self.buckets.get((gx, gy), ()))
        for i in near:
            px, py = self.xy[i]
            if (x - px) ** 2 + (y - py) ** 2 < min_d2:
                return False
        return True

    def add(self, x, y):
        self.xy[self.n] = (x, y)
        self.buckets.setdefault(self.key(x, y), []).append(self.n)
        self.n += 1


def sample_spawns(region, count: int, radius: float, pref_speed: float, clearance_time: float,
                  rng: np.random.Generator, existing=None) -> np.ndarray:
    """`count` points uniform in the rectangle `region` with pairwise distance
    >= 2*radius + pref_speed*clearance_time, by rejection (scenario.py:328-389).
    `existing` rows (x, y, contribution) are agents already placed, possibly of another
    class; a new point keeps own_contribution + their contribution from each, where a
    contribution is radius + pref_speed*clearance_time/2. Every attempt consumes exactly
    two doubles of `rng` (x first), accepted or not."""
    x0, y0, x1, y1 = (float(v) for v in region)
    if x0 >= x1 or y0 >= y1:
        raise ScenarioError(f"spawn region {region!r} is degenerate")
    if clearance_time < 0:
        raise ScenarioError("clearance_time must be >= 0")
    contrib = radius + pref_speed * clearance_time / 2.0
    min_dist = 2.0 * contrib
    area = (x1 - x0) * (y1 - y0)
    if count > 1 and count * math.pi * (min_dist / 2.0) ** 2 > HEX_PACKING * area:
        raise ScenarioError(f"region area {area:.3g} m^2 cannot hold {count} agents at minimum "
                            f"spacing {min_dist:.3g} m")
    others = None
    if existing is not None:
        others = np.asarray(existing, dtype=np.float64)
        if others.size == 0:
            others = None
    reach2 = None if others is None else (contrib + others[:, 2]) ** 2
    placed = _Placed(count, min_dist if min_dist > 0 else 1.0)
    min_d2 = min_dist ** 2
    for i in range(count):
        for _ in range(SPAWN_ATTEMPTS_PER_POINT):
            x = x0 + (x1 - x0) * rng.random()
            y = y0 + (y1 - y0) * rng.random()
            if not placed.clear_of(x, y, min_d2):
                continue
            if others is not None and np.any((others[:, 0] - x) ** 2 + (others[:, 1] - y) ** 2 < reach2):
                continue
            placed.add(x, y)
            break
        else:
            raise ScenarioError(f"could not place agent {i + 1} of {count} in region {region!r} "
                                f"after {SPAWN_ATTEMPTS_PER_POINT} attempts ({i} placed); "
                                "the region is too dense for the requested spacing")
    return placed.xy


def sample_goal_points(region, count: int, rng: np.random.Generator) -> np.ndarray:
    """Uniform goals in the end region, from the same stream as the spawns, x then y per
    point (scenario.py:392-401)."""
    x0, y0, x1, y1 = (float(v) for v in region)
    u = rng.random(2 * count).reshape(count, 2)     # same doubles as 2*count scalar draws
    return np.column_stack([x0 + (x1 - x0) * u[:, 0], y0 + (y1 - y0) * u[:, 1]])


def spawn_arrays(config: ScenarioConfig) -> dict:
    """The spawned crowd of `config` as structure-of-arrays (what init_state needs):
    regions in order, placement chained across regions so cross-region and cross-class
    pairs respect the clearance rule too, ids in region order (scenario.py:404-428)."""
    rng = np.random.default_rng(config.seed)
    pos, goal, cls, rad, pref, maxs = [], [], [], [], [], []
    chained = np.empty((0, 3))
    for region in config.regions:
        p = config.class_params[region.agent_class]
        spawns = sample_spawns(region.spawn, region.count, p.radius, p.pref_speed, config.clearance_time,
                               rng, existing=chained if chained.shape[0] else None)
        goals = sample_goal_points(region.goal, region.count, rng)
        contrib = p.radius + p.pref_speed * config.clearance_time / 2.0
        chained = np.vstack([chained, np.column_stack([spawns, np.full(region.count, contrib)])])
        pos.append(spawns)
        goal.append(goals)
        cls.append(np.full(region.count, int(region.agent_class), dtype=np.int64))
        rad.append(np.full(region.count, p.radius))
        pref.append(np.full(region.count, p.pref_speed))
        maxs.append(np.full(region.count, p.max_speed))

    def cat(parts, shape, dtype=np.float64):
        return np.concatenate(parts).astype(dtype) if parts else np.empty(shape, dtype=dtype)

    n = sum(r.count for r in config.regions)
    return dict(ids=np.arange(n, dtype=np.int64), positions=cat(pos, (0, 2)), goals=cat(goal, (0, 2)),
                class_codes=cat(cls, 0, np.int64), radii=cat(rad, 0), pref_speeds=cat(pref, 0),
                max_speeds=cat(maxs, 0))


def build_agents(config: ScenarioConfig) -> list:
    """Spawn every region's agents deterministically from the config seed
    (scenario.py:404-428) -> list of Agent, velocity zero."""
    a = spawn_arrays(config)
    return [Agent(id=int(a["ids"][i]), position=a["positions"][i], velocity=np.zeros(2),
                  radius=float(a["radii"][i]), pref_speed=float(a["pref_speeds"][i]),
                  max_speed=float(a["max_speeds"][i]), goal=a["goals"][i],
                  agent_class=AgentClass(int(a["class_codes"][i]))) for i in range(a["ids"].shape[0])]


# ---------------------------------------------------------------------------
# trajectory and metrics files (scenario.py:434-519)
# ---------------------------------------------------------------------------

def atomic_write_text(path, write_fn):
    """Write through a temporary file in the destination directory, then rename."""
    path = os.fspath(path)
    fd, tmp = tempfile.mkstemp(dir=os.path.dirname(path) or ".", suffix=".tmp")
    try:
        with os.fdopen(fd, "w", encoding="utf-8", newline="") as f:
            write_fn(f)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


_EOL = "\r\n"            # csv.writer's default row terminator, which the reference's files carry


def _frame_rows(log: FrameLog) -> str:
    """All CSV rows of one frame. Floats are written with repr() (shortest round-trip
    form), so reading the file back reproduces the arrays exactly."""
    head = f"{int(log.frame)},{float(log.time)!r},"
    ids = np.asarray(log.ids).tolist()
    labels = [AgentClass(int(c)).label for c in np.asarray(log.classes).tolist()]
    pos = np.asarray(log.positions, dtype=np.float64).reshape(-1, 2).tolist()
    vel = np.asarray(log.velocities, dtype=np.float64).reshape(-1, 2).tolist()
    rad = np.asarray(log.radii, dtype=np.float64).tolist()
    return "".join(f"{head}{int(i)},{c},{p[0]!r},{p[1]!r},{v[0]!r},{v[1]!r},{r!r}{_EOL}"
                   for i, c, p, v, r in zip(ids, labels, pos, vel, rad))


def write_trajectories(logs, path) -> None:
    """One row per (frame, agent): frame,time,agent_id,class,x,y,vx,vy,radius."""
    def emit(f):
        f.write(",".join(TRAJECTORY_COLUMNS) + _EOL)
        for log in logs:
            f.write(_frame_rows(log))
    atomic_write_text(path, emit)


def read_trajectories(path) -> list:
    """Inverse of write_trajectories (scenario.py:469-501)."""
    with open(path, "r", encoding="utf-8", newline="") as f:
        lines = f.read().splitlines()
    header = lines[0].split(",") if lines else None
    if header != TRAJECTORY_COLUMNS:
        raise ValueError(f"{path}: unexpected trajectory header {header!r}")
    logs, start = [], 1
    rows = [ln.split(",") for ln in lines[1:] if ln]
    frames = [int(r[0]) for r in rows]
    i = 0
    while i < len(rows):
        j = i
        while j < len(rows) and frames[j] == frames[i]:
            j += 1
        chunk = rows[i:j]
        logs.append(FrameLog(
            frame=frames[i], time=float(chunk[0][1]),
            ids=np.array([int(r[2]) for r in chunk], dtype=np.int64),
            classes=np.array([int(AgentClass.from_label(r[3])) for r in chunk], dtype=np.int8),
            positions=np.array([[float(r[4]), float(r[5])] for r in chunk], dtype=np.float64).reshape(-1, 2),
            velocities=np.array([[float(r[6]), float(r[7])] for r in chunk], dtype=np.float64).reshape(-1, 2),
            radii=np.array([float(r[8]) for r in chunk], dtype=np.float64)))
        i = j
    del start
    return logs


def write_metrics_summary(summary, path) -> None:
    """One record per run (scenario.py:504-519)."""
    def emit(f):
        f.write(",".join(METRICS_COLUMNS) + _EOL)
        f.write(",".join([str(int(summary.total_collisions)), repr(float(summary.min_separation)),
                          repr(float(summary.mean_frame_ms)), repr(float(summary.p95_frame_ms)),
                          str(int(summary.agents)), str(int(summary.seed))]) + _EOL)
    atomic_write_text(path, emit)
