"""The paper's 2-way and 4-way crossing experiments as scenario documents
(pkg/src/orcasim/crossings.py:94-143): opposing rectangular spawn / goal regions give
head-on streams, the 4-way variant adds side-on streams. Geometry follows the reference's
sizing rule exactly (spawn area per agent = 6 x squared class spacing, at least 8 m x 8 m,
at most 120 m across), so a (kind, agents per arm, vehicle fraction, seed) tuple means the
same scenario -- and, through scenario.spawn_arrays, the same spawned crowd -- in both
implementations (tests/golden/scenario_*.json).
"""

from __future__ import annotations

import math

from .scenario import scenario_from_dict
from .types import DEFAULT_CLASS_PARAMS, DEFAULTS, AgentClass, ScenarioConfig

__all__ = ["two_way_dict", "four_way_dict", "crossing_config", "arm_size", "split_counts"]

AREA_PER_AGENT = 6.0      # in squared class spacings        crossings.py:20-22
SMALLEST_SIDE = 8.0
WIDEST_ARM = 120.0
CORRIDOR_GAP = 24.0       # free space between opposing arms  crossings.py:106, 125


def split_counts(per_arm: int, vehicle_fraction: float):
    """-> (pedestrians, vehicles) of one arm."""
    vehicles = int(round(per_arm * vehicle_fraction))
    return per_arm - vehicles, vehicles


def _class_spacing(cls: AgentClass, clearance_time: float) -> float:
    radius, pref_speed, _ = DEFAULT_CLASS_PARAMS[cls]
    return 2.0 * radius + pref_speed * clearance_time


def arm_size(per_arm: int, vehicle_fraction: float, clearance_time: float = DEFAULTS["clearance_time"],
             size_for_worst_class: bool = False):
    """(width across the stream, depth along it) of one arm's rectangles."""
    peds, vehs = split_counts(per_arm, vehicle_fraction)
    sp = _class_spacing(AgentClass.PEDESTRIAN, clearance_time)
    sv = _class_spacing(AgentClass.VEHICLE, clearance_time)
    if size_for_worst_class:
        widest = max(sp, sv)
        area = AREA_PER_AGENT * per_arm * widest * widest
    else:
        area = AREA_PER_AGENT * (peds * sp * sp + vehs * sv * sv)
    area = max(area, SMALLEST_SIDE * SMALLEST_SIDE)
    width = min(WIDEST_ARM, math.sqrt(area))
    return width, area / width


def _arm(width, depth, gap, axis, sign, peds, vehs):
    """Region documents of one arm: spawn on the -sign side of `axis`, goal opposite."""
    near, far = gap / 2.0, gap / 2.0 + depth
    along_spawn = sorted((-sign * far, -sign * near))
    along_goal = sorted((sign * near, sign * far))
    across = (-width / 2.0, width / 2.0)
    if axis == "x":
        spawn = [along_spawn[0], across[0], along_spawn[1], across[1]]
        goal = [along_goal[0], across[0], along_goal[1], across[1]]
    else:
        spawn = [across[0], along_spawn[0], across[1], along_spawn[1]]
        goal = [across[0], along_goal[0], across[1], along_goal[1]]
    return [{"spawn": list(spawn), "goal": list(goal), "agent_class": label, "count": count}
            for label, count in (("pedestrian", peds), ("vehicle", vehs)) if count]


def _document(kind_axes, per_arm, vehicle_fraction, seed, arm_width, arm_depth, size_for_worst_class,
              gap_for, overrides):
    clearance = overrides.get("clearance_time", DEFAULTS["clearance_time"])
    width, depth = (arm_size(per_arm, vehicle_fraction, clearance, size_for_worst_class)
                    if per_arm else (SMALLEST_SIDE, SMALLEST_SIDE))
    width = arm_width if arm_width is not None else width
    depth = arm_depth if arm_depth is not None else depth
    peds, vehs = split_counts(per_arm, vehicle_fraction)
    doc = {"format_version": 1, "seed": int(seed),
           "responsibility": {"pedestrian|pedestrian": 0.5, "vehicle|vehicle": 0.5,
                              "pedestrian|vehicle": 1.0, "vehicle|pedestrian": 0.0},
           "regions": []}
    doc.update(overrides)
    for axis in kind_axes:
        for sign in (1, -1):
            doc["regions"].extend(_arm(width, depth, gap_for(width), axis, sign, peds, vehs))
    return doc


def two_way_dict(per_side: int, vehicle_fraction: float = 0.0, seed: int = 0, arm_width=None,
                 arm_depth=None, size_for_worst_class: bool = False, **overrides) -> dict:
    """Two opposing crowds crossing a shared corridor (crossings.py:94-110)."""
    return _document("x", per_side, vehicle_fraction, seed, arm_width, arm_depth, size_for_worst_class,
                     lambda width: CORRIDOR_GAP, overrides)


def four_way_dict(per_arm: int, vehicle_fraction: float = 0.0, seed: int = 0, arm_width=None,
                  arm_depth=None, size_for_worst_class: bool = False, **overrides) -> dict:
    """Four crowds crossing one centre; perpendicular arms are kept disjoint
    (crossings.py:113-132)."""
    return _document("xy", per_arm, vehicle_fraction, seed, arm_width, arm_depth, size_for_worst_class,
                     lambda width: max(CORRIDOR_GAP, width + 8.0), overrides)


def crossing_config(kind: str, per_arm: int, vehicle_fraction: float = 0.0, seed: int = 0,
                    **kwargs) -> ScenarioConfig:
    makers = {"two_way": two_way_dict, "four_way": four_way_dict}
    if kind not in makers:
        raise ValueError(f"unknown crossing kind {kind!r} (expected two_way or four_way)")
    return scenario_from_dict(makers[kind](per_arm, vehicle_fraction, seed, **kwargs),
                              source=f"<{kind} crossing>")
