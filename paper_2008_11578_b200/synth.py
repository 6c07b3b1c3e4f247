"""Synthetic inputs for parity tests and benchmarks.

* plaza_crowd: a square plaza of side sqrt(N/density) filled with pedestrians
  and vehicles on a jittered lattice (centres never coincide), goals uniform in
  the plaza, velocities = random heading x pref_speed x U(0,1). Every float is
  rounded to float32 and up-cast to float64 so the float64 CPU oracle and the
  FP32 device state see identical inputs. The state is built directly as a
  SimState, the way the reference's own tests do (pkg/tests/test_engine.py:72-74).
* lp_batch: CSR-packed closest-point problems in the layout of
  _kernels.solve_range (pkg/src/orcasim/_kernels.py:306-312); the feasible mix
  is the witness-disc construction of pkg/tests/oracles.py:237-257 and the
  unconstrained mix is pkg/tests/oracles.py:260-268, both vectorised.
"""

from __future__ import annotations

import math

import numpy as np

from .types import DEFAULT_CLASS_PARAMS, AgentClass, ScenarioConfig, SimState

__all__ = ["plaza_crowd", "blobs_crowd", "make_workload", "lp_batch", "CONFIGS", "CONFIG_PARAMS"]

# BASELINE.json configs -> (pedestrians, vehicles, density per m^2)
CONFIGS = {
    "config1_1k": (1024, 0, 0.25),
    "config2_16k": (16384, 256, 0.25),
    "config3_262k_d1": (262144, 4096, 1.0),
    "config3_262k_d2": (262144, 4096, 2.0),
    "plaza_1m": (1032192, 16384, 0.25),
    "config5_8m": (8388608, 131072, 0.25),
    # config 3 at neighbor_radius = 3 m (same neighbour sets at these densities,
    # the reference's CPU cost drops ~4x; engine.py:211-213)
    "config3_262k_d1_nr3": (262144, 4096, 1.0),
    "config3_262k_d2_nr3": (262144, 4096, 2.0),
    # NON-uniform crowd: Gaussian blobs with a 10x density contrast (0.1 .. 1.0 /m2, mean ~0.25),
    # four crossing streams -- the worst case for a search grid planned from the mean density
    "blobs_1m": (1032192, 16384, 0.25),
}

# ScenarioConfig fields a named workload overrides, and the generator it uses
CONFIG_PARAMS = {
    "config3_262k_d1_nr3": {"neighbor_radius": 3.0},
    "config3_262k_d2_nr3": {"neighbor_radius": 3.0},
}
GENERATORS = {"blobs_1m": "blobs"}


def make_workload(name: str, seed: int = 0, origin=(0.0, 0.0)):
    """(state, config) of a named workload of CONFIGS."""
    n_ped, n_veh, density = CONFIGS[name]
    cfg = ScenarioConfig(**CONFIG_PARAMS.get(name, {}))
    if GENERATORS.get(name) == "blobs":
        return blobs_crowd(n_ped, n_veh, seed=seed, config=cfg, origin=origin)
    return plaza_crowd(n_ped, n_veh, density=density, seed=seed, config=cfg, origin=origin)


def _f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def plaza_crowd(n_ped: int, n_veh: int = 0, density: float = 0.25, seed: int = 0,
                config: ScenarioConfig | None = None, origin=(0.0, 0.0),
                round_f32: bool = True) -> tuple[SimState, ScenarioConfig]:
    """Random mixed crowd at `density` agents/m^2; returns (state, config)."""
    cfg = config if config is not None else ScenarioConfig()
    n = int(n_ped) + int(n_veh)
    rng = np.random.default_rng(seed)
    side = math.sqrt(max(n, 1) / density)
    m = max(1, math.ceil(math.sqrt(max(n, 1))))
    pitch = side / m
    slots = rng.permutation(m * m)[:n]
    sx = (slots % m).astype(np.float64)
    sy = (slots // m).astype(np.float64)
    jitter = rng.uniform(-0.3, 0.3, size=(n, 2))
    pos = np.empty((n, 2))
    pos[:, 0] = origin[0] + (sx + 0.5 + jitter[:, 0]) * pitch
    pos[:, 1] = origin[1] + (sy + 0.5 + jitter[:, 1]) * pitch
    goals = np.empty((n, 2))
    goals[:, 0] = origin[0] + rng.uniform(0.0, side, size=n)
    goals[:, 1] = origin[1] + rng.uniform(0.0, side, size=n)

    cls = np.zeros(n, dtype=np.int64)
    if n_veh:
        cls[rng.permutation(n)[:n_veh]] = int(AgentClass.VEHICLE)
    params = np.array([DEFAULT_CLASS_PARAMS[AgentClass(c)] for c in (0, 1)])
    radii = params[cls, 0]
    pref = params[cls, 1]
    maxs = params[cls, 2]
    heading = rng.uniform(0.0, 2.0 * math.pi, size=n)
    speed = pref * rng.uniform(0.0, 1.0, size=n)
    vel = np.column_stack([np.cos(heading) * speed, np.sin(heading) * speed])
    gtol = np.array([cfg.goal_tolerance_for(AgentClass(int(c))) for c in (0, 1)])[cls]

    if round_f32:
        pos, vel, goals = _f32(pos), _f32(vel), _f32(goals)
        radii, pref, maxs, gtol = _f32(radii), _f32(pref), _f32(maxs), _f32(gtol)
        # float32 rounding of a jittered lattice cannot merge two centres
        # (pitch >> ulp), but make the guarantee explicit:
        key = pos[:, 0] * 1.0e7 + pos[:, 1]
        assert np.unique(key).shape[0] == n or n == 0

    state = SimState(frame=0, time=0.0, ids=np.arange(n, dtype=np.int64), positions=pos,
                     velocities=vel, radii=radii, pref_speeds=pref, max_speeds=maxs,
                     goals=goals, goal_tols=gtol, class_codes=cls,
                     rng_state=None, lp_fallbacks=0)
    return state, cfg


def blobs_crowd(n_ped: int, n_veh: int = 0, seed: int = 0, config: ScenarioConfig | None = None,
                origin=(0.0, 0.0), rho_max: float = 1.0, contrast: float = 10.0, blobs: int = 24,
                mean_density: float = 0.25) -> tuple[SimState, ScenarioConfig]:
    """A NON-uniform crowd: density rho_max/contrast in the open, rising to rho_max inside
    `blobs` Gaussian clusters, tuned to `mean_density` overall. Agents sit on slots of a fine
    jittered lattice (pitch 1/sqrt(rho_max)) thinned with probability rho(x, y)/rho_max, so
    centres never coincide. Goals: four crossing streams -- each agent walks half a plaza in
    the direction its quadrant faces (east, north, west, south)."""
    cfg = config if config is not None else ScenarioConfig()
    n = int(n_ped) + int(n_veh)
    rng = np.random.default_rng(seed)
    side = math.sqrt(max(n, 1) / mean_density)
    pitch = 1.0 / math.sqrt(rho_max)
    m = max(2, int(math.ceil(side / pitch)))
    side = m * pitch
    gx, gy = np.meshgrid(np.arange(m, dtype=np.float32), np.arange(m, dtype=np.float32), indexing="ij")
    cx, cy = (gx.ravel() + 0.5) * pitch, (gy.ravel() + 0.5) * pitch
    # blob widths chosen so the blobs hold ~ (mean - floor) of the mass
    floor = rho_max / contrast
    sigma = math.sqrt(max(mean_density - floor, 1e-3) * side * side / (blobs * 2.0 * math.pi * (rho_max - floor)))
    centres = rng.uniform(0.1 * side, 0.9 * side, size=(blobs, 2))
    bump = np.zeros(cx.shape[0], dtype=np.float32)
    for bx, by in centres:
        bump = np.maximum(bump, np.exp(-(((cx - bx) ** 2 + (cy - by) ** 2) / (2.0 * sigma * sigma))).astype(np.float32))
    p = (floor + (rho_max - floor) * bump) / rho_max
    key = rng.random(cx.shape[0]) / p                 # the n smallest keys: slots kept ~ proportionally to p
    if n > key.shape[0]:
        raise ValueError("blobs_crowd: rho_max too small for this many agents")
    slots = np.argpartition(key, n - 1)[:n] if n < key.shape[0] else np.arange(n)
    slots = slots[rng.permutation(n)]                 # storage order unrelated to space
    jitter = rng.uniform(-0.3, 0.3, size=(n, 2))
    pos = np.empty((n, 2))
    pos[:, 0] = origin[0] + cx[slots] + jitter[:, 0] * pitch
    pos[:, 1] = origin[1] + cy[slots] + jitter[:, 1] * pitch
    rel = pos - (np.asarray(origin) + side / 2)
    quadrant = (np.arctan2(rel[:, 1], rel[:, 0]) // (math.pi / 2)).astype(np.int64) % 4
    heading = quadrant * (math.pi / 2) + rng.normal(scale=0.2, size=n)
    goals = pos + np.column_stack([np.cos(heading), np.sin(heading)]) * (side / 2)

    cls = np.zeros(n, dtype=np.int64)
    if n_veh:
        cls[rng.permutation(n)[:n_veh]] = int(AgentClass.VEHICLE)
    params = np.array([DEFAULT_CLASS_PARAMS[AgentClass(c)] for c in (0, 1)])
    radii, pref, maxs = params[cls, 0], params[cls, 1], params[cls, 2]
    speed = pref * rng.uniform(0.3, 1.0, size=n)
    vel = np.column_stack([np.cos(heading) * speed, np.sin(heading) * speed])
    gtol = np.array([cfg.goal_tolerance_for(AgentClass(int(c))) for c in (0, 1)])[cls]
    pos, vel, goals = _f32(pos), _f32(vel), _f32(goals)
    radii, pref, maxs, gtol = _f32(radii), _f32(pref), _f32(maxs), _f32(gtol)
    state = SimState(frame=0, time=0.0, ids=np.arange(n, dtype=np.int64), positions=pos,
                     velocities=vel, radii=radii, pref_speeds=pref, max_speeds=maxs,
                     goals=goals, goal_tols=gtol, class_codes=cls, rng_state=None, lp_fallbacks=0)
    return state, cfg


def lp_batch(n: int, k_min: int = 8, k_max: int = 64, infeasible_frac: float = 0.0,
             seed: int = 0, round_f32: bool = True):
    """n closest-point problems, k ~ U{k_min..k_max} constraints each.

    Problems are "feasible" (witness disc, oracles.py:237-257) except a random
    fraction `infeasible_frac` drawn as unconstrained geometry
    (oracles.py:260-268; almost always infeasible at k >= 8).
    Returns (coff i64[n+1], cpts f64[m,2], cnrm f64[m,2], tgt f64[n,2],
    caps f64[n], seeds u64[n]). With round_f32 every float (normals included,
    which leaves them unit to ~6e-8) is float32-representable so an FP32 device
    path and the float64 oracle see identical inputs; solve_range itself does
    not validate normals (only the object API does, lp.py:115-130).
    """
    rng = np.random.default_rng(seed)
    ks = rng.integers(k_min, k_max + 1, size=n)
    coff = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(ks, out=coff[1:])
    m = int(coff[-1])
    owner = np.repeat(np.arange(n), ks)

    cap = 0.5 + 2.5 * rng.random(n)
    rho = cap * (0.03 + 0.27 * rng.random(n))
    ang = 2 * np.pi * rng.random(n)
    rad = (cap - rho) * np.sqrt(rng.random(n))
    cx, cy = rad * np.cos(ang), rad * np.sin(ang)

    a = 2 * np.pi * rng.random(m)
    nx, ny = np.cos(a), np.sin(a)
    slack = 2.0 * rng.random(m) ** 2
    shift = rng.normal(size=m) * cap[owner]
    off = rho[owner] + slack
    px = cx[owner] - off * nx + shift * (-ny)
    py = cy[owner] - off * ny + shift * nx

    if infeasible_frac > 0.0:
        bad = rng.random(n) < infeasible_frac
        badc = bad[owner]
        rnd = rng.normal(size=(m, 2)) * 1.2
        px = np.where(badc, rnd[:, 0], px)
        py = np.where(badc, rnd[:, 1], py)

    tgt = rng.normal(size=(n, 2)) * cap[:, None]
    seeds = rng.integers(0, 2**63, size=n, dtype=np.uint64)
    cpts = np.column_stack([px, py])
    cnrm = np.column_stack([nx, ny])
    if round_f32:
        cpts, cnrm, tgt, cap = _f32(cpts), _f32(cnrm), _f32(tgt), _f32(cap)
    return coff, np.ascontiguousarray(cpts), np.ascontiguousarray(cnrm), tgt, cap, seeds
