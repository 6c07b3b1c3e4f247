"""Drop-in replacement for the reference's per-frame step, running on a B200.

Public surface (same names, arguments and error behaviour as the reference's
pkg/src/orcasim/engine.py):

    init_state(config[, agents])  engine.py:173-191
    step(state, config, worker_count=1, work_unit_steps=4096)
                                  engine.py:298-308 -> (SimState, FrameMetrics)
    problem_seed(agent_id, frame) engine.py:40-43
    desired_velocity(agent, dt)   engine.py:118-130

plus `Simulation`, a device-resident stepping handle for runs that do not want
a host round trip per frame (the reference's run() loop, engine.py:333-346,
without the Python between frames).

Everything numerical happens in liborca_b200.so (hand-written sm_100a CUDA,
reached through the C ABI of include/orca_b200.h). There is no CPU fallback:
without the library or without a CUDA device these functions raise.

`worker_count` / `work_unit_steps` are accepted for signature compatibility and
ignored: the reference guarantees results independent of both (engine.py:7-8).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import time as _time

import numpy as np

from . import _lib
from ._lib import OrcaError, OrcaInfo, OrcaParams, check, load, precision_code, ptr
from .types import (AgentClass, FrameLog, FrameMetrics, RunResult, RunSummary, ScenarioConfig,
                    SimState)

__all__ = ["Simulation", "init_state", "step", "run", "problem_seed", "desired_velocity",
           "DEFAULT_PRECISION", "COLLISION_TOLERANCE", "DEFAULT_WORK_UNIT_STEPS"]

COLLISION_TOLERANCE = 1e-6          # engine.py:36 (applied inside k_min_sep)
DEFAULT_WORK_UNIT_STEPS = 4096      # engine.py:37
MASK64 = (1 << 64) - 1

# "f64" (default of every reference-shaped entry point: step, run, the CLI): FP64 state and
#   arithmetic, bit-identical to the reference on ANY float64 input -- trajectories, arrival
#   frames and CSV files equal the reference's byte for byte.
# "mixed" (opt-in; what bench.py times): FP32 device state, FP64 arithmetic -- the reference's
#   branches and results for float32-representable inputs, rounded once to FP32 on store.
#   float64 inputs that float32 cannot hold are ROUNDED on upload: positions then differ from
#   the reference's by up to an FP32 ulp, and two distinct float64 centres closer than that
#   collapse (the step then raises the coincident-centres error).
# "f32" (opt-in): FP32 state and arithmetic (fastest; ill-conditioned LPs may differ > 1e-4 m/s).
# Binning and neighbour-ordering keys are FP64 in every mode.
DEFAULT_PRECISION = os.environ.get("ORCA_B200_PRECISION", "f64")


def _mix64(z: int) -> int:
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return (z ^ (z >> 31)) & MASK64


def problem_seed(agent_id: int, frame: int) -> int:
    """Shuffle seed of one agent's LP in one frame (engine.py:40-43)."""
    return _mix64(((frame & 0xFFFFFFFF) << 32) | (agent_id & 0xFFFFFFFF)) & MASK64


def desired_velocity(agent, dt: float) -> np.ndarray:
    """engine.py:118-130 for one AgentState-like object (host-side helper)."""
    if dt <= 0:
        raise ValueError(f"dt must be positive, got {dt!r}")
    dx = agent.goal[0] - agent.position[0]
    dy = agent.goal[1] - agent.position[1]
    dist = math.sqrt(dx * dx + dy * dy)
    if dist == 0.0:
        return np.zeros(2)
    speed = min(agent.pref_speed, dist / dt)
    scale = speed / dist
    return np.array([dx * scale, dy * scale])


_torch = None


def _host_empty(shape, dtype=np.float64):
    """Readback buffers. With PyTorch available they come from its caching pinned-memory
    allocator (cheap after the first call), so device->host copies run at PCIe speed;
    the numpy array keeps its tensor alive. ORCA_B200_PINNED=0 forces plain numpy."""
    global _torch
    if _torch is None:
        _torch = False
        if os.environ.get("ORCA_B200_PINNED", "1") != "0":
            try:
                import torch
                _torch = torch
            except Exception:       # torch is optional plumbing here
                _torch = False
    if _torch:
        try:
            tdt = {np.dtype(np.float64): _torch.float64, np.dtype(np.int64): _torch.int64}[np.dtype(dtype)]
            return _torch.empty(shape, dtype=tdt, pin_memory=True).numpy()
        except Exception:
            pass
    return np.empty(shape, dtype=dtype)


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a if shape is None else a.reshape(shape)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _params_from_config(config, remove_arrivals: bool, compute_metrics: bool) -> OrcaParams:
    p = OrcaParams()
    p.dt = float(config.dt)
    p.tau = float(config.tau)
    p.neighbor_radius = float(config.neighbor_radius)
    p.avoidance_margin = float(config.avoidance_margin)
    fm = np.asarray(config.responsibility.as_array(), dtype=np.float64)
    if fm.shape != (2, 2):
        raise ValueError(f"responsibility matrix must be 2x2, got {fm.shape}")
    for i in range(4):
        p.fmat[i] = float(fm.flat[i])
    p.max_neighbors = int(config.max_neighbors)
    p.remove_arrivals = 1 if remove_arrivals else 0
    p.compute_metrics = 1 if compute_metrics else 0
    return p


class Simulation:
    """A device-resident crowd: upload once, step many times, read back.

        sim = Simulation(config, capacity=state.active_count)
        sim.load(state)
        sim.run(100)                  # 100 frames, no host round trips
        state = sim.state()           # SimState of numpy float64 / int64 arrays

    remove_arrivals / compute_metrics select the parts of engine._advance that
    sit next to the steering step proper (arrival removal engine.py:251-255,
    metrics engine.py:270-286).
    """

    def __init__(self, config: ScenarioConfig, capacity: int, precision=None, device: int = 0,
                 remove_arrivals: bool = True, compute_metrics: bool = False, stream=None):
        self._L = load()
        self._h = C.c_void_p()
        self.precision = precision_code(DEFAULT_PRECISION if precision is None else precision)
        self.capacity = int(capacity)
        self.device = int(device)
        check(self._L.orca_create(C.byref(self._h), self.device, self.capacity, self.precision))
        self._rng_state = None
        self._dt = float(config.dt)
        self.set_config(config, remove_arrivals, compute_metrics)
        if stream is not None:
            self.set_stream(stream)

    # -- lifetime -----------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None) is not None and self._h:
            self._L.orca_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- configuration ------------------------------------------------------
    def set_config(self, config, remove_arrivals: bool = True, compute_metrics: bool = False):
        self._params = _params_from_config(config, remove_arrivals, compute_metrics)
        self._dt = float(config.dt)
        check(self._L.orca_set_params(self._h, C.byref(self._params)), self._h)

    def set_stream(self, stream):
        """Run on an existing CUDA stream (an int handle or a torch.cuda.Stream)."""
        handle = getattr(stream, "cuda_stream", stream)
        check(self._L.orca_set_stream(self._h, C.c_void_p(int(handle) if handle else None)), self._h)

    # -- state --------------------------------------------------------------
    def load(self, state: SimState):
        n = int(np.asarray(state.ids).shape[0])
        self._keep = (_i64(state.ids), _f64(state.positions, (n, 2)), _f64(state.velocities, (n, 2)),
                      _f64(state.radii), _f64(state.pref_speeds), _f64(state.max_speeds),
                      _f64(state.goals, (n, 2)), _f64(state.goal_tols), _i64(state.class_codes))
        check(self._L.orca_upload(self._h, n, int(state.frame), *[ptr(a) for a in self._keep]), self._h)
        self._rng_state = getattr(state, "rng_state", None)
        self._state_type = type(state)

    def load_pv(self, positions, velocities, frame: int):
        pos, vel = _f64(positions), _f64(velocities)
        n = pos.shape[0] if pos.ndim == 2 else pos.size // 2
        self._keep_pv = (pos, vel)
        check(self._L.orca_upload_pv(self._h, n, int(frame), ptr(pos), ptr(vel)), self._h)

    def step(self):
        check(self._L.orca_step(self._h), self._h)

    def run(self, steps: int):
        check(self._L.orca_run(self._h, int(steps)), self._h)

    def run_logged(self, steps: int, n_bound: int, with_trajectories: bool = False):
        """Up to `steps` frames with NO host synchronisation in between (orca_run_logged), then
        one readback of what engine.run needs per frame. `n_bound`: an upper bound on the rows
        active during these frames (the current agent count). Returns
          records  structured array (_lib.FRAME_RECORD_DTYPE), one row per frame actually
                   stepped -- fewer than `steps` when the crowd fully arrived,
          traj     float64 [rows, 4] (x, y, vx, vy), the frames' un-compacted results back to
                   back (records["rows_before"] rows each), or None,
          arrivals (ids int64[m], frames int64[m]) of the agents removed during these frames."""
        steps, n_bound = int(steps), max(int(n_bound), 1)
        rec = np.empty(max(steps, 1), dtype=_lib.FRAME_RECORD_DTYPE)
        traj = _host_empty((steps * n_bound, 4)) if with_trajectories else None
        arr_ids, arr_frames = np.empty(n_bound, dtype=np.int64), np.empty(n_bound, dtype=np.int64)
        n_rec, n_traj, n_arr = C.c_int64(), C.c_int64(), C.c_int64()
        self._raise_like_reference(self._L.orca_run_logged(
            self._h, steps, ptr(rec), C.byref(n_rec), ptr(traj), steps * n_bound if with_trajectories else 0,
            C.byref(n_traj), ptr(arr_ids), ptr(arr_frames), n_bound, C.byref(n_arr)))
        m = int(n_arr.value)
        return (rec[:int(n_rec.value)], traj[:int(n_traj.value)] if with_trajectories else None,
                (arr_ids[:m], arr_frames[:m]))

    def sync(self):
        self._raise_like_reference(self._L.orca_sync(self._h))

    def reorder_rows(self):
        """Lay the resident rows out in cell-sorted order now (orca_reorder_rows); invisible
        to every host-facing array."""
        check(self._L.orca_reorder_rows(self._h), self._h)

    def info(self) -> OrcaInfo:
        info = OrcaInfo()
        self._raise_like_reference(self._L.orca_get_info(self._h, C.byref(info)))
        return info

    def _raise_like_reference(self, rc: int):
        if rc in (_lib.ORCA_ECOINCIDENT, _lib.ORCA_ERANGE):
            # engine.py:239-245 / engine.py:152-153 raise plain ValueError with this text
            raise ValueError(self._L.orca_last_error(self._h).decode())
        check(rc, self._h)

    def profile_stages(self, enable: bool = True):
        """Record CUDA events at the stage boundaries of every following step."""
        check(self._L.orca_profile_stages(self._h, 1 if enable else 0), self._h)

    def stage_ms(self):
        """-> ({stage name: accumulated ms}, steps covered) since the last call."""
        ms = (C.c_double * _lib.ORCA_N_STAGES)()
        steps = C.c_int64()
        check(self._L.orca_get_stage_ms(self._h, ms, C.byref(steps)), self._h)
        return {name: float(ms[i]) for i, name in enumerate(_lib.STAGE_NAMES)}, int(steps.value)

    def _L_active(self) -> int:
        return int(self.info().active_agents)

    def state(self, state_type=None) -> SimState:
        info = self.info()
        n = int(info.active_agents)
        ids = _host_empty(n, np.int64)
        pos, vel, goals = _host_empty((n, 2)), _host_empty((n, 2)), _host_empty((n, 2))
        radii, pref, maxs, gtol = _host_empty(n), _host_empty(n), _host_empty(n), _host_empty(n)
        cls = _host_empty(n, np.int64)
        self._raise_like_reference(self._L.orca_download(
            self._h, ptr(ids), ptr(pos), ptr(vel), ptr(radii), ptr(pref), ptr(maxs), ptr(goals),
            ptr(gtol), ptr(cls)))
        mk = state_type or getattr(self, "_state_type", SimState)
        frame = int(info.frame)
        return mk(frame=frame, time=frame * self._dt, ids=ids, positions=pos, velocities=vel,
                  radii=radii, pref_speeds=pref, max_speeds=maxs, goals=goals, goal_tols=gtol,
                  class_codes=cls, rng_state=self._rng_state, lp_fallbacks=int(info.lp_fallbacks))

    def positions_velocities(self):
        n = int(self._L_active())
        pos, vel = _host_empty((n, 2)), _host_empty((n, 2))
        self._raise_like_reference(self._L.orca_download_pv(self._h, ptr(pos), ptr(vel)))
        return pos, vel

    def last_step_positions_velocities(self, n_pre: int):
        """Un-compacted result of the last step for every row active during that frame,
        arrivals included (what the reference logs per frame, engine.py:257-263)."""
        pos, vel = _host_empty((n_pre, 2)), _host_empty((n_pre, 2))
        self._raise_like_reference(self._L.orca_download_last_step_pv(self._h, int(n_pre), ptr(pos), ptr(vel)))
        return pos, vel

    def last_step_kept(self, n_pre: int) -> np.ndarray:
        """bool[n_pre]: which storage rows of the last step's input survived its arrival
        removal (orca_download_last_step_kept)."""
        kept = np.empty(int(n_pre), dtype=np.uint8)
        self._raise_like_reference(self._L.orca_download_last_step_kept(self._h, int(n_pre), ptr(kept)))
        return kept.astype(bool)

    def ids(self):
        n = self._L_active()
        ids = np.empty(n, dtype=np.int64)
        self._raise_like_reference(self._L.orca_download(self._h, ptr(ids), *([None] * 8)))
        return ids

    def step_host(self, positions, velocities, frame: int, out_pos=None, out_vel=None,
                  out_status=None):
        """One frame through host buffers (orca_step_host): H2D of positions and
        velocities, the step, D2H of the results. Needs remove_arrivals=False."""
        pos, vel = _f64(positions), _f64(velocities)
        n = pos.shape[0]
        out_pos = np.empty((n, 2)) if out_pos is None else out_pos
        out_vel = np.empty((n, 2)) if out_vel is None else out_vel
        self._raise_like_reference(self._L.orca_step_host(
            self._h, n, int(frame), ptr(pos), ptr(vel), ptr(out_pos), ptr(out_vel), ptr(out_status)))
        return out_pos, out_vel

    def advance_host(self, positions, velocities, frame: int):
        """One frame of engine._advance through host buffers with overlapped copies
        (orca_advance_host): -> (new_positions, new_velocities, info). The returned arrays
        are the first info.active_agents rows of pinned buffers sized for the input."""
        pos, vel = _f64(positions), _f64(velocities)
        n = pos.shape[0] if pos.ndim == 2 else pos.size // 2
        self._keep_pv = (pos, vel)
        out_pos, out_vel = _host_empty((n, 2)), _host_empty((n, 2))
        info = OrcaInfo()
        self._raise_like_reference(self._L.orca_advance_host(
            self._h, n, int(frame), ptr(pos), ptr(vel), ptr(out_pos), ptr(out_vel), C.byref(info)))
        m = int(info.active_agents)
        return out_pos[:m], out_vel[:m], info

    def attributes(self):
        """The seven per-agent arrays a step never changes, as resident now (after a frame
        that removed agents: the compacted ones), in _STATIC order."""
        n = self._L_active()
        ids, cls = _host_empty(n, np.int64), _host_empty(n, np.int64)
        goals = _host_empty((n, 2))
        radii, pref, maxs, gtol = _host_empty(n), _host_empty(n), _host_empty(n), _host_empty(n)
        self._raise_like_reference(self._L.orca_download(
            self._h, ptr(ids), None, None, ptr(radii), ptr(pref), ptr(maxs), ptr(goals), ptr(gtol), ptr(cls)))
        return ids, radii, pref, maxs, goals, gtol, cls

    def debug_last_step(self, n: int, max_neighbors: int):
        """Parity taps of the last step (orca_debug_last_step), storage-row order."""
        k = max(int(max_neighbors), 1)
        out = dict(cell_ix=np.empty(n, dtype=np.int64), cell_iy=np.empty(n, dtype=np.int64),
                   nb_rows=np.full((n, k), -1, dtype=np.int64), nb_count=np.empty(n, dtype=np.int64),
                   out_v=np.empty((n, 2)), status=np.empty(n, dtype=np.int64),
                   failed_at=np.empty(n, dtype=np.int64), des=np.empty((n, 2)))
        self._raise_like_reference(self._L.orca_debug_last_step(
            self._h, n, ptr(out["cell_ix"]), ptr(out["cell_iy"]), ptr(out["nb_rows"]),
            ptr(out["nb_count"]), ptr(out["out_v"]), ptr(out["status"]), ptr(out["failed_at"]),
            ptr(out["des"])))
        if max_neighbors == 0:
            out["nb_rows"] = out["nb_rows"][:, :0]
        return out


# ---------------------------------------------------------------------------
# reference-shaped functions
# ---------------------------------------------------------------------------

def init_state(config: ScenarioConfig, agents=None) -> SimState:
    """Start agents at their desired velocities (engine.py:173-191).

    Without `agents` the crowd is spawned from config.regions with the reference's seeded
    sampling (scenario.spawn_arrays: same seed, same crowd, bit for bit). `agents` may
    instead be a list of already spawned agents (objects with id, position, radius,
    pref_speed, max_speed, goal, agent_class -- e.g. orcasim.AgentState)."""
    if agents is None:
        agents = getattr(config, "agents", None)
    if agents is None:
        from .scenario import spawn_arrays
        a = spawn_arrays(config)
        ids, positions, goals, codes = a["ids"], a["positions"], a["goals"], a["class_codes"]
        radii, pref, maxs = a["radii"], a["pref_speeds"], a["max_speeds"]
        n = ids.shape[0]
    else:
        n = len(agents)
        ids = np.array([a.id for a in agents], dtype=np.int64)
        positions = np.array([a.position for a in agents], dtype=np.float64).reshape(n, 2)
        radii = np.array([a.radius for a in agents], dtype=np.float64)
        pref = np.array([a.pref_speed for a in agents], dtype=np.float64)
        maxs = np.array([a.max_speed for a in agents], dtype=np.float64)
        goals = np.array([a.goal for a in agents], dtype=np.float64).reshape(n, 2)
        codes = np.array([int(a.agent_class) for a in agents], dtype=np.int64)
    tol_of = {int(c): config.goal_tolerance_for(AgentClass(int(c))) for c in np.unique(codes)}
    gtols = np.array([tol_of[int(c)] for c in codes], dtype=np.float64)
    # engine.py:133-139 (host-side setup, once per run)
    d = goals - positions
    dist = np.sqrt(d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1])
    speed = np.minimum(pref, dist / config.dt)
    safe = np.where(dist > 0.0, dist, 1.0)
    scale = np.where(dist > 0.0, speed / safe, 0.0)
    velocities = d * scale[:, None]
    return SimState(frame=0, time=0.0, ids=ids, positions=positions, velocities=velocities,
                    radii=radii, pref_speeds=pref, max_speeds=maxs, goals=goals, goal_tols=gtols,
                    class_codes=codes, rng_state=np.random.default_rng(config.seed))


_handles: dict = {}
_STATIC = ("ids", "radii", "pref_speeds", "max_speeds", "goals", "goal_tols", "class_codes")


def _handle_for(config, n: int, precision, device: int) -> Simulation:
    """step() keeps one device handle per (device, precision) and grows it on demand."""
    key = (device, precision_code(DEFAULT_PRECISION if precision is None else precision))
    sim = _handles.get(key)
    if sim is None or sim.capacity < n:
        if sim is not None:
            sim.close()
        cap = max(1024, int(n * 1.25))
        sim = Simulation(config, cap, precision=key[1], device=device,
                         remove_arrivals=True, compute_metrics=True)
        sim._resident = None
        _handles[key] = sim
        _prewarm_host_buffers(n)       # the allocator pools by rounded size: warm the size in use
    return sim


def _prewarm_host_buffers(n: int):
    """Page-locking host memory costs ~0.3 ms per MB the first time. A step() loop needs,
    live at once, the returned state and the previous one: 2 x (pos, vel) always and, on
    a frame that removes arrived agents, 2 x the seven attribute arrays as well. Allocate
    and release them once so the caching pinned allocator serves every later call,
    including the first frame with arrivals, from its pool."""
    bufs = []
    for _ in range(2):
        bufs += [_host_empty((n, 2)) for _ in range(3)]                 # positions, velocities, goals
        bufs += [_host_empty(n) for _ in range(4)]                      # radii, pref, max, tolerances
        bufs += [_host_empty(n, np.int64) for _ in range(2)]            # ids, classes
    del bufs


def step(state: SimState, config: ScenarioConfig, worker_count: int = 1,
         work_unit_steps: int = DEFAULT_WORK_UNIT_STEPS, *, precision=None, device: int = 0,
         reuse_resident: bool = True):
    """Advance one frame on the GPU; returns (new_state, FrameMetrics) exactly
    like the reference's engine.step (engine.py:298-308). `state` is not
    modified. Raises ValueError with the reference's messages for coincident
    centres (engine.py:239-245) and out-of-range positions (engine.py:152-153).

    Host traffic: positions and velocities go up and come back every call. The
    per-agent attributes a step never changes (ids, radii, speeds, goals, tolerances,
    classes) stay resident on the device between calls when `state` carries the very
    array objects the previous call returned (the usual `state, m = step(state, cfg)`
    loop); the returned state shares those arrays with the input when nobody arrived and
    otherwise holds the input's own float64 values, compacted (the device keeps float64
    copies of the attributes next to an FP32 state, so nothing comes back rounded). Pass reuse_resident=False if you mutate them in
    place between calls."""
    del worker_count, work_unit_steps  # results do not depend on them (engine.py:7-8)
    t0 = _time.perf_counter()
    n = int(np.asarray(state.ids).shape[0])
    sim = _handle_for(config, n, precision, device)
    sim.set_config(config, remove_arrivals=True, compute_metrics=True)
    static = tuple(getattr(state, f) for f in _STATIC)
    res = getattr(sim, "_resident", None)
    if not (reuse_resident and res is not None and len(res) == len(static)
            and all(a is b for a, b in zip(res, static)) and sim._L_active() == n):
        sim.load(state)                     # everything goes up (104 B/agent), then pos/vel again below
        h2d = 136 * n
    else:
        h2d = 32 * n                        # positions + velocities only
    sim._rng_state = getattr(state, "rng_state", None)
    sim._state_type = type(state)
    sim._resident = None
    # positions/velocities in, step, positions/velocities out, copies overlapped with the
    # bin build / the metrics (orca_advance_host); raises the reference's ValueError on
    # device-side errors
    pos, vel, info = sim.advance_host(state.positions, state.velocities, state.frame)
    frame = int(info.frame)
    d2h = 32 * n
    if int(info.removed_agents) == 0:
        new_static = static if reuse_resident else tuple(np.array(a, copy=True) for a in static)
    else:
        # compacted on the device (engine.py:288-294) and read back from its float64 copies of
        # what the host uploaded -- bit for bit the caller's own values in every precision mode
        # (3 ms for a million agents; compacting seven arrays with a mask on the host takes 20+)
        new_static = sim.attributes()
        d2h += 72 * int(info.active_agents)
    new_state = type(state)(frame=frame, time=frame * float(config.dt), positions=pos, velocities=vel,
                            rng_state=getattr(state, "rng_state", None),
                            lp_fallbacks=int(info.lp_fallbacks), **dict(zip(_STATIC, new_static)))
    step.last_traffic = (h2d, d2h)          # bytes copied host->device, device->host by this call
    sim._resident = tuple(getattr(new_state, f) for f in _STATIC)
    wall_ms = (_time.perf_counter() - t0) * 1e3
    n2 = new_state.ids.shape[0]
    min_sep = float(info.min_separation) if n2 >= 2 else float("inf")
    metrics = FrameMetrics(frame=new_state.frame, wall_ms=wall_ms, min_separation=min_sep,
                           collision_count=int(info.collision_count) if n2 >= 2 else 0,
                           active_agents=int(n2))
    return new_state, metrics


RUN_CHUNK_FRAMES = 64                 # frames between host synchronisations in run()
RUN_CHUNK_TRAJ_BYTES = 256 << 20      # ... fewer when trajectories of a large crowd are recorded


def run(config: ScenarioConfig, worker_count: int = 1, record_trajectories: bool = True,
        work_unit_steps: int = DEFAULT_WORK_UNIT_STEPS, *, agents=None, state: SimState | None = None,
        precision=None, device: int = 0) -> RunResult:
    """Step until every agent reaches its goal or the frame guard trips (engine.py:311-370).
    The crowd stays on the device for the whole run and the HOST IS NOT IN THE FRAME LOOP: frames
    are issued in chunks of up to RUN_CHUNK_FRAMES (orca_run_logged); the per-frame metrics, the
    fallback counts, who arrived when and -- when record_trajectories is set -- every frame's
    positions and velocities accumulate in device buffers and are read back once per chunk (one
    synchronisation per chunk; `run.last_host_syncs` counts them). A frame that would start with no
    agents left is never stepped, exactly like the reference's loop. FrameMetrics.wall_ms is the
    chunk's wall time divided by its frames (a per-frame wall time needs a per-frame sync).
    `agents` / `state` supply an already spawned crowd; otherwise it is sampled from config.regions
    with the reference's seeded sampler. summary.terminated is False when the guard stopped the run."""
    del worker_count, work_unit_steps
    if state is None:
        state = init_state(config, agents)
    n0 = state.active_count
    agent_records = [{"id": int(state.ids[i]), "agent_class": AgentClass(int(state.class_codes[i])),
                      "spawn": state.positions[i].copy(), "goal": state.goals[i].copy(),
                      "radius": float(state.radii[i])} for i in range(n0)]
    guard = config.frame_guard()
    logs, metrics, arrival, fallbacks = [], [], {}, 0
    ids = np.ascontiguousarray(state.ids, dtype=np.int64)
    classes = np.asarray(state.class_codes).astype(np.int8)
    radii = np.ascontiguousarray(state.radii, dtype=np.float64)
    frame, dt = int(state.frame), float(config.dt)
    sim = Simulation(config, capacity=max(n0, 1), precision=precision, device=device,
                     remove_arrivals=True, compute_metrics=True)
    run.last_host_syncs = 0
    try:
        sim.load(state)
        while ids.shape[0] > 0 and frame < guard:
            chunk = min(RUN_CHUNK_FRAMES, guard - frame)
            if record_trajectories:
                chunk = max(1, min(chunk, RUN_CHUNK_TRAJ_BYTES // (32 * ids.shape[0])))
            t0 = _time.perf_counter()
            recs, traj, (arr_ids, arr_frames) = sim.run_logged(chunk, ids.shape[0], record_trajectories)
            run.last_host_syncs += 1
            wall_ms = (_time.perf_counter() - t0) * 1e3 / max(len(recs), 1)
            row0 = 0
            for r in recs:
                frame = int(r["frame"])
                n_pre = int(r["rows_before"])
                if record_trajectories:
                    block = traj[row0:row0 + n_pre]
                    row0 += n_pre
                    logs.append(FrameLog(frame=frame, time=frame * dt, ids=ids.copy(), classes=classes.copy(),
                                         positions=np.ascontiguousarray(block[:, 0:2]),
                                         velocities=np.ascontiguousarray(block[:, 2:4]), radii=radii.copy()))
                if int(r["removed_agents"]):
                    gone_ids = arr_ids[arr_frames == frame]
                    for agent_id in gone_ids:
                        arrival[int(agent_id)] = frame * dt
                    keep = ~np.isin(ids, gone_ids, assume_unique=True)
                    ids, classes, radii = ids[keep], classes[keep], radii[keep]
                n2 = int(r["active_agents"])
                metrics.append(FrameMetrics(
                    frame=frame, wall_ms=wall_ms,
                    min_separation=float(r["min_separation"]) if n2 >= 2 else float("inf"),
                    collision_count=int(r["collision_count"]) if n2 >= 2 else 0, active_agents=n2))
                fallbacks += int(r["lp_fallbacks"])
            if len(recs) < chunk:          # the device stopped stepping: nobody is left
                break
        final_state = sim.state(type(state))
    finally:
        sim.close()
    wall = np.array([m.wall_ms for m in metrics]) if metrics else np.zeros(1)
    class_of = {rec["id"]: rec["agent_class"] for rec in agent_records}
    travel = {}
    for cls in AgentClass:
        times = [t for agent_id, t in arrival.items() if class_of[agent_id] == cls]
        if times:
            travel[cls] = float(np.mean(times))
    summary = RunSummary(
        total_collisions=int(sum(m.collision_count for m in metrics)),
        min_separation=float(min((m.min_separation for m in metrics), default=np.inf)),
        mean_frame_ms=float(wall.mean()), p95_frame_ms=float(np.percentile(wall, 95)), agents=n0,
        seed=config.seed, frames=frame, terminated=ids.shape[0] == 0, arrived=len(arrival),
        total_fallbacks=fallbacks, mean_travel_time=travel)
    return RunResult(frame_logs=logs, frame_metrics=metrics, summary=summary,
                     agent_records=agent_records, final_state=final_state)
