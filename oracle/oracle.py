"""ctypes front-end of the CPU oracle (oracle/orca_oracle.c).

TEST INFRASTRUCTURE ONLY -- see the header of orca_oracle.c.  Nothing under
paper_2008_11578_b200/ imports this module; it is used by tests/, by
__graft_entry__.smoke() as the checker and by bench.py's CPU-baseline legs.

Parity status: PINNED against the reference run in the build container
(oracle/gen_golden.py -> tests/golden/*.npz, checked by
tests/test_oracle_golden.py) and against the reference tests' known answers.

The functions mirror the reference's own call structure so parity tests read
like the reference's tests ("E" = pkg/src/orcasim/engine.py,
"K" = pkg/src/orcasim/_kernels.py, "L" = pkg/src/orcasim/lp.py):

    grid_arrays          E:149-161        frame_solve      K:493-556 via E:229-237
    desired_velocities   E:133-139        advance / step   E:194-308
    solve_range          K:306-336        solve_one        K:290-303 (L:152-165)
    vo_exit              K:343-419        shuffle_order    K:43-54  (L:101-112)
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
import time as _time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liborca_oracle.so")

COLLISION_TOLERANCE = 1e-6          # E:36
DEFAULT_WORK_UNIT_STEPS = 4096      # E:37

_lib = None


def build(force: bool = False) -> str:
    """Compile liborca_oracle.so with the committed Makefile (gcc only)."""
    src = os.path.join(_HERE, "orca_oracle.c")
    stale = (not os.path.exists(_LIB_PATH)
             or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src))
    if force or stale:
        subprocess.run(["make", "-C", _HERE, "-B"], check=True,
                       stdout=subprocess.DEVNULL)
    return _LIB_PATH


_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


def lib():
    global _lib
    if _lib is not None:
        return _lib
    build()
    L = C.CDLL(_LIB_PATH)
    i64, f64, u64, vp = C.c_int64, C.c_double, C.c_uint64, C.c_void_p
    L.oracle_mix64.restype = u64
    L.oracle_mix64.argtypes = [u64]
    L.oracle_problem_seed.restype = u64
    L.oracle_problem_seed.argtypes = [i64, i64]
    L.oracle_shuffle_into.restype = None
    L.oracle_shuffle_into.argtypes = [_i64p, i64, u64]
    L.oracle_solve_one.restype = C.c_int
    L.oracle_solve_one.argtypes = [_f64p, _f64p, i64, f64, f64, f64, u64, _f64p, _i64p, _i64p]
    L.oracle_least_penetration.restype = C.c_int
    L.oracle_least_penetration.argtypes = [_f64p, _f64p, i64, i64, f64, f64, f64, _f64p]
    L.oracle_solve_range.restype = C.c_int
    L.oracle_solve_range.argtypes = [_i64p, _f64p, _f64p, _f64p, _f64p, _u64p, _f64p, _i64p,
                                     _i64p, i64, i64]
    L.oracle_solve_batch.restype = C.c_int
    L.oracle_solve_batch.argtypes = [_i64p, _f64p, _f64p, _f64p, _f64p, _u64p, _f64p, _i64p,
                                     _i64p, i64, i64]
    L.oracle_vo_exit.restype = C.c_int
    L.oracle_vo_exit.argtypes = [f64, f64, f64, f64, f64, f64, f64, _f64p]
    L.oracle_grid_arrays.restype = i64
    L.oracle_grid_arrays.argtypes = [_f64p, i64, f64, _i64p, _i64p, _i64p, vp, vp]
    L.oracle_collect_neighbors.restype = i64
    L.oracle_collect_neighbors.argtypes = [i64, _f64p, _i64p, _i64p, _i64p, i64, _i64p, f64, i64,
                                           f64, i64, _f64p, _i64p, _i64p]
    L.oracle_frame_solve.restype = C.c_int
    L.oracle_frame_solve.argtypes = [_f64p, _f64p, _f64p, _f64p, _i64p, _i64p, _f64p, _f64p,
                                     _i64p, _i64p, i64, _i64p, f64, i64, f64, i64, f64, f64, i64,
                                     _f64p, _i64p, _i64p, _i64p, i64, i64, i64, vp, vp, vp]
    L.oracle_desired_velocities.restype = None
    L.oracle_desired_velocities.argtypes = [_f64p, _f64p, _f64p, f64, i64, _f64p]
    L.oracle_integrate.restype = None
    L.oracle_integrate.argtypes = [_f64p, _f64p, f64, _f64p, _f64p, i64, _f64p, _u8p]
    L.oracle_min_sep.restype = None
    L.oracle_min_sep.argtypes = [_f64p, _f64p, _i64p, _i64p, _i64p, i64, _i64p, f64, i64, f64,
                                 f64, i64, C.POINTER(f64), C.POINTER(i64)]
    _lib = L
    return L


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------------------
# LP / VO object-level helpers
# ---------------------------------------------------------------------------

def mix64(z: int) -> int:
    return int(lib().oracle_mix64(z & (2**64 - 1)))


def problem_seed(agent_id: int, frame: int) -> int:
    """E:40-43 (argument order of the public function)."""
    return int(lib().oracle_problem_seed(frame, agent_id))


def shuffle_order(count: int, seed: int) -> list[int]:
    perm = np.empty(max(count, 1), dtype=np.int64)
    lib().oracle_shuffle_into(perm, count, seed & (2**64 - 1))
    return [int(v) for v in perm[:count]]


def solve_one(pts, nrm, target, cap, seed=0):
    """-> (velocity[2], status, failed_at); K:290-303."""
    pts = _f64(pts).reshape(-1, 2)
    nrm = _f64(nrm).reshape(-1, 2)
    k = pts.shape[0]
    if k == 0:
        pts = np.zeros((1, 2))
        nrm = np.zeros((1, 2))
    out = np.empty(2)
    status = np.empty(1, dtype=np.int64)
    failed = np.empty(1, dtype=np.int64)
    rc = lib().oracle_solve_one(pts, nrm, k, float(cap), float(target[0]), float(target[1]),
                                int(seed) & (2**64 - 1), out, status, failed)
    assert rc == 0
    return out, int(status[0]), int(failed[0])


def least_penetration(pts, nrm, cap, start_index=0, warm_start=(0.0, 0.0)):
    """L:168-190 (identity order)."""
    pts = _f64(pts).reshape(-1, 2)
    nrm = _f64(nrm).reshape(-1, 2)
    k = pts.shape[0]
    if k == 0:
        pts = np.zeros((1, 2))
        nrm = np.zeros((1, 2))
    out = np.empty(2)
    rc = lib().oracle_least_penetration(pts, nrm, k, int(start_index), float(cap),
                                        float(warm_start[0]), float(warm_start[1]), out)
    assert rc == 0
    return out


def solve_range(coff, cpts, cnrm, tgt, caps, seeds, worker_count: int = 1):
    """K:306-336 over the whole batch -> (out_v[n,2], status[n], failed_at[n])."""
    coff = _i64(coff)
    n = coff.shape[0] - 1
    cpts = _f64(cpts).reshape(-1, 2)
    cnrm = _f64(cnrm).reshape(-1, 2)
    if cpts.shape[0] == 0:
        cpts = np.zeros((1, 2))
        cnrm = np.zeros((1, 2))
    tgt = _f64(tgt).reshape(-1, 2)
    caps = _f64(caps)
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    out_v = np.empty((max(n, 1), 2))
    status = np.empty(max(n, 1), dtype=np.int64)
    failed = np.empty(max(n, 1), dtype=np.int64)
    if n > 0:
        rc = lib().oracle_solve_batch(coff, cpts, cnrm, tgt, caps, seeds, out_v, status, failed,
                                      n, int(worker_count))
        assert rc == 0
    return out_v[:n], status[:n], failed[:n]


def vo_exit(rel_pos, rel_vel, combined_radius, tau, dt):
    """-> (u[2], normal[2], ok); K:343-419."""
    out = np.empty(4)
    ok = lib().oracle_vo_exit(float(rel_pos[0]), float(rel_pos[1]), float(rel_vel[0]),
                              float(rel_vel[1]), float(combined_radius), float(tau), float(dt), out)
    return out[:2].copy(), out[2:].copy(), bool(ok)


# ---------------------------------------------------------------------------
# grid + frame
# ---------------------------------------------------------------------------

def grid_arrays(positions, cell_size, with_cells: bool = False):
    """E:149-161 -> (order, ukeys, starts[, cell_ix, cell_iy])."""
    pos = _f64(positions).reshape(-1, 2)
    n = pos.shape[0]
    order = np.empty(max(n, 1), dtype=np.int64)
    ukeys = np.empty(max(n, 1), dtype=np.int64)
    starts = np.empty(n + 1, dtype=np.int64)
    cix = np.empty(max(n, 1), dtype=np.int64)
    ciy = np.empty(max(n, 1), dtype=np.int64)
    nc = lib().oracle_grid_arrays(pos if n else np.zeros((1, 2)), n, float(cell_size), order,
                                  ukeys, starts, _ptr(cix), _ptr(ciy))
    if nc == -2:
        raise ValueError("agent position out of indexable grid range")  # E:153
    assert nc >= 0
    res = (order[:n], ukeys[:nc].copy(), starts[:nc + 1].copy())
    if with_cells:
        res = res + (cix[:n], ciy[:n])
    return res


def desired_velocities(positions, goals, pref_speeds, dt):
    pos = _f64(positions).reshape(-1, 2)
    n = pos.shape[0]
    des = np.empty((n, 2))
    if n:
        lib().oracle_desired_velocities(pos, _f64(goals).reshape(-1, 2), _f64(pref_speeds),
                                        float(dt), n, des)
    return des


class FrameSolve:
    """Everything frame_solve_range writes, plus the debug taps."""

    __slots__ = ("out_v", "status", "failed_at", "err", "nb_rows", "nb_count", "constraints",
                 "cell_ix", "cell_iy", "des")


def frame_solve(state, config, worker_count: int = 1,
                work_unit_steps: int = DEFAULT_WORK_UNIT_STEPS, debug: bool = False,
                rows: int | None = None) -> FrameSolve:
    """Grid build + desired velocity + K.frame_solve_range over all agents,
    exactly as engine._advance wires them (E:211-237). With debug=True also
    returns each agent's ordered neighbour rows and ORCA constraints.
    rows=R solves only agents [0, R) (grid and desired velocities still cover
    the whole crowd) -- the bounded sample bench.py times on the host cores."""
    n = int(np.asarray(state.ids).shape[0])
    max_n = int(config.max_neighbors)
    cell_size = float(config.neighbor_radius)                               # E:211
    reach = int(math.ceil(config.neighbor_radius / cell_size))              # E:212
    rad2 = float(config.neighbor_radius) * float(config.neighbor_radius)    # E:213
    pos = _f64(state.positions).reshape(-1, 2)
    vel = _f64(state.velocities).reshape(-1, 2)
    order, ukeys, starts, cix, ciy = grid_arrays(pos, cell_size, with_cells=True)
    des = desired_velocities(pos, state.goals, state.pref_speeds, config.dt)
    fmat = _f64(config.responsibility.as_array())
    avoid = _f64(state.radii) + 0.5 * float(config.avoidance_margin)        # E:227

    out = FrameSolve()
    out.out_v = np.empty((n, 2))
    out.status = np.empty(n, dtype=np.int64)
    out.failed_at = np.empty(n, dtype=np.int64)
    out.err = np.empty(n, dtype=np.int64)
    out.cell_ix, out.cell_iy, out.des = cix, ciy, des
    out.nb_rows = out.nb_count = out.constraints = None
    n_solved = n if rows is None else min(int(rows), n)
    if debug:
        out.nb_rows = np.empty((n_solved, max(max_n, 1)), dtype=np.int64)
        out.nb_count = np.empty(n_solved, dtype=np.int64)
        # debug="lists": neighbour lists only (the constraint dump is 512 B/agent)
        out.constraints = None if debug == "lists" else np.empty((n_solved, max(max_n, 1), 4))
    if n == 0:
        return out
    rc = lib().oracle_frame_solve(
        pos, vel, avoid, _f64(state.max_speeds), _i64(state.class_codes), _i64(state.ids), fmat,
        des, _i64(order), ukeys, ukeys.shape[0], starts, cell_size, reach, rad2, max_n,
        float(config.tau), float(config.dt), int(state.frame), out.out_v, out.status,
        out.failed_at, out.err, n_solved, int(worker_count),
        int(work_unit_steps),
        _ptr(out.nb_rows), _ptr(out.nb_count), _ptr(out.constraints))
    assert rc == 0
    if debug and max_n == 0:
        out.nb_rows = out.nb_rows[:, :0]
        out.constraints = out.constraints[:, :0]
    return out


def min_separation(positions, radii, ids, cell_size, rad2, reach=1):
    """E:270-286 -> (min_separation, collision_count)."""
    pos = _f64(positions).reshape(-1, 2)
    n = pos.shape[0]
    if n < 2:
        return float("inf"), 0
    order, ukeys, starts = grid_arrays(pos, cell_size)
    best = C.c_double()
    cnt = C.c_int64()
    lib().oracle_min_sep(pos, _f64(radii), _i64(ids), _i64(order), ukeys, ukeys.shape[0], starts,
                         float(cell_size), int(reach), float(rad2), COLLISION_TOLERANCE, n,
                         C.byref(best), C.byref(cnt))
    return float(best.value), int(cnt.value)


def advance(state, config, worker_count: int = 1,
            work_unit_steps: int = DEFAULT_WORK_UNIT_STEPS, with_metrics: bool = True):
    """engine._advance (E:194-295) without the FrameLog. Returns
    (new_state, min_separation, collision_count, fallback_count, removed_ids).
    new_state is built with type(state), so any SimState-shaped dataclass works."""
    n = int(np.asarray(state.ids).shape[0])
    frame_new = state.frame + 1
    dt = float(config.dt)
    mk = type(state)
    if n == 0:                                                              # E:202-209
        new_state = mk(frame=frame_new, time=frame_new * dt, ids=state.ids,
                       positions=state.positions, velocities=state.velocities,
                       radii=state.radii, pref_speeds=state.pref_speeds,
                       max_speeds=state.max_speeds, goals=state.goals,
                       goal_tols=state.goal_tols, class_codes=state.class_codes,
                       rng_state=getattr(state, "rng_state", None))
        return new_state, float("inf"), 0, 0, state.ids

    fs = frame_solve(state, config, worker_count, work_unit_steps)
    ids = _i64(state.ids)
    bad = np.flatnonzero(fs.err >= 0)                                       # E:239-245
    if bad.size:
        i = int(bad[0])
        j = int(fs.err[i])
        raise ValueError(
            f"frame {frame_new}: agents {int(ids[i])} and {int(ids[j])} "
            "have exactly coincident centers; avoidance direction is undefined")
    fallback_count = int(np.count_nonzero(fs.status))                       # E:247

    pos = _f64(state.positions).reshape(-1, 2)
    goals = _f64(state.goals).reshape(-1, 2)
    new_pos = np.empty((n, 2))
    arrived8 = np.empty(n, dtype=np.uint8)
    lib().oracle_integrate(pos, fs.out_v, dt, goals, _f64(state.goal_tols), n, new_pos, arrived8)
    arrived = arrived8.astype(bool)
    keep = ~arrived
    removed_ids = ids[arrived]

    kept_pos = new_pos[keep]
    kept_ids = ids[keep]
    kept_radii = _f64(state.radii)[keep]
    min_sep, collisions = float("inf"), 0
    if with_metrics and kept_pos.shape[0] >= 2:
        cell_size = float(config.neighbor_radius)
        min_sep, collisions = min_separation(kept_pos, kept_radii, kept_ids, cell_size,
                                             cell_size * cell_size)
    new_state = mk(frame=frame_new, time=frame_new * dt, ids=kept_ids, positions=kept_pos,
                   velocities=fs.out_v[keep], radii=kept_radii,
                   pref_speeds=_f64(state.pref_speeds)[keep],
                   max_speeds=_f64(state.max_speeds)[keep], goals=goals[keep],
                   goal_tols=_f64(state.goal_tols)[keep],
                   class_codes=_i64(state.class_codes)[keep],
                   rng_state=getattr(state, "rng_state", None), lp_fallbacks=fallback_count)
    return new_state, min_sep, collisions, fallback_count, removed_ids


def step(state, config, worker_count: int = 1, work_unit_steps: int = DEFAULT_WORK_UNIT_STEPS):
    """engine.step (E:298-308) -> (new_state, dict of FrameMetrics fields)."""
    t0 = _time.perf_counter()
    new_state, min_sep, collisions, _fb, _removed = advance(state, config, worker_count,
                                                            work_unit_steps)
    wall_ms = (_time.perf_counter() - t0) * 1e3
    metrics = dict(frame=new_state.frame, wall_ms=wall_ms, min_separation=min_sep,
                   collision_count=collisions, active_agents=int(new_state.ids.shape[0]))
    return new_state, metrics
