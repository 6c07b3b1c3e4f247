"""Host-side stand-in for the CUDA handle in the strip protocol tests (TEST
INFRASTRUCTURE: the product binds StripDriver to the C ABI via DeviceStripOps).

OracleStripOps keeps one rank's agent table in numpy, packs / appends the same
96-byte records as orca_strip_pack / orca_strip_append, and steps with the CPU
oracle exactly the way the device does: owned + ghost agents are searched, only
owned agents are solved and integrated, ghosts are dropped after the step.
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2008_11578_b200._lib import RECORD_BYTES, RECORD_DTYPE  # noqa: E402
from paper_2008_11578_b200.types import SimState  # noqa: E402

FIELDS = ("ids", "positions", "velocities", "radii", "pref_speeds", "max_speeds", "goals",
          "goal_tols", "class_codes")


def take(state, mask):
    return SimState(frame=state.frame, time=state.time,
                    **{f: getattr(state, f)[mask].copy() for f in FIELDS})


def to_records(state, mask):
    n = int(mask.sum())
    r = np.zeros(n, dtype=RECORD_DTYPE)
    r["x"], r["y"] = state.positions[mask, 0], state.positions[mask, 1]
    r["vx"], r["vy"] = state.velocities[mask, 0], state.velocities[mask, 1]
    r["radius"], r["pref_speed"] = state.radii[mask], state.pref_speeds[mask]
    r["max_speed"], r["goal_tol"] = state.max_speeds[mask], state.goal_tols[mask]
    r["goal_x"], r["goal_y"] = state.goals[mask, 0], state.goals[mask, 1]
    r["id"], r["class_code"] = state.ids[mask], state.class_codes[mask]
    return r


def append_records(state, r):
    cat = np.concatenate
    state.ids = cat([state.ids, r["id"]])
    state.positions = cat([state.positions, np.column_stack([r["x"], r["y"]])])
    state.velocities = cat([state.velocities, np.column_stack([r["vx"], r["vy"]])])
    state.radii = cat([state.radii, r["radius"]])
    state.pref_speeds = cat([state.pref_speeds, r["pref_speed"]])
    state.max_speeds = cat([state.max_speeds, r["max_speed"]])
    state.goals = cat([state.goals, np.column_stack([r["goal_x"], r["goal_y"]])])
    state.goal_tols = cat([state.goal_tols, r["goal_tol"]])
    state.class_codes = cat([state.class_codes, r["class_code"]])


class OracleStripOps:
    def __init__(self, state, cfg):
        self.state, self.cfg = state, cfg
        self.n_owned = state.ids.shape[0]

    def pack(self, x_lo, x_hi, remove, buf):
        st = self.state
        n = st.ids.shape[0]
        mask = np.zeros(n, dtype=bool)
        x = st.positions[: self.n_owned, 0]
        mask[: self.n_owned] = (x >= x_lo) & (x < x_hi)
        rec = to_records(st, mask)
        assert rec.nbytes <= buf.numel()
        buf.numpy()[: rec.nbytes] = rec.view(np.uint8)
        if remove and rec.shape[0]:
            assert n == self.n_owned, "cannot remove rows while ghosts are resident"
            self.state = take(st, ~mask)
            self.n_owned = self.state.ids.shape[0]
        return rec.shape[0]

    def append(self, buf, count, ghost):
        if not count:
            return
        rec = buf.numpy()[: count * RECORD_BYTES].view(RECORD_DTYPE).copy()
        if not ghost:
            assert self.state.ids.shape[0] == self.n_owned
        append_records(self.state, rec)
        if not ghost:
            self.n_owned += count

    def step(self):
        st, cfg = self.state, self.cfg
        m = self.n_owned
        fs = O.frame_solve(st, cfg, rows=m)
        assert np.all(fs.err[:m] == -1)
        owned = np.zeros(st.ids.shape[0], dtype=bool)
        owned[:m] = True
        new = take(st, owned)
        new.positions = st.positions[:m] + fs.out_v[:m] * cfg.dt      # engine.py:249
        new.velocities = fs.out_v[:m].copy()
        new.frame = st.frame + 1
        new.time = new.frame * cfg.dt
        self.state = new
        self.n_owned = m


def reference_run(state, cfg, steps):
    """Single-domain reference: `steps` frames without arrival removal."""
    st = take(state, np.ones(state.ids.shape[0], dtype=bool))
    for _ in range(steps):
        fs = O.frame_solve(st, cfg, worker_count=4)
        st.positions = st.positions + fs.out_v * cfg.dt
        st.velocities = fs.out_v
        st.frame += 1
    return st


def make_crowd(seed=0, n_ped=700, n_veh=60, density=0.35):
    """A crowd whose agents stream across x so strips see steady migration."""
    from paper_2008_11578_b200.synth import plaza_crowd
    st, cfg = plaza_crowd(n_ped, n_veh, density=density, seed=seed)
    rng = np.random.default_rng(seed + 1)
    side = float(st.positions[:, 0].max())
    # goals on the far side: left half heads right and vice versa
    left = st.positions[:, 0] < side / 2
    gx = np.where(left, side * (0.75 + 0.25 * rng.random(left.shape[0])),
                  side * 0.25 * rng.random(left.shape[0]))
    st.goals[:, 0] = gx.astype(np.float32)
    st.velocities[:, 0] = (np.where(left, 1.0, -1.0) * st.pref_speeds).astype(np.float32)
    st.velocities[:, 1] = 0.0
    return st, cfg


def gloo_worker(rank, world, port, steps, out_dir):
    """Entry point of one spawned rank (torch.multiprocessing.spawn)."""
    import torch
    import torch.distributed as dist

    from paper_2008_11578_b200.parallel.strips import StripDriver, strip_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        st, cfg = make_crowd()
        bounds = strip_bounds(st.positions[:, 0], world)
        b = [-np.inf] + list(bounds) + [np.inf]
        mine = (st.positions[:, 0] >= b[rank]) & (st.positions[:, 0] < b[rank + 1])
        ops = OracleStripOps(take(st, mine), cfg)
        drv = StripDriver(ops, rank, world, bounds, cfg.neighbor_radius, torch.device("cpu"),
                          halo_capacity=st.ids.shape[0])
        for _ in range(steps):
            drv.step()
        out = ops.state
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), ids=out.ids, positions=out.positions,
                 velocities=out.velocities, frame=out.frame, lo=drv.lo, hi=drv.hi,
                 **{k: v for k, v in drv.stats.items()})
        dist.barrier()
    finally:
        dist.destroy_process_group()
