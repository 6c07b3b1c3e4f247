"""Host-side stand-in for the CUDA handle in the strip protocol tests (TEST
INFRASTRUCTURE: the product binds StripDriver to the C ABI via DeviceStripOps).

OracleStripOps keeps one rank's agent table in numpy, fills / reads the same slabs
as orca_strip_pack_halo / orca_strip_step / orca_strip_append_slab, and steps with the
CPU oracle exactly the way the device does: owned + ghost agents are searched, only
owned agents are solved and integrated, ghosts are dropped after the step, agents whose
new x left the strip go to the migrant slabs.
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2008_11578_b200._lib import (HALO_DTYPE_F64, RECORD_BYTES, RECORD_DTYPE,  # noqa: E402
                                        SLAB_HEADER_BYTES, SLAB_HEADER_DTYPE)
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


def _header(slab):
    return slab.numpy()[:SLAB_HEADER_BYTES].view(SLAB_HEADER_DTYPE)


def _records(slab, dtype, cap):
    return slab.numpy()[SLAB_HEADER_BYTES:SLAB_HEADER_BYTES + cap * dtype.itemsize].view(dtype)


class OracleStripOps:
    """The ops interface of StripDriver (DeviceStripOps) on host memory: the same slabs
    (32-byte header with the count + records), halo records in the FP64 layout."""

    halo_record_bytes = HALO_DTYPE_F64.itemsize

    def __init__(self, state, cfg):
        self.state, self.cfg = state, cfg
        self.n_owned = state.ids.shape[0]
        self.ghosts = self.migrants = 0
        self.overflow = False

    def configure(self, x_lo, x_hi, vmax_floor, slack_rows):
        self.lo, self.hi = x_lo, x_hi

    def pack_halo(self, reach, slab_left, slab_right, cap):
        st = self.state
        assert st.ids.shape[0] == self.n_owned, "ghost rows are resident"
        x = st.positions[:, 0]
        for slab, mask in ((slab_left, x < self.lo + reach), (slab_right, x >= self.hi - reach)):
            if slab is None:
                continue
            n = int(mask.sum())
            h = _header(slab)
            h["count"], h["overflow"] = n, 0
            rec = _records(slab, HALO_DTYPE_F64, cap)
            m = min(n, cap)
            rec["x"][:m], rec["y"][:m] = st.positions[mask, 0][:m], st.positions[mask, 1][:m]
            rec["vx"][:m], rec["vy"][:m] = st.velocities[mask, 0][:m], st.velocities[mask, 1][:m]
            rec["radius"][:m], rec["id"][:m] = st.radii[mask][:m], st.ids[mask][:m]
            rec["class_code"][:m] = st.class_codes[mask][:m]

    def append_slab(self, slab, cap, kind):
        """kind 0: immigrants (owned); 1: a received halo (ghosts); 2: own emigrants as ghosts."""
        h = _header(slab)
        count = int(h["count"][0])
        if count > cap or int(h["overflow"][0]):
            self.overflow = True
        count = min(count, cap)
        if kind == 1:
            g = _records(slab, HALO_DTYPE_F64, cap)[:count]
            rec = np.zeros(count, dtype=RECORD_DTYPE)
            for f in ("x", "y", "vx", "vy", "radius", "id", "class_code"):
                rec[f] = g[f]
            rec["goal_x"], rec["goal_y"] = g["x"], g["y"]
            self.ghosts += count
        else:
            rec = _records(slab, RECORD_DTYPE, cap)[:count].copy()
            if kind == 0:
                assert self.state.ids.shape[0] == self.n_owned
                self.migrants += count
        append_records(self.state, rec)
        if kind == 0:
            self.n_owned += count

    def step(self, mig_left, mig_right, cap):
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
        x = new.positions[:, 0]
        keep = np.ones(m, dtype=bool)
        for slab, mask in ((mig_left, x < self.lo), (mig_right, x >= self.hi)):
            if slab is None:
                assert not mask.any()
                continue
            rec = to_records(new, mask)
            h = _header(slab)
            h["count"], h["overflow"] = rec.shape[0], int(rec.shape[0] > cap)
            if rec.shape[0] > cap:
                self.overflow = True
            k = min(rec.shape[0], cap)
            _records(slab, RECORD_DTYPE, cap)[:k] = rec[:k]
            keep &= ~mask
        self.state = take(new, keep)
        self.n_owned = self.state.ids.shape[0]

    def resync(self):
        if self.overflow:
            raise RuntimeError("strip exchange: a slab overflowed")

    def stats(self):
        return self.ghosts, self.migrants


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


def crowd_for(world):
    """Strips must be at least neighbor_radius + max_speed*dt wide: a wider plaza for 3 strips."""
    return make_crowd() if world <= 2 else make_crowd(n_ped=1150, n_veh=80)


def gloo_worker(rank, world, port, steps, out_dir):
    """Entry point of one spawned rank (torch.multiprocessing.spawn)."""
    import torch
    import torch.distributed as dist

    from paper_2008_11578_b200.parallel.strips import StripDriver, strip_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        st, cfg = crowd_for(world)
        bounds = strip_bounds(st.positions[:, 0], world)
        b = [-np.inf] + list(bounds) + [np.inf]
        mine = (st.positions[:, 0] >= b[rank]) & (st.positions[:, 0] < b[rank + 1])
        ops = OracleStripOps(take(st, mine), cfg)
        drv = StripDriver(ops, rank, world, bounds, cfg.neighbor_radius, torch.device("cpu"),
                          halo_capacity=st.ids.shape[0], vmax=float(st.max_speeds.max()), dt=cfg.dt,
                          resync_every=4)
        for _ in range(steps):
            drv.step()
        drv.flush()
        out = ops.state
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), ids=out.ids, positions=out.positions,
                 velocities=out.velocities, frame=out.frame, lo=drv.lo, hi=drv.hi,
                 halo_recv=ops.stats()[0], migr_recv=ops.stats()[1], host_syncs=drv.host_syncs)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def gpu_gloo_worker(rank, world, port, steps, out_dir, precision, transport="sendrecv"):
    """One of several ranks sharing cuda:0: the CUDA handle behind DeviceStripOps; the slabs are
    staged through the host and sent over gloo ("sendrecv"), or written by each process's kernel
    into its neighbours' windows through CUDA IPC ("window") (tests/test_gpu_strips.py)."""
    import torch
    import torch.distributed as dist

    from paper_2008_11578_b200 import Simulation
    from paper_2008_11578_b200.parallel.strips import DeviceStripOps, StripDriver, strip_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        st, cfg = make_crowd(seed=4, n_ped=4000, n_veh=200, density=0.5)
        n = st.ids.shape[0]
        bounds = strip_bounds(st.positions[:, 0], world)
        b = [-np.inf] + list(bounds) + [np.inf]
        mine = (st.positions[:, 0] >= b[rank]) & (st.positions[:, 0] < b[rank + 1])
        with Simulation(cfg, capacity=2 * n, precision=precision, remove_arrivals=False) as sim:
            sim.load(take(st, mine))
            drv = StripDriver(DeviceStripOps(sim), rank, world, bounds, cfg.neighbor_radius,
                              torch.device("cuda", 0), halo_capacity=n, migrant_capacity=n // 4,
                              vmax=float(st.max_speeds.max()), dt=cfg.dt, resync_every=4,
                              transport="sendrecv" if transport == "window_fail" else transport)
            if transport == "window_fail":
                # rank 1 cannot map its neighbour's window: connect_windows must raise THERE, return on the
                # other ranks, and leave nobody behind in a collective; everyone then falls back to send/recv
                # together, the way bench.py --transport auto does
                def make(tr):
                    return StripDriver(drv.ops, rank, world, bounds, cfg.neighbor_radius, torch.device("cuda", 0),
                                       halo_capacity=n, migrant_capacity=n // 4, vmax=float(st.max_speeds.max()),
                                       dt=cfg.dt, resync_every=4, transport=tr)
                drv = make("window")
                if rank == 1:
                    def refuse(*_a, **_k):
                        raise RuntimeError("no peer access (simulated)")
                    drv.ops.window_open = refuse
                failed = 0.0
                try:
                    drv.connect_windows()
                except RuntimeError as exc:
                    assert rank == 1 and "simulated" in str(exc)
                    failed = 1.0
                bad = torch.tensor([failed], dtype=torch.float64)
                dist.all_reduce(bad)
                assert float(bad.item()) == 1.0
                drv.close()
                drv = make("sendrecv")
                assert drv._stage
            elif transport == "window":
                drv.connect_windows()
            else:
                assert drv._stage
            for _ in range(steps):
                drv.step()
            drv.flush()
            out = sim.state()
            g, m = drv.ops.stats()
            torch.cuda.synchronize()
            dist.barrier()           # nobody frees a window its neighbour may still be writing
            drv.close()
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), ids=out.ids, positions=out.positions,
                 velocities=out.velocities, halo_recv=g, migr_recv=m)
        dist.barrier()
    finally:
        dist.destroy_process_group()
