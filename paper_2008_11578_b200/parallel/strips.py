"""Strip-decomposed stepping: the crowd is cut into vertical strips along x, one
rank (one GPU) per strip; every step neighbouring strips swap halo agents before
the solve and migrating agents after it.

The reference has no multi-process path at all; what must hold is
its synchronous-update rule: an agent's new velocity depends
only on the pre-step snapshot of the agents within neighbor_radius, so a rank that
sees its owned agents plus every foreign agent within neighbor_radius of its strip
computes exactly what a single device would. Per step and per rank:

  1. halo     pack owned agents with x in [lo, lo+nr] / [hi-nr, hi)   (C ABI:
              orca_strip_pack) and send them left / right; append what arrives
              as ghosts (orca_strip_append, ghost=1)
  2. step     orca_step solves owned agents only and drops the ghosts
  3. migrate  pack-and-remove owned agents whose new x left [lo, hi), send,
              append arrivals as owned rows

The exchange is point-to-point with the two adjacent strips only (counts first,
then the 96-byte records as raw bytes); there is no collective on the data path.
`StripDriver` holds this protocol and is written against a small ops interface so
the same code runs on NCCL with the CUDA handle (DeviceStripOps) and, in the CPU
tests, on gloo with a host-side stand-in (tests/strip_ops_cpu.py).

Constraint: a strip must be wider than neighbor_radius + max_speed*dt (an agent
may cross at most one boundary per step, and a halo reaches one strip deep).
"""

from __future__ import annotations

import ctypes as C
import json
import math
import time

import numpy as np
import torch
import torch.distributed as dist

from .._lib import RECORD_BYTES, check, load

__all__ = ["DeviceStripOps", "StripDriver", "strip_bounds", "run_bench"]


def strip_bounds(x: np.ndarray, world: int) -> np.ndarray:
    """Interior strip boundaries (world-1 values) that split the agents evenly:
    quantiles of the x coordinates. Strip r owns x in [b[r-1], b[r]) with
    b[-1] = -inf and b[world-1] = +inf."""
    if world <= 1:
        return np.zeros(0)
    qs = np.arange(1, world) / world
    return np.quantile(np.asarray(x, dtype=np.float64), qs)


class DeviceStripOps:
    """pack / append on a Simulation's resident state through the C ABI."""

    def __init__(self, sim):
        self.sim = sim
        self._L = load()

    def pack(self, x_lo: float, x_hi: float, remove: bool, buf: torch.Tensor) -> int:
        count = C.c_int64()
        cap = buf.numel() // RECORD_BYTES
        check(self._L.orca_strip_pack(self.sim._h, float(x_lo), float(x_hi), 1 if remove else 0,
                                      C.c_void_p(buf.data_ptr()), cap, C.byref(count)), self.sim._h)
        return int(count.value)

    def append(self, buf: torch.Tensor, count: int, ghost: bool):
        if count:
            check(self._L.orca_strip_append(self.sim._h, C.c_void_p(buf.data_ptr()), int(count),
                                            1 if ghost else 0), self.sim._h)

    def step(self):
        self.sim.step()

    def reorder(self):
        self.sim.reorder_rows()


class StripDriver:
    """One rank's side of the strip protocol."""

    def __init__(self, ops, rank: int, world: int, bounds, neighbor_radius: float, device,
                 halo_capacity: int, group=None):
        self.ops, self.rank, self.world, self.group = ops, rank, world, group
        b = [-math.inf] + [float(v) for v in bounds] + [math.inf]
        assert len(b) == world + 1 and all(b[i] <= b[i + 1] for i in range(world))
        self.lo, self.hi = b[rank], b[rank + 1]
        self.left = rank - 1 if rank > 0 else None
        self.right = rank + 1 if rank < world - 1 else None
        # halo reach with a relative margin: including a few extra agents is harmless,
        # missing one that sits exactly at distance neighbor_radius is not
        self.reach = float(neighbor_radius) * (1.0 + 1e-9) + 1e-9
        self.device = device
        nbytes = int(halo_capacity) * RECORD_BYTES
        mk = lambda: torch.empty(nbytes, dtype=torch.uint8, device=device)  # noqa: E731
        self.send = {"left": mk(), "right": mk()}
        self.recv = {"left": mk(), "right": mk()}
        self.capacity = int(halo_capacity)
        self.stats = {"halo_sent": 0, "halo_recv": 0, "migr_sent": 0, "migr_recv": 0}
        self.frames = 0
        self.reorder_every = 64      # frames between row reorderings (no ghosts resident then)

    # -- one exchange with both neighbours --------------------------------------
    def _swap(self, counts: dict) -> dict:
        """Send self.send[side][:counts[side]] to that side, receive into self.recv.
        Returns the received counts. Counts travel first, then the payloads."""
        peers = {"left": self.left, "right": self.right}
        cnt_out = {s: torch.tensor([counts.get(s, 0)], dtype=torch.int64, device=self.device)
                   for s in peers}
        cnt_in = {s: torch.zeros(1, dtype=torch.int64, device=self.device) for s in peers}
        ops = []
        for s, p in peers.items():
            if p is not None:
                ops.append(dist.P2POp(dist.isend, cnt_out[s], p, group=self.group))
                ops.append(dist.P2POp(dist.irecv, cnt_in[s], p, group=self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        got = {s: int(cnt_in[s].item()) if peers[s] is not None else 0 for s in peers}
        ops = []
        for s, p in peers.items():
            if p is None:
                continue
            if got[s] > self.capacity:
                raise RuntimeError(f"rank {self.rank}: {got[s]} records from the {s} exceed the "
                                   f"exchange capacity {self.capacity}")
            if counts.get(s, 0):
                ops.append(dist.P2POp(dist.isend, self.send[s][:counts[s] * RECORD_BYTES], p,
                                      group=self.group))
            if got[s]:
                ops.append(dist.P2POp(dist.irecv, self.recv[s][:got[s] * RECORD_BYTES], p,
                                      group=self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            if self.device.type == "cuda":
                # the append kernels run on the handle's stream, the NCCL copies on torch's:
                # make the received records globally visible before anyone reads them
                torch.cuda.current_stream(self.device).synchronize()
        return got

    # -- protocol phases (split so a test can drive two ranks in one process) ------
    def pack_halo(self) -> dict:
        counts = {}
        if self.left is not None:
            counts["left"] = self.ops.pack(self.lo, self.lo + self.reach, False, self.send["left"])
        if self.right is not None:
            counts["right"] = self.ops.pack(self.hi - self.reach, self.hi, False, self.send["right"])
        self.stats["halo_sent"] += sum(counts.values())
        return counts

    def unpack_halo(self, got: dict):
        for s in ("left", "right"):
            self.ops.append(self.recv[s], got.get(s, 0), True)
        self.stats["halo_recv"] += sum(got.values())

    def pack_migrants(self) -> dict:
        counts = {}
        if self.left is not None:
            counts["left"] = self.ops.pack(-math.inf, self.lo, True, self.send["left"])
        if self.right is not None:
            counts["right"] = self.ops.pack(self.hi, math.inf, True, self.send["right"])
        self.stats["migr_sent"] += sum(counts.values())
        return counts

    def unpack_migrants(self, got: dict):
        for s in ("left", "right"):
            self.ops.append(self.recv[s], got.get(s, 0), False)
        self.stats["migr_recv"] += sum(got.values())

    def exchange_halo(self):
        self.unpack_halo(self._swap(self.pack_halo()))

    def migrate(self):
        self.unpack_migrants(self._swap(self.pack_migrants()))

    def step(self):
        """One frame of the whole strip-decomposed crowd, as seen by this rank."""
        if self.reorder_every and self.frames % self.reorder_every == 0 and hasattr(self.ops, "reorder"):
            self.ops.reorder()       # rows in cell order: memory coherence only, results unchanged
        self.frames += 1
        self.exchange_halo()
        self.ops.step()
        self.migrate()


# ---------------------------------------------------------------------------
# bench.py --gpus N (torchrun, one rank per GPU)
# ---------------------------------------------------------------------------

def run_bench(args, rank: int, world: int, local: int):
    """Weak scaling: every rank owns one `workload` plaza; the plazas sit side by
    side along x and form one crowd of world * n agents with halo exchange and
    migration every step. Prints the JSON line on rank 0."""
    from .. import Simulation
    from ..synth import CONFIGS, plaza_crowd

    n_ped, n_veh, density = CONFIGS[args.workload]
    n_local = n_ped + n_veh
    side = math.sqrt(n_local / density)
    state, cfg = plaza_crowd(n_ped, n_veh, density=density, seed=100 + rank, origin=(rank * side, 0.0))
    state.ids = state.ids + rank * n_local
    # goals anywhere in the whole crowd's plaza, so agents do cross strip boundaries
    rng = np.random.default_rng(1000 + rank)
    state.goals[:, 0] = rng.uniform(0.0, world * side, size=n_local).astype(np.float32)
    bounds = [side * r for r in range(1, world)]
    device = torch.device("cuda", local)
    stream = torch.cuda.Stream(device)
    torch.cuda.set_stream(stream)       # NCCL ops order themselves against the current stream
    capacity = int(n_local * 1.15) + 65536
    sim = Simulation(cfg, capacity=capacity, precision=args.precision, device=local,
                     remove_arrivals=False, stream=stream)
    sim.load(state)
    halo_cap = int(4 * cfg.neighbor_radius * side * density) + 65536
    drv = StripDriver(DeviceStripOps(sim), rank, world, bounds, cfg.neighbor_radius, device, halo_cap)

    for _ in range(max(args.warmup, 3)):
        drv.step()
    sim.sync()
    l0 = sim.info().kernel_launches
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = args.make_sampler() if hasattr(args, "make_sampler") else None
    if sampler is not None:
        sampler.__enter__()
    e0.record(stream)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        drv.step()
    e1.record(stream)
    sim.sync()
    torch.cuda.synchronize()
    wall_ms = (time.perf_counter() - t0) * 1e3
    if sampler is not None:
        sampler.__exit__(None, None, None)
    ms = torch.tensor([max(e0.elapsed_time(e1), 0.0), wall_ms], device=device, dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    info = sim.info()
    tot = torch.tensor([float(info.active_agents), float(info.kernel_launches - l0),
                        float(drv.stats["halo_sent"]), float(drv.stats["migr_sent"])],
                       device=device, dtype=torch.float64)
    dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    dist.barrier()

    # ---- e2e: the same step with this rank's positions / velocities going up from pinned host
    # memory and coming back every frame (what a host-side caller of a strip-decomposed crowd pays)
    e2e_steps = max(3, min(args.steps, getattr(args, "e2e_steps", 20)))
    pos, vel = sim.positions_velocities()
    h2d = d2h = 0
    for k in range(2 + e2e_steps):
        if k == 2:
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            h2d = d2h = 0
        sim.load_pv(pos, vel, int(sim.info().frame))
        h2d += pos.nbytes + vel.nbytes
        drv.step()
        pos, vel = sim.positions_velocities()
        d2h += pos.nbytes + vel.nbytes
    torch.cuda.synchronize()
    e2e = torch.tensor([(time.perf_counter() - t0) * 1e3 / e2e_steps], device=device, dtype=torch.float64)
    dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    io = torch.tensor([float(h2d), float(d2h), float(sim.info().active_agents)], device=device, dtype=torch.float64)
    dist.all_reduce(io, op=dist.ReduceOp.SUM)

    # ---- roofline of the dominant kernel on rank 0 (same definition as the N=1 line)
    sim.profile_stages(True)
    for _ in range(5):
        drv.step()
    stage_ms, covered = sim.stage_ms()
    sim.profile_stages(False)
    stage_ms = {k: v / max(covered, 1) for k, v in stage_ms.items()}
    dist.barrier()
    if rank == 0:
        import os
        hbm_peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
        pk = os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))),
                          "MEASURED_PEAKS.json")
        if os.path.exists(pk):
            with open(pk) as f:
                hbm_peak, peak_src = float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
        solve_bytes = (16 + 32 + 1 + 4 * 16 + 1 + 16 + 16 + 2 + 1) * n_local     # bench.py SOLVE_BYTES_PER_AGENT
        achieved = solve_bytes / (max(stage_ms["solve"], 1e-9) * 1e-3) / 1e9
        ms_step = float(ms[0]) / args.steps
        n_total = int(tot[0])
        line = {"metric": "agent_steps_per_s", "value": n_total / ms_step * 1e3, "unit": "agent-steps/s",
                "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
                "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": {"mixed": "f32 state / f64 arithmetic", "f32": "f32", "f64": "f64"}[args.precision],
                "data": "synthetic",
                "config": {"workload": args.workload, "agents_per_gpu": n_local, "agents_total": n_total,
                           "parallelism": f"x-strips={world}, halo+migration over NCCL send/recv",
                           "precision": args.precision, "density_per_m2": density,
                           "halo_records_per_step": float(tot[2]) / args.steps,
                           "migrants_per_step": float(tot[3]) / args.steps,
                           "cache": "state advances every step; working set > L2"},
                "gpu_launches": int(tot[1]), "host_wall_ms_per_step": float(ms[1]) / args.steps,
                "stages_ms": stage_ms,
                "clocks": sampler.summary() if sampler is not None else None,
                "e2e": {"value": float(io[2]) / float(e2e[0]) * 1e3, "unit": "agent-steps/s",
                        "ms_per_step": float(e2e[0]), "h2d_bytes_per_step": int(float(io[0]) / e2e_steps),
                        "d2h_bytes_per_step": int(float(io[1]) / e2e_steps),
                        "call": "per rank and frame: Simulation.load_pv(host pos, vel) -> StripDriver.step() "
                                "(halo exchange, orca_step, migration) -> Simulation.positions_velocities()"},
                "roofline": {"bound": "hbm", "kernel": "k_solve" if args.precision == "f32" else "k_solve_group",
                             "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                             "traffic": None, "peak_source": peak_src,
                             "algorithmic_bytes_per_launch": solve_bytes,
                             "note": "rank 0's dominant kernel; the step is issue/latency bound (DESIGN.md s5)"},
                "cpu_baseline": None,
                "note": "multi-GPU line: device-timed max over ranks; cpu_baseline is reported by the N=1 run"}
        print(json.dumps(line), flush=True)
    sim.close()
