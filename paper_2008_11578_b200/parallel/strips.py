"""Strip-decomposed stepping: the crowd is cut into vertical strips along x, one
rank (one GPU) per strip; every step neighbouring strips swap halo agents before
the solve and migrating agents after it.

The reference has no multi-process path at all; what must hold is
its synchronous-update rule: an agent's new velocity depends
only on the pre-step snapshot of the agents within neighbor_radius, so a rank that
sees its owned agents plus every foreign agent within neighbor_radius of its strip
computes exactly what a single device would. Per frame and per rank, ONE exchange with each
adjacent strip:

  1. append   what the last exchange brought: immigrants as owned rows, the neighbour's halo as
              ghost rows -- and this rank's OWN emigrants of the last step as ghosts too (an agent
              that just crossed the edge is still within neighbor_radius of it, so the neighbour
              never has to send it back)
  2. step     orca_strip_step solves the owned agents, then ONE compaction drops the ghosts, the
              arrivals and the owned agents whose new x left the strip -- those go into the
              EMIGRANT SLABS as full 96-byte records
  3. halo     the owned agents within neighbor_radius of a strip edge, at their NEW positions, are
              packed into that side's HALO SLAB (32-byte records: position, velocity, radius,
              class, id)
  4. exchange emigrant + halo slab of each side travel together: with transport "window" this
              strip's kernel copies the used part of them into the neighbour's memory (peer
              mapping, CUDA IPC) and raises a flag the neighbour's stream waits on; with
              "sendrecv" the whole buffers go through one grouped send/recv

The host is not in this loop. A slab is a fixed-capacity device buffer whose 32-byte header
carries the record count; the packing kernels count with atomics, the receiving side needs no
size from the host, the appending kernels read the count from the header.
The exchange is ordered against the handle's stream on the device and involves the two
adjacent strips only -- no collective on the data path. The host keeps a launch bound that
stays FIXED between two synchronisations (row count last seen + slack), so the frames in
between replay one captured CUDA graph, and re-synchronises every `resync_every` frames
(default 16), which is also when a slab overflow -- a sticky device-side flag -- surfaces as an
error.

`StripDriver` holds this protocol and is written against a small ops interface so
the same code runs on NCCL with the CUDA handle (DeviceStripOps) and, in the CPU
tests, on gloo with a host-side stand-in (tests/strip_ops_cpu.py).

Constraint, checked at construction: every interior strip must be at least
neighbor_radius + max_speed*dt wide (a halo reaches one strip deep, and an agent
may cross at most one boundary per step). Frame metrics (min separation,
collisions) are per handle and would miss pairs that straddle strips:
compute_metrics is not supported under strips (orca_strip_step refuses it).
"""

from __future__ import annotations

import ctypes as C
import json
import math
import os
import time

import numpy as np
import torch
import torch.distributed as dist

from .._lib import ORCA_IPC_HANDLE_BYTES, RECORD_BYTES, SLAB_HEADER_BYTES, check, load

__all__ = ["DeviceStripOps", "StripDriver", "strip_bounds", "check_strip_widths", "state_hash",
           "run_bench"]


def strip_bounds(x: np.ndarray, world: int, min_width: float = 0.0) -> np.ndarray:
    """Interior strip boundaries (world-1 values) that split the agents evenly:
    quantiles of the x coordinates. Strip r owns x in [b[r-1], b[r]) with
    b[-1] = -inf and b[world-1] = +inf. With min_width > 0 the boundaries are
    validated (see check_strip_widths)."""
    if world <= 1:
        return np.zeros(0)
    qs = np.arange(1, world) / world
    b = np.quantile(np.asarray(x, dtype=np.float64), qs)
    if min_width > 0.0:
        check_strip_widths(b, min_width)
    return b


def check_strip_widths(bounds, min_width: float):
    """Raise ValueError if an interior strip is narrower than min_width
    (= neighbor_radius + max_speed*dt): its halo would have to reach two strips
    deep and an agent could cross two boundaries in one step -- the results would
    silently differ from a single device."""
    b = np.asarray(bounds, dtype=np.float64)
    if b.size and np.any(np.diff(b) < 0):
        raise ValueError(f"strip boundaries must be non-decreasing, got {b.tolist()}")
    w = np.diff(b)
    if w.size and float(w.min()) < min_width:
        k = int(np.argmin(w))
        raise ValueError(f"strip {k + 1} is {float(w[k]):.6g} m wide; strips must be at least "
                         f"neighbor_radius + max_speed*dt = {min_width:.6g} m wide "
                         "(use fewer strips for a crowd this clustered)")


_MIX = np.uint64(0x9E3779B97F4A7C15)


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def state_hash(ids, positions, velocities) -> int:
    """Order-independent 64-bit digest of {id: (position bits, velocity bits)}: the sum
    (mod 2^64) of a per-agent mix. Equal for a strip-decomposed crowd and the single-device
    run exactly when every agent's position and velocity agree bit for bit, whatever the
    row order and whichever rank holds the agent (per-rank digests add up)."""
    ids = np.ascontiguousarray(ids, dtype=np.int64).view(np.uint64)
    p = np.ascontiguousarray(positions, dtype=np.float64).view(np.uint64).reshape(-1, 2)
    v = np.ascontiguousarray(velocities, dtype=np.float64).view(np.uint64).reshape(-1, 2)
    with np.errstate(over="ignore"):
        h = _mix64(ids * _MIX + np.uint64(1))
        for col in (p[:, 0], p[:, 1], v[:, 0], v[:, 1]):
            h = _mix64(h ^ (col + _MIX))
        return int(h.sum(dtype=np.uint64))


class DeviceStripOps:
    """The slab protocol on a Simulation's resident state through the C ABI."""

    def __init__(self, sim, stream=None):
        """`stream`: the torch.cuda.Stream the exchange is ordered on (default: the current
        one). The handle is moved onto it: the packing / appending kernels and the send/recv
        of the slabs must follow each other on ONE stream, since nothing else orders them."""
        self.sim = sim
        self._L = load()
        self.halo_record_bytes = int(self._L.orca_strip_halo_record_bytes(sim._h))
        dev = torch.device("cuda", sim.device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(dev)
        if not self.stream.cuda_stream:      # the legacy default stream: orca_set_stream reads 0 as
            self.stream = torch.cuda.Stream(dev)   # "the handle's own stream" -- take a real one
        sim.set_stream(self.stream)

    def configure(self, x_lo: float, x_hi: float, vmax_floor: float, slack_rows: int):
        check(self._L.orca_strip_configure(self.sim._h, float(x_lo), float(x_hi), float(vmax_floor),
                                           int(slack_rows)), self.sim._h)

    @staticmethod
    def _p(t):
        return C.c_void_p(t.data_ptr()) if t is not None else None

    # -- the exchange through peer memory (orca_strip_window_*) --
    def window_create(self, side_bytes: int):
        """Allocate this handle's window (two receive buffers of side_bytes per side + flags):
        (CUDA IPC handle as 64 bytes -- for neighbours in other processes --, base address -- for
        neighbours in this process)."""
        h = (C.c_ubyte * ORCA_IPC_HANDLE_BYTES)()
        base = C.c_void_p()
        check(self._L.orca_strip_window_create(self.sim._h, int(side_bytes), h, C.byref(base)), self.sim._h)
        return bytes(h), int(base.value)

    def window_open(self, side: int, ipc_handle: bytes | None = None, base: int | None = None):
        buf = (C.c_ubyte * ORCA_IPC_HANDLE_BYTES).from_buffer_copy(ipc_handle) if ipc_handle is not None else None
        check(self._L.orca_strip_window_open(self.sim._h, int(side), buf,
                                             C.c_void_p(base) if base is not None else None), self.sim._h)

    def window_push(self, side: int, send, mig_cap: int, halo_cap: int, exchange: int):
        check(self._L.orca_strip_window_push(self.sim._h, int(side), self._p(send), int(mig_cap), int(halo_cap),
                                             int(exchange)), self.sim._h)

    def window_wait(self, side: int, exchange: int) -> int:
        out = C.c_void_p()
        check(self._L.orca_strip_window_wait(self.sim._h, int(side), int(exchange), C.byref(out)), self.sim._h)
        return int(out.value)

    def window_close(self):
        check(self._L.orca_strip_window_close(self.sim._h), self.sim._h)

    def pack_halo(self, reach: float, slab_left, slab_right, cap: int):
        check(self._L.orca_strip_pack_halo(self.sim._h, float(reach), self._p(slab_left),
                                           self._p(slab_right), int(cap)), self.sim._h)

    def append_slab(self, slab, cap: int, kind: int):
        """kind 0: immigrants (agent records) as owned rows; 1: a received halo as ghosts;
        2: this handle's own emigrants (agent records) as ghosts."""
        check(self._L.orca_strip_append_slab(self.sim._h, self._p(slab), int(cap), int(kind)), self.sim._h)

    def step(self, mig_left, mig_right, cap: int):
        check(self._L.orca_strip_step(self.sim._h, self._p(mig_left), self._p(mig_right), int(cap)),
              self.sim._h)

    def resync(self):
        """The one host synchronisation: tightens the host's row bound and raises if a
        slab or the handle overflowed (or on the reference's own errors)."""
        self.sim.sync()

    def stats(self):
        g, m = C.c_int64(), C.c_int64()
        check(self._L.orca_strip_stats(self.sim._h, C.byref(g), C.byref(m)), self.sim._h)
        return int(g.value), int(m.value)

    def reorder(self):
        self.sim.reorder_rows()


class _DevAddr:
    """A raw device address where the ops expect a tensor (a slot of the handle's window)."""

    __slots__ = ("addr",)

    def __init__(self, addr: int):
        self.addr = int(addr)

    def data_ptr(self) -> int:
        return self.addr


class StripDriver:
    """One rank's side of the strip protocol."""

    SIDES = ("left", "right")

    def __init__(self, ops, rank: int, world: int, bounds, neighbor_radius: float, device,
                 halo_capacity: int, migrant_capacity: int | None = None, group=None,
                 vmax: float = 0.0, dt: float = 0.0, resync_every: int = 16, transport: str = "sendrecv"):
        """transport: "sendrecv" -- the slabs travel through torch.distributed (NCCL between GPUs;
        gloo, staged through the host, when several ranks share one); "window" -- every strip writes
        its slabs into its neighbours' memory (orca_strip_window_*, CUDA IPC / peer mappings: one
        node) and the receiving stream waits on a flag: no library call per frame at all. After
        construction a "window" driver must be connected: connect_windows() (ranks = processes)
        or connect_local() (several drivers in one process)."""
        if transport not in ("sendrecv", "window"):
            raise ValueError(f"transport must be 'sendrecv' or 'window', got {transport!r}")
        self.ops, self.rank, self.world, self.group = ops, rank, world, group
        self.transport = transport
        b = [-math.inf] + [float(v) for v in bounds] + [math.inf]
        if len(b) != world + 1:
            raise ValueError(f"{world} strips need {world - 1} interior boundaries, got {len(b) - 2}")
        # halo reach with a relative margin: including a few extra agents is harmless,
        # missing one that sits exactly at distance neighbor_radius is not
        self.reach = float(neighbor_radius) * (1.0 + 1e-9) + 1e-9
        check_strip_widths(b[1:-1], self.reach + float(vmax) * float(dt))
        self.lo, self.hi = b[rank], b[rank + 1]
        self.peer = {"left": rank - 1 if rank > 0 else None,
                     "right": rank + 1 if rank < world - 1 else None}
        self.device = torch.device(device)
        self.halo_cap = int(halo_capacity)
        self.mig_cap = int(migrant_capacity if migrant_capacity is not None else halo_capacity)
        hb = SLAB_HEADER_BYTES + self.halo_cap * int(ops.halo_record_bytes)
        mb = SLAB_HEADER_BYTES + self.mig_cap * RECORD_BYTES
        self._mb = mb
        # per side ONE send and ONE receive buffer: [emigrant slab | halo slab]
        def buffers():
            return {s: (torch.zeros(mb + hb, dtype=torch.uint8, device=self.device)
                        if self.peer[s] is not None else None) for s in self.SIDES}
        view = lambda d, lo, hi: {s: (t[lo:hi] if t is not None else None) for s, t in d.items()}  # noqa: E731
        self.send = buffers()
        self.send_mig, self.send_halo = view(self.send, 0, mb), view(self.send, mb, mb + hb)
        if transport == "window":
            # the receive buffers live in this handle's window, where the neighbours write them;
            # recv_mig / recv_halo are filled in (as addresses) by the wait of each exchange
            self.recv = {s: None for s in self.SIDES}
            self.recv_mig, self.recv_halo = dict(self.recv), dict(self.recv)
        else:
            self.recv = buffers()
            self.recv_mig, self.recv_halo = view(self.recv, 0, mb), view(self.recv, mb, mb + hb)
        self.exchanges = 0               # exchanges issued so far (the index of the next one)
        self._connected = transport != "window"
        self._immigrants_done = False    # flush() has already appended the pending immigrants
        self.frames = 0
        self.reorder_every = 64          # frames between row reorderings (no ghosts resident then)
        self.resync_every = int(resync_every)
        self.host_syncs = 0
        self._pending = False            # an exchange has happened and its slabs are not appended yet
        # gloo moves host memory only: device slabs are staged through the host (the 2-process
        # test on one GPU); NCCL sends them as they are
        self._stage = (self.device.type == "cuda" and dist.is_available() and dist.is_initialized()
                       and dist.get_backend(group) == "gloo")
        # rows that may be appended on top of the count the host last saw: two halos at any time,
        # immigrants of every frame until the next synchronisation
        slack = 2 * self.halo_cap + 2 * self.mig_cap * (max(self.resync_every, 1) + 1)
        ops.configure(self.lo, self.hi, float(vmax), slack)
        if transport == "window":
            self.window_handle, self.window_base = ops.window_create(mb + hb)

    # -- "window" transport: map the neighbours' windows ------------------------------
    def connect_windows(self):
        """Ranks are processes: every rank publishes (host name, device, IPC handle) and maps the
        windows of its two neighbours. One all_gather of a few bytes, at set-up only."""
        import socket
        mine = (socket.gethostname(), self.window_handle)
        everyone = [None] * self.world
        dist.all_gather_object(everyone, mine, group=self.group)
        failure = None
        try:
            for k, s in enumerate(self.SIDES):
                p = self.peer[s]
                if p is None:
                    continue
                if everyone[p][0] != mine[0]:
                    raise RuntimeError(f"strip {self.rank} and strip {p} are on different hosts ({mine[0]}, "
                                       f"{everyone[p][0]}): the window transport maps peer memory and needs one "
                                       "node; use transport='sendrecv'")
                self.ops.window_open(k, ipc_handle=everyone[p][1])
        except Exception as exc:            # noqa: BLE001 -- re-raised below, after the collective
            failure = exc
        # (every rank reaches this barrier whether or not its own mapping worked: a rank that raised
        #  before it would leave the others waiting in a collective it never joins)
        dist.barrier(group=self.group)      # nobody pushes into a window its owner has not created yet
        if failure is not None:
            raise failure
        self._connected = True

    def connect_local(self, left=None, right=None):
        """Several drivers in ONE process (tests, one process driving several GPUs): the
        neighbours' windows are given by their drivers."""
        for k, other in enumerate((left, right)):
            if (other is None) != (self.peer[self.SIDES[k]] is None):
                raise ValueError(f"strip {self.rank}: neighbour on side {self.SIDES[k]} does not match the layout")
            if other is not None:
                self.ops.window_open(k, base=other.window_base)
        self._connected = True

    def close(self):
        """Unmap / free the window (after every rank has finished its frames)."""
        if self.transport == "window" and self._connected:
            self.ops.window_close()
            self._connected = False

    # -- one exchange with both neighbours: fixed-size buffers, one grouped call ----
    def _swap(self):
        p2p, staged = [], []
        for s in self.SIDES:
            p = self.peer[s]
            if p is None:
                continue
            if self._stage:
                out = self.send[s].cpu()                 # (synchronises: test transport only)
                inn = torch.empty_like(out)
                staged.append((self.recv[s], inn))
                p2p += [dist.P2POp(dist.isend, out, p, group=self.group),
                        dist.P2POp(dist.irecv, inn, p, group=self.group)]
            else:
                p2p += [dist.P2POp(dist.isend, self.send[s], p, group=self.group),
                        dist.P2POp(dist.irecv, self.recv[s], p, group=self.group)]
        if not p2p:
            return
        # NCCL: the grouped send/recv is ordered after the packing kernels through the current
        # stream, and wait() makes the current stream (= the handle's) wait for it -- the host
        # does not block. gloo (CPU tests): wait() blocks until the bytes are there.
        for w in dist.batch_isend_irecv(p2p):
            w.wait()
        for dst, src in staged:
            dst.copy_(src)

    def exchange(self):
        if self.transport == "window":
            if not self._connected:
                raise RuntimeError("window transport: call connect_windows() / connect_local() first")
            # the used part of [emigrants | halo] goes straight into the neighbour's window, then its flag
            for k, s in enumerate(self.SIDES):
                if self.peer[s] is not None:
                    self.ops.window_push(k, self.send[s], self.mig_cap, self.halo_cap, self.exchanges)
        else:
            stream = getattr(self.ops, "stream", None)
            if stream is None:
                self._swap()
            else:
                with torch.cuda.stream(stream):  # the handle's stream is the current one for the transport
                    self._swap()
        self.mark_exchanged()

    def mark_exchanged(self):
        """The slabs of one more exchange are on their way / in place (also called by tests that
        move the buffers themselves)."""
        self.exchanges += 1
        self._pending = True
        self._immigrants_done = False

    def _await_exchange(self):
        """window transport: the handle's stream waits for the last exchange of both neighbours;
        the slabs are then where the neighbours wrote them."""
        if self.transport != "window":
            return
        for k, s in enumerate(self.SIDES):
            if self.peer[s] is not None:
                addr = self.ops.window_wait(k, self.exchanges - 1)
                self.recv_mig[s], self.recv_halo[s] = _DevAddr(addr), _DevAddr(addr + self._mb)

    # -- protocol phases (split so a test can drive several ranks in one process) ------
    def append_received(self):
        """Phase 1: immigrants as owned rows, then the ghosts (received halo, own emigrants)."""
        if not self._pending:
            return
        self._await_exchange()
        if not self._immigrants_done:
            for s in self.SIDES:
                if self.peer[s] is not None:
                    self.ops.append_slab(self.recv_mig[s], self.mig_cap, 0)
        for s in self.SIDES:
            if self.peer[s] is not None:
                self.ops.append_slab(self.recv_halo[s], self.halo_cap, 1)
                self.ops.append_slab(self.send_mig[s], self.mig_cap, 2)
        self._pending = False

    def step_and_pack(self):
        """Phases 2 and 3: the step with its emigrant slabs, then the halo of the new positions."""
        self.ops.step(self.send_mig["left"], self.send_mig["right"], self.mig_cap)
        self.ops.pack_halo(self.reach, self.send_halo["left"], self.send_halo["right"], self.halo_cap)

    def _zero_header(self, slab):
        stream = getattr(self.ops, "stream", None)
        if stream is None:
            slab[:SLAB_HEADER_BYTES].zero_()
        else:
            with torch.cuda.stream(stream):      # ordered with the handle's kernels
                slab[:SLAB_HEADER_BYTES].zero_()

    def prime(self):
        """Before the first frame: nobody has emigrated yet, the halo of the initial positions
        goes out (the emigrant slabs travel empty)."""
        for s in self.SIDES:
            if self.peer[s] is not None:
                self._zero_header(self.send_mig[s])
        self.ops.pack_halo(self.reach, self.send_halo["left"], self.send_halo["right"], self.halo_cap)

    def begin_frame(self):
        if self.reorder_every and self.frames % self.reorder_every == 0 and hasattr(self.ops, "reorder"):
            self.ops.reorder()       # rows in cell order: memory coherence only, results unchanged
        self.frames += 1

    def end_frame(self):
        if self.resync_every and self.frames % self.resync_every == 0:
            self.resync()

    def resync(self):
        self.host_syncs += 1
        self.ops.resync()

    def flush(self):
        """Append what the last exchange brought as OWNED rows only (the immigrants), so that
        the resident state is the strip's agents and nothing else -- before reading it back."""
        if self._pending and not self._immigrants_done:
            self._await_exchange()
            for s in self.SIDES:
                if self.peer[s] is not None:
                    self.ops.append_slab(self.recv_mig[s], self.mig_cap, 0)
            self._immigrants_done = True     # (a later append_received must not add them again)
        self.resync()

    def step(self):
        """One frame of the whole strip-decomposed crowd, as seen by this rank."""
        if self.frames == 0 and not self._pending:
            self.prime()
            self.exchange()
        self.begin_frame()
        self.append_received()
        self.step_and_pack()
        self.exchange()
        self.end_frame()


# ---------------------------------------------------------------------------
# bench.py --gpus N (one rank per GPU)
# ---------------------------------------------------------------------------

def _select(state, mask):
    fields = ("ids", "positions", "velocities", "radii", "pref_speeds", "max_speeds", "goals",
              "goal_tols", "class_codes")
    return type(state)(frame=state.frame, time=state.time, rng_state=None, lp_fallbacks=0,
                       **{f: np.ascontiguousarray(getattr(state, f)[mask]) for f in fields})


def _slab_capacities(cfg, n_local: int, height: float, density: float, vmax: float):
    """Records per slab: 2x the expected halo population of one edge (edge length x reach x
    density) and 16x the expected per-frame migrants, with floors."""
    halo = int(2.0 * cfg.neighbor_radius * height * density) + 8192
    mig = int(16.0 * vmax * cfg.dt * height * density) + 4096
    return min(halo, n_local + 8192), min(mig, n_local + 4096)


def _strip_sim(cfg, state, args, local, stream, halo_cap, mig_cap, resync_every):
    from .. import Simulation
    n_local = state.active_count
    capacity = n_local + 2 * halo_cap + 2 * mig_cap * (resync_every + 1) + max(131072, n_local // 8)
    sim = Simulation(cfg, capacity=capacity, precision=args.precision, device=local,
                     remove_arrivals=False, compute_metrics=False, stream=stream)
    sim.load(state)
    return sim


def _timed(drv, sim, stream, steps, device, sampler=None):
    """K frames between a barrier + synchronize on both sides; (device ms, host wall ms),
    each the max over ranks."""
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if sampler is not None:
        sampler.__enter__()
    syncs0 = drv.host_syncs
    e0.record(stream)
    t0 = time.perf_counter()
    for _ in range(steps):
        drv.step()
    e1.record(stream)
    t_enq = (time.perf_counter() - t0) * 1e3
    sim.sync()
    torch.cuda.synchronize()
    wall_ms = (time.perf_counter() - t0) * 1e3
    if sampler is not None:
        sampler.__exit__(None, None, None)
    ms = torch.tensor([max(e0.elapsed_time(e1), 0.0), wall_ms, t_enq, float(drv.host_syncs - syncs0)],
                      device=_rdev(device), dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    dist.barrier()
    return [float(v) for v in ms]


def _rdev(device):
    """Where the (set-up / reporting) reductions live: on the GPU with NCCL, on the host with gloo."""
    return device if dist.get_backend() == "nccl" else torch.device("cpu")


def _gather_hash(sim, device):
    """Sum over ranks of the per-rank state_hash (mod 2^64) and the total agent count."""
    st = sim.state()
    h = state_hash(st.ids, st.positions, st.velocities)
    t = torch.tensor([h - (1 << 64) if h >= (1 << 63) else h, st.ids.shape[0]], dtype=torch.int64,
                     device=_rdev(device))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)          # int64 addition wraps: mod 2^64
    return int(t[0].item()) & ((1 << 64) - 1), int(t[1].item())


def run_bench(args, rank: int, world: int, local: int):
    """bench.py --gpus N. Two modes (--scaling):

    weak    every rank owns one `workload` plaza; the plazas sit side by side along x and
            form ONE crowd of world * n agents with halo exchange and migration every step.
    strong  ONE `workload` crowd (BASELINE config 5: config5_8m) cut into `world` strips at
            the quantiles of x.

    Either way the line carries `bit_equal_vs_1gpu`: after the timed frames the id-keyed digest
    of (position, velocity) over all ranks is compared with the digest of the same crowd stepped
    the same number of frames on ONE device by rank 0 (SURVEY.md s8(e) correctness gate; the
    multi-rank analogue of pkg/tests/test_engine.py:197). Skipped (null) when the whole crowd
    does not fit rank 0's GPU next to its strip, or with --no-verify. Returns the JSON line (a
    dict) on rank 0, None elsewhere."""
    from .. import Simulation
    from ..synth import CONFIGS, make_workload

    n_ped, n_veh, density = CONFIGS[args.workload]
    n_cfg = n_ped + n_veh
    strong = getattr(args, "scaling", "weak") == "strong"
    side = math.sqrt(n_cfg / density)
    device = torch.device("cuda", local)
    stream = torch.cuda.Stream(device)
    torch.cuda.set_stream(stream)       # NCCL ops order themselves against the current stream
    if strong:
        whole, cfg = make_workload(args.workload, seed=100)
        vmax = float(whole.max_speeds.max())
        bounds = strip_bounds(whole.positions[:, 0], world)
        b = [-math.inf] + [float(v) for v in bounds] + [math.inf]
        x = whole.positions[:, 0]
        state = _select(whole, (x >= b[rank]) & (x < b[rank + 1]))
        if rank != 0 or getattr(args, "no_verify", False):
            whole = None
    else:
        state, cfg = make_workload(args.workload, seed=100 + rank, origin=(rank * side, 0.0))
        state.ids = state.ids + rank * n_cfg
        # goals anywhere in the whole crowd's plaza, so agents do cross strip boundaries
        rng = np.random.default_rng(1000 + rank)
        state.goals[:, 0] = rng.uniform(0.0, world * side, size=n_cfg).astype(np.float32)
        bounds = [side * r for r in range(1, world)]
        vmax = float(state.max_speeds.max())
        whole = None
    n_local = state.active_count
    rdev = _rdev(device)
    vm = torch.tensor([vmax], dtype=torch.float64, device=rdev)
    dist.all_reduce(vm, op=dist.ReduceOp.MAX)      # set-up only; nothing collective per frame
    vmax = float(vm.item())
    resync_every = 16
    halo_cap, mig_cap = _slab_capacities(cfg, n_local, side, density, vmax)
    sim = _strip_sim(cfg, state, args, local, stream, halo_cap, mig_cap, resync_every)
    ops = DeviceStripOps(sim, stream)

    def make_driver(transport):
        return StripDriver(ops, rank, world, bounds, cfg.neighbor_radius, device, halo_cap, mig_cap, vmax=vmax,
                           dt=cfg.dt, resync_every=resync_every, transport=transport)

    # transport: peer-memory windows by default (one node: every rank maps its neighbours' windows
    # through CUDA IPC); if ANY rank cannot map its neighbour, all fall back to send/recv together
    want = getattr(args, "transport", "auto")
    transport_note = None
    if want in ("auto", "window") and world > 1:
        drv = make_driver("window")
        err = ""
        try:
            drv.connect_windows()
        except Exception as exc:             # noqa: BLE001 -- reported in the line, see below
            err = f"{type(exc).__name__}: {exc}"
        bad = torch.tensor([1.0 if err else 0.0], dtype=torch.float64, device=rdev)
        dist.all_reduce(bad, op=dist.ReduceOp.SUM)
        if float(bad.item()) > 0:
            if want == "window":
                raise RuntimeError(f"--transport window: {int(bad.item())} rank(s) could not map a neighbour's "
                                   f"window ({err or 'see the other ranks'})")
            drv.close()
            transport_note = "peer-memory windows unavailable, send/recv instead" + (f" ({err})" if err else "")
            drv = make_driver("sendrecv")
    else:
        drv = make_driver("sendrecv")

    warm = max(args.warmup, 3)
    for _ in range(warm):
        drv.step()
    drv.resync()
    for _ in range(2):      # (the handle adapts at a synchronisation: keep the re-capture out of the timed frames)
        drv.step()
    drv.resync()
    warm += 2
    l0 = sim.info().kernel_launches
    g0, m0 = drv.ops.stats()
    sampler = args.make_sampler() if hasattr(args, "make_sampler") else None
    dev_ms, wall_ms, enq_ms, syncs = _timed(drv, sim, stream, args.steps, device, sampler)
    drv.flush()
    info = sim.info()
    g1, m1 = drv.ops.stats()
    tot = torch.tensor([float(info.active_agents), float(info.kernel_launches - l0), float(g1 - g0),
                        float(m1 - m0)], device=rdev, dtype=torch.float64)
    dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    frames_done = warm + args.steps

    # ---- correctness gate: id-keyed digest over all ranks vs the same crowd on ONE device ----
    verify = None
    if not getattr(args, "no_verify", False):
        drv.flush()
        got_hash, got_n = _gather_hash(sim, device)
        want = torch.zeros(2, dtype=torch.int64, device=rdev)
        if rank == 0:
            if strong:
                ref_state = whole
            else:
                # the weak-scaling crowd is the concatenation of every rank's plaza (same seeds)
                parts = []
                for r in range(world):
                    st_r, _ = make_workload(args.workload, seed=100 + r, origin=(r * side, 0.0))
                    st_r.ids = st_r.ids + r * n_cfg
                    st_r.goals[:, 0] = np.random.default_rng(1000 + r).uniform(
                        0.0, world * side, size=n_cfg).astype(np.float32)
                    parts.append(st_r)
                ref_state = parts[0]
                if world > 1:
                    for f in ("ids", "positions", "velocities", "radii", "pref_speeds", "max_speeds", "goals",
                              "goal_tols", "class_codes"):
                        setattr(ref_state, f, np.concatenate([getattr(p, f) for p in parts]))
            n_ref = ref_state.active_count
            free_b, _total = torch.cuda.mem_get_info(device)
            if n_ref * 1200 < free_b:                  # ~0.8 KB/agent resident + staging
                with Simulation(cfg, capacity=n_ref, precision=args.precision, device=local,
                                remove_arrivals=False, compute_metrics=False, stream=stream) as ref:
                    ref.load(ref_state)
                    ref.run(frames_done)
                    rs = ref.state()
                h = state_hash(rs.ids, rs.positions, rs.velocities)
                want[0] = h - (1 << 64) if h >= (1 << 63) else h
                want[1] = rs.ids.shape[0]
            else:
                want[1] = -1
            del ref_state
        dist.broadcast(want, src=0)
        if int(want[1].item()) >= 0:
            want_hash = int(want[0].item()) & ((1 << 64) - 1)
            verify = {"bit_equal_vs_1gpu": bool(got_hash == want_hash and got_n == int(want[1].item())),
                      "frames": frames_done, "agents": got_n,
                      "digest": f"{got_hash:016x}", "digest_1gpu": f"{want_hash:016x}"}
        else:
            verify = {"bit_equal_vs_1gpu": None, "note": "the whole crowd does not fit rank 0's GPU"}
    whole = None
    dist.barrier()

    # ---- e2e: the same step with this rank's positions / velocities going up from pinned host
    # memory and coming back every frame (what a host-side caller of a strip-decomposed crowd pays)
    e2e_steps = max(3, min(args.steps, getattr(args, "e2e_steps", 20)))
    drv.flush()
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
        drv.flush()
        pos, vel = sim.positions_velocities()
        d2h += pos.nbytes + vel.nbytes
    torch.cuda.synchronize()
    e2e = torch.tensor([(time.perf_counter() - t0) * 1e3 / e2e_steps], device=rdev, dtype=torch.float64)
    dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    io = torch.tensor([float(h2d), float(d2h), float(sim.info().active_agents)], device=rdev, dtype=torch.float64)
    dist.all_reduce(io, op=dist.ReduceOp.SUM)

    # ---- roofline of the dominant kernel on rank 0 (same definition as the N=1 line)
    sim.profile_stages(True)
    for _ in range(5):
        drv.step()
    stage_ms, covered = sim.stage_ms()
    sim.profile_stages(False)
    stage_ms = {k: v / max(covered, 1) for k, v in stage_ms.items()}
    dist.barrier()
    line = None
    if rank == 0:
        hbm_peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
        pk = os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))),
                          "MEASURED_PEAKS.json")
        try:
            with open(pk) as f:
                hbm_peak, peak_src = float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
        except Exception:
            pass
        solve_bytes = (16 + 32 + 1 + 4 * 16 + 1 + 16 + 16 + 2 + 1) * n_local     # bench.py SOLVE_BYTES_PER_AGENT
        achieved = solve_bytes / (max(stage_ms["solve"], 1e-9) * 1e-3) / 1e9
        ms_step = dev_ms / args.steps
        n_total = int(tot[0])
        line = {"metric": "agent_steps_per_s", "value": n_total / ms_step * 1e3, "unit": "agent-steps/s",
                "n_gpus": world, "steps": args.steps, "warmup": warm,
                "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong" if strong else "weak",
                "vs_baseline": None,
                "dtype": {"mixed": "f32 state / f64 arithmetic", "f32": "f32", "f64": "f64",
                          "cert32": "f32 state / certified f32 solve, f64 result"}[args.precision],
                "data": "synthetic",
                "config": {"workload": args.workload, "pedestrians": n_ped, "vehicles": n_veh,
                           "density_per_m2": density, "neighbor_radius": cfg.neighbor_radius,
                           "max_neighbors": cfg.max_neighbors, "dt": cfg.dt, "tau": cfg.tau},
                "parallelism": {"layout": f"x-strips={world}", "agents_rank0": n_local, "agents_total": n_total,
                                "transport": drv.transport,
                                "exchange": ("fixed-capacity slabs with device-side counts; each strip's kernel "
                                             "writes the used part of its slabs into the adjacent strips' memory "
                                             "(CUDA IPC peer mapping) and raises a flag the receiving stream waits "
                                             "on: no library call, no collective per frame"
                                             if drv.transport == "window" else
                                             "fixed-capacity slabs, device-side counts, grouped send/recv "
                                             "with the adjacent strips; no collective per frame"),
                                "transport_note": transport_note,
                                "backend": dist.get_backend() + (
                                    " (set-up and timing reductions only)" if drv.transport == "window" else
                                    " (slabs staged through the host: several ranks share a GPU)" if drv._stage
                                    else ""),
                                "halo_record_bytes": drv.ops.halo_record_bytes, "migrant_record_bytes": RECORD_BYTES,
                                "halo_slab_records": halo_cap, "migrant_slab_records": mig_cap,
                                "halo_records_per_step": float(tot[2]) / args.steps,
                                "migrants_per_step": float(tot[3]) / args.steps,
                                "host_syncs_per_step": syncs / args.steps,
                                "host_wall_ms_per_step": wall_ms / args.steps,
                                "host_enqueue_ms_per_step": enq_ms / args.steps},
                "precision": args.precision,
                "cache": "state advances every step; working set > L2, no flush",
                "verify": verify,
                "gpu_launches": int(tot[1]), "host_wall_ms_per_step": wall_ms / args.steps,
                "stages_ms": stage_ms,
                "clocks": sampler.summary() if sampler is not None else None,
                "e2e": {"value": float(io[2]) / float(e2e[0]) * 1e3, "unit": "agent-steps/s",
                        "ms_per_step": float(e2e[0]), "h2d_bytes_per_step": int(float(io[0]) / e2e_steps),
                        "d2h_bytes_per_step": int(float(io[1]) / e2e_steps),
                        "call": "per rank and frame: Simulation.load_pv(host pos, vel) -> StripDriver.step() "
                                "(halo exchange, orca_strip_step, migration) -> Simulation.positions_velocities()"},
                "roofline": {"bound": "hbm", "kernel": "k_solve" if args.precision == "f32" else "k_solve_group",
                             "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                             "traffic": None, "peak_source": peak_src,
                             "algorithmic_bytes_per_launch": solve_bytes,
                             "note": "rank 0's dominant kernel; the step is issue/latency bound (DESIGN.md s5)"},
                "cpu_baseline": None,
                "note": "multi-GPU line: device-timed max over ranks; cpu_baseline is reported by the N=1 run"}
    torch.cuda.synchronize()
    dist.barrier()          # (window transport: nobody frees a window a neighbour may still be writing)
    drv.close()
    sim.close()
    return line if rank == 0 else None
