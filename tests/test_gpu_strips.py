"""Strip decomposition through the C ABI on one GPU: two (three) handles on cuda:0
play adjacent strips and swap their record buffers device-to-device in place of the
NCCL send/recv of parallel/strips.py (same StripDriver phases, same kernels). The
decomposed crowd must equal the single-handle run bit for bit, keyed by id."""

import numpy as np
import pytest
import torch

import strip_ops_cpu as S
from paper_2008_11578_b200 import Simulation
import ctypes as C

from paper_2008_11578_b200 import _lib
from paper_2008_11578_b200._lib import RECORD_BYTES, RECORD_DTYPE, OrcaError
from paper_2008_11578_b200.parallel.strips import DeviceStripOps, StripDriver, state_hash, strip_bounds

pytestmark = pytest.mark.gpu

SIDE = {"left": "right", "right": "left"}


def lockstep(drivers, steps, reorder_every=3):
    """Drive all ranks phase by phase; rank r's `right` buffer goes to rank r+1's `left`
    (a device-to-device copy on the legacy stream in place of the NCCL send/recv). Drivers on
    the window transport exchange for real: every handle's kernel writes into its neighbours'
    windows and their streams wait on the flags -- no synchronisation from here."""
    def exchange():
        if drivers[0].transport == "window":
            for d in drivers:
                d.exchange()
            return
        torch.cuda.synchronize()
        for d in drivers:
            for side in ("left", "right"):
                if d.peer[side] is not None:
                    drivers[d.peer[side]].recv[SIDE[side]].copy_(d.send[side])
        torch.cuda.synchronize()
        for d in drivers:
            d.mark_exchanged()

    for d in drivers:
        d.reorder_every = reorder_every
    if drivers[0].frames == 0:
        for d in drivers:
            d.prime()
        exchange()
    for _ in range(steps):
        for d in drivers:
            d.begin_frame()
        for d in drivers:
            d.append_received()
        for d in drivers:
            d.step_and_pack()
        exchange()
        for d in drivers:
            d.end_frame()
    for d in drivers:
        d.flush()


def build_strips(st, cfg, precision, world, halo_cap, mig_cap, resync_every=4, capacity=None,
                 transport="sendrecv"):
    n = st.ids.shape[0]
    bounds = strip_bounds(st.positions[:, 0], world)
    b = [-np.inf] + list(bounds) + [np.inf]
    sims, drivers = [], []
    for r in range(world):
        mine = (st.positions[:, 0] >= b[r]) & (st.positions[:, 0] < b[r + 1])
        sim = Simulation(cfg, capacity=capacity or 2 * n, precision=precision, remove_arrivals=False)
        sim.load(S.take(st, mine))
        sims.append(sim)
        drivers.append(StripDriver(DeviceStripOps(sim), r, world, bounds, cfg.neighbor_radius,
                                   torch.device("cuda", 0), halo_cap, mig_cap,
                                   vmax=float(st.max_speeds.max()), dt=cfg.dt, resync_every=resync_every,
                                   transport=transport))
    if transport == "window":
        for r, d in enumerate(drivers):
            d.connect_local(drivers[r - 1] if r > 0 else None, drivers[r + 1] if r + 1 < world else None)
    return sims, drivers, b


@pytest.mark.parametrize("precision,world,transport", [("f64", 2, "sendrecv"), ("mixed", 3, "sendrecv"),
                                                       ("f32", 2, "sendrecv"), ("f64", 3, "window"),
                                                       ("mixed", 4, "window"), ("cert32", 2, "window")])
def test_strips_on_device_equal_single_handle(precision, world, transport):
    st, cfg = S.make_crowd(seed=4, n_ped=4000, n_veh=200, density=0.5)
    n = st.ids.shape[0]
    steps = 8
    with Simulation(cfg, capacity=n, precision=precision, remove_arrivals=False) as ref:
        ref.load(st)
        ref.run(steps)
        want = ref.state()
    sims, drivers, b = build_strips(st, cfg, precision, world, halo_cap=n, mig_cap=n // 4, transport=transport)
    assert drivers[0].ops.halo_record_bytes == (64 if precision == "f64" else 32)
    lockstep(drivers, steps)
    parts = [s.state() for s in sims]
    for r, p in enumerate(parts):
        assert p.frame == steps
        assert np.all((p.positions[:, 0] >= b[r]) & (p.positions[:, 0] < b[r + 1]))
    ids = np.concatenate([p.ids for p in parts])
    order, ref_order = np.argsort(ids), np.argsort(want.ids)
    assert np.array_equal(ids[order], want.ids[ref_order])
    for f in ("positions", "velocities", "goals", "radii", "max_speeds", "class_codes"):
        got = np.concatenate([getattr(p, f) for p in parts])[order]
        assert np.array_equal(got, getattr(want, f)[ref_order]), f
    stats = [d.ops.stats() for d in drivers]
    assert sum(g for g, _m in stats) > 0 and sum(m for _g, m in stats) > 0     # both paths exercised
    assert sum(int(s.info().lp_fallbacks) for s in sims) == want.lp_fallbacks
    assert all(d.host_syncs <= steps // 4 + 1 for d in drivers)                # (+1: the final flush)
    # the digest bench.py compares across ranks
    assert sum(state_hash(p.ids, p.positions, p.velocities) for p in parts) % (1 << 64) == \
        state_hash(want.ids, want.positions, want.velocities)
    for s in sims:
        s.close()


def test_strips_with_arrival_removal_equal_single_handle():
    """Arrivals are removed by the strip that owns the agent, in the same compaction that drops
    ghosts and migrants; who is left, and where, equals the single-handle run."""
    st, cfg = S.make_crowd(seed=9, n_ped=3000, n_veh=100, density=0.5)
    rng = np.random.default_rng(2)
    near = rng.random(st.ids.shape[0]) < 0.4  # 40 % of the agents: a goal 5.5 .. 7.5 m ahead, tolerance 6 m,
    ang = rng.uniform(0, 2 * np.pi, near.sum())  # so they arrive one after the other during the run
    dist = rng.uniform(5.5, 7.5, near.sum())
    st.goals[near] = (st.positions[near] + np.column_stack([np.cos(ang), np.sin(ang)]) * dist[:, None]
                      ).astype(np.float32)
    st.goal_tols[near] = 6.0
    n = st.ids.shape[0]
    steps = 12
    with Simulation(cfg, capacity=n, precision="f64", remove_arrivals=True) as ref:
        ref.load(st)
        ref.run(steps)
        want = ref.state()
    assert 0 < want.ids.shape[0] < n
    sims, drivers, _b = build_strips(st, cfg, "f64", 2, halo_cap=n, mig_cap=n // 4)
    for s in sims:
        s.set_config(cfg, remove_arrivals=True, compute_metrics=False)
    lockstep(drivers, steps)
    parts = [s.state() for s in sims]
    ids = np.concatenate([p.ids for p in parts])
    order, ref_order = np.argsort(ids), np.argsort(want.ids)
    assert np.array_equal(ids[order], want.ids[ref_order])
    assert np.array_equal(np.concatenate([p.positions for p in parts])[order], want.positions[ref_order])
    assert np.array_equal(np.concatenate([p.velocities for p in parts])[order], want.velocities[ref_order])
    for s in sims:
        s.close()


def test_window_wait_gives_up_with_an_error_instead_of_hanging(monkeypatch):
    """A neighbour that never delivers: the receiving stream's wait is bounded and the failure
    surfaces as ORCA_ETIMEOUT at the next synchronisation."""
    monkeypatch.setenv("ORCA_WINDOW_TIMEOUT_MS", "200")
    st, cfg = S.make_crowd(seed=4, n_ped=2000, n_veh=100, density=0.5)
    n = st.ids.shape[0]
    sims, drivers, _b = build_strips(st, cfg, "mixed", 2, halo_cap=n, mig_cap=n // 4, transport="window")
    d0 = drivers[0]
    d0.prime()
    d0.exchange()                    # strip 0 delivers, strip 1 never does
    d0.begin_frame()
    d0.append_received()             # waits for strip 1's exchange 0 on the device
    with pytest.raises(OrcaError) as e:
        d0.resync()
    assert e.value.code == _lib.ORCA_ETIMEOUT and "did not arrive" in str(e.value)
    # refusals of the window calls themselves
    L = _lib.load()
    assert L.orca_strip_window_push(sims[1]._h, 0, None, 8, 8, 0) == _lib.ORCA_EINVAL       # no send buffer
    assert L.orca_strip_window_push(sims[1]._h, 1, C.c_void_p(drivers[1].send["left"].data_ptr()), 8, 8, 0) \
        == _lib.ORCA_EINVAL                                                                   # no neighbour there
    assert L.orca_strip_window_push(sims[1]._h, 0, C.c_void_p(drivers[1].send["left"].data_ptr()), 8, 8, 3) \
        == _lib.ORCA_EINVAL                                                                   # out of order
    out = C.c_void_p()
    assert L.orca_strip_window_wait(sims[1]._h, 0, 5, C.byref(out)) == _lib.ORCA_EINVAL      # out of order
    for s in sims:
        s.close()


def test_slab_overflow_is_reported_not_silent():
    st, cfg = S.make_crowd(seed=4, n_ped=4000, n_veh=200, density=0.5)
    # halo slabs far too small for the ~1,000 agents within neighbor_radius of the edge
    sims, drivers, _b = build_strips(st, cfg, "mixed", 2, halo_cap=16, mig_cap=4096, resync_every=0)
    with pytest.raises(OrcaError) as ei:
        lockstep(drivers, 1)
    assert ei.value.code == -5 and "overflow" in str(ei.value)
    for s in sims:
        s.close()
    # emigrant slabs too small: the rows that do not fit stay put and the flag is raised
    sims, drivers, _b = build_strips(st, cfg, "mixed", 2, halo_cap=8192, mig_cap=1, resync_every=0)
    with pytest.raises(OrcaError) as ei:
        lockstep(drivers, 6)
    assert ei.value.code == -5
    for s in sims:
        s.close()


def test_halo_slab_layout_and_refusals():
    st, cfg = S.make_crowd(seed=5, n_ped=600, n_veh=40)
    n = st.ids.shape[0]
    mid = float(np.median(st.positions[:, 0]))
    for precision, dtype in (("mixed", _lib.HALO_DTYPE_F32), ("f64", _lib.HALO_DTYPE_F64)):
        with Simulation(cfg, capacity=2 * n, precision=precision, remove_arrivals=False) as sim:
            sim.load(st)
            ops = DeviceStripOps(sim)
            assert ops.halo_record_bytes == dtype.itemsize
            with pytest.raises(OrcaError):
                ops.pack_halo(3.0, None, None, n)                     # not configured yet
            with pytest.raises(OrcaError):
                ops.append_slab(torch.zeros(64, dtype=torch.uint8, device="cuda"), 1, 1)
            ops.configure(-np.inf, mid, 2.0, 2 * n)
            slab = torch.zeros(_lib.SLAB_HEADER_BYTES + n * dtype.itemsize, dtype=torch.uint8, device="cuda")
            ops.pack_halo(cfg.neighbor_radius, None, slab, n)
            raw = slab.cpu().numpy()
            hdr = raw[:32].view(_lib.SLAB_HEADER_DTYPE)
            mask = st.positions[:, 0] >= mid - cfg.neighbor_radius    # owned or not: the handle holds all rows
            assert int(hdr["count"][0]) == int(mask.sum()) and int(hdr["overflow"][0]) == 0
            rec = raw[32:32 + int(hdr["count"][0]) * dtype.itemsize].view(dtype)
            o, ro = np.argsort(rec["id"]), np.argsort(st.ids[mask])
            assert np.array_equal(rec["id"][o], st.ids[mask][ro])
            for f, src in (("x", st.positions[mask, 0]), ("vy", st.velocities[mask, 1]), ("radius", st.radii[mask]),
                           ("class_code", st.class_codes[mask])):
                assert np.array_equal(rec[f][o].astype(np.float64), src[ro].astype(np.float64)), f
            # ghosts from a slab: invisible to readback, dropped by the strip step
            # (the same agents, nudged aside and renamed so that no two centres coincide)
            rec["x"] += 0.37
            rec["id"] += 10**6
            slab.copy_(torch.from_numpy(raw))
            ops.append_slab(slab, n, 1)
            assert int(sim.info().active_agents) == n
            with pytest.raises(OrcaError):
                ops.append_slab(slab, n, 0)                           # owned rows cannot follow ghosts
            sim.set_config(cfg, remove_arrivals=False, compute_metrics=True)
            mig = torch.zeros(_lib.SLAB_HEADER_BYTES + n * RECORD_BYTES, dtype=torch.uint8, device="cuda")
            with pytest.raises(OrcaError) as ei:
                ops.step(None, mig, n)                                # metrics would miss cross-strip pairs
            assert ei.value.code == -6
            sim.set_config(cfg, remove_arrivals=False, compute_metrics=False)
            ops.step(None, mig, n)
            left = sim.state()
            moved = mig.cpu().numpy()
            cnt = int(moved[:32].view(_lib.SLAB_HEADER_DTYPE)["count"][0])
            out = moved[32:32 + cnt * RECORD_BYTES].view(RECORD_DTYPE)
            assert left.ids.shape[0] + cnt == n                       # every agent is in exactly one place
            assert np.all(left.positions[:, 0] < mid) and np.all(out["x"] >= mid)
            assert np.array_equal(np.sort(np.concatenate([left.ids, out["id"]])), np.sort(st.ids))
            # own emigrants stay as ghosts (kind 2); immigrants (kind 0) come back as owned rows
            ops.append_slab(mig, n, 2)
            assert int(sim.info().active_agents) == n - cnt
            ops.step(None, mig, n)                                    # drops the ghosts again
            with Simulation(cfg, capacity=2 * n, precision=precision, remove_arrivals=False) as other:
                other.load(S.take(st, np.arange(n) < 4))
                o2 = DeviceStripOps(other)
                o2.configure(mid, np.inf, 2.0, 2 * n)
                back = torch.from_numpy(moved).cuda()
                o2.append_slab(back, n, 0)
                got = other.state()
                assert got.ids.shape[0] == 4 + cnt and np.array_equal(got.ids[4:], out["id"])
                assert np.array_equal(got.goals[4:, 0], out["goal_x"]) and np.array_equal(got.radii[4:], out["radius"])


@pytest.mark.parametrize("world,transport", [(2, "sendrecv"), (2, "window"), (3, "window"), (2, "window_fail")])
def test_processes_sharing_one_gpu(tmp_path, world, transport):
    """The real device ops under the real multi-process protocol: the ranks are processes that
    share cuda:0. "sendrecv": the slabs are staged through host memory and travel over gloo (NCCL
    refuses two ranks on one device). "window": every process maps its neighbours' windows through
    CUDA IPC handles, its kernels write the slabs there and raise the flags the neighbours'
    streams wait on (gloo carries the 64-byte handles at set-up, nothing per frame). Equal to
    the single-handle run, keyed by id. "window_fail": one rank cannot map its neighbour's window --
    it raises, nobody hangs, and all ranks fall back to send/recv together."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    steps = 6
    mp.spawn(S.gpu_gloo_worker, args=(world, port, steps, str(tmp_path), "mixed", transport), nprocs=world,
             join=True)
    st, cfg = S.make_crowd(seed=4, n_ped=4000, n_veh=200, density=0.5)
    with Simulation(cfg, capacity=st.ids.shape[0], precision="mixed", remove_arrivals=False) as ref:
        ref.load(st)
        ref.run(steps)
        want = ref.state()
    import os
    parts = [np.load(os.path.join(tmp_path, f"rank{r}.npz")) for r in range(world)]
    ids = np.concatenate([p["ids"] for p in parts])
    order, ref_order = np.argsort(ids), np.argsort(want.ids)
    assert np.array_equal(ids[order], want.ids[ref_order])
    assert np.array_equal(np.concatenate([p["positions"] for p in parts])[order], want.positions[ref_order])
    assert np.array_equal(np.concatenate([p["velocities"] for p in parts])[order], want.velocities[ref_order])
    assert sum(int(p["migr_recv"]) for p in parts) > 0 and sum(int(p["halo_recv"]) for p in parts) > 0


class HostCountOps:
    """orca_strip_pack / orca_strip_append: the variant that reports its count to the host."""

    def __init__(self, sim):
        self.sim, self._L = sim, _lib.load()

    def pack(self, x_lo, x_hi, remove, buf):
        count = C.c_int64()
        _lib.check(self._L.orca_strip_pack(self.sim._h, float(x_lo), float(x_hi), 1 if remove else 0,
                                           C.c_void_p(buf.data_ptr()), buf.numel() // RECORD_BYTES,
                                           C.byref(count)), self.sim._h)
        return int(count.value)

    def append(self, buf, count, ghost):
        _lib.check(self._L.orca_strip_append(self.sim._h, C.c_void_p(buf.data_ptr()), int(count),
                                             1 if ghost else 0), self.sim._h)


def test_pack_record_layout_and_errors():
    st, cfg = S.make_crowd(seed=5, n_ped=300, n_veh=20)
    n = st.ids.shape[0]
    with Simulation(cfg, capacity=n + 64, precision="f64", remove_arrivals=False) as sim:
        sim.load(st)
        ops = HostCountOps(sim)
        buf = torch.empty(n * RECORD_BYTES, dtype=torch.uint8, device="cuda")
        mid = float(np.median(st.positions[:, 0]))
        c = ops.pack(-np.inf, mid, False, buf)
        mask = st.positions[:, 0] < mid
        assert c == int(mask.sum())
        rec = buf[: c * RECORD_BYTES].cpu().numpy().view(RECORD_DTYPE)
        want = S.to_records(st, mask)                         # storage order is preserved
        for name in RECORD_DTYPE.names:
            assert np.array_equal(rec[name], want[name]), name
        # too small a buffer: error, nothing removed
        small = torch.empty(4 * RECORD_BYTES, dtype=torch.uint8, device="cuda")
        with pytest.raises(OrcaError) as ei:
            ops.pack(-np.inf, mid, True, small)
        assert ei.value.code == -5 and int(sim.info().active_agents) == n
        # ghosts: appended, invisible to readback, dropped by the step
        g = rec[:10].copy()
        g["x"] += 0.37                                         # distinct centres, distinct ids
        g["id"] += 10**6
        gbuf = torch.from_numpy(g.view(np.uint8).copy()).cuda()
        ops.append(gbuf, 10, True)
        assert int(sim.info().active_agents) == n
        with pytest.raises(OrcaError):
            ops.append(buf, 1, False)                          # owned rows cannot follow ghosts
        with pytest.raises(OrcaError):
            ops.pack(-np.inf, mid, True, buf)                  # no removal while ghosts are resident
        sim.step()
        assert int(sim.info().active_agents) == n and sim.state().ids.shape[0] == n
        # migration round trip: remove the left half, put it back as owned rows
        c = ops.pack(-np.inf, mid, True, buf)
        assert int(sim.info().active_agents) == n - c
        ops.append(buf, c, False)
        back = sim.state()
        assert np.array_equal(np.sort(back.ids), np.sort(st.ids))


def test_bench_gpus_2_launches_its_ranks_and_verifies_against_one_gpu():
    """`python bench.py --gpus 2` outside torchrun: it starts its own two ranks (they share this
    box's GPU, so the set-up runs over gloo), the strips exchange through peer-memory windows, and
    the one JSON line on stdout carries the digest check against the same crowd on one GPU."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "6", "--warmup", "3",
                          "--workload", "config2_16k"], capture_output=True, text=True, timeout=900, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout[-2000:]          # stdout carries the line and nothing else
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["scaling"] == "weak" and line["metric"] == "agent_steps_per_s"
    assert line["parallelism"]["transport"] == "window"
    assert line["verify"]["bit_equal_vs_1gpu"] is True and line["verify"]["agents"] == 2 * 16640
    assert line["parallelism"]["host_syncs_per_step"] <= 0.5 and line["gpu_launches"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
