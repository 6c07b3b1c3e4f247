"""Strip decomposition through the C ABI on one GPU: two (three) handles on cuda:0
play adjacent strips and swap their record buffers device-to-device in place of the
NCCL send/recv of parallel/strips.py (same StripDriver phases, same kernels). The
decomposed crowd must equal the single-handle run bit for bit, keyed by id."""

import numpy as np
import pytest
import torch

import strip_ops_cpu as S
from paper_2008_11578_b200 import Simulation
from paper_2008_11578_b200._lib import RECORD_BYTES, RECORD_DTYPE, OrcaError
from paper_2008_11578_b200.parallel.strips import DeviceStripOps, StripDriver, strip_bounds

pytestmark = pytest.mark.gpu

SIDE = {"left": "right", "right": "left"}


def lockstep(drivers, steps):
    """Drive all ranks phase by phase; rank r's `right` buffer goes to rank r+1's `left`."""
    def swap(counts):
        got = [dict() for _ in drivers]
        for r, d in enumerate(drivers):
            for side, c in counts[r].items():
                peer = r - 1 if side == "left" else r + 1
                dst = drivers[peer].recv[SIDE[side]]
                dst[: c * RECORD_BYTES].copy_(d.send[side][: c * RECORD_BYTES])
                got[peer][SIDE[side]] = c
        torch.cuda.synchronize()
        return got

    for k in range(steps):
        if k % 3 == 0:                     # what StripDriver.step does every reorder_every frames
            for d in drivers:
                d.ops.reorder()
        got = swap([d.pack_halo() for d in drivers])
        for d, g in zip(drivers, got):
            d.unpack_halo(g)
        for d in drivers:
            d.ops.step()
        got = swap([d.pack_migrants() for d in drivers])
        for d, g in zip(drivers, got):
            d.unpack_migrants(g)


@pytest.mark.parametrize("precision,world", [("f64", 2), ("mixed", 3)])
def test_strips_on_device_equal_single_handle(precision, world):
    st, cfg = S.make_crowd(seed=4, n_ped=4000, n_veh=200, density=0.5)
    n = st.ids.shape[0]
    steps = 8
    with Simulation(cfg, capacity=n, precision=precision, remove_arrivals=False) as ref:
        ref.load(st)
        ref.run(steps)
        want = ref.state()
    bounds = strip_bounds(st.positions[:, 0], world)
    b = [-np.inf] + list(bounds) + [np.inf]
    sims, drivers = [], []
    for r in range(world):
        mine = (st.positions[:, 0] >= b[r]) & (st.positions[:, 0] < b[r + 1])
        sim = Simulation(cfg, capacity=n, precision=precision, remove_arrivals=False)
        sim.load(S.take(st, mine))
        sims.append(sim)
        drivers.append(StripDriver(DeviceStripOps(sim), r, world, bounds, cfg.neighbor_radius,
                                   torch.device("cuda", 0), halo_capacity=n))
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
    assert sum(d.stats["migr_sent"] for d in drivers) > 0
    assert sum(d.stats["halo_sent"] for d in drivers) > 0
    assert sum(int(s.info().lp_fallbacks) for s in sims) == want.lp_fallbacks
    for s in sims:
        s.close()


def test_pack_record_layout_and_errors():
    st, cfg = S.make_crowd(seed=5, n_ped=300, n_veh=20)
    n = st.ids.shape[0]
    with Simulation(cfg, capacity=n + 64, precision="f64", remove_arrivals=False) as sim:
        sim.load(st)
        ops = DeviceStripOps(sim)
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
