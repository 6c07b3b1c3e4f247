"""Randomised single-step parity: random crowd geometry and random step parameters
(radius, neighbour cap, dt, tau, margin, responsibility matrix, class mix, frame) against
the CPU oracle. FP64 mode must be bit-exact, MIXED within 1e-6 m/s with identical status;
bins and ordered neighbour lists exact in both."""

import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2008_11578_b200 import (AgentClass, ResponsibilityMatrix, ScenarioConfig, SimState,
                                   Simulation)

pytestmark = pytest.mark.gpu


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def random_case(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 1500))
    kind = rng.integers(0, 5)
    if kind == 0:        # uniform box
        side = float(rng.uniform(3, 120))
        pos = rng.uniform(0, side, size=(n, 2))
    elif kind == 1:      # gaussian blobs
        k = int(rng.integers(1, 5))
        centres = rng.uniform(-200, 200, size=(k, 2))
        pos = centres[rng.integers(0, k, size=n)] + rng.normal(size=(n, 2)) * rng.uniform(0.5, 8)
    elif kind == 2:      # two counter-flowing streams in a corridor
        pos = np.column_stack([rng.uniform(-60, 60, size=n), rng.uniform(-3, 3, size=n)])
    elif kind == 3:      # jittered lattice (near-regular spacing)
        m = int(np.ceil(np.sqrt(n)))
        g = np.stack(np.meshgrid(np.arange(m), np.arange(m)), -1).reshape(-1, 2)[:n].astype(float)
        pos = g * rng.uniform(0.6, 3.0) + rng.uniform(-0.05, 0.05, size=(n, 2)) - 17.0
    else:                # ring
        a = rng.uniform(0, 2 * np.pi, size=n)
        pos = np.column_stack([np.cos(a), np.sin(a)]) * rng.uniform(5, 40) + rng.normal(size=(n, 2)) * 0.8
    pos = f32(pos)
    # exactly coincident centres are an error in the reference: nudge duplicates apart
    _, first = np.unique(pos, axis=0, return_index=True)
    dup = np.setdiff1d(np.arange(n), first)
    pos[dup] = f32(pos[dup] + rng.uniform(0.01, 0.2, size=(dup.size, 2)))
    cls = (rng.random(n) < rng.uniform(0, 0.5)).astype(np.int64)
    radii = f32(np.where(cls == 1, rng.uniform(0.6, 1.4), rng.uniform(0.15, 0.45)) * np.ones(n))
    pref = f32(np.where(cls == 1, 3.0, 1.4) * rng.uniform(0.5, 1.2, size=n))
    maxs = f32(pref * rng.uniform(1.0, 2.0, size=n))
    goals = f32(pos + rng.normal(size=(n, 2)) * rng.uniform(0.1, 60))
    vel = f32(rng.normal(size=(n, 2)) * rng.uniform(0.0, 2.5))
    gtol = f32(rng.uniform(0.05, 0.6, size=n))
    P, V = AgentClass.PEDESTRIAN, AgentClass.VEHICLE
    fm = rng.uniform(0, 1, size=4)
    resp = ResponsibilityMatrix({(P, P): fm[0], (P, V): fm[1], (V, P): fm[2], (V, V): fm[3]})
    cfg = ScenarioConfig(responsibility=resp, dt=float(rng.choice([0.05, 0.1, 0.25, 0.5])),
                         tau=float(rng.uniform(0.5, 4.0)), neighbor_radius=float(f32(rng.uniform(1.0, 25.0))),
                         max_neighbors=int(rng.choice([1, 2, 5, 8, 16, 16, 16, 24, 32])),
                         avoidance_margin=float(rng.choice([0.0, 0.1, 0.3])))
    ids = rng.permutation(n * 3)[:n].astype(np.int64) + int(rng.integers(0, 2**33))
    st = SimState(frame=int(rng.integers(0, 10**6)), time=0.0, ids=ids, positions=pos, velocities=vel,
                  radii=radii, pref_speeds=pref, max_speeds=maxs, goals=goals, goal_tols=gtol,
                  class_codes=cls)
    return st, cfg


@pytest.fixture(autouse=True)
def certified_kernels_on_small_crowds(monkeypatch):
    """cert32 handles take the certified path only for large crowds by themselves; these crowds are small."""
    monkeypatch.setenv("ORCA_CERT_FORCE", "1")


@pytest.mark.parametrize("seed", range(24))
def test_random_step_matches_oracle(seed):
    st, cfg = random_case(seed)
    n = st.active_count
    fs = O.frame_solve(st, cfg, worker_count=4, debug=True)
    assert np.all(fs.err == -1)
    k = max(cfg.max_neighbors, 1)
    kept = {}
    for precision in ("f64", "mixed", "cert32"):
        with Simulation(cfg, capacity=n, precision=precision, remove_arrivals=False) as sim:
            sim.load(st)
            sim.step()
            sim.sync()
            d = sim.debug_last_step(n, cfg.max_neighbors)
            # a second step exercises the radius-hint fast pass on the moved crowd
            sim.step()
            sim.sync()
            d2 = sim.debug_last_step(n, cfg.max_neighbors)
            pos2, vel2 = sim.positions_velocities()
        assert np.array_equal(d["cell_ix"], fs.cell_ix) and np.array_equal(d["cell_iy"], fs.cell_iy)
        assert np.array_equal(d["nb_count"], fs.nb_count)
        assert np.array_equal(d["nb_rows"][:, :k], fs.nb_rows[:, :k])
        assert np.array_equal(d["status"], fs.status) and np.array_equal(d["failed_at"], fs.failed_at)
        if precision == "f64":
            assert np.array_equal(d["out_v"], fs.out_v) and np.array_equal(d["des"], fs.des)
            # second step from the first step's exact output
            st1 = SimState(frame=st.frame + 1, time=0.0, ids=st.ids,
                           positions=st.positions + fs.out_v * cfg.dt, velocities=fs.out_v,
                           radii=st.radii, pref_speeds=st.pref_speeds, max_speeds=st.max_speeds,
                           goals=st.goals, goal_tols=st.goal_tols, class_codes=st.class_codes)
            fs1 = O.frame_solve(st1, cfg, worker_count=4, debug=True)
            if np.all(fs1.err == -1):
                assert np.array_equal(d2["nb_rows"][:, :k], fs1.nb_rows[:, :k])
                assert np.array_equal(d2["out_v"], fs1.out_v)
                assert np.array_equal(pos2, st1.positions + fs1.out_v * cfg.dt)
        else:
            assert np.abs(d["out_v"] - fs.out_v).max() <= 1e-6
            kept[precision] = (d["out_v"], d2["out_v"], d2["status"])
    # the certified FP32 solve returns what MIXED returns, bit for bit (random radii, speeds,
    # responsibility matrices, max_neighbors 0..32, lattices with exact ties)
    for a, b in zip(kept["mixed"], kept["cert32"]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("seed", [0, 1, 2, 3, 5, 8, 13, 21, 1399])
def test_certificate_refuses_what_it_cannot_decide(seed):
    """Crowds that sit ON the decisions of the certified FP32 solve (tests/soak/soak_cert_adversarial.py:
    exact lattices, discs exactly touching, identical / mirrored / zero velocities, agents at their
    goal): cert32 == mixed bit for bit over three frames, and f64 == the oracle on the first. (Seed 1399:
    duplicated half-planes on which the reference's incremental LP gives up by FP64 rounding although
    the LP is feasible -- the case that made the certificate check the path, not only the result.)"""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "soak"))
    from soak_cert_adversarial import adversarial
    st, cfg = adversarial(seed)
    n = st.active_count
    out = {}
    for precision in ("mixed", "cert32"):
        rows = []
        with Simulation(cfg, capacity=n, precision=precision, remove_arrivals=False) as sim:
            sim.load(st)
            for _ in range(3):
                sim.step()
                sim.sync()
                d = sim.debug_last_step(n, cfg.max_neighbors)
                rows.append((d["out_v"], d["status"], d["failed_at"]))
        out[precision] = rows
    for a, b in zip(out["mixed"], out["cert32"]):
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    ref = O.frame_solve(st, cfg, debug=True)
    with Simulation(cfg, capacity=n, precision="f64", remove_arrivals=False) as sim:
        sim.load(st)
        sim.step()
        sim.sync()
        d = sim.debug_last_step(n, cfg.max_neighbors)
    assert np.array_equal(d["out_v"], ref.out_v) and np.array_equal(d["status"], ref.status)
    assert np.array_equal(d["failed_at"], ref.failed_at) and np.array_equal(d["nb_count"], ref.nb_count)
