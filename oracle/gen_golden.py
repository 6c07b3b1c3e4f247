#!/usr/bin/env python
"""Generate tests/golden/*.npz by RUNNING THE REFERENCE ITSELF.

TEST INFRASTRUCTURE ONLY. Run in the build container (where /root/reference is
mounted read-only); the GPU box never runs this, it only reads the committed
fixtures:

    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/gen_golden.py

Every array saved here is an output of the unmodified reference package
(`orcasim`, imported from /root/reference/pkg/src) or a seeded input fed to it.
tests/test_oracle_golden.py pins oracle/orca_oracle.c against these fixtures bit
for bit; the GPU parity tests then compare the CUDA path both with the fixtures
directly and with the pinned oracle on larger seeded inputs.

Fixtures (all small, compressed):
  kat.npz            shuffle permutations, problem seeds, VO exits and LP
                     known answers (the cases of pkg/tests/test_lp.py:23-100,
                     122-127 and pkg/tests/test_orca.py:25-50) + random VO/LP.
  lp_batch_*.npz     K.solve_range over CSR-packed random batches, k in [8,64],
                     feasible / mixed / infeasible.
  frame_*.npz        engine._advance on seeded plaza crowds incl. per-agent
                     cell (ix,iy), ordered neighbour rows, constraints, out_v,
                     status, failed_at, new state, metrics.
  run_*.npz          whole engine.run() of the built-in 2-way / 4-way crossings: the crowd
                     the reference spawned, its guard, summary, per-frame metrics,
                     arrival times and sampled trajectories.
  scenario_cases.json, traj_two_way_12.csv, agents_two_way_12.csv
                     crossing documents, spawned crowds, validation messages and CSV
                     bytes of the reference's scenario / crossings / cli modules.
  api_cases.npz      the object-level operators (orca.gather_constraints, grid.query_neighbors,
                     lp.solve_least_penetration) on seeded inputs.
  chain_1k.npz       config 1: 100 consecutive reference steps of 1,024
                     pedestrians (each input = previous output rounded to
                     float32 so an FP32 device state sees identical inputs);
                     positions/velocities stored for every step.
"""

from __future__ import annotations

import math
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, REF_SRC)
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import orcasim._kernels as K  # noqa: E402
import orcasim.engine as E  # noqa: E402
from orcasim.lp import shuffle_order  # noqa: E402
from orcasim.scenario import ScenarioConfig as RefConfig  # noqa: E402

from paper_2008_11578_b200.synth import lp_batch, plaza_crowd  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def ref_config(**kw) -> RefConfig:
    from orcasim.orca import AgentClass, ResponsibilityMatrix
    from orcasim.scenario import DEFAULT_CLASS_PARAMS, ClassParams
    cfg = RefConfig(regions=[],
                    class_params={c: ClassParams(*p) for c, p in DEFAULT_CLASS_PARAMS.items()},
                    responsibility=ResponsibilityMatrix.default())
    for k, v in kw.items():
        setattr(cfg, k, v)
    return cfg


def ref_state(st) -> E.SimState:
    return E.SimState(frame=st.frame, time=st.time, ids=st.ids, positions=st.positions,
                      velocities=st.velocities, radii=st.radii, pref_speeds=st.pref_speeds,
                      max_speeds=st.max_speeds, goals=st.goals, goal_tols=st.goal_tols,
                      class_codes=st.class_codes, rng_state=None)


# ---------------------------------------------------------------------------

def gen_kat():
    out = {}
    ks, seeds, perms = [], [], []
    for k in (0, 1, 2, 5, 16, 33, 64):
        for seed in (0, 1, 2**63 - 1, 1234567890123456789, 0xDEADBEEFCAFEF00D):
            perm = np.empty(max(k, 1), dtype=np.int64)
            K.shuffle_into(perm, k, np.uint64(seed))
            assert list(perm[:k]) == shuffle_order(k, seed)
            row = np.full(64, -1, dtype=np.int64)
            row[:k] = perm[:k]
            ks.append(k)
            seeds.append(seed)
            perms.append(row)
    out["shuffle_k"] = np.array(ks, dtype=np.int64)
    out["shuffle_seed"] = np.array(seeds, dtype=np.uint64)
    out["shuffle_perm"] = np.array(perms)

    fr = np.array([0, 1, 2, 99, 12345, 2**31 - 1], dtype=np.int64)
    ag = np.array([0, 1, 7, 1023, 2**31 - 1, 2**32 + 5], dtype=np.int64)
    ps = np.empty((fr.size, ag.size), dtype=np.uint64)
    for a, f in enumerate(fr):
        for b, g in enumerate(ag):
            ps[a, b] = K._problem_seed(np.int64(f), np.int64(g))
            if g < 2**32:
                assert int(ps[a, b]) == E.problem_seed(int(g), int(f))
    out["seed_frames"], out["seed_ids"], out["seed_values"] = fr, ag, ps

    # VO exits: the three known answers of test_orca.py:25-50 then random ones
    rng = np.random.default_rng(31)
    cases = [(10.0, 0.0, 0.0, 0.0, 0.5, 2.0, 0.1),
             (2.0, 0.0, 2.0, 0.0, 1.0, 1.0, 0.1),
             (0.4, 0.0, 0.0, 0.0, 0.5, 2.0, 0.1),
             (0.0, 0.0, 1.0, 0.0, 0.5, 2.0, 0.1)]
    for _ in range(4000):
        d = 0.05 + 12.0 * rng.random()
        a = 2 * np.pi * rng.random()
        comb = 0.2 + 2.2 * rng.random()
        tau = 0.5 + 3.0 * rng.random()
        rv = rng.normal(size=2) * 3.0
        cases.append((d * math.cos(a), d * math.sin(a), rv[0], rv[1], comb, tau, 0.1))
    cases = f32(np.array(cases))
    vo = np.empty((cases.shape[0], 5))
    for i, c in enumerate(cases):
        ux, uy, nx, ny, ok = K.vo_exit(*c)
        vo[i] = (ux, uy, nx, ny, float(ok))
    assert np.allclose(vo[0, :4], [4.75, 0, -1, 0]) and np.allclose(vo[1, :4], [-1, 0, -1, 0])
    assert np.allclose(vo[2, :4], [-1, 0, -1, 0]) and vo[3, 4] == 0.0
    out["vo_in"], out["vo_out"] = cases, vo

    # LP known answers (test_lp.py:23-43, 77-100): solve_closest_point / least_penetration
    from orcasim.lp import (HalfPlaneConstraint, LpProblem, solve_closest_point,
                            solve_least_penetration)

    def hp(p, n):
        return HalfPlaneConstraint(np.asarray(p, float), np.asarray(n, float))

    r1 = solve_closest_point(LpProblem([], (1.0, 0.5), 2.0))
    r2 = solve_closest_point(LpProblem([], (3.0, 4.0), 2.5))
    r3 = solve_closest_point(LpProblem([hp((0, 1), (0, 1))], (0.7, 0.2), 5.0))
    out["lp_kat_closest"] = np.array([r1.velocity, r2.velocity, r3.velocity])
    band_f = [hp((0, -1), (0, 1)), hp((0, 1), (0, -1))]
    band_e = [hp((0, 1), (0, 1)), hp((0, -1), (0, -1))]
    tri = []
    for deg in (90, 210, 330):
        n = np.array([math.cos(math.radians(deg)), math.sin(math.radians(deg))])
        tri.append(hp(n, n))
    out["lp_kat_lpen"] = np.array([
        solve_least_penetration(band_f, 5.0, 0, (0.3, 2.0)),
        solve_least_penetration(band_f, 5.0, 0, (-0.2, 0.4)),
        solve_least_penetration(band_e, 5.0, 0, (0.3, 2.0)),
        solve_least_penetration(tri, 5.0, 0, (0.4, -0.3))])
    out["lp_kat_tri_nrm"] = np.array([c.normal for c in tri])
    np.savez_compressed(os.path.join(OUT, "kat.npz"), **out)
    print("kat.npz", {k: v.shape for k, v in out.items()})


def gen_lp_batches():
    for name, frac, n, seed in (("feasible", 0.0, 600, 1), ("mixed", 0.5, 600, 2),
                                ("infeasible", 1.0, 600, 3), ("small_k", 0.3, 1500, 4)):
        kmin, kmax = (0, 16) if name == "small_k" else (8, 64)
        coff, cpts, cnrm, tgt, caps, seeds = lp_batch(n, kmin, kmax, frac, seed=seed)
        out_v = np.empty((n, 2))
        status = np.empty(n, dtype=np.int64)
        failed = np.empty(n, dtype=np.int64)
        K.solve_range(coff, cpts, cnrm, tgt, caps, seeds, out_v, status, failed, 0, n)
        np.savez_compressed(os.path.join(OUT, f"lp_batch_{name}.npz"), coff=coff,
                            cpts=cpts.astype(np.float32), cnrm=cnrm.astype(np.float32),
                            tgt=tgt.astype(np.float32), caps=caps.astype(np.float32),
                            seeds=seeds, out_v=out_v, status=status.astype(np.int8),
                            failed=failed.astype(np.int16))
        print(f"lp_batch_{name}.npz fallback frac {status.mean():.3f}")


def frame_debug(state, cfg):
    """What engine._advance computes before integration, plus the per-agent
    neighbour rows / constraints (via K._collect_neighbors and K.vo_exit, the
    same calls frame_solve_range makes, K:515-541)."""
    n = state.active_count
    cell = cfg.neighbor_radius
    reach = int(math.ceil(cfg.neighbor_radius / cell))
    rad2 = cfg.neighbor_radius * cfg.neighbor_radius
    order, ukeys, starts = E._grid_arrays(state.positions, cell)
    ix = np.floor(state.positions[:, 0] / cell).astype(np.int64)
    iy = np.floor(state.positions[:, 1] / cell).astype(np.int64)
    max_n = cfg.max_neighbors
    nb_rows = np.full((n, max(max_n, 1)), -1, dtype=np.int64)
    nb_cnt = np.zeros(n, dtype=np.int64)
    nb_d2 = np.empty(max(max_n, 1))
    nb_id = np.empty(max(max_n, 1), dtype=np.int64)
    nb_ix = np.empty(max(max_n, 1), dtype=np.int64)
    cons = np.zeros((n, max(max_n, 1), 4))
    fmat = cfg.responsibility.as_array()
    avoid = state.radii + 0.5 * cfg.avoidance_margin
    for i in range(n):
        c = 0
        if max_n > 0:
            c = K._collect_neighbors(i, state.positions, state.ids, order, ukeys, starts, cell,
                                     reach, rad2, max_n, nb_d2, nb_id, nb_ix)
        nb_cnt[i] = c
        nb_rows[i, :c] = nb_ix[:c]
        for t in range(c):
            j = nb_ix[t]
            rp = state.positions[j] - state.positions[i]
            rv = state.velocities[i] - state.velocities[j]
            ux, uy, nx, ny, ok = K.vo_exit(rp[0], rp[1], rv[0], rv[1], avoid[i] + avoid[j],
                                           cfg.tau, cfg.dt)
            assert ok
            f = fmat[state.class_codes[i], state.class_codes[j]]
            cons[i, t] = (state.velocities[i, 0] + f * ux, state.velocities[i, 1] + f * uy, nx, ny)
    des = E._desired_velocities(state.positions, state.goals, state.pref_speeds, cfg.dt)
    out_v = np.empty((n, 2))
    status = np.empty(n, dtype=np.int64)
    failed = np.empty(n, dtype=np.int64)
    err = np.empty(n, dtype=np.int64)
    K.frame_solve_range(state.positions, state.velocities, avoid, state.max_speeds,
                        state.class_codes, state.ids, fmat, des, order, ukeys, starts, cell, reach,
                        rad2, max_n, cfg.tau, cfg.dt, state.frame, out_v, status, failed, err, 0, n)
    return dict(cell_ix=ix, cell_iy=iy, nb_rows=nb_rows, nb_count=nb_cnt, cons=cons, des=des,
                out_v=out_v, status=status, failed=failed, err=err)


def save_frame(name, state, cfg, extra=None):
    dbg = frame_debug(state, cfg)
    new_state, _log, min_sep, coll, fb, removed = E._advance(ref_state(state), cfg, 1, 4096, False)
    # the fused kernel inside _advance must agree with the composed debug run
    keep = ~np.isin(state.ids, removed)
    assert np.array_equal(new_state.velocities, dbg["out_v"][keep])
    d = dict(
        frame=np.int64(state.frame), ids=state.ids, positions=state.positions.astype(np.float32),
        velocities=state.velocities.astype(np.float32), radii=state.radii.astype(np.float32),
        pref_speeds=state.pref_speeds.astype(np.float32),
        max_speeds=state.max_speeds.astype(np.float32), goals=state.goals.astype(np.float32),
        goal_tols=state.goal_tols.astype(np.float32), class_codes=state.class_codes.astype(np.int8),
        dt=cfg.dt, tau=cfg.tau, neighbor_radius=cfg.neighbor_radius,
        max_neighbors=np.int64(cfg.max_neighbors), avoidance_margin=cfg.avoidance_margin,
        fmat=cfg.responsibility.as_array(),
        cell_ix=dbg["cell_ix"].astype(np.int32), cell_iy=dbg["cell_iy"].astype(np.int32),
        nb_rows=dbg["nb_rows"].astype(np.int32), nb_count=dbg["nb_count"].astype(np.int8),
        cons=dbg["cons"], des=dbg["des"], out_v=dbg["out_v"], status=dbg["status"].astype(np.int8),
        failed=dbg["failed"].astype(np.int8),
        new_ids=new_state.ids, new_positions=new_state.positions,
        new_velocities=new_state.velocities, removed_ids=removed,
        min_separation=np.float64(min_sep), collision_count=np.int64(coll),
        lp_fallbacks=np.int64(fb))
    # inputs must be float32-representable (so an FP32 device state is exact)
    for k in ("positions", "velocities", "radii", "pref_speeds", "max_speeds", "goals",
              "goal_tols"):
        assert np.array_equal(d[k].astype(np.float64), getattr(state, k)), k
    if extra:
        d.update(extra)
    np.savez_compressed(os.path.join(OUT, f"frame_{name}.npz"), **d)
    print(f"frame_{name}.npz n={state.active_count} fallbacks={fb} removed={removed.size} "
          f"min_sep={min_sep:.4f} coll={coll}")


def gen_frames():
    # mixed plaza, default parameters (config 2 in miniature)
    st, _ = plaza_crowd(480, 32, density=0.25, seed=11)
    save_frame("mixed_512", st, ref_config())
    # dense crowd: most agents take the fallback (config 3 in miniature)
    st, _ = plaza_crowd(700, 20, density=2.0, seed=12)
    st.frame = 7
    save_frame("dense_720", st, ref_config())
    # small radius / few neighbours, non-default responsibility, agents near their goals
    from orcasim.orca import AgentClass, ResponsibilityMatrix
    P, V = AgentClass.PEDESTRIAN, AgentClass.VEHICLE
    resp = ResponsibilityMatrix({(P, P): 0.5, (V, V): 0.5, (P, V): 0.75, (V, P): 0.25})
    st, _ = plaza_crowd(300, 60, density=0.6, seed=13, origin=(-20.0, -13.0))
    rng = np.random.default_rng(5)
    near = rng.permutation(360)[:60]
    st.goals[near] = f32(st.positions[near] + rng.normal(size=(60, 2)) * 0.2)
    st.frame = 3
    save_frame("odd_360", st, ref_config(neighbor_radius=f32(4.0).item(), max_neighbors=5,
                                          tau=1.5, dt=0.25, avoidance_margin=0.0,
                                          responsibility=resp))
    # sparse: many agents with no / few neighbours, negative coordinates
    st, _ = plaza_crowd(200, 10, density=0.004, seed=14, origin=(-150.0, -90.0))
    save_frame("sparse_210", st, ref_config())


def gen_chain():
    st, _ = plaza_crowd(1024, 0, density=0.25, seed=1)
    cfg = ref_config()
    state = ref_state(st)
    n0 = state.active_count
    steps = 100
    pos_in = np.full((steps, n0, 2), np.nan, dtype=np.float32)
    vel_in = np.full((steps, n0, 2), np.nan, dtype=np.float32)
    out_v = np.full((steps, n0, 2), np.nan)
    status = np.full((steps, n0), -1, dtype=np.int8)
    active = np.zeros(steps, dtype=np.int64)
    fallbacks = np.zeros(steps, dtype=np.int64)
    min_sep = np.zeros(steps)
    coll = np.zeros(steps, dtype=np.int64)
    for s in range(steps):
        ids = state.ids
        active[s] = ids.shape[0]
        pos_in[s, ids] = state.positions
        vel_in[s, ids] = state.velocities
        dbg = frame_debug(state, cfg)
        out_v[s, ids] = dbg["out_v"]
        status[s, ids] = dbg["status"]
        new_state, _log, ms, cc, fb, _removed = E._advance(state, cfg, 1, 4096, False)
        fallbacks[s], min_sep[s], coll[s] = fb, ms, cc
        # next input = this output rounded to float32 (identical inputs for FP32 device state)
        new_state.positions = f32(new_state.positions)
        new_state.velocities = f32(new_state.velocities)
        state = new_state
    np.savez_compressed(os.path.join(OUT, "chain_1k.npz"), pos_in=pos_in, vel_in=vel_in,
                        out_v=out_v, status=status, active=active, fallbacks=fallbacks,
                        min_sep=min_sep, collisions=coll,
                        goals=st.goals.astype(np.float32), radii=st.radii.astype(np.float32),
                        pref_speeds=st.pref_speeds.astype(np.float32),
                        max_speeds=st.max_speeds.astype(np.float32),
                        goal_tols=st.goal_tols.astype(np.float32))
    print("chain_1k.npz active", active[[0, -1]], "fallbacks/step", fallbacks.mean())


def gen_scenarios():
    """The callers either side of the step, from the reference:
    crossing scenario documents, the crowds its seeded sampler spawns from them, frame
    guards, validation messages for broken documents, and the bytes of its CSV writers."""
    import hashlib
    import json
    import tempfile

    import orcasim.scenario as S
    from orcasim.cli import _write_agents_csv
    from orcasim.crossings import arm_size, four_way_dict, two_way_dict

    cases = []
    for kind, per_arm, vf, seed, kw in (
            ("two_way", 40, 0.1, 3, {}), ("four_way", 24, 0.25, 5, {}), ("four_way", 625, 0.0, 0, {}),
            ("two_way", 300, 0.5, 11, {}), ("four_way", 60, 0.3, 2, {"size_for_worst_class": True}),
            ("two_way", 25, 1.0, 7, {"arm_width": 30.0, "arm_depth": 50.0, "clearance_time": 0.8}),
            ("four_way", 10, 0.5, 1, {"dt": 0.05, "tau": 3.0, "max_frames": 77, "goal_tolerance": 0.4}),
            ("two_way", 0, 0.0, 0, {})):
        maker = two_way_dict if kind == "two_way" else four_way_dict
        doc = maker(per_arm, vf, seed, **kw)
        cfg = S.scenario_from_dict(doc, source=f"<{kind} crossing>")
        st = E.init_state(cfg)
        cases.append(dict(kind=kind, per_arm=per_arm, vehicle_fraction=vf, seed=seed, kwargs=kw, doc=doc,
                          guard=cfg.frame_guard(), warnings=cfg.warnings,
                          arm_size=list(arm_size(per_arm, vf, kw.get("clearance_time", 0.5),
                                                 kw.get("size_for_worst_class", False))),
                          ids=st.ids.tolist(), positions=st.positions.tolist(), goals=st.goals.tolist(),
                          velocities=st.velocities.tolist(), radii=st.radii.tolist(),
                          pref_speeds=st.pref_speeds.tolist(), max_speeds=st.max_speeds.tolist(),
                          goal_tols=st.goal_tols.tolist(), class_codes=st.class_codes.tolist()))
        print(f"scenario {kind} per_arm={per_arm} vf={vf} seed={seed}: {st.active_count} agents, guard {cfg.frame_guard()}")

    # validation: broken documents and the reference's message for each
    good = two_way_dict(4, 0.5, 1)
    broken = []

    def bad(label, mutate):
        doc = json.loads(json.dumps(good))
        doc = mutate(doc) or doc
        try:
            S.scenario_from_dict(doc, source="<t>")
            msg = None
        except S.ScenarioError as exc:
            msg = str(exc)
        broken.append(dict(label=label, doc=doc, message=msg))

    bad("not a mapping", lambda d: [1, 2])
    bad("version", lambda d: d.update(format_version=2))
    bad("unknown top-level", lambda d: d.update(speed=3))
    bad("dt string", lambda d: d.update(dt="fast"))
    bad("dt zero", lambda d: d.update(dt=0))
    bad("dt inf", lambda d: d.update(dt=float("inf")))
    bad("tau bool", lambda d: d.update(tau=True))
    bad("clearance negative", lambda d: d.update(clearance_time=-1))
    bad("margin negative", lambda d: d.update(avoidance_margin=-0.5))
    bad("max_neighbors float", lambda d: d.update(max_neighbors=3.5))
    bad("seed float", lambda d: d.update(seed=1.5))
    bad("max_frames zero", lambda d: d.update(max_frames=0))
    bad("goal_tolerance negative", lambda d: d.update(goal_tolerance=-1.0))
    bad("classes unknown", lambda d: d.update(classes={"bicycle": {"radius": 1}}))
    bad("classes not mapping", lambda d: d.update(classes={"vehicle": 3}))
    bad("class unknown field", lambda d: d.update(classes={"vehicle": {"mass": 3}}))
    bad("pref above max", lambda d: d.update(classes={"pedestrian": {"pref_speed": 9.0}}))
    bad("regions missing", lambda d: d.pop("regions") and None)
    bad("region not mapping", lambda d: d["regions"].__setitem__(0, 5))
    bad("region unknown field", lambda d: d["regions"][0].update(colour="red"))
    bad("rect short", lambda d: d["regions"][0].update(spawn=[0, 1, 2]))
    bad("rect degenerate", lambda d: d["regions"][0].update(goal=[5, 0, 1, 3]))
    bad("rect nan", lambda d: d["regions"][0].update(goal=[0, 0, float("nan"), 3]))
    bad("region class", lambda d: d["regions"][0].update(agent_class="tram"))
    bad("region class type", lambda d: d["regions"][0].update(agent_class=7))
    bad("count negative", lambda d: d["regions"][0].update(count=-2))
    bad("responsibility list", lambda d: d.update(responsibility=[1]))
    bad("responsibility key", lambda d: d.update(responsibility={"pedestrian": 1.0}))
    bad("responsibility value", lambda d: d["responsibility"].update({"pedestrian|vehicle": "all"}))
    bad("responsibility range", lambda d: d["responsibility"].update({"pedestrian|vehicle": 1.5}))
    bad("responsibility missing", lambda d: d["responsibility"].pop("vehicle|pedestrian") and None)
    bad("unguaranteed pair (warning only)", lambda d: d["responsibility"].update({"pedestrian|vehicle": 0.3}))
    bad("too dense", lambda d: d["regions"][0].update(count=100000))
    warn_cfg = S.scenario_from_dict({**json.loads(json.dumps(good)),
                                     "responsibility": {**good["responsibility"], "pedestrian|vehicle": 0.3,
                                                        "vehicle|vehicle": 0.2}}, source="<w>")
    # spawn failures surface at build time
    dense = json.loads(json.dumps(good))
    dense["regions"][0]["count"] = 100000
    try:
        S.build_agents(S.scenario_from_dict(dense, source="<t>"))
        dense_msg = None
    except S.ScenarioError as exc:
        dense_msg = str(exc)

    # CSV bytes of the reference's writers on a short reference run
    from orcasim.crossings import crossing_config
    cfg = crossing_config("two_way", 6, 0.34, seed=9)
    cfg.max_frames = 12
    res = E.run(cfg, worker_count=1, record_trajectories=True)
    with tempfile.TemporaryDirectory() as tmp:
        S.write_trajectories(res.frame_logs, os.path.join(tmp, "t.csv"))
        S.write_metrics_summary(res.summary, os.path.join(tmp, "m.csv"))
        _write_agents_csv(res, os.path.join(tmp, "a.csv"))
        traj_csv = open(os.path.join(tmp, "t.csv"), "rb").read()
        metrics_csv = open(os.path.join(tmp, "m.csv"), "rb").read()
        agents_csv = open(os.path.join(tmp, "a.csv"), "rb").read()
    with open(os.path.join(OUT, "traj_two_way_12.csv"), "wb") as f:
        f.write(traj_csv)
    with open(os.path.join(OUT, "agents_two_way_12.csv"), "wb") as f:
        f.write(agents_csv)

    # sha256 of the full trajectory files of the two whole-run fixtures (run_*.npz)
    run_sha = {}
    for name, kind, per_arm, vf, seed in (("two_way_80", "two_way", 40, 0.1, 3),
                                          ("four_way_96", "four_way", 24, 0.25, 5)):
        r = E.run(crossing_config(kind, per_arm, vf, seed), worker_count=2, record_trajectories=True)
        with tempfile.TemporaryDirectory() as tmp:
            S.write_trajectories(r.frame_logs, os.path.join(tmp, "t.csv"))
            _write_agents_csv(r, os.path.join(tmp, "a.csv"))
            run_sha[name] = dict(trajectories=hashlib.sha256(open(os.path.join(tmp, "t.csv"), "rb").read()).hexdigest(),
                                 agents=hashlib.sha256(open(os.path.join(tmp, "a.csv"), "rb").read()).hexdigest(),
                                 kind=kind, per_arm=per_arm, vehicle_fraction=vf, seed=seed,
                                 frames=r.summary.frames)
    with open(os.path.join(OUT, "scenario_cases.json"), "w") as f:
        json.dump(dict(cases=cases, broken=broken, warnings_two_pairs=warn_cfg.warnings,
                       dense_build_message=dense_msg,
                       short_run=dict(kind="two_way", per_arm=6, vehicle_fraction=0.34, seed=9, max_frames=12,
                                      metrics_csv_head=metrics_csv.decode().splitlines()[0],
                                      total_collisions=res.summary.total_collisions,
                                      min_separation=res.summary.min_separation, frames=res.summary.frames),
                       run_sha=run_sha), f)
    print("scenario_cases.json:", len(cases), "cases,", len(broken), "broken documents")


def gen_api():
    """api_cases.npz: the reference's OBJECT-level operators on seeded inputs --
    orca.gather_constraints, grid.query_neighbors, lp.solve_least_penetration and
    lp.solve_batch -- for the host wrappers of paper_2008_11578_b200 (orca.py, grid.py, lp.py)."""
    import orcasim
    from orcasim import AgentClass, AgentState, HalfPlaneConstraint, ResponsibilityMatrix
    rng = np.random.default_rng(77)
    n = 160
    pos = rng.uniform(0.0, 30.0, size=(n, 2))
    pos[5] = pos[4] + np.array([0.3, 0.0])                     # an overlapping pair (dt-horizon disc)
    vel = rng.normal(size=(n, 2))
    cls = (rng.random(n) < 0.15).astype(np.int64)
    radius = np.where(cls == 1, 1.0, 0.25) * (1.0 + 0.1 * rng.random(n))
    ids = rng.permutation(1000)[:n].astype(np.int64)
    agents = [AgentState(id=int(ids[i]), position=pos[i], velocity=vel[i], radius=float(radius[i]),
                         pref_speed=1.0, max_speed=2.0, goal=pos[i] + 1.0, agent_class=AgentClass(int(cls[i])))
              for i in range(n)]
    grid = orcasim.rebuild(agents, 4.0)
    out = {"ids": ids, "positions": pos, "velocities": vel, "radii": radius, "class_codes": cls,
           "grid_cells": np.array(sorted(grid.cells), dtype=np.int64), "grid_population": np.int64(grid.population)}
    for radius_q, max_count in ((6.0, 8), (3.5, 16), (9.0, 32), (50.0, 5)):
        rows = np.full((n, max_count), -1, dtype=np.int64)
        for i, a in enumerate(agents):
            nb = orcasim.query_neighbors(grid, agents, a.id, radius_q, max_count)
            rows[i, :len(nb)] = [b.id for b in nb]
        out[f"nb_ids_r{radius_q:g}_m{max_count}"] = rows
    matrix = ResponsibilityMatrix.default()
    cons_pts, cons_nrm, cons_cnt = np.zeros((n, 16, 2)), np.zeros((n, 16, 2)), np.zeros(n, dtype=np.int64)
    for i, a in enumerate(agents):
        nb = orcasim.query_neighbors(grid, agents, a.id, 6.0, 16)
        cs = orcasim.gather_constraints(a, nb, matrix, 2.0, 0.1)
        cons_cnt[i] = len(cs)
        for t, c in enumerate(cs):
            cons_pts[i, t], cons_nrm[i, t] = c.point, c.normal
    out.update(cons_pts=cons_pts, cons_nrm=cons_nrm, cons_cnt=cons_cnt)
    # least penetration on random (mostly infeasible) constraint sets, the given order, several warm starts
    lp_k, lp_pts, lp_nrm, lp_cap, lp_start, lp_warm, lp_out = [], [], [], [], [], [], []
    for case in range(60):
        k = int(rng.integers(0, 20))
        ang = rng.uniform(0, 2 * np.pi, k)
        nrm = np.column_stack([np.cos(ang), np.sin(ang)])
        pts = rng.normal(size=(k, 2)) * 1.2
        cap = float(0.5 + 2.0 * rng.random())
        start = int(rng.integers(0, k + 1))
        warm = rng.normal(size=2) * 0.5
        cs = [HalfPlaneConstraint(pts[t], nrm[t]) for t in range(k)]
        v = orcasim.solve_least_penetration(cs, cap, start_index=start, warm_start=warm)
        row_p, row_n = np.zeros((20, 2)), np.zeros((20, 2))
        row_p[:k], row_n[:k] = pts, nrm
        lp_k.append(k); lp_pts.append(row_p); lp_nrm.append(row_n); lp_cap.append(cap)
        lp_start.append(start); lp_warm.append(warm); lp_out.append(v)
    out.update(lp_k=np.array(lp_k), lp_pts=np.array(lp_pts), lp_nrm=np.array(lp_nrm), lp_cap=np.array(lp_cap),
               lp_start=np.array(lp_start), lp_warm=np.array(lp_warm), lp_out=np.array(lp_out))
    np.savez_compressed(os.path.join(OUT, "api_cases.npz"), **out)
    print("api_cases.npz", {k: getattr(v, "shape", None) for k, v in out.items()})


def main():
    os.makedirs(OUT, exist_ok=True)
    if os.environ.get("GEN_ONLY_API"):
        return gen_api()
    if os.environ.get("GEN_ONLY_RUN"):
        return gen_run()
    if os.environ.get("GEN_ONLY_PAPER"):
        return gen_run_paper()
    if os.environ.get("GEN_ONLY_SCENARIO"):
        return gen_scenarios()
    gen_kat()
    gen_lp_batches()
    gen_frames()
    gen_chain()
    gen_run()
    gen_run_paper()
    gen_scenarios()
    gen_api()


def gen_run():
    """Whole reference runs (engine.run) of the built-in crossing scenarios: the spawned
    crowd (the reference's own seeded sampling), the guard, and everything run() reports."""
    from orcasim.crossings import crossing_config
    for name, kind, per_arm, vf, seed in (("two_way_80", "two_way", 40, 0.1, 3),
                                          ("four_way_96", "four_way", 24, 0.25, 5)):
        cfg = crossing_config(kind, per_arm, vf, seed)
        st = E.init_state(cfg)
        res = E.run(cfg, worker_count=2, record_trajectories=True)
        s = res.summary
        nf = len(res.frame_metrics)
        n0 = st.active_count
        # trajectories: positions of every 10th frame (padded with NaN for removed agents)
        sample = list(range(0, nf, 10)) + [nf - 1]
        traj = np.full((len(sample), n0, 4), np.nan)
        row_of = {int(a): i for i, a in enumerate(st.ids)}
        for k, f in enumerate(sample):
            log = res.frame_logs[f]
            rows = [row_of[int(a)] for a in log.ids]
            traj[k, rows, :2] = log.positions
            traj[k, rows, 2:] = log.velocities
        arr_ids = np.array(sorted(row_of), dtype=np.int64)
        # arrival time per agent id, NaN if it never arrived
        arrival = np.full(n0, np.nan)
        last_seen = {}
        for log in res.frame_logs:
            for a in log.ids:
                last_seen[int(a)] = log.time
        if s.terminated or s.arrived:
            final_ids = set(int(a) for a in res.final_state.ids)
            for a, t in last_seen.items():
                if a not in final_ids:
                    arrival[row_of[a]] = t
        np.savez_compressed(
            os.path.join(OUT, f"run_{name}.npz"),
            ids=st.ids, positions=st.positions, velocities=st.velocities, radii=st.radii,
            pref_speeds=st.pref_speeds, max_speeds=st.max_speeds, goals=st.goals,
            goal_tols=st.goal_tols, class_codes=st.class_codes.astype(np.int8),
            dt=cfg.dt, tau=cfg.tau, neighbor_radius=cfg.neighbor_radius,
            max_neighbors=np.int64(cfg.max_neighbors), avoidance_margin=cfg.avoidance_margin,
            fmat=cfg.responsibility.as_array(), guard=np.int64(cfg.frame_guard()), seed=np.int64(cfg.seed),
            frames=np.int64(s.frames), terminated=np.bool_(s.terminated), arrived=np.int64(s.arrived),
            total_collisions=np.int64(s.total_collisions), min_separation=np.float64(s.min_separation),
            total_fallbacks=np.int64(s.total_fallbacks),
            travel_ped=np.float64(s.mean_travel_time.get(E.AgentClass.PEDESTRIAN, np.nan)),
            travel_veh=np.float64(s.mean_travel_time.get(E.AgentClass.VEHICLE, np.nan)),
            m_min_sep=np.array([m.min_separation for m in res.frame_metrics]),
            m_coll=np.array([m.collision_count for m in res.frame_metrics], dtype=np.int64),
            m_active=np.array([m.active_agents for m in res.frame_metrics], dtype=np.int64),
            arrival=arrival, sample_frames=np.array(sample, dtype=np.int64), traj=traj,
            final_ids=res.final_state.ids)
        print(f"run_{name}.npz agents={n0} frames={s.frames} terminated={s.terminated} "
              f"arrived={s.arrived} collisions={s.total_collisions} fallbacks={s.total_fallbacks}")


def _mix64(z):
    z = z.astype(np.uint64, copy=True)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def frame_digest(ids, positions, velocities) -> int:
    """Order-independent 64-bit digest of {id: (position bits, velocity bits)} -- the function of
    paper_2008_11578_b200.parallel.strips.state_hash, restated here so that the generator needs
    nothing but the reference."""
    mix = np.uint64(0x9E3779B97F4A7C15)
    ids = np.ascontiguousarray(ids, dtype=np.int64).view(np.uint64)
    p = np.ascontiguousarray(positions, dtype=np.float64).view(np.uint64).reshape(-1, 2)
    v = np.ascontiguousarray(velocities, dtype=np.float64).view(np.uint64).reshape(-1, 2)
    with np.errstate(over="ignore"):
        h = _mix64(ids * mix + np.uint64(1))
        for col in (p[:, 0], p[:, 1], v[:, 0], v[:, 1]):
            h = _mix64(h ^ (col + mix))
        return int(h.sum(dtype=np.uint64))


def gen_run_paper():
    """The paper's own experiment scale: 2- and 4-way crossings of
    2,500 agents, run to termination by the reference. Too long for per-frame trajectories in a
    fixture: every frame is pinned by an id-keyed 64-bit digest of (position, velocity) of the agents
    active in it, plus the per-frame metrics and the run summary."""
    from orcasim.crossings import crossing_config
    for name, kind, per_arm, vf, seed in (("paper_four_way_2500", "four_way", 625, 0.1, 11),
                                          ("paper_two_way_2500", "two_way", 1250, 0.1, 12)):
        cfg = crossing_config(kind, per_arm, vf, seed)
        st = E.init_state(cfg)
        res = E.run(cfg, worker_count=os.cpu_count() or 1, record_trajectories=True)
        s = res.summary
        digests = np.array([frame_digest(l.ids, l.positions, l.velocities) for l in res.frame_logs], dtype=np.uint64)
        np.savez_compressed(
            os.path.join(OUT, f"run_{name}.npz"),
            ids=st.ids, positions=st.positions, velocities=st.velocities, radii=st.radii,
            pref_speeds=st.pref_speeds, max_speeds=st.max_speeds, goals=st.goals,
            goal_tols=st.goal_tols, class_codes=st.class_codes.astype(np.int8),
            dt=cfg.dt, tau=cfg.tau, neighbor_radius=cfg.neighbor_radius,
            max_neighbors=np.int64(cfg.max_neighbors), avoidance_margin=cfg.avoidance_margin,
            fmat=cfg.responsibility.as_array(), guard=np.int64(cfg.frame_guard()), seed=np.int64(cfg.seed),
            frames=np.int64(s.frames), terminated=np.bool_(s.terminated), arrived=np.int64(s.arrived),
            total_collisions=np.int64(s.total_collisions), min_separation=np.float64(s.min_separation),
            total_fallbacks=np.int64(s.total_fallbacks),
            travel_ped=np.float64(s.mean_travel_time.get(E.AgentClass.PEDESTRIAN, np.nan)),
            travel_veh=np.float64(s.mean_travel_time.get(E.AgentClass.VEHICLE, np.nan)),
            m_min_sep=np.array([m.min_separation for m in res.frame_metrics]),
            m_coll=np.array([m.collision_count for m in res.frame_metrics], dtype=np.int64),
            m_active=np.array([m.active_agents for m in res.frame_metrics], dtype=np.int64),
            digests=digests, final_ids=res.final_state.ids)
        print(f"run_{name}.npz agents={st.active_count} frames={s.frames} terminated={s.terminated} "
              f"arrived={s.arrived} collisions={s.total_collisions} fallbacks={s.total_fallbacks}")


if __name__ == "__main__":
    main()
