"""Small end-to-end exercise of every kernel family for compute-sanitizer runs:
    compute-sanitizer --tool memcheck  python scripts/sanitize_probe.py
    compute-sanitizer --tool racecheck python scripts/sanitize_probe.py
"""
import os, sys
import numpy as np
os.environ["ORCA_CERT_FORCE"] = "1"   # the certified kernels on small crowds too
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2008_11578_b200 import Simulation, LpBatch, step
from paper_2008_11578_b200.synth import plaza_crowd, lp_batch

for prec in ("mixed", "cert32", "f32", "f64"):
    for dens in (0.3, 2.0):
        st, cfg = plaza_crowd(3000, 100, density=dens, seed=3)
        rng = np.random.default_rng(1)
        close = rng.permutation(st.active_count)[:300]
        st.goals[close] = st.positions[close] + rng.normal(size=(300, 2)) * 0.5
        with Simulation(cfg, capacity=st.active_count, precision=prec, remove_arrivals=True, compute_metrics=True) as sim:
            sim.load(st)
            sim.run(4)
            s2 = sim.state()
            pos, vel, info = sim.advance_host(s2.positions, s2.velocities, s2.frame)
            sim.reorder_rows()
            sim.step()
            sim.sync()
        print(prec, dens, "ok", s2.active_count, int(info.active_agents))
# a queue long enough for the 4-lanes-per-agent fallback instance and the lane-per-entry exact search
st, cfg = plaza_crowd(40000, 800, density=1.5, seed=6)
with Simulation(cfg, capacity=st.active_count, precision="mixed", remove_arrivals=False) as sim:
    sim.load(st)
    sim.run(3)
    print("dense 40k ok, fallbacks", int(sim.info().lp_fallbacks))
cur, cfg = plaza_crowd(2000, 50, density=0.5, seed=4)
for _ in range(3):
    cur, m = step(cur, cfg)
coff, cpts, cnrm, tgt, caps, seeds = lp_batch(4000, 8, 64, 0.5, seed=5)
for prec in ("f64", "f32"):
    b = LpBatch(coff, cpts, cnrm, tgt, caps, seeds, precision=prec)
    b.solve()
    v, stt, fa = b.results()
    b.close()
print("lp done", m.active_agents, int(stt.sum()))

# round 2: chunked pipeline on two streams (ORCA_CHUNKS forces it on a small crowd), the device-side
# frame log, the slab protocol of the strip decomposition (two handles in lock step), the taps
import torch
sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ["ORCA_CHUNKS"] = "2"
st, cfg = plaza_crowd(6000, 200, density=0.8, seed=8)
rng = np.random.default_rng(2)
close = rng.permutation(st.active_count)[:500]
st.goals[close] = st.positions[close] + rng.normal(size=(500, 2)) * 0.5
for prec in ("cert32", "mixed"):
    with Simulation(cfg, capacity=st.active_count, precision=prec, remove_arrivals=True, compute_metrics=True) as sim:
        sim.load(st)
        recs, traj, arr = sim.run_logged(6, st.active_count, with_trajectories=True)
        kept = sim.last_step_kept(int(recs[-1]["rows_before"]))
        s2 = sim.state()
    print("chunks + frame log", prec, len(recs), traj.shape, arr[0].shape, int(kept.sum()), s2.active_count)
del os.environ["ORCA_CHUNKS"]
import strip_ops_cpu as S
from test_gpu_strips import build_strips, lockstep
st, cfg = S.make_crowd(seed=4, n_ped=4000, n_veh=200, density=0.5)
for prec, world, transport in (("mixed", 2, "sendrecv"), ("f64", 3, "sendrecv"), ("mixed", 3, "window"),
                               ("f64", 2, "window")):
    sims, drivers, _b = build_strips(st, cfg, prec, world, halo_cap=st.ids.shape[0], mig_cap=2000, resync_every=3,
                                     transport=transport)
    lockstep(drivers, 7)
    print("strips", prec, world, transport, [s.state().ids.shape[0] for s in sims], [d.ops.stats() for d in drivers])
    for s_ in sims:
        s_.close()
from paper_2008_11578_b200 import HalfPlaneConstraint, solve_least_penetration
from paper_2008_11578_b200.grid import neighbor_lists, neighbor_lists_all
rows, cnt = neighbor_lists(st.ids, st.positions, 5.0, 12)
off, allrows = neighbor_lists_all(st.ids, st.positions, 6.0)          # the uncapped query (CSR)
print("neighbor_lists_all", off[-1], allrows.shape)
ang = rng.uniform(0, 6.28, 9)
v = solve_least_penetration([HalfPlaneConstraint(rng.normal(size=2), (np.cos(a), np.sin(a))) for a in ang], 1.5,
                            start_index=3, warm_start=(0.1, 0.2))
print("probe done", rows.shape, int(cnt.sum()), v)
