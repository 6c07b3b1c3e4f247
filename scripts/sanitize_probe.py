"""Small end-to-end exercise of every kernel family for compute-sanitizer runs:
    compute-sanitizer --tool memcheck  python scripts/sanitize_probe.py
    compute-sanitizer --tool racecheck python scripts/sanitize_probe.py
"""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2008_11578_b200 import Simulation, LpBatch, step
from paper_2008_11578_b200.synth import plaza_crowd, lp_batch

for prec in ("mixed", "f32", "f64"):
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
print("probe done", m.active_agents, int(stt.sum()))
