import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2008_11578_b200 import engine as E
from paper_2008_11578_b200.synth import plaza_crowd
st, cfg = plaza_crowd(1032192, 16384, density=0.25, seed=100)
n = st.active_count
cur = st
for _ in range(3):
    cur, m = E.step(cur, cfg)
from paper_2008_11578_b200 import Simulation
sim = Simulation(cfg, capacity=n, remove_arrivals=False, compute_metrics=True)
sim.load(cur)
def T(f, reps=5):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); r = f(); ts.append((time.perf_counter() - t0) * 1e3)
    return min(ts), r
print("host_empty x2", T(lambda: (E._host_empty((n, 2)), E._host_empty((n, 2))))[0])
print("np.empty x2", T(lambda: (np.empty((n, 2)), np.empty((n, 2))))[0])
print("set_config", T(lambda: sim.set_config(cfg, False, True))[0])
print("load_pv", T(lambda: (sim.load_pv(cur.positions, cur.velocities, 5), sim.sync()))[0])
print("step+sync", T(lambda: (sim.step(), sim.sync()))[0])
print("info", T(lambda: sim.info())[0])
print("positions_velocities", T(lambda: sim.positions_velocities())[0])
pos, vel = E._host_empty((n, 2)), E._host_empty((n, 2))
from paper_2008_11578_b200._lib import ptr
print("download_pv into pinned", T(lambda: sim._L.orca_download_pv(sim._h, ptr(pos), ptr(vel)))[0])
pos2, vel2 = np.empty((n, 2)), np.empty((n, 2))
print("download_pv into pageable", T(lambda: sim._L.orca_download_pv(sim._h, ptr(pos2), ptr(vel2)))[0])
print("full step()", T(lambda: E.step(cur, cfg))[0])
t0 = time.perf_counter()
c = cur
for _ in range(10):
    c, m = E.step(c, cfg)
print("loop avg", (time.perf_counter() - t0) * 100)
c = cur
ts = []
for _ in range(30):
    t0 = time.perf_counter()
    n0 = c.active_count
    c, m = E.step(c, cfg)
    ts.append(((time.perf_counter() - t0) * 1e3, n0 - c.active_count, E.step.last_traffic))
print("per-iteration ms / removed / traffic:", [(round(a, 2), b, t[0] // n, t[1] // n) for a, b, t in ts])
