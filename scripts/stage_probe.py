"""Stage times (ms/step) of the resident step with arrival removal and metrics on, as engine.step runs it."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2008_11578_b200 import Simulation
from paper_2008_11578_b200.synth import plaza_crowd
st, cfg = plaza_crowd(1032192, 16384, density=0.25, seed=100)
for rem, met in ((False, False), (True, False), (True, True)):
    sim = Simulation(cfg, capacity=st.active_count, remove_arrivals=rem, compute_metrics=met)
    sim.load(st); sim.run(10); sim.sync()
    sim.profile_stages(True); sim.run(50); ms, cov = sim.stage_ms(); sim.profile_stages(False)
    print(rem, met, {k: round(v / cov, 4) for k, v in ms.items()}, "total", round(sum(ms.values()) / cov, 4), "n", sim.info().active_agents)
    sim.close()
