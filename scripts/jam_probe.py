"""Long resident run of the jammed crowd (2 /m2): does an FP32 state reach the reference's
coincident-centres error (two agents rounded onto the same float32 position) where FP64 does not?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_11578_b200 import Simulation
from paper_2008_11578_b200.synth import make_workload
for prec in ("cert32", "mixed", "f64"):
    st, cfg = make_workload("config3_262k_d2", seed=100)
    sim = Simulation(cfg, capacity=st.active_count, precision=prec, remove_arrivals=False, compute_metrics=False)
    sim.load(st)
    done = 0
    try:
        for k in range(12):
            sim.run(50); sim.sync(); done += 50
        print(prec, "ran", done, "frames, no error")
    except Exception as e:
        print(prec, "error after", done, "+<=50 frames:", str(e)[:200])
    sim.close()
