import sys, os, numpy as np, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import oracle as O
from paper_2008_11578_b200 import Simulation
from paper_2008_11578_b200.synth import make_workload
import torch
for name in sys.argv[1:]:
    st, cfg = make_workload(name, seed=100)
    n = st.active_count
    fs = O.frame_solve(st, cfg, worker_count=16, debug="lists")
    for prec in ("mixed", "cert32"):
        with Simulation(cfg, capacity=n, precision=prec, remove_arrivals=False) as sim:
            sim.load(st); sim.step(); sim.sync()
            info = sim.info()
            d = sim.debug_last_step(n, cfg.max_neighbors)
            dv = np.abs(d["out_v"] - fs.out_v).max(axis=1)
            print(name, prec, "flips", int((d["status"] != fs.status).sum()), "failed_at diffs", int((d["failed_at"] != fs.failed_at).sum()),
                  "max dv %.3e" % dv.max(), ">1e-6:", int((dv > 1e-6).sum()), "fallbacks", int(info.lp_fallbacks), "uncertified", int(info.solve_queue), "of", n)
            if prec == "cert32":
                sim.load(st)
            stream = None
            sim.run(10); sim.sync()
            sim.profile_stages(True); sim.run(30); ms, cov = sim.stage_ms(); sim.profile_stages(False)
            print("   stages", {k: round(v / cov, 4) for k, v in ms.items()}, "total", round(sum(ms.values()) / cov, 4))
            t0=time.perf_counter(); sim.run(50); sim.sync(); print("   wall ms/step", (time.perf_counter()-t0)*1e3/50, "uncert last", int(sim.info().solve_queue))
