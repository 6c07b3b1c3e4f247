"""Resident ms/step of the named workloads and ms/solve of the LP mixes (development tooling).
    python scripts/perf_probe.py [precision] workload ..."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_11578_b200 import LpBatch, Simulation  # noqa: E402
from paper_2008_11578_b200.synth import CONFIGS, lp_batch, make_workload  # noqa: E402

LP = {"lp_1m_feasible": 0.0, "lp_1m_half": 0.5, "lp_1m_infeasible": 1.0}
prec = "mixed"
for name in sys.argv[1:]:
    if name in ("mixed", "f64", "f32", "cert32"):
        prec = name
        continue
    stream = torch.cuda.Stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if name in LP:
        args = lp_batch(1 << 20, 8, 64, LP[name], seed=5)
        for p in ("f64", "f32"):
            bt = LpBatch(*args, precision=p, stream=stream)
            for _ in range(3):
                bt.solve()
            bt.results()
            a.record(stream)
            for _ in range(10):
                bt.solve()
            b.record(stream)
            bt.results()
            torch.cuda.synchronize()
            print(f"{name:22s} {p:6s} {a.elapsed_time(b) / 10:8.3f} ms/solve", flush=True)
            bt.close()
        continue
    st, cfg = make_workload(name, seed=100)
    with Simulation(cfg, capacity=st.active_count, precision=prec, remove_arrivals=False, stream=stream) as sim:
        sim.load(st)
        sim.run(10)
        sim.sync()
        a.record(stream)
        sim.run(50)
        b.record(stream)
        sim.sync()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 50
        sim.profile_stages(True)
        sim.run(20)
        stg, cov = sim.stage_ms()
        sim.profile_stages(False)
        print(f"{name:22s} {prec:6s} {ms:8.4f} ms/step  " + " ".join(f"{k}={v / cov:.3f}" for k, v in stg.items()),
              flush=True)
