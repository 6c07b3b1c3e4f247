"""Per-step device time over a long resident run (CUDA events around every orca_step on the handle's stream):
where do reorder frames, graph captures and the crowd's own evolution show?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2008_11578_b200 import Simulation
from paper_2008_11578_b200.synth import make_workload
wl = sys.argv[1] if len(sys.argv) > 1 else "plaza_1m"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 300
st, cfg = make_workload(wl, seed=100)
stream = torch.cuda.Stream()
sim = Simulation(cfg, capacity=st.active_count, precision=os.environ.get("PREC", "cert32"), remove_arrivals=False,
                 compute_metrics=False, stream=stream)
sim.load(st)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
ev[0].record(stream)
for i in range(steps):
    sim.step()
    ev[i + 1].record(stream)
sim.sync()
ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
for b in range(0, steps, 16):
    seg = ms[b:b + 16]
    print(f"{b:4d}: " + " ".join(f"{x:.3f}" for x in seg))
print("fallbacks last step", sim.info().lp_fallbacks)
