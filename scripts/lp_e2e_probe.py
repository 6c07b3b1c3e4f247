import sys, os, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2008_11578_b200 import solve_range
from paper_2008_11578_b200.synth import lp_batch
keep=[]
def pin(a):
    a=np.ascontiguousarray(a); t=torch.from_numpy(a.view(np.int64) if a.dtype==np.uint64 else a).pin_memory(); keep.append(t); return t.numpy().view(a.dtype)
for frac in (0.0, 1.0):
    args=[pin(a) for a in lp_batch(1<<20, 8, 64, frac, seed=5)]
    solve_range(*args)
    for rep in range(3):
        t0=time.perf_counter(); solve_range(*args); print(frac, "pinned", round((time.perf_counter()-t0)*1e3,1), "ms")
