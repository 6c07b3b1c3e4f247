#!/usr/bin/env python
"""Development probe (not part of the product): parity census + quick timings on
the GPU box. Writes gpurun_out/probe.json and prints a summary."""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import FRAME_FIXTURES, LP_FIXTURES, load_golden, state_from_frame_fixture  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2008_11578_b200 import Simulation, solve_range  # noqa: E402
from paper_2008_11578_b200.synth import lp_batch, plaza_crowd  # noqa: E402

out = {}


def census(dv, st_g, st_o):
    return dict(n=int(dv.size), max=float(dv.max()) if dv.size else 0.0,
                p50=float(np.median(dv)) if dv.size else 0.0,
                p99=float(np.quantile(dv, 0.99)) if dv.size else 0.0,
                gt1e4=int((dv > 1e-4).sum()), status_diff=int((st_g != st_o).sum()))


def frame_case(name, state, cfg, ref):
    n = state.active_count
    res = {}
    for prec in ("f64", "f32"):
        with Simulation(cfg, capacity=n, precision=prec, remove_arrivals=False) as sim:
            sim.load(state)
            sim.step()
            sim.sync()
            d = sim.debug_last_step(n, cfg.max_neighbors)
        dv = np.abs(d["out_v"] - ref["out_v"]).max(axis=1)
        r = census(dv, d["status"], ref["status"])
        r.update(cells=bool(np.array_equal(d["cell_ix"], ref["cell_ix"]) and np.array_equal(d["cell_iy"], ref["cell_iy"])),
                 nb=bool(np.array_equal(d["nb_rows"], ref["nb_rows"]) and np.array_equal(d["nb_count"], ref["nb_count"])),
                 des_exact=bool(np.array_equal(d["des"], ref["des"])),
                 v_exact=bool(np.array_equal(d["out_v"], ref["out_v"])),
                 failed_exact=bool(np.array_equal(d["failed_at"], ref["failed"])))
        res[prec] = r
        print(name, prec, r, flush=True)
    out[name] = res


for fx in FRAME_FIXTURES:
    g = load_golden(fx)
    st, cfg = state_from_frame_fixture(g)
    frame_case(fx, st, cfg, dict(out_v=g["out_v"], status=g["status"].astype(np.int64), cell_ix=g["cell_ix"],
                                 cell_iy=g["cell_iy"], nb_rows=g["nb_rows"].astype(np.int64)[:, :max(int(g["max_neighbors"]), 1)],
                                 nb_count=g["nb_count"].astype(np.int64), des=g["des"],
                                 failed=g["failed"].astype(np.int64)))

for fx in LP_FIXTURES:
    g = load_golden(fx)
    for prec in ("f64", "f32"):
        v, st, fa = solve_range(g["coff"], g["cpts"], g["cnrm"], g["tgt"], g["caps"], g["seeds"], precision=prec)
        dv = np.abs(v - g["out_v"]).max(axis=1)
        r = census(dv, st, g["status"].astype(np.int64))
        r.update(v_exact=bool(np.array_equal(v, g["out_v"])), failed_exact=bool(np.array_equal(fa, g["failed"].astype(np.int64))))
        out[f"{fx}:{prec}"] = r
        print(fx, prec, r, flush=True)

# bigger scenes against the C oracle
for name, (nped, nveh, dens) in {"16k": (16384, 256, 0.25), "66k_d1": (65536, 1024, 1.0)}.items():
    st, cfg = plaza_crowd(nped, nveh, density=dens, seed=2)
    t0 = time.time()
    fs = O.frame_solve(st, cfg, worker_count=os.cpu_count(), debug=True)
    print(name, "oracle s", time.time() - t0, flush=True)
    frame_case(name, st, cfg, dict(out_v=fs.out_v, status=fs.status, cell_ix=fs.cell_ix, cell_iy=fs.cell_iy,
                                   nb_rows=fs.nb_rows, nb_count=fs.nb_count, des=fs.des, failed=fs.failed_at))

# timings
import torch  # noqa: E402

for name, (nped, nveh, dens) in {"16k": (16384, 256, 0.25), "262k_d1": (262144, 4096, 1.0),
                                 "1m": (1032192, 16384, 0.25)}.items():
    st, cfg = plaza_crowd(nped, nveh, density=dens, seed=3)
    for prec in ("f32", "f64"):
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            with Simulation(cfg, capacity=st.active_count, precision=prec, remove_arrivals=False, stream=stream) as sim:
                sim.load(st)
                sim.run(3)
                sim.sync()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                sim.run(10)
                e1.record(stream)
                sim.sync()
                ms = e0.elapsed_time(e1) / 10
                info = sim.info()
        out[f"time:{name}:{prec}"] = dict(ms_per_step=ms, agent_steps_per_s=st.active_count / ms * 1e3,
                                          fallbacks=int(info.lp_fallbacks), grid=(info.grid_nx, info.grid_ny, info.grid_cell))
        print("time", name, prec, out[f"time:{name}:{prec}"], flush=True)

for frac in (0.0, 0.5, 1.0):
    coff, cpts, cnrm, tgt, caps, seeds = lp_batch(1 << 18, 8, 64, frac, seed=5)
    from paper_2008_11578_b200 import LpBatch
    for prec in ("f32", "f64"):
        stream = torch.cuda.Stream()
        b = LpBatch(coff, cpts, cnrm, tgt, caps, seeds, precision=prec, stream=stream)
        b.solve()
        b.results()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            b.solve()
        e1.record(stream)
        b.results()
        ms = e0.elapsed_time(e1) / 5
        out[f"lp_time:{frac}:{prec}"] = dict(ms=ms, lps_per_s=b.n / ms * 1e3)
        print("lp time", frac, prec, out[f"lp_time:{frac}:{prec}"], flush=True)
        b.close()

os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "probe.json"), "w") as f:
    json.dump(out, f, indent=1, default=str)
