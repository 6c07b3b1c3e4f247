#!/usr/bin/env python
"""BASELINE config 4: batched LP microbench -- 1,048,576 independent 2-D LPs with 8..64
half-plane constraints each (mean 36), three mixes (all feasible / half / all
unconstrained-geometry, i.e. ~99.7 % infeasible), through orca_lp_batch_* with the batch
resident on the device; the CPU port of the reference's solve_range runs beside it on a
bounded sample. Prints one JSON object per (mix, precision).

    python scripts/bench_lp.py [--n 1048576] [--repeats 5] [--cpu-n 65536]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2008_11578_b200 import LpBatch  # noqa: E402
from paper_2008_11578_b200.synth import lp_batch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 20)
ap.add_argument("--repeats", type=int, default=5)
ap.add_argument("--cpu-n", type=int, default=1 << 16)
args = ap.parse_args()
hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
threads = os.cpu_count() or 1

for name, frac in (("feasible", 0.0), ("mixed", 0.5), ("infeasible", 1.0)):
    coff, cpts, cnrm, tgt, caps, seeds = lp_batch(args.n, 8, 64, frac, seed=5)
    m = int(coff[-1])
    # CPU port on a bounded sample of the same batch
    cn = min(args.cpu_n, args.n)
    sub = (coff[:cn + 1], cpts[:coff[cn]], cnrm[:coff[cn]], tgt[:cn], caps[:cn], seeds[:cn])
    O.solve_range(*sub, worker_count=threads)
    t0 = time.perf_counter()
    cv, cst, cfa = O.solve_range(*sub, worker_count=threads)
    cpu_rate = cn / (time.perf_counter() - t0)
    for prec in ("f64", "f32"):
        stream = torch.cuda.Stream()
        b = LpBatch(coff, cpts, cnrm, tgt, caps, seeds, precision=prec, stream=stream)
        for _ in range(3):
            b.solve()
        v, st, fa = b.results()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.repeats):
            b.solve()
        e1.record(stream)
        b.results()
        ms = e0.elapsed_time(e1) / args.repeats
        b.close()
        dv = np.abs(v[:cn] - cv).max(axis=1)
        rs = 4 if prec == "f32" else 8
        alg_bytes = (4 * rs) * m + (3 * rs + 8 + 8 + 16 + 16) * args.n      # constraints + per-LP in/out
        print(json.dumps({
            "mix": name, "precision": prec, "n_lps": args.n, "constraints": m, "ms": ms,
            "lps_per_s": args.n / ms * 1e3, "constraints_per_s": m / ms * 1e3,
            "fallback_frac": float((st != 0).mean()),
            "hbm_frac_of_measured": alg_bytes / (ms * 1e-3) / 1e9 / hbm,
            "parity_vs_cpu_port": {"n": cn, "status_flips": int((st[:cn] != cst).sum()),
                                   "bit_exact": bool(np.array_equal(v[:cn], cv)),
                                   "max_abs_dv": float(dv.max()), "gt_1e-4": int((dv > 1e-4).sum())},
            "cpu_port": {"lps_per_s": cpu_rate, "threads": threads, "sample": cn}}), flush=True)
