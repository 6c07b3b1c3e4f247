#!/usr/bin/env python
"""Benchmark of the ORCA steering step (BASELINE.json: agent-steps/s and ms/step
at 1M agents).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--workload plaza_1m] [--precision mixed|f32|f64]

One "step" is one frame of the steering step (bin build, neighbour gather, ORCA
half-planes, LP + least-penetration fallback, integration) over the whole
synthetic crowd. Prints ONE JSON line on rank 0.

  value        agent-steps/s with the crowd resident in HBM (orca_step x K)
  e2e          the same metric through the drop-in call a reference user makes,
               engine.step(state, config): host SimState in, host SimState +
               FrameMetrics out (arrival removal and metrics included), with
               the H2D / D2H copies inside the timed region
  roofline     the dominant kernel of the step, timed live with CUDA events on
               the launching stream (orca_profile_stages), against the measured
               HBM peak of MEASURED_PEAKS.json
  roofline.traffic / roofline.ncu   DRAM bytes per launch and issue / pipe utilisation of
               that kernel from the committed ncu capture (profiles/traffic.json)
  cpu_baseline oracle/orca_oracle.c (a C port of the reference's step, pinned
               bit-exactly to the reference) on this box's host cores: one whole
               step of the same crowd, all host threads
  extras       context: the other precision modes on this workload and BASELINE
               config 5 (8.5 M agents) resident on this one GPU (--no-extras skips)
  --impl reference   times that CPU port as the reference arm (the Python+numba
               reference itself cannot travel to the GPU box)

--workload lp_1m_feasible | lp_1m_half | lp_1m_infeasible: the batched-LP microbench of
BASELINE config 4 (metric LP/s), same JSON contract.

Multi-GPU (torchrun, one rank per GPU): the plaza is cut into x-strips, one per
rank, with per-step halo exchange and migration over NCCL (parallel/strips.py);
weak scaling: every rank owns `workload` agents.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2008_11578_b200.synth import CONFIGS, make_workload  # noqa: E402

# algorithmic bytes
STEP_BYTES_PER_AGENT = 64          # read 44 + write 20, FP32 state
GATHER_BYTES_PER_AGENT = 8 + 4 + 4 * 16 + 1   # read (x,y) + cell id, write 16 neighbour slots + count
SOLVE_BYTES_PER_AGENT = 16 + 32 + 1 + 4 * 16 + 1 + 16 + 16 + 2 + 1  # sorted snapshot, des/max/avoid, class, lists, goal, out pv, status, arrived
BINS_BYTES_PER_AGENT = 16 + 4 + 4 + (16 + 16 + 8 + 1 + 8) + (8 + 16 + 32 + 4 + 4 + 1)  # bbox+count pass, scatter reads, scatter writes


def load_traffic(workload, precision, kernel):
    """ncu-measured DRAM bytes per launch of `kernel` (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f).get(f"{workload}/{precision}", {})
        return t.get(kernel), t.get("source"), t.get("ncu", {}).get(kernel)
    except Exception:
        return None, None, None


def load_peaks():
    """Measured HBM copy bandwidth of this pool's B200s (MEASURED_PEAKS.json, driver-written), else
    the fallback B200_PROFILING.md states."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            peaks = json.load(f)
        for key in ("hbm_gbs", "hbm_gb_s", "hbm_GBs", "hbm"):
            if key in peaks and float(peaks[key]) > 0:
                return float(peaks[key]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        pass
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Samples SM clock and throttle reasons through NVML while the timed region runs."""

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._thr = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = int(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        names = {"hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
                 "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
                 "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
                 "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4)}
        while not self._stop.is_set():
            try:
                self.samples.append(int(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)))
                try:
                    mask = int(nv.nvmlDeviceGetCurrentClocksEventReasons(self._h))
                except Exception:
                    mask = int(nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h))
                for k, bit in names.items():
                    if mask & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self._nv is not None:
            self._thr = threading.Thread(target=self._run, daemon=True)
            self._thr.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thr is not None:
            self._thr.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def build_workload(name: str, rank: int = 0, world: int = 1):
    n_ped, n_veh, density = CONFIGS[name]
    state, cfg = make_workload(name, seed=100 + rank)
    if os.environ.get("ORCA_BENCH_SORTED"):
        # experiment: storage rows in spatial (column-major cell) order instead of random order
        c = float(os.environ["ORCA_BENCH_SORTED"])
        key = np.floor(state.positions[:, 0] / c) * 1e6 + np.floor(state.positions[:, 1] / c)
        o = np.argsort(key, kind="stable")
        for f in ("ids", "positions", "velocities", "radii", "pref_speeds", "max_speeds", "goals", "goal_tols",
                  "class_codes"):
            setattr(state, f, np.ascontiguousarray(getattr(state, f)[o]))
    return state, cfg, dict(workload=name, pedestrians=n_ped, vehicles=n_veh, density_per_m2=density,
                            neighbor_radius=cfg.neighbor_radius, max_neighbors=cfg.max_neighbors,
                            dt=cfg.dt, tau=cfg.tau)


def cpu_port_rate(state, cfg, rows: int, threads: int, repeats: int = 1):
    """agent-steps/s of the oracle port, from a bounded sample: the whole-crowd part of
    the step (grid build, desired velocities) is timed in full, the per-agent part
    (neighbour query, ORCA, LP, integration) on agents [0, rows) and scaled by n/rows.
    Returns (agent-steps/s of a full step, seconds of CPU wall time spent per repeat)."""
    from oracle import oracle as O
    O.lib()
    n = state.active_count
    best_full, spent = None, 0.0
    for _ in range(repeats):
        t0 = time.perf_counter()
        O.frame_solve(state, cfg, worker_count=threads, rows=0)
        t_common = time.perf_counter() - t0
        t0 = time.perf_counter()
        fs = O.frame_solve(state, cfg, worker_count=threads, rows=rows)
        _ = state.positions[:rows] + fs.out_v[:rows] * cfg.dt      # engine.py:249
        t_rows = max(time.perf_counter() - t0 - t_common, 1e-9)
        full = t_common + t_rows * (n / rows)
        spent = t_common * 2 + t_rows
        best_full = full if best_full is None else min(best_full, full)
    return n / best_full, spent


def numba_reference(state, cfg, budget_s: float = 40.0):
    """The UNMODIFIED reference (Python + numba, installed into baseline/_ref by
    __graft_entry__.build(); git-ignored, travels with the snapshot) through ITS OWN public
    engine.step (pkg/src/orcasim/engine.py:298; arrival removal and frame metrics included, as
    in this repository's e2e), after its own JIT warm-up (pkg/src/orcasim/bench.py:55-58), at
    worker_count = all host cores and 1, on the crowd the GPU arm was timed on. The state and
    config objects of this package mirror the reference's field for field, so they are passed
    as they are. Returns a dict for cpu_baseline["reference_numba"]."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "orcasim")):
        return {"unavailable": "baseline/_ref/orcasim is not installed (run __graft_entry__.build() "
                               "where /root/reference exists)"}
    try:
        import tempfile
        os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_"))
        if ref_dir not in sys.path:
            sys.path.insert(0, ref_dir)
        from orcasim import bench as rbench
        from orcasim import engine as rengine
        t0 = time.perf_counter()
        rbench.warmup()
        warm_s = time.perf_counter() - t0
        n = state.active_count
        threads = os.cpu_count() or 1
        out = {"kind": "reference", "impl": "orcasim 0.1.0 (numba %s), engine.step" % __import__("numba").__version__,
               "agents": n, "jit_warmup_s": round(warm_s, 2), "unit": "agent-steps/s"}
        spent = 0.0
        for w in (threads, 1):
            times = []
            while len(times) < 3 and spent < budget_s * (0.6 if w == threads else 1.0):
                t0 = time.perf_counter()
                rengine.step(state, cfg, worker_count=w)
                times.append(time.perf_counter() - t0)
                spent += times[-1]
                if len(times) == 1 and times[0] * 2 > budget_s * 0.5:
                    break
            if times:
                out[f"workers_{w}"] = {"value": n / min(times), "s_per_step": min(times), "steps_timed": len(times)}
        return out
    except Exception as e:      # the reference arm must never take the GPU line down
        return {"unavailable": f"{type(e).__name__}: {e}"}


def paper_scale_run(device):
    """The paper's own experiment: a 4-way crossing of 2,500 agents
    (10 % vehicles) from spawn to the last arrival through `run(config)` -- spawn sampling, every
    frame with arrival removal and metrics, trajectories recorded -- in this package (f64: the
    reference's bits, tests/test_gpu_run.py) and, where baseline/_ref is installed, in the
    unmodified reference with all host cores. Wall-clock, the whole call."""
    from paper_2008_11578_b200 import crossing_config, run
    out = {"scenario": "four_way crossing, 625 agents per arm, vehicle fraction 0.1, seed 11; run to termination"}
    cfg = crossing_config("four_way", 625, 0.1, seed=11)
    run(crossing_config("four_way", 8, 0.1, seed=1), device=device)          # (library / context warm-up)
    t0 = time.perf_counter()
    res = run(cfg, record_trajectories=True, device=device)
    t = time.perf_counter() - t0
    out["ours_f64"] = {"frames": res.summary.frames, "arrived": res.summary.arrived, "wall_s": t,
                       "ms_per_frame": t / max(res.summary.frames, 1) * 1e3}
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref_dir, "orcasim")):
        try:
            if ref_dir not in sys.path:
                sys.path.insert(0, ref_dir)
            from orcasim import bench as rbench
            from orcasim import crossings as rcross
            from orcasim import engine as rengine
            rbench.warmup()
            rcfg = rcross.crossing_config("four_way", 625, 0.1, seed=11)
            threads = os.cpu_count() or 1
            t0 = time.perf_counter()
            rres = rengine.run(rcfg, worker_count=threads, record_trajectories=True)
            t = time.perf_counter() - t0
            out["reference_numba"] = {"frames": rres.summary.frames, "arrived": rres.summary.arrived, "wall_s": t,
                                      "ms_per_frame": t / max(rres.summary.frames, 1) * 1e3, "workers": threads}
            out["same_frames_and_arrivals"] = bool(rres.summary.frames == res.summary.frames
                                                   and rres.summary.arrived == res.summary.arrived)
        except Exception as e:      # noqa: BLE001 -- context only, never takes the line down
            out["reference_numba"] = {"unavailable": f"{type(e).__name__}: {e}"}
    return out


def parity_census(state, cfg, precisions, device):
    """One frame of the benchmarked crowd from its initial state in each precision mode against
    the CPU oracle on EVERY agent (run after the timed region; the oracle is the checker only):
    status flips, agents beyond the 1e-4 m/s gate, worst |dv|, and whether bins and ordered
    neighbour lists are bit-identical (north_star: "LP tie/degenerate cases counted and reported")."""
    from oracle import oracle as O
    from paper_2008_11578_b200 import Simulation
    n = state.active_count
    fs = O.frame_solve(state, cfg, worker_count=os.cpu_count() or 1, debug="lists")
    out = {"agents": n, "oracle": "oracle/orca_oracle.c, one frame from the initial state, every agent",
           "fallbacks_oracle": int((fs.status != 0).sum())}
    for prec in precisions:
        with Simulation(cfg, capacity=n, precision=prec, device=device, remove_arrivals=False) as sim:
            sim.load(state)
            sim.step()
            sim.sync()
            d = sim.debug_last_step(n, cfg.max_neighbors)
        dv = np.abs(d["out_v"] - fs.out_v).max(axis=1)
        out[prec] = {"status_flips": int((d["status"] != fs.status).sum()),
                     "failed_at_diffs": int((d["failed_at"] != fs.failed_at).sum()),
                     "over_1e-4": int((dv > 1e-4).sum()), "max_dv": float(dv.max()),
                     "bit_exact_velocities": bool(np.array_equal(d["out_v"], fs.out_v)),
                     "bins_and_neighbour_lists_bit_exact": bool(
                         np.array_equal(d["cell_ix"], fs.cell_ix) and np.array_equal(d["cell_iy"], fs.cell_iy)
                         and np.array_equal(d["nb_rows"], fs.nb_rows))}
    return out


def run_reference(args):
    """--impl reference: the CPU port of the reference step on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    state, cfg, wl = build_workload(args.workload)
    threads = os.cpu_count() or 1
    n = state.active_count
    rows = min(n, args.cpu_rows if args.cpu_rows > 0 else 262144)
    for _ in range(max(args.warmup, 1)):
        cpu_port_rate(state, cfg, min(rows, 8192), threads)
    rates = []
    for _ in range(args.steps):
        rate, _spent = cpu_port_rate(state, cfg, rows, threads)
        rates.append(rate)
    value = float(np.median(rates))
    t_step = n / value
    sample = (f"per step: grid build + desired velocities over all {n} agents, per-agent solve on rows "
              f"[0,{rows}) scaled by n/rows; oracle/orca_oracle.c with {threads} pthreads")
    line = {"impl": "reference", "metric": "agent_steps_per_s", "value": value, "unit": "agent-steps/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": wl,
            "cpu_baseline": {"value": value, "unit": "agent-steps/s", "cores": threads, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "agent-steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "note": "ms_per_step is the full-crowd step time extrapolated from the bounded sample"}
    print(json.dumps(line), flush=True)


def pinned_like(torch, arr):
    t = torch.empty(arr.shape, dtype={np.dtype("float64"): torch.float64,
                                      np.dtype("int64"): torch.int64}[arr.dtype]).pin_memory()
    out = t.numpy()
    out[...] = arr
    return t, out


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2008_11578_b200 import Simulation
    from paper_2008_11578_b200 import engine as E

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise RuntimeError("bench.py needs a CUDA device; there is no CPU fallback")
    ndev = torch.cuda.device_count()
    if world > 1 or os.environ.get("ORCA_BENCH_FORCE_STRIPS"):
        # the strip-decomposed path; ORCA_BENCH_FORCE_STRIPS=1 runs it with a single rank
        # (no neighbours) to smoke-test the NCCL plumbing on a one-GPU box.
        # One rank per GPU over NCCL. With fewer GPUs than ranks (a functional run of the
        # multi-process protocol on a smaller box) the ranks share devices, which NCCL refuses:
        # the slabs are then staged through the host and travel over gloo -- labelled in the line.
        if "MASTER_ADDR" not in os.environ:
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", RANK="0", WORLD_SIZE="1")
        backend = os.environ.get("ORCA_STRIPS_BACKEND") or ("nccl" if ndev >= world else "gloo")
        local = local % ndev
        torch.cuda.set_device(local)
        # NCCL prints its version banner on stdout (at communicator creation): keep file
        # descriptor 1 for the ONE JSON line
        sys.stdout.flush()
        saved_stdout = os.dup(1)
        os.dup2(2, 1)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
        from paper_2008_11578_b200.parallel import strips
        args.make_sampler = lambda: ClockSampler(local)
        line = None
        try:
            line = strips.run_bench(args, rank, world, local)
        finally:
            dist.destroy_process_group()
            sys.stdout.flush()
            try:                              # NCCL's banner sits in libc's stdout buffer: flush it to stderr
                import ctypes
                ctypes.CDLL(None).fflush(None)
            except Exception:
                pass
            os.dup2(saved_stdout, 1)
            os.close(saved_stdout)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    torch.cuda.set_device(local)

    state, cfg, wl = build_workload(args.workload)
    n = state.active_count
    stream = torch.cuda.Stream()
    hbm_peak, peak_src = load_peaks()

    # ---- resident: K steps of orca_step on the state in HBM -------------------
    sim = Simulation(cfg, capacity=n, precision=args.precision, device=local, remove_arrivals=False,
                     compute_metrics=False, stream=stream)
    sim.load(state)
    sim.run(max(args.warmup, 3))
    sim.sync()
    # (the handle adapts at a synchronisation -- ORCA_CERT32 picks its path from the fallback count it
    #  sees there -- and a changed path means a new graph capture and first launches of other kernels:
    #  a second, short warm-up keeps those one-off costs out of the timed region)
    sim.run(2)
    sim.sync()
    l0 = sim.info().kernel_launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        e0.record(stream)
        sim.run(args.steps)
        e1.record(stream)
        sim.sync()
        torch.cuda.synchronize()
    ms_step = e0.elapsed_time(e1) / args.steps
    info = sim.info()
    launches = int(info.kernel_launches - l0)
    value = n / ms_step * 1e3

    # ---- per-stage timing, second pass (CUDA events at stage boundaries) -------
    sim.profile_stages(True)
    sim.run(args.steps)
    stage_ms, covered = sim.stage_ms()
    sim.profile_stages(False)
    stage_pass_error = None
    try:                 # a sticky device-side error of the second pass (e.g. the reference's coincident-centres
        sim.sync()       # error deep into a jammed FP32-state run) is reported, not hidden
    except Exception as e:
        stage_pass_error = str(e)[:200]
    stage_ms = {k: v / max(covered, 1) for k, v in stage_ms.items()}
    stage_bytes = {"bins": BINS_BYTES_PER_AGENT, "gather": GATHER_BYTES_PER_AGENT,
                   "solve": SOLVE_BYTES_PER_AGENT}
    dom = max(("bins", "gather", "solve", "fallback"), key=lambda k: stage_ms[k])
    dom_bytes = stage_bytes.get(dom, SOLVE_BYTES_PER_AGENT) * n
    achieved = dom_bytes / (stage_ms[dom] * 1e-3) / 1e9
    fallbacks = int(info.lp_fallbacks)
    sim.close()
    if args.resident_only:
        print(json.dumps({"metric": "agent_steps_per_s", "value": value, "ms_per_step": ms_step,
                          "stages_ms": stage_ms, "gpu_launches": launches, "n": n,
                          "precision": args.precision, "note": "resident-only run",
                          **({"stages_error": stage_pass_error} if stage_pass_error else {})}), flush=True)
        return

    # ---- e2e: engine.step(state, config), host in / host out -------------------
    keep = []
    pinned = {}
    for name in ("ids", "positions", "velocities", "radii", "pref_speeds", "max_speeds", "goals",
                 "goal_tols", "class_codes"):
        t, arr = pinned_like(torch, np.ascontiguousarray(getattr(state, name)))
        keep.append(t)
        pinned[name] = arr
    host_state = type(state)(frame=0, time=0.0, rng_state=None, lp_fallbacks=0, **pinned)
    e2e_steps = max(3, min(args.steps, args.e2e_steps))
    cur = host_state
    for _ in range(5):      # warm-up: first full upload, graph capture (the pinned pool is pre-warmed)
        cur, _m = E.step(cur, cfg, precision=args.precision, device=local)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h2d = d2h = 0
    per_call = []
    for _ in range(e2e_steps):
        tc = time.perf_counter()
        cur, metrics = E.step(cur, cfg, precision=args.precision, device=local)
        per_call.append((time.perf_counter() - tc) * 1e3)
        # bytes actually copied: positions + velocities always; the 7 attribute arrays
        # (72 B/agent) only when not already resident / re-read after arrivals
        h2d += E.step.last_traffic[0]
        d2h += E.step.last_traffic[1]
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
    e2e_value = n / e2e_ms * 1e3
    print("e2e per-call ms:", " ".join(f"{t:.2f}" for t in per_call), file=sys.stderr)

    # ---- e2e through the C ABI with pinned buffers (positions/velocities only) ---
    sim = Simulation(cfg, capacity=n, precision=args.precision, device=local, remove_arrivals=False,
                     stream=stream)
    sim.load(state)
    tp_in, pos_in = pinned_like(torch, state.positions)
    tv_in, vel_in = pinned_like(torch, state.velocities)
    tp_out, pos_out = pinned_like(torch, state.positions)
    tv_out, vel_out = pinned_like(torch, state.velocities)
    ts_out, st_out = pinned_like(torch, np.zeros(n, dtype=np.int64))
    for _ in range(2):
        sim.step_host(pos_in, vel_in, 0, pos_out, vel_out, st_out)
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        sim.step_host(pos_in, vel_in, k, pos_out, vel_out, st_out)
        pos_in, pos_out = pos_out, pos_in
        vel_in, vel_out = vel_out, vel_in
    abi_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
    sim.close()

    # ---- CPU baseline: the oracle port on a bounded sample ------------------------
    threads = os.cpu_count() or 1
    rows = n if args.cpu_rows <= 0 else min(n, args.cpu_rows)   # default: the whole crowd, no extrapolation
    cpu_port_rate(state, cfg, min(rows, 8192), threads)          # warm the page cache / threads
    cpu_value, _ = cpu_port_rate(state, cfg, rows, threads, repeats=3)
    cpu1_value, _ = cpu_port_rate(state, cfg, max(1024, min(rows, 65536)), 1)

    dom_kernel = {"bins": "k_scatter", "gather": "k_gather_fast32",
                  "solve": {"f32": "k_solve", "cert32": "k_solve_cert"}.get(args.precision, "k_solve_group"),
                  "fallback": "k_fallback_coop"}[dom]
    traffic, traffic_src, ncu_util = load_traffic(args.workload, args.precision, dom_kernel)
    # ---- context lines the driver sees too: the other precision modes on this workload, every
    # other BASELINE config resident on this one GPU, a NON-uniform crowd, the LP microbench
    extras = {}
    census = None
    if not args.no_extras:
        def resident(st, cf, precision, steps, warm=5):
            with Simulation(cf, capacity=st.active_count, precision=precision, device=local,
                            remove_arrivals=False, compute_metrics=False, stream=stream) as sm:
                sm.load(st)
                sm.run(warm)
                sm.sync()
                sm.run(2)          # (see run_ours: adaptation happens at a synchronisation)
                sm.sync()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                sm.run(steps)
                b.record(stream)
                sm.sync()
                torch.cuda.synchronize()
                inf = sm.info()
                ms = a.elapsed_time(b) / steps
                return {"agents": st.active_count, "ms_per_step": ms,
                        "agent_steps_per_s": st.active_count / ms * 1e3,
                        "fallback_fraction": float(inf.lp_fallbacks) / max(st.active_count, 1),
                        "fast_gather_reject_fraction": float(inf.gather_queue) / max(st.active_count, 1)}
        extras["precision_modes_ms_per_step"] = {
            p: resident(state, cfg, p, 50)["ms_per_step"] for p in PRECISIONS if p != args.precision}
        if args.workload == "plaza_1m":
            other = {}
            for name, steps in (("config1_1k", 200), ("config2_16k", 200), ("config3_262k_d1", 50),
                                ("config3_262k_d2", 50), ("config3_262k_d1_nr3", 50), ("config3_262k_d2_nr3", 50),
                                ("blobs_1m", 50), ("config5_8m", 20)):
                st2, cf2, _ = build_workload(name)
                other[name] = resident(st2, cf2, args.precision, steps)
                other[name]["precision"] = args.precision
                del st2
            extras["other_configs_resident"] = other
            extras["config5_8m_single_gpu"] = other["config5_8m"]
            extras["lp_1m_resident_ms"] = {k: lp_resident(k, "f64", local, stream, 10)
                                           for k in sorted(LP_WORKLOADS)}
            extras["paper_scale_run"] = paper_scale_run(local)
        census = parity_census(state, cfg, [args.precision] + [p for p in ("mixed", "cert32", "f32")
                                                               if p != args.precision], local)
        ref_numba = numba_reference(state, cfg)
    else:
        ref_numba = {"skipped": "--no-extras"}

    dtype = DTYPES[args.precision]
    line = {
        "metric": "agent_steps_per_s", "value": value, "unit": "agent-steps/s", "n_gpus": 1,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype,
        "data": "synthetic", "config": wl, "precision": args.precision,
        "cache": "state advances every step; per-step working set ~%.0f MB > 126 MB L2, no flush"
                 % (n * 260 / 1e6),
        "lp_fallbacks_last_step": fallbacks, "parity": census, "clocks": clocks.summary(),
        "e2e": {"value": e2e_value, "unit": "agent-steps/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": h2d // e2e_steps, "d2h_bytes_per_step": d2h // e2e_steps,
                "call": "paper_2008_11578_b200.engine.step(state, config) -- full drop-in incl. "
                        "arrival removal and metrics; input arrays in pinned host memory",
                "c_abi_step_host": {"value": n / abi_ms * 1e3, "ms_per_step": abi_ms,
                                    "h2d_bytes_per_step": 32 * n, "d2h_bytes_per_step": 40 * n}},
        "gpu_launches": launches,
        "stages_ms": stage_ms,
        "stages_note": "per-stage CUDA events, plain launches, the stages one after the other; the timed step replays "
                       "a CUDA graph in which gather / solve / fallback run as a two-chunk pipeline on two streams, "
                       "so the stages add up to more than ms_per_step",
        **({"stages_error": stage_pass_error} if stage_pass_error else {}),
        "extras": extras,
        "roofline": {"bound": "hbm", "kernel": dom_kernel,
                     "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                     "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
                     "ncu": ncu_util,   # what actually bounds it: issue slots (ipc of 4), FP64 pipe, lanes, warps
                     "algorithmic_bytes_per_launch": dom_bytes,
                     "duration_ms": stage_ms[dom],
                     "duration_source": f"CUDA events on the handle's stream around the '{dom}' stage in this run "
                                        "(plain launches, one chunk: ONE launch of the kernel per step"
                                        + (", plus k_shuffle and the FP64 pass over the few percent it queues -- "
                                           "the stage's time is charged to the kernel whole)" if dom == "solve"
                                           else ")"),
                     "step_frac": STEP_BYTES_PER_AGENT * n / (ms_step * 1e-3) / 1e9 / hbm_peak,
                     "note": "the step is issue/latency bound, not HBM bound (DESIGN.md s5); "
                             "fractions are reported against the HBM roofline as the contract asks"},
        "cpu_baseline": {"value": cpu_value, "unit": "agent-steps/s", "cores": threads, "kind": "port",
                         "sample": f"one step: grid build + desired velocities over all {n} agents, "
                                   f"per-agent solve on rows [0,{rows}) scaled by n/rows; "
                                   f"oracle/orca_oracle.c ({threads} pthreads); "
                                   f"1 thread: {cpu1_value:.3e} agent-steps/s",
                         "reference_numba": ref_numba},
    }
    print(json.dumps(line), flush=True)


PRECISIONS = ("mixed", "cert32", "f32", "f64")
DTYPES = {"mixed": "f32 state / f64 arithmetic", "f32": "f32", "f64": "f64",
          "cert32": "f32 state / f32 arithmetic with an f64-evaluated, certified result (f64 otherwise)"}

LP_WORKLOADS = {"lp_1m_feasible": 0.0, "lp_1m_half": 0.5, "lp_1m_infeasible": 1.0}


def lp_resident(workload, prec, local, stream, steps):
    """ms per solve of the resident 1,048,576-LP batch of BASELINE config 4 (for `extras`)."""
    import torch

    from paper_2008_11578_b200 import LpBatch
    from paper_2008_11578_b200.synth import lp_batch
    coff, cpts, cnrm, tgt, caps, seeds = lp_batch(1 << 20, 8, 64, LP_WORKLOADS[workload], seed=5)
    b = LpBatch(coff, cpts, cnrm, tgt, caps, seeds, precision=prec, device=local, stream=stream)
    del cpts, cnrm
    for _ in range(3):
        b.solve()
    b.results()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        b.solve()
    e1.record(stream)
    _v, status, _f = b.results()
    torch.cuda.synchronize()
    b.close()
    return {"ms_per_solve": e0.elapsed_time(e1) / steps, "precision": prec,
            "fallback_fraction": float((status != 0).mean())}


def run_lp(args):
    """BASELINE config 4: 1,048,576 independent 2-D LPs with 8..64 half-plane constraints each
    (the CSR layout of _kernels.solve_range), all feasible / half / (almost) all infeasible.
    One step = one solve of the whole batch. value: batch resident on the device; e2e: the
    reference-shaped call lp.solve_range(host arrays) -> host arrays."""
    import torch

    from paper_2008_11578_b200 import LpBatch, solve_range
    from paper_2008_11578_b200.synth import lp_batch

    if not torch.cuda.is_available():
        raise RuntimeError("bench.py needs a CUDA device; there is no CPU fallback")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    n = 1 << 20
    frac = LP_WORKLOADS[args.workload]
    coff, cpts, cnrm, tgt, caps, seeds = lp_batch(n, 8, 64, frac, seed=5)
    m = int(coff[-1])
    prec = "f32" if args.precision == "f32" else "f64"
    hbm_peak, peak_src = load_peaks()
    stream = torch.cuda.Stream()
    b = LpBatch(coff, cpts, cnrm, tgt, caps, seeds, precision=prec, device=local, stream=stream)
    for _ in range(max(args.warmup, 3)):
        b.solve()
    b.results()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            b.solve()
        e1.record(stream)
        _v, status, _f = b.results()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    b.close()
    e2e_steps = max(3, min(args.steps, 5))
    keep = []
    def pin(a):      # the contract's e2e copies its inputs from pinned host memory
        a = np.ascontiguousarray(a)
        t = torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).pin_memory()
        keep.append(t)
        return t.numpy().view(a.dtype)
    coff, cpts, cnrm, tgt, caps, seeds = (pin(a) for a in (coff, cpts, cnrm, tgt, caps, seeds))
    solve_range(coff, cpts, cnrm, tgt, caps, seeds, precision=prec, device=local)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        solve_range(coff, cpts, cnrm, tgt, caps, seeds, precision=prec, device=local)
    e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
    h2d = coff.nbytes + cpts.nbytes + cnrm.nbytes + tgt.nbytes + caps.nbytes + seeds.nbytes
    d2h = n * (16 + 8 + 8)
    # CPU port of solve_range on a bounded sample of the same batch
    from oracle import oracle as O
    threads = os.cpu_count() or 1
    cn = min(n, 1 << 17)
    sub = (coff[:cn + 1], cpts[:coff[cn]], cnrm[:coff[cn]], tgt[:cn], caps[:cn], seeds[:cn])
    O.solve_range(*sub, worker_count=threads)
    t0 = time.perf_counter()
    for _ in range(3):
        O.solve_range(*sub, worker_count=threads)
    cpu_rate = 3 * cn / (time.perf_counter() - t0)
    rs = 4 if prec == "f32" else 8
    alg_bytes = (4 * rs) * m + (3 * rs + 8 + 8 + 16 + 16) * n      # constraints + per-LP in/out
    achieved = alg_bytes / (ms * 1e-3) / 1e9
    line = {"metric": "lp_per_s", "value": n / ms * 1e3, "unit": "LP/s", "n_gpus": 1, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": prec, "data": "synthetic",
            "config": {"workload": args.workload, "lps": n, "constraints": m, "k": "U{8..64}",
                       "infeasible_fraction_requested": frac, "fallback_fraction": float((status != 0).mean()),
                       "constraints_per_s": m / ms * 1e3,
                       "cache": f"batch of {alg_bytes / 1e6:.0f} MB > 126 MB L2, no flush"},
            "clocks": clocks.summary(),
            "e2e": {"value": n / e2e_ms * 1e3, "unit": "LP/s", "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "call": "paper_2008_11578_b200.lp.solve_range(host CSR arrays) -> host arrays"},
            "gpu_launches": 2 * args.steps,
            "roofline": {"bound": "hbm", "kernel": "k_lp_batch" + ("+k_lp_batch_fallback" if frac > 0 else ""),
                         "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                         "traffic": None, "peak_source": peak_src, "algorithmic_bytes_per_launch": alg_bytes,
                         "note": "thread-per-problem incremental LP: issue/latency bound, not HBM bound"},
            "cpu_baseline": {"value": cpu_rate, "unit": "LP/s", "cores": threads, "kind": "port",
                             "sample": f"oracle/orca_oracle.c solve_range on the first {cn} problems of the batch, "
                                       f"{threads} pthreads, 3 repeats"}}
    print(json.dumps(line), flush=True)


def self_launch(args):
    """python bench.py --gpus N (N > 1) outside torchrun: start N ranks of this script, one per
    GPU, the way the driver's own multi-GPU launch does, and pass their exit code on."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="plaza_1m", choices=sorted(CONFIGS) + sorted(LP_WORKLOADS))
    ap.add_argument("--precision", default="cert32", choices=list(PRECISIONS),
                    help="cert32 (default): FP32 state, certified FP32 solve with an FP64-evaluated result -- the "
                         "results of `mixed` bit for bit, checked against the oracle on every agent in the line's "
                         "`parity`; mixed: FP32 state, FP64 arithmetic; f64: bit-identical to the reference; f32")
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--cpu-rows", type=int, default=0,
                    help="agents the CPU port solves per step (0: the whole crowd for cpu_baseline, "
                         "262144 per step for --impl reference)")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the context measurements (other precision modes, 8.5 M agents on one GPU)")
    ap.add_argument("--resident-only", action="store_true",
                    help="only the HBM-resident timing (for runs under ncu)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="--gpus N > 1: weak = one `workload` plaza per GPU (default), strong = ONE "
                         "`workload` crowd cut into N strips (BASELINE config 5: --workload config5_8m)")
    ap.add_argument("--transport", default="auto", choices=["auto", "window", "sendrecv"],
                    help="--gpus N > 1, how the strips' slabs travel: window = each strip's kernel writes them "
                         "into its neighbours' memory (CUDA IPC peer mapping, flags; no library call per frame), "
                         "sendrecv = grouped NCCL send/recv (gloo, staged through the host, when ranks share a "
                         "GPU); auto = window, send/recv if a neighbour's window cannot be mapped")
    ap.add_argument("--no-verify", action="store_true",
                    help="--gpus N > 1: skip the bit-equality check against the same crowd on one GPU")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.workload not in LP_WORKLOADS:
        if args.impl != "reference":   # (the CPU arm is one process whatever N is)
            sys.exit(self_launch(args))
    if args.workload in LP_WORKLOADS:
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "the reference arm times the steering step; "
                              "the LP microbench line carries its CPU port rate as cpu_baseline"}))
        else:
            run_lp(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
