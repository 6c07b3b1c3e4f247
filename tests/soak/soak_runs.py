"""Soak of whole frames with arrival removal and metrics at mid size (development tooling; uses the
oracle): random crowd size 5k-60k, density 0.05-3 /m2, vehicle share, goals close enough that agents
keep arriving; 6 resident frames in f64 must equal oracle.advance bit for bit (state, metrics,
fallback counts), the same frames through orca_advance_host as well, mixed within 1e-6 m/s of it
frame by frame.   python tests/soak/soak_runs.py [first_seed] [count]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
os.environ.setdefault("ORCA_REORDER_EVERY", "3")

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2008_11578_b200 import Simulation  # noqa: E402
from paper_2008_11578_b200.synth import plaza_crowd  # noqa: E402

first = int(sys.argv[1]) if len(sys.argv) > 1 else 0
count = int(sys.argv[2]) if len(sys.argv) > 2 else 60
bad, t0 = [], time.time()
BUDGET = float(os.environ.get("ORCA_SOAK_SECONDS", "0"))
for seed in range(first, first + count):
    if BUDGET and time.time() - t0 > BUDGET:     # ORCA_SOAK_SECONDS: stop here, report what ran
        count = seed - first
        break
    rng = np.random.default_rng(seed)
    n_ped = int(rng.integers(5000, 60000))
    n_veh = int(rng.integers(0, n_ped // 8))
    dens = float(np.exp(rng.uniform(np.log(0.05), np.log(3.0))))
    st, cfg = plaza_crowd(n_ped, n_veh, density=dens, seed=seed + 7)
    n = st.active_count
    close = rng.permutation(n)[: n // 10]
    st.goals[close] = (st.positions[close] + rng.normal(size=(close.size, 2)) * 0.5).astype(np.float32)
    try:
        ref = st
        with Simulation(cfg, capacity=n, precision="f64", remove_arrivals=True, compute_metrics=True) as sim, \
                Simulation(cfg, capacity=n, precision="f64", remove_arrivals=True, compute_metrics=True) as host, \
                Simulation(cfg, capacity=n, precision="mixed", remove_arrivals=True, compute_metrics=True) as mix:
            sim.load(st)
            host.load(st)
            mix.load(st)
            for k in range(6):
                prev = ref
                ref, sep, coll, fb, _ = O.advance(ref, cfg, worker_count=16)
                sim.step()
                info = sim.info()
                got = (int(info.active_agents), float(info.min_separation) if ref.active_count >= 2 else sep,
                       int(info.collision_count), int(info.lp_fallbacks))
                assert got == (ref.active_count, sep, coll, fb), f"frame {k}: {got} vs {(ref.active_count, sep, coll, fb)}"
                pos, vel, hinfo = host.advance_host(prev.positions, prev.velocities, prev.frame)
                assert np.array_equal(pos, ref.positions) and np.array_equal(vel, ref.velocities), f"frame {k}: host step"
                # mixed: fed the f64 state rounded to float32, one frame, against the oracle on the same input
                p32 = prev.positions.astype(np.float32).astype(np.float64)
                v32 = prev.velocities.astype(np.float32).astype(np.float64)
                if k == 0:
                    mref, *_ = O.advance(type(prev)(**{**prev.__dict__, "positions": p32, "velocities": v32}), cfg,
                                         worker_count=16)
                    mpos, mvel, minfo = mix.advance_host(p32, v32, prev.frame)
                    assert int(minfo.active_agents) == mref.active_count, f"frame {k}: mixed count"
                    assert np.abs(mvel - mref.velocities).max() <= 1e-6, f"frame {k}: mixed velocities"
            final = sim.state()
            for f in ("ids", "positions", "velocities", "goals", "radii", "class_codes"):
                assert np.array_equal(getattr(final, f), getattr(ref, f)), f
    except (AssertionError, ValueError) as e:
        if "coincident" in str(e):
            continue
        bad.append((seed, repr(e)[:200]))
        print("FAIL", seed, n, round(dens, 3), repr(e)[:200], flush=True)
print("soak done:", count, "seeds from", first, "- failures:", len(bad), "in", round(time.time() - t0), "s")
