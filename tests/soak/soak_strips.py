"""Soak of the strip decomposition on one GPU (development tooling): 2-4 handles on cuda:0 play
adjacent strips with device-to-device buffer swaps in place of NCCL (tests/test_gpu_strips.py),
random crowds / densities / strip counts, 12 frames with a row reordering every third frame; the
decomposed crowd must equal the single-handle run bit for bit, keyed by id.
    python tests/soak/soak_strips.py [first_seed] [count] [sendrecv|window|both]
"window": the handles exchange through their peer-memory windows (kernels write the neighbour's
window and raise its flag) instead of the test's buffer swaps; "both" alternates by seed."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import strip_ops_cpu as S  # noqa: E402
from test_gpu_strips import build_strips, lockstep  # noqa: E402
from paper_2008_11578_b200 import Simulation  # noqa: E402
from paper_2008_11578_b200.parallel.strips import strip_bounds  # noqa: E402

first = int(sys.argv[1]) if len(sys.argv) > 1 else 0
count = int(sys.argv[2]) if len(sys.argv) > 2 else 40
mode = sys.argv[3] if len(sys.argv) > 3 else "sendrecv"
bad, t0, ran = [], time.time(), 0
BUDGET = float(os.environ.get("ORCA_SOAK_SECONDS", "0"))
for seed in range(first, first + count):
    if BUDGET and time.time() - t0 > BUDGET:     # ORCA_SOAK_SECONDS: stop here, report what ran
        count = seed - first
        break
    rng = np.random.default_rng(seed)
    world = int(rng.integers(2, 5))
    precision = ["f64", "mixed"][seed % 2]
    n_ped, n_veh = int(rng.integers(3000, 12000)), int(rng.integers(0, 600))
    dens = float(np.exp(rng.uniform(np.log(0.1), np.log(1.5))))
    st, cfg = S.make_crowd(seed=seed, n_ped=n_ped, n_veh=n_veh, density=dens)
    n, steps = st.ids.shape[0], 12
    try:
        with Simulation(cfg, capacity=n, precision=precision, remove_arrivals=False) as ref:
            ref.load(st)
            ref.run(steps)
            want = ref.state()
        bounds = strip_bounds(st.positions[:, 0], world)
        b = [-np.inf] + list(bounds) + [np.inf]
        if min(b[i + 1] - b[i] for i in range(world)) < cfg.neighbor_radius + 1.0:
            continue                                   # strips must be wider than the halo reach (StripDriver checks)
        sims, drivers, _b = build_strips(st, cfg, precision, world, halo_cap=n, mig_cap=n,
                                         resync_every=int(rng.integers(1, 6)), capacity=5 * n,
                                         transport=mode if mode != "both" else ("window", "sendrecv")[(seed // 2) % 2])
        lockstep(drivers, steps)
        ran += 1
        parts = [s.state() for s in sims]
        ids = np.concatenate([p.ids for p in parts])
        order, ref_order = np.argsort(ids), np.argsort(want.ids)
        assert np.array_equal(ids[order], want.ids[ref_order]), "ids"
        for f in ("positions", "velocities", "goals", "radii", "max_speeds", "class_codes"):
            got = np.concatenate([getattr(p, f) for p in parts])[order]
            assert np.array_equal(got, getattr(want, f)[ref_order]), f
        assert sum(int(s.info().lp_fallbacks) for s in sims) == want.lp_fallbacks, "fallbacks"
        for s in sims:
            s.close()
    except (AssertionError, ValueError, RuntimeError) as e:
        if "coincident" in str(e):
            continue
        bad.append((seed, repr(e)[:200]))
        print("FAIL", seed, world, precision, n, round(dens, 3), repr(e)[:200], flush=True)
print("soak done:", count, "seeds from", first, f"({ran} decomposed runs)", "- failures:", len(bad), "in",
      round(time.time() - t0), "s")
