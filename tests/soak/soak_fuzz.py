"""Soak of the randomised parity tests over many more seeds than the test-suite runs
(development tooling; imports the tests, which use the oracle):
    python tests/soak/soak_fuzz.py [first_seed] [count] [adversarial]
Per seed: tests/test_gpu_fuzz.py::test_random_step_matches_oracle, then five resident frames
(radius-hint fast pass, exact-search queue, row reordering every 2 frames) of the same random
crowd in f64 and mixed, every frame against the oracle fed the device's own state. With
"adversarial" the crowds are those of soak_cert_adversarial.py (exact lattices, touching discs,
identical / mirrored velocities) instead of the random ones."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)
os.environ.setdefault("ORCA_REORDER_EVERY", "2")
os.environ.setdefault("ORCA_CERT_FORCE", "1")     # the certified kernels on small crowds too

import numpy as np  # noqa: E402

import test_gpu_fuzz as F  # noqa: E402
from test_gpu_step import check_against, oracle_ref  # noqa: E402
from paper_2008_11578_b200 import SimState, Simulation  # noqa: E402

first = int(sys.argv[1]) if len(sys.argv) > 1 else 24
count = int(sys.argv[2]) if len(sys.argv) > 2 else 400
adv = len(sys.argv) > 3 and sys.argv[3] == "adversarial"
if adv:
    sys.path.insert(0, os.path.join(ROOT, "tests", "soak"))
    from soak_cert_adversarial import adversarial  # noqa: E402
bad, t0 = [], time.time()
BUDGET = float(os.environ.get("ORCA_SOAK_SECONDS", "0"))
for seed in range(first, first + count):
    if BUDGET and time.time() - t0 > BUDGET:     # ORCA_SOAK_SECONDS: stop here, report what ran
        count = seed - first
        break
    try:
        if adv:
            st, cfg = adversarial(seed)
        else:
            F.test_random_step_matches_oracle(seed)
            st, cfg = F.random_case(seed)
        n = st.active_count
        for precision in ("f64", "mixed"):
            with Simulation(cfg, capacity=n, precision=precision, remove_arrivals=False) as sim:
                sim.load(st)
                cur = st
                for k in range(5):
                    ref = oracle_ref(cur, cfg, workers=4)
                    sim.step()
                    sim.sync()
                    d = sim.debug_last_step(n, cfg.max_neighbors)
                    d["lp_fallbacks"] = int(sim.info().lp_fallbacks)
                    check_against(d, ref, precision, f"seed {seed} frame {k}")
                    pos, vel = sim.positions_velocities()
                    cur = SimState(frame=cur.frame + 1, time=0.0, ids=st.ids, positions=pos, velocities=vel,
                                   radii=st.radii, pref_speeds=st.pref_speeds, max_speeds=st.max_speeds,
                                   goals=st.goals, goal_tols=st.goal_tols, class_codes=st.class_codes)
    except AssertionError as e:
        if str(e) == "":          # oracle_ref's bare `assert np.all(fs.err == -1)`: two agents ended a
            continue              # frame on exactly the same spot -- an error in the reference as well
        bad.append((seed, repr(e)[:160]))
        print("FAIL", seed, repr(e)[:160], flush=True)
    except ValueError as e:       # the reference's own error (coincident centres after a frame)
        if "coincident" not in str(e):
            bad.append((seed, repr(e)[:160]))
            print("FAIL", seed, repr(e)[:160], flush=True)
print("soak done:", count, "seeds from", first, "- failures:", len(bad), "in", round(time.time() - t0), "s")
