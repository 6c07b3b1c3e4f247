"""Soak of ORCA_CERT32 (development tooling): random crowds of every density, max_neighbors,
responsibility matrix and radius mix (tests/test_gpu_fuzz.random_case) plus mid-size plazas and
blobs, several resident frames each; cert32 must equal mixed BIT FOR BIT on every agent and frame
(a mis-certified agent would show as a different velocity or status), and mixed is checked against
the oracle elsewhere (soak_fuzz.py). Prints the share of agents the certificate accepted.
    python tests/soak/soak_cert.py [first_seed] [count]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)

os.environ["ORCA_CERT_FORCE"] = "1"     # small crowds too

import numpy as np  # noqa: E402

import test_gpu_fuzz as F  # noqa: E402
from paper_2008_11578_b200 import Simulation  # noqa: E402
from paper_2008_11578_b200.synth import blobs_crowd, plaza_crowd  # noqa: E402

first = int(sys.argv[1]) if len(sys.argv) > 1 else 0
count = int(sys.argv[2]) if len(sys.argv) > 2 else 400
bad, t0, agents, queued = [], time.time(), 0, 0
BUDGET = float(os.environ.get("ORCA_SOAK_SECONDS", "0"))
for seed in range(first, first + count):
    if BUDGET and time.time() - t0 > BUDGET:     # ORCA_SOAK_SECONDS: stop here, report what ran
        count = seed - first
        break
    rng = np.random.default_rng(10_000 + seed)
    kind = seed % 4
    if kind == 3:
        dens = float(np.exp(rng.uniform(np.log(0.05), np.log(3.0))))
        st, cfg = plaza_crowd(int(rng.integers(2000, 40000)), int(rng.integers(0, 800)), density=dens, seed=seed)
    elif kind == 2:
        st, cfg = blobs_crowd(int(rng.integers(5000, 40000)), int(rng.integers(0, 500)), seed=seed)
    else:
        st, cfg = F.random_case(seed)
    n = st.active_count
    frames = 4
    try:
        out = {}
        for precision in ("mixed", "cert32"):
            rows = []
            with Simulation(cfg, capacity=n, precision=precision, remove_arrivals=False) as sim:
                sim.load(st)
                for _ in range(frames):
                    sim.step()
                    sim.sync()
                    d = sim.debug_last_step(n, cfg.max_neighbors)
                    info = sim.info()
                    rows.append((d["out_v"], d["status"], d["failed_at"], int(info.lp_fallbacks), int(info.solve_queue)))
            out[precision] = rows
        for k, (a, b) in enumerate(zip(out["mixed"], out["cert32"])):
            assert np.array_equal(a[0], b[0]), f"velocities, frame {k}"
            assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2]) and a[3] == b[3], f"status, frame {k}"
            agents += n
            queued += b[4]
    except ValueError as e:       # the reference's own error (coincident centres after a frame)
        if "coincident" not in str(e):
            bad.append((seed, repr(e)[:160]))
            print("FAIL", seed, repr(e)[:160], flush=True)
    except AssertionError as e:
        bad.append((seed, repr(e)[:160]))
        print("FAIL", seed, n, repr(e)[:160], flush=True)
print("cert32 soak done:", count, "seeds from", first, "- failures:", len(bad), "in", round(time.time() - t0), "s;",
      f"{agents} agent-frames, {queued} ({queued / max(agents, 1):.1%}) went through the FP64 kernels")
