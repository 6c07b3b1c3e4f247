"""Strip decomposition on the adversarial crowds of soak_cert_adversarial.py (development tooling):
exact lattices put whole columns of agents ON a strip boundary (x == bound: the owner is the strip
with x_lo <= x < x_hi on every rank alike) and at exactly neighbor_radius from it; 2-4 handles on one
GPU, both transports, 8 frames; the decomposed crowd must equal the single handle bit for bit.
    python tests/soak/soak_strips_adversarial.py [first_seed] [count]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tests", "soak"))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from soak_cert_adversarial import adversarial  # noqa: E402
from test_gpu_strips import build_strips, lockstep  # noqa: E402
from paper_2008_11578_b200 import Simulation  # noqa: E402
from paper_2008_11578_b200.parallel.strips import strip_bounds  # noqa: E402


def main():
    first = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    count = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    bad, t0, ran = [], time.time(), 0
    budget = float(os.environ.get("ORCA_SOAK_SECONDS", "0"))   # stop after this many seconds, report what ran
    for seed in range(first, first + count):
        if budget and time.time() - t0 > budget:
            count = seed - first
            break
        st, cfg = adversarial(seed)
        st.goal_tols[:] = 0.25
        n, steps = st.active_count, 8
        world = 2 + seed % 3
        precision = ["f64", "mixed", "cert32"][seed % 3]
        bounds = strip_bounds(st.positions[:, 0], world)
        b = [-np.inf] + list(bounds) + [np.inf]
        if world > 2 and min(b[i + 1] - b[i] for i in range(1, world - 1)) < cfg.neighbor_radius + 1.0:
            world = 2
            bounds = strip_bounds(st.positions[:, 0], world)
        try:
            with Simulation(cfg, capacity=n, precision=precision, remove_arrivals=False) as ref:
                ref.load(st)
                ref.run(steps)
                want = ref.state()
            sims, drivers, _b = build_strips(st, cfg, precision, world, halo_cap=n, mig_cap=n, resync_every=3,
                                             capacity=5 * n, transport=("window", "sendrecv")[seed % 2])
            lockstep(drivers, steps)
            ran += 1
            parts = [s.state() for s in sims]
            ids = np.concatenate([p.ids for p in parts])
            order, ref_order = np.argsort(ids), np.argsort(want.ids)
            assert np.array_equal(ids[order], want.ids[ref_order]), "ids"
            for f in ("positions", "velocities"):
                got = np.concatenate([getattr(p, f) for p in parts])[order]
                assert np.array_equal(got, getattr(want, f)[ref_order]), f
            assert sum(int(s.info().lp_fallbacks) for s in sims) == want.lp_fallbacks, "fallbacks"
            for s in sims:
                s.close()
        except (AssertionError, ValueError, RuntimeError) as e:
            if "coincident" in str(e) or "strips must be at least" in str(e):
                continue
            bad.append((seed, repr(e)[:200]))
            print("FAIL", seed, world, precision, n, repr(e)[:200], flush=True)
    print("adversarial strips soak done:", count, "seeds from", first, f"({ran} decomposed runs)", "- failures:",
          len(bad), "in", round(time.time() - t0), "s")


if __name__ == "__main__":
    main()
