"""Adversarial soak of ORCA_CERT32 (development tooling): crowds built to sit ON the decisions the
certificate has to guard -- exact lattices (every distance tied), discs exactly touching or
overlapping by one ulp (the overlap branch K:357 at equality), zero and identical velocities
(|w| = |rp| / tau exactly, w parallel to rp: the arc / leg test K:395 and the leg side K:404 at
zero), mirror-symmetric pairs (parallel and anti-parallel half-planes in one LP), goals exactly
along a neighbour's tangent, agents at their goal (zero preferred velocity), speeds exactly at the
cap. float32-representable values throughout, so that `mixed` and `cert32` see the same inputs.
cert32 must equal mixed BIT FOR BIT on every agent and frame.
With a third argument "oracle" the same crowds go through the f64 mode against the CPU oracle
instead (one frame: status, failed_at, velocities bit for bit, ordered neighbour lists).
    python tests/soak/soak_cert_adversarial.py [first_seed] [count] [oracle]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)
os.environ["ORCA_CERT_FORCE"] = "1"

import numpy as np  # noqa: E402

from paper_2008_11578_b200 import Simulation  # noqa: E402
from paper_2008_11578_b200.synth import plaza_crowd  # noqa: E402


def adversarial(seed):
    rng = np.random.default_rng(77_000 + seed)
    side = int(rng.integers(12, 40))
    st, cfg = plaza_crowd(side * side, 0, density=0.5, seed=seed)
    n = st.active_count
    radius = float(np.float32(rng.choice([0.25, 0.3, 0.5])))
    margin = float(cfg.avoidance_margin)
    touch = 2.0 * radius + margin                       # combined avoid radii exactly
    pitch = float(np.float32(rng.choice([touch, touch * (1 + 2 ** -20), touch * (1 - 2 ** -20), 2 * touch,
                                         1.0, 0.75, 1.5])))
    gx, gy = np.meshgrid(np.arange(side), np.arange(side), indexing="ij")
    pos = np.stack([gx.ravel(), gy.ravel()], axis=1).astype(np.float64)[:n] * pitch
    kind = int(rng.integers(0, 6))
    if kind == 1:                                      # hexagonal-ish: every second row shifted by half a pitch
        pos[:, 0] += (np.arange(n) // side % 2) * (pitch / 2)
    if kind == 2:                                      # a few exact duplicates of a distance pattern, jitter on a power of two grid
        pos += rng.integers(-2, 3, size=pos.shape) * (pitch / 8)
        _u, first = np.unique(pos, axis=0, return_index=True)
        keep = np.sort(first)
        pos = pos[keep]
    n = pos.shape[0]
    for f in ("ids", "radii", "pref_speeds", "max_speeds", "goal_tols", "class_codes"):
        setattr(st, f, getattr(st, f)[:n].copy())
    st.radii[:] = radius
    st.positions = pos.astype(np.float32).astype(np.float64)
    vmode = int(rng.integers(0, 5))
    speed = float(np.float32(rng.choice([0.0, 0.5, 1.0, float(st.max_speeds[0])])))
    if vmode == 0:
        vel = np.zeros((n, 2))
    elif vmode == 1:                                   # everybody the same velocity: rv = 0 for every pair
        vel = np.tile([speed, 0.0], (n, 1))
    elif vmode == 2:                                   # rows moving against each other: mirror pairs
        vel = np.zeros((n, 2))
        vel[:, 0] = np.where((np.arange(n) // side) % 2 == 0, speed, -speed)
    elif vmode == 3:                                   # along the lattice diagonals
        vel = np.tile([speed, speed], (n, 1)) * np.where(np.arange(n) % 2 == 0, 1.0, -1.0)[:, None]
    else:
        vel = rng.choice([-1.0, 0.0, 1.0], size=(n, 2)) * speed
    st.velocities = vel.astype(np.float32).astype(np.float64)
    gmode = int(rng.integers(0, 4))
    if gmode == 0:                                     # at the goal already: zero preferred velocity
        goals = st.positions.copy()
    elif gmode == 1:                                   # straight through the neighbour ahead
        goals = st.positions + np.array([pitch * side, 0.0])
    elif gmode == 2:                                   # everyone to the centre: head-on everywhere
        goals = np.tile(st.positions.mean(axis=0), (n, 1))
    else:
        goals = st.positions[rng.permutation(n)]       # somebody else's lattice site
    st.goals = goals.astype(np.float32).astype(np.float64)
    st.goal_tols[:] = 0.0
    return st, cfg


def main():
    first = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    count = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    bad, t0, agents, queued, ran = [], time.time(), 0, 0, 0
    budget = float(os.environ.get("ORCA_SOAK_SECONDS", "0"))   # stop after this many seconds, report what ran
    if len(sys.argv) > 3 and sys.argv[3] == "oracle":
        from oracle import oracle as O
        for seed in range(first, first + count):
            if budget and time.time() - t0 > budget:
                count = seed - first
                break
            st, cfg = adversarial(seed)
            n = st.active_count
            try:
                ref = O.frame_solve(st, cfg, debug=True)
            except ValueError:
                continue                                   # coincident centres in the initial crowd
            with Simulation(cfg, capacity=n, precision="f64", remove_arrivals=False) as sim:
                sim.load(st)
                sim.step()
                sim.sync()
                d = sim.debug_last_step(n, cfg.max_neighbors)
            ran += 1
            ok = (np.array_equal(d["out_v"], ref.out_v) and np.array_equal(d["status"], ref.status)
                  and np.array_equal(d["failed_at"], ref.failed_at) and np.array_equal(d["nb_count"], ref.nb_count))
            for i in range(n):
                ok = ok and np.array_equal(d["nb_rows"][i, :d["nb_count"][i]], ref.nb_rows[i, :ref.nb_count[i]])
            if not ok:
                bad.append(seed)
                print("FAIL", seed, n, flush=True)
            agents += n
        print("adversarial f64-vs-oracle soak done:", count, "seeds from", first, f"({ran} ran)", "- failures:", len(bad),
              "in", round(time.time() - t0), "s;", agents, "agents")
        sys.exit(1 if bad else 0)
    for seed in range(first, first + count):
        if budget and time.time() - t0 > budget:
            count = seed - first
            break
        st, cfg = adversarial(seed)
        n = st.active_count
        try:
            out = {}
            for precision in ("mixed", "cert32"):
                rows = []
                with Simulation(cfg, capacity=n, precision=precision, remove_arrivals=False) as sim:
                    sim.load(st)
                    for _ in range(3):
                        sim.step()
                        sim.sync()
                        d = sim.debug_last_step(n, cfg.max_neighbors)
                        info = sim.info()
                        rows.append((d["out_v"], d["status"], d["failed_at"], int(info.lp_fallbacks), int(info.solve_queue)))
                out[precision] = rows
            ran += 1
            for k, (a, b) in enumerate(zip(out["mixed"], out["cert32"])):
                assert np.array_equal(a[0], b[0]), f"velocities, frame {k}: {int((a[0] != b[0]).any(axis=1).sum())} agents"
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
    print("adversarial cert32 soak done:", count, "seeds from", first, f"({ran} ran to the end)", "- failures:", len(bad),
          "in", round(time.time() - t0), "s;",
          f"{agents} agent-frames, {queued} ({queued / max(agents, 1):.1%}) went through the FP64 kernels")


if __name__ == "__main__":
    main()
