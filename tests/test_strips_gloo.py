"""Multi-rank strip protocol on CPU: world_size 2 and 3 over gloo, with the oracle
standing in for the device (tests/strip_ops_cpu.py). The strip-decomposed run must
equal the single-domain reference run bit for bit, keyed by agent id -- the
multi-rank analogue of the reference's worker-count independence tests
(pkg/tests/test_engine.py:197-204)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import strip_ops_cpu as S
from paper_2008_11578_b200.parallel.strips import strip_bounds


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_strips_equal_single_domain(world, tmp_path):
    steps = 6
    mp.spawn(S.gloo_worker, args=(world, free_port(), steps, str(tmp_path)), nprocs=world, join=True)
    st, cfg = S.crowd_for(world)
    ref = S.reference_run(st, cfg, steps)
    got_ids, got_pos, got_vel = [], [], []
    migrated = halo = 0
    for r in range(world):
        z = np.load(os.path.join(tmp_path, f"rank{r}.npz"))
        assert int(z["frame"]) == steps
        # ownership is consistent after the last migration
        assert np.all((z["positions"][:, 0] >= z["lo"]) & (z["positions"][:, 0] < z["hi"]))
        got_ids.append(z["ids"])
        got_pos.append(z["positions"])
        got_vel.append(z["velocities"])
        migrated += int(z["migr_recv"])
        halo += int(z["halo_recv"])
        assert int(z["host_syncs"]) <= steps // 4 + 1       # the host is not in the per-frame loop
    ids = np.concatenate(got_ids)
    order = np.argsort(ids)
    assert np.array_equal(ids[order], np.sort(ref.ids))            # nobody lost or duplicated
    ref_order = np.argsort(ref.ids)
    assert np.array_equal(np.concatenate(got_pos)[order], ref.positions[ref_order])
    assert np.array_equal(np.concatenate(got_vel)[order], ref.velocities[ref_order])
    assert migrated > 0 and halo > 0                                # the test exercised both paths


def test_strip_bounds_balance():
    rng = np.random.default_rng(0)
    x = rng.normal(size=10000) * 50
    b = strip_bounds(x, 4)
    assert b.shape == (3,) and np.all(np.diff(b) > 0)
    counts = np.histogram(x, bins=[-np.inf, *b, np.inf])[0]
    assert counts.max() - counts.min() <= 2
    assert strip_bounds(x, 1).shape == (0,)


def test_narrow_strips_are_rejected():
    from paper_2008_11578_b200.parallel.strips import check_strip_widths
    check_strip_widths([10.0, 30.0, 50.0], 15.2)
    with pytest.raises(ValueError, match="wide"):
        check_strip_widths([10.0, 20.0, 50.0], 15.2)
    with pytest.raises(ValueError, match="non-decreasing"):
        check_strip_widths([10.0, 5.0], 1.0)
    x = np.concatenate([np.zeros(1000), np.full(1000, 3.0), np.full(1000, 6.0), np.full(1000, 100.0)])
    with pytest.raises(ValueError):     # a clustered crowd: the quantiles are 3 m apart
        strip_bounds(x + np.random.default_rng(0).random(4000), 4, min_width=15.2)


def test_state_hash_is_order_and_partition_independent():
    from paper_2008_11578_b200.parallel.strips import state_hash
    rng = np.random.default_rng(3)
    ids = rng.permutation(5000).astype(np.int64)
    pos, vel = rng.normal(size=(5000, 2)), rng.normal(size=(5000, 2))
    h = state_hash(ids, pos, vel)
    p = rng.permutation(5000)
    assert state_hash(ids[p], pos[p], vel[p]) == h
    a, b = p[:1234], p[1234:]
    assert (state_hash(ids[a], pos[a], vel[a]) + state_hash(ids[b], pos[b], vel[b])) % (1 << 64) == h
    vel2 = vel.copy()
    vel2[17, 1] = np.nextafter(vel2[17, 1], 1.0)
    assert state_hash(ids, pos, vel2) != h
