"""Pin the CPU oracle (oracle/orca_oracle.c) to the reference, bit for bit.

The fixtures in tests/golden/ are outputs of the unmodified reference package run
in the build container by oracle/gen_golden.py. Everything here is float64 and
every comparison is exact (np.array_equal) unless stated.
"""

import numpy as np
import pytest

from helpers import FRAME_FIXTURES, LP_FIXTURES, load_golden, state_from_frame_fixture
from oracle import oracle as O


def test_shuffle_matches_reference_permutations():
    g = load_golden("kat.npz")
    for k, seed, row in zip(g["shuffle_k"], g["shuffle_seed"], g["shuffle_perm"]):
        assert O.shuffle_order(int(k), int(seed)) == [int(v) for v in row[:k]]


def test_problem_seed_matches_reference():
    g = load_golden("kat.npz")
    for a, f in enumerate(g["seed_frames"]):
        for b, i in enumerate(g["seed_ids"]):
            assert O.problem_seed(int(i), int(f)) == int(g["seed_values"][a, b])


def test_vo_exit_bitwise():
    g = load_golden("kat.npz")
    for c, want in zip(g["vo_in"], g["vo_out"]):
        u, n, ok = O.vo_exit(c[0:2], c[2:4], c[4], c[5], c[6])
        assert ok == bool(want[4])
        assert np.array_equal(np.concatenate([u, n]), want[:4])


def test_vo_exit_known_answers():
    # pkg/tests/test_orca.py:25-50
    u, n, ok = O.vo_exit((10, 0), (0, 0), 0.5, 2.0, 0.1)
    np.testing.assert_allclose(u, [4.75, 0], atol=1e-12)
    np.testing.assert_allclose(n, [-1, 0], atol=1e-12)
    u, n, ok = O.vo_exit((2, 0), (2, 0), 1.0, 1.0, 0.1)
    np.testing.assert_allclose(u, [-1, 0], atol=1e-12)
    u, n, ok = O.vo_exit((0.4, 0), (0, 0), 0.5, 2.0, 0.1)
    np.testing.assert_allclose(u, [-1, 0], atol=1e-12)
    np.testing.assert_allclose(n, [-1, 0], atol=1e-12)
    assert O.vo_exit((0, 0), (1, 0), 0.5, 2.0, 0.1)[2] is False


def test_lp_known_answers():
    # pkg/tests/test_lp.py:23-43 and :77-100
    g = load_golden("kat.npz")
    e = np.zeros((0, 2))
    v, st, fa = O.solve_one(e, e, (1.0, 0.5), 2.0)
    assert np.array_equal(v, [1.0, 0.5]) and st == 0 and fa == -1
    v, _, _ = O.solve_one(e, e, (3.0, 4.0), 2.5)
    np.testing.assert_allclose(v, [1.5, 2.0], atol=1e-12)
    assert np.array_equal(v, g["lp_kat_closest"][1])
    v, _, _ = O.solve_one([(0, 1)], [(0, 1)], (0.7, 0.2), 5.0)
    np.testing.assert_allclose(v, [0.7, 1.0], atol=1e-12)
    band_f = ([(0, -1), (0, 1)], [(0, 1), (0, -1)])
    band_e = ([(0, 1), (0, -1)], [(0, 1), (0, -1)])
    tri_n = g["lp_kat_tri_nrm"]
    got = [O.least_penetration(*band_f, 5.0, 0, (0.3, 2.0)),
           O.least_penetration(*band_f, 5.0, 0, (-0.2, 0.4)),
           O.least_penetration(*band_e, 5.0, 0, (0.3, 2.0)),
           O.least_penetration(tri_n, tri_n, 5.0, 0, (0.4, -0.3))]
    assert np.array_equal(np.array(got), g["lp_kat_lpen"])
    np.testing.assert_allclose(got[0], [0.3, 1.0], atol=1e-9)
    np.testing.assert_allclose(got[2], [0.3, 0.0], atol=1e-9)
    np.testing.assert_allclose(got[3], [0.0, 0.0], atol=1e-9)


@pytest.mark.parametrize("name", LP_FIXTURES)
def test_solve_range_bitwise(name):
    g = load_golden(name)
    for workers in (1, 4):
        v, st, fa = O.solve_range(g["coff"], g["cpts"], g["cnrm"], g["tgt"], g["caps"],
                                  g["seeds"], worker_count=workers)
        assert np.array_equal(st, g["status"])
        assert np.array_equal(fa, g["failed"])
        assert np.array_equal(v, g["out_v"])


@pytest.mark.parametrize("name", FRAME_FIXTURES)
def test_frame_bitwise(name):
    g = load_golden(name)
    st, cfg = state_from_frame_fixture(g)
    for workers in (1, 3):
        fs = O.frame_solve(st, cfg, worker_count=workers, debug=True)
        assert np.array_equal(fs.cell_ix, g["cell_ix"])
        assert np.array_equal(fs.cell_iy, g["cell_iy"])
        assert np.array_equal(fs.nb_count, g["nb_count"])
        assert np.array_equal(fs.nb_rows, g["nb_rows"])
        assert np.array_equal(fs.des, g["des"])
        assert np.array_equal(fs.constraints, g["cons"])
        assert np.array_equal(fs.status, g["status"])
        assert np.array_equal(fs.failed_at, g["failed"])
        assert np.array_equal(fs.out_v, g["out_v"])
        assert np.all(fs.err == -1)


@pytest.mark.parametrize("name", FRAME_FIXTURES)
def test_advance_bitwise(name):
    g = load_golden(name)
    st, cfg = state_from_frame_fixture(g)
    new, min_sep, coll, fb, removed = O.advance(st, cfg)
    assert new.frame == st.frame + 1 and new.time == new.frame * cfg.dt
    assert np.array_equal(new.ids, g["new_ids"])
    assert np.array_equal(new.positions, g["new_positions"])
    assert np.array_equal(new.velocities, g["new_velocities"])
    assert np.array_equal(removed, g["removed_ids"])
    assert min_sep == float(g["min_separation"])
    assert coll == int(g["collision_count"])
    assert fb == int(g["lp_fallbacks"]) == new.lp_fallbacks


def test_chain_100_steps_bitwise():
    """Config 1: 100 consecutive steps of 1,024 pedestrians; each input is the
    previous output rounded to float32 (gen_golden.gen_chain)."""
    from paper_2008_11578_b200.synth import plaza_crowd
    g = load_golden("chain_1k.npz")
    st, cfg = plaza_crowd(1024, 0, density=0.25, seed=1)
    f32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    for s in range(100):
        ids = st.ids
        assert ids.shape[0] == int(g["active"][s])
        assert np.array_equal(st.positions, g["pos_in"][s][ids].astype(np.float64))
        assert np.array_equal(st.velocities, g["vel_in"][s][ids].astype(np.float64))
        fs = O.frame_solve(st, cfg)
        assert np.array_equal(fs.out_v, g["out_v"][s][ids])
        assert np.array_equal(fs.status, g["status"][s][ids])
        st, min_sep, coll, fb, _ = O.advance(st, cfg)
        assert (fb, coll) == (int(g["fallbacks"][s]), int(g["collisions"][s]))
        assert min_sep == float(g["min_sep"][s])
        st.positions, st.velocities = f32(st.positions), f32(st.velocities)


def test_coincident_centres_error_text():
    # pkg/tests/test_engine.py:279 / engine.py:239-245
    from paper_2008_11578_b200.synth import plaza_crowd
    st, cfg = plaza_crowd(16, 0, density=0.25, seed=3)
    st.positions[5] = st.positions[9]
    with pytest.raises(ValueError, match=r"frame 1: agents 5 and 9 have exactly coincident"):
        O.advance(st, cfg)


def test_grid_range_error():
    with pytest.raises(ValueError, match="out of indexable grid range"):
        O.grid_arrays(np.array([[1e12, 0.0]]), 1.0)


@pytest.mark.parametrize("name", ["run_two_way_80.npz", "run_four_way_96.npz", "run_paper_four_way_2500.npz",
                                  "run_paper_two_way_2500.npz"])
def test_whole_run_bitwise(name):
    """The oracle stepped in a loop reproduces the reference's engine.run of the built-in
    crossing scenarios (spawned crowd taken from the fixture): frames, arrivals, metrics."""
    from paper_2008_11578_b200.types import (AgentClass, ResponsibilityMatrix, ScenarioConfig,
                                             SimState)
    g = load_golden(name)
    fm = g["fmat"]
    P, V = AgentClass.PEDESTRIAN, AgentClass.VEHICLE
    cfg = ScenarioConfig(responsibility=ResponsibilityMatrix({(P, P): fm[0, 0], (P, V): fm[0, 1],
                                                              (V, P): fm[1, 0], (V, V): fm[1, 1]}),
                         dt=float(g["dt"]), tau=float(g["tau"]), neighbor_radius=float(g["neighbor_radius"]),
                         max_neighbors=int(g["max_neighbors"]), avoidance_margin=float(g["avoidance_margin"]))
    st = SimState(frame=0, time=0.0, ids=g["ids"].astype(np.int64), positions=g["positions"],
                  velocities=g["velocities"], radii=g["radii"], pref_speeds=g["pref_speeds"],
                  max_speeds=g["max_speeds"], goals=g["goals"], goal_tols=g["goal_tols"],
                  class_codes=g["class_codes"].astype(np.int64))
    f = 0
    fallbacks = collisions = 0
    while st.ids.shape[0] > 0 and st.frame < int(g["guard"]):
        st, sep, coll, fb, _removed = O.advance(st, cfg)
        assert sep == g["m_min_sep"][f] and coll == g["m_coll"][f] and st.ids.shape[0] == g["m_active"][f]
        fallbacks += fb
        collisions += coll
        f += 1
    assert f == int(g["frames"]) and fallbacks == int(g["total_fallbacks"])
    assert collisions == int(g["total_collisions"])
