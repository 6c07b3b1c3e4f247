"""The reference's OBJECT-level operators through the host wrappers of this package
(orca.py, grid.py, lp.py), against outputs of the reference itself
(tests/golden/api_cases.npz, written by oracle/gen_golden.gen_api from orcasim):

    gather_constraints / build_orca_halfplane / compute_vo_exit   pkg/src/orcasim/orca.py:145-196
    rebuild / query_neighbors                                      pkg/src/orcasim/grid.py:34-83
    solve_least_penetration                                        pkg/src/orcasim/lp.py:168-190

Everything numerical runs on the device (orca_vo_exit_batch, orca_neighbor_query,
orca_least_penetration); FP64, so the comparison is array_equal."""

import numpy as np
import pytest

from helpers import load_golden
from paper_2008_11578_b200 import (AgentClass, AgentState, HalfPlaneConstraint, ResponsibilityMatrix, VoExit,
                                   build_orca_halfplane, compute_vo_exit, gather_constraints, query_neighbors,
                                   rebuild, solve_least_penetration)
from paper_2008_11578_b200.grid import neighbor_lists

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def crowd():
    g = load_golden("api_cases.npz")
    agents = [AgentState(id=int(g["ids"][i]), position=g["positions"][i], velocity=g["velocities"][i],
                         radius=float(g["radii"][i]), pref_speed=1.0, max_speed=2.0, goal=g["positions"][i] + 1.0,
                         agent_class=AgentClass(int(g["class_codes"][i]))) for i in range(g["ids"].shape[0])]
    return g, agents


def test_rebuild_and_query_neighbors_equal_the_reference(crowd):
    g, agents = crowd
    grid = rebuild(agents, 4.0)
    assert grid.population == int(g["grid_population"])
    assert np.array_equal(np.array(sorted(grid.cells), dtype=np.int64), g["grid_cells"])
    assert grid.cell_of(agents[0].position) in grid.cells
    for key in [k for k in g if k.startswith("nb_ids_")]:
        radius, max_count = float(key.split("_r")[1].split("_m")[0]), int(key.split("_m")[1])
        for i in (0, 4, 5, 77, len(agents) - 1):
            nb = query_neighbors(grid, agents, agents[i].id, radius, max_count)
            want = g[key][i]
            assert [b.id for b in nb] == [int(x) for x in want[want >= 0]], (key, i)
        rows, count = neighbor_lists(g["ids"], g["positions"], radius, max_count)     # every agent at once
        got = np.where(rows >= 0, g["ids"][np.maximum(rows, 0)], -1)
        assert np.array_equal(got, g[key]) and np.array_equal(count, (g[key] >= 0).sum(axis=1))
    assert query_neighbors(grid, agents, agents[0].id, 6.0, 0) == []
    with pytest.raises(KeyError):
        query_neighbors(grid, agents, -12345, 6.0, 4)
    with pytest.raises(ValueError, match="radius must be positive"):
        query_neighbors(grid, agents, agents[0].id, 0.0, 4)
    with pytest.raises(ValueError, match="max_count must be >= 0"):
        query_neighbors(grid, agents, agents[0].id, 1.0, -1)
    with pytest.raises(ValueError, match="cell_size must be positive"):
        rebuild(agents, 0.0)


def test_gather_constraints_equal_the_reference(crowd):
    g, agents = crowd
    grid = rebuild(agents, 4.0)
    matrix = ResponsibilityMatrix.default()
    for i, a in enumerate(agents):
        nb = query_neighbors(grid, agents, a.id, 6.0, 16)
        cs = gather_constraints(a, nb, matrix, 2.0, 0.1)
        assert len(cs) == int(g["cons_cnt"][i])
        for t, c in enumerate(cs):
            assert isinstance(c, HalfPlaneConstraint)
            assert np.array_equal(c.point, g["cons_pts"][i, t]) and np.array_equal(c.normal, g["cons_nrm"][i, t]), (i, t)
    a, b = agents[4], agents[5]                                   # the overlapping pair
    one = build_orca_halfplane(a, b, 0.5, 2.0, 0.1)
    ex = compute_vo_exit(b.position - a.position, a.velocity - b.velocity, a.radius + b.radius, 2.0, 0.1)
    assert isinstance(ex, VoExit) and np.array_equal(one.point, a.velocity + 0.5 * ex.u)
    assert np.array_equal(one.normal, ex.normal)
    with pytest.raises(ValueError, match="cannot avoid itself"):
        build_orca_halfplane(a, a, 0.5, 2.0, 0.1)
    with pytest.raises(ValueError, match="outside"):
        build_orca_halfplane(a, b, 1.5, 2.0, 0.1)
    with pytest.raises(ValueError, match="coincident agent centers"):
        compute_vo_exit((0.0, 0.0), (1.0, 0.0), 1.0, 2.0, 0.1)
    with pytest.raises(ValueError, match="must all be positive"):
        compute_vo_exit((1.0, 0.0), (1.0, 0.0), 1.0, 0.0, 0.1)
    twin = AgentState(id=10**6, position=a.position, velocity=a.velocity, radius=0.3, pref_speed=1.0, max_speed=2.0,
                      goal=a.goal)
    with pytest.raises(ValueError, match=f"neighbor {10**6}: coincident"):
        gather_constraints(a, [b, twin], matrix, 2.0, 0.1)


def test_solve_least_penetration_equals_the_reference():
    g = load_golden("api_cases.npz")
    for c in range(g["lp_k"].shape[0]):
        k = int(g["lp_k"][c])
        cs = [HalfPlaneConstraint(g["lp_pts"][c, t], g["lp_nrm"][c, t]) for t in range(k)]
        v = solve_least_penetration(cs, float(g["lp_cap"][c]), start_index=int(g["lp_start"][c]),
                                    warm_start=g["lp_warm"][c])
        assert np.array_equal(v, g["lp_out"][c]), c
    with pytest.raises(ValueError, match="speed_cap must be positive"):
        solve_least_penetration([], 0.0)
    with pytest.raises(ValueError, match="out of range"):
        solve_least_penetration([], 1.0, start_index=1)
    with pytest.raises(ValueError, match="warm_start is non-finite"):
        solve_least_penetration([], 1.0, warm_start=(np.nan, 0.0))


def test_query_neighbors_without_a_cap_matches_brute_force():
    """max_count beyond the step's 32 (the reference's tests ask for 300 and 10**9): complete
    lists from orca_neighbor_query_all, ordered by (d2, id) with exact ties, against a brute-force
    scan in the reference's arithmetic (grid.py:60-83)."""
    from paper_2008_11578_b200.grid import neighbor_lists_all
    rng = np.random.default_rng(5)
    n = 700
    pos = np.round(rng.uniform(-20.0, 20.0, size=(n, 2)) * 4.0) / 4.0     # a 0.25 m lattice: many equal distances
    _u, first = np.unique(pos, axis=0, return_index=True)
    pos = pos[np.sort(first)]
    n = pos.shape[0]
    ids = rng.permutation(10 * n)[:n].astype(np.int64)
    for radius in (0.9, 3.0, 7.5):
        off, rows = neighbor_lists_all(ids, pos, radius)
        assert off.shape == (n + 1,) and off[0] == 0 and off[-1] == rows.shape[0]
        for i in range(0, n, 7):
            d = pos - pos[i]
            d2 = d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]
            cand = [j for j in range(n) if j != i and not d2[j] > radius * radius]
            cand.sort(key=lambda j: (d2[j], ids[j]))
            assert rows[off[i]:off[i + 1]].tolist() == cand, (radius, i)
    agents = [AgentState(int(ids[i]), pos[i], (0.0, 0.0), 0.25, 1.4, 2.0, (0.0, 0.0)) for i in range(n)]
    g = rebuild(agents, 3.0)
    full = query_neighbors(g, agents, int(ids[3]), 7.5, 10**9)
    assert len(full) > 32
    assert [a.id for a in query_neighbors(g, agents, int(ids[3]), 7.5, 40)] == [a.id for a in full[:40]]
    assert [a.id for a in query_neighbors(g, agents, int(ids[3]), 7.5, 16)] == [a.id for a in full[:16]]
    # an empty crowd and a crowd nobody is near anybody in
    off, rows = neighbor_lists_all(np.zeros(0, np.int64), np.zeros((0, 2)), 1.0)
    assert off.tolist() == [0] and rows.shape == (0,)
    off, rows = neighbor_lists_all(np.arange(3), np.array([[0.0, 0.0], [50.0, 0.0], [0.0, 50.0]]), 1.0)
    assert off.tolist() == [0, 0, 0, 0] and rows.shape == (0,)


def test_simstate_agents_are_the_rows_as_agent_states():
    from paper_2008_11578_b200 import crossing_config, init_state
    cfg = crossing_config("two_way", 6, 0.5, seed=3)
    st = init_state(cfg)
    agents = st.agents
    assert len(agents) == st.active_count
    for i, a in enumerate(agents):
        assert a.id == int(st.ids[i]) and np.array_equal(a.position, st.positions[i])
        assert np.array_equal(a.goal, st.goals[i]) and a.radius == float(st.radii[i])
        assert int(a.agent_class) == int(st.class_codes[i])
    agents[0].position[0] += 1.0                     # copies, not views
    assert agents[0].position[0] != st.positions[0, 0]


def test_neighbor_query_all_reports_the_capacity_it_needs():
    """The C entry point with a buffer that is too small: ORCA_ECAPACITY, with the offsets and the
    total already valid, so that one retry with `total` entries succeeds (grid.neighbor_lists_all)."""
    import ctypes as C
    from paper_2008_11578_b200 import _lib
    L = _lib.load()
    rng = np.random.default_rng(9)
    n = 300
    pos = rng.uniform(0.0, 12.0, size=(n, 2))
    ids = np.arange(n, dtype=np.int64)
    off = np.zeros(n + 1, dtype=np.int64)
    total = C.c_int64(-1)
    rc = L.orca_neighbor_query_all(0, n, _lib.ptr(ids), _lib.ptr(pos), 2.0, 0, _lib.ptr(off), None, C.byref(total))
    assert rc == _lib.ORCA_ECAPACITY and total.value > 0 and off[-1] == total.value
    rows = np.empty(total.value, dtype=np.int64)
    rc = L.orca_neighbor_query_all(0, n, _lib.ptr(ids), _lib.ptr(pos), 2.0, total.value, _lib.ptr(off),
                                   _lib.ptr(rows), C.byref(total))
    assert rc == 0
    d = pos[:, None, :] - pos[None, :, :]
    within = (d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1] <= 4.0) & ~np.eye(n, dtype=bool)
    assert np.array_equal(np.diff(off), within.sum(axis=1))
    # bad arguments are refused, not dereferenced
    assert L.orca_neighbor_query_all(0, n, _lib.ptr(ids), _lib.ptr(pos), -1.0, 0, _lib.ptr(off), None,
                                     C.byref(total)) == _lib.ORCA_EINVAL
    assert L.orca_neighbor_query_all(0, n, _lib.ptr(ids), _lib.ptr(pos), 2.0, 0, _lib.ptr(off), None, None) \
        == _lib.ORCA_EINVAL
