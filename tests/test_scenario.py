"""The callers and file formats either side of the steering step (SURVEY.md s8(f) rows
3-4) against fixtures produced by the reference's own scenario / crossings / cli modules
(oracle/gen_golden.gen_scenarios): crossing documents, the crowd the seeded sampler spawns
(bit for bit), frame guards, validation messages, CSV bytes. CPU only."""

import hashlib
import json
import os

import numpy as np
import pytest

from helpers import GOLDEN as GOLDEN_DIR
from paper_2008_11578_b200 import (AgentClass, ScenarioError, build_agents, crossing_config, four_way_dict,
                                   init_state, read_trajectories, scenario_from_dict, two_way_dict,
                                   write_trajectories)
from paper_2008_11578_b200 import cli
from paper_2008_11578_b200.crossings import arm_size
from paper_2008_11578_b200.scenario import write_metrics_summary
from paper_2008_11578_b200.types import RunSummary

with open(os.path.join(GOLDEN_DIR, "scenario_cases.json")) as f:
    G = json.load(f)


def same(a, b):
    """dict / list equality where NaN == NaN."""
    if isinstance(a, dict):
        return isinstance(b, dict) and a.keys() == b.keys() and all(same(a[k], b[k]) for k in a)
    if isinstance(a, (list, tuple)):
        return isinstance(b, (list, tuple)) and len(a) == len(b) and all(same(x, y) for x, y in zip(a, b))
    if isinstance(a, float) and isinstance(b, float) and a != a:
        return b != b
    return a == b


@pytest.mark.parametrize("case", G["cases"], ids=lambda c: f"{c['kind']}-{c['per_arm']}-{c['seed']}")
def test_crossing_documents_and_spawned_crowd_match_reference(case):
    maker = two_way_dict if case["kind"] == "two_way" else four_way_dict
    doc = maker(case["per_arm"], case["vehicle_fraction"], case["seed"], **case["kwargs"])
    assert same(doc, case["doc"])
    assert list(arm_size(case["per_arm"], case["vehicle_fraction"], case["kwargs"].get("clearance_time", 0.5),
                         case["kwargs"].get("size_for_worst_class", False))) == case["arm_size"]
    cfg = crossing_config(case["kind"], case["per_arm"], case["vehicle_fraction"], case["seed"], **case["kwargs"])
    assert cfg.frame_guard() == case["guard"] and cfg.warnings == case["warnings"]
    st = init_state(cfg)                         # spawns with the seeded sampler
    for key in ("ids", "class_codes"):
        assert np.array_equal(getattr(st, key), np.array(case[key], dtype=np.int64)), key
    for key in ("positions", "goals", "velocities"):
        assert np.array_equal(getattr(st, key), np.array(case[key], dtype=np.float64).reshape(-1, 2)), key
    for key in ("radii", "pref_speeds", "max_speeds", "goal_tols"):
        assert np.array_equal(getattr(st, key), np.array(case[key], dtype=np.float64)), key
    assert st.frame == 0 and st.time == 0.0 and st.lp_fallbacks == 0


def test_build_agents_objects():
    case = G["cases"][1]
    agents = build_agents(crossing_config(case["kind"], case["per_arm"], case["vehicle_fraction"], case["seed"]))
    assert [a.id for a in agents] == case["ids"]
    assert np.array_equal(np.array([a.position for a in agents]), np.array(case["positions"]))
    assert [int(a.agent_class) for a in agents] == case["class_codes"]
    assert all(np.array_equal(a.velocity, np.zeros(2)) for a in agents)


@pytest.mark.parametrize("item", G["broken"], ids=lambda b: b["label"])
def test_validation_messages_match_reference(item):
    if item["message"] is None:
        cfg = scenario_from_dict(item["doc"], source="<t>")
        assert cfg.regions
    else:
        with pytest.raises(ScenarioError) as exc:
            cfg = scenario_from_dict(item["doc"], source="<t>")
            build_agents(cfg)                    # density is checked when spawning
        assert str(exc.value) == item["message"]


def test_warnings_and_spawn_failure_text():
    good = two_way_dict(4, 0.5, 1)
    doc = {**good, "responsibility": {**good["responsibility"], "pedestrian|vehicle": 0.3, "vehicle|vehicle": 0.2}}
    assert scenario_from_dict(doc, source="<w>").warnings == G["warnings_two_pairs"]
    dense = json.loads(json.dumps(good))
    dense["regions"][0]["count"] = 100000
    with pytest.raises(ScenarioError) as exc:
        build_agents(scenario_from_dict(dense, source="<t>"))
    assert str(exc.value) == G["dense_build_message"]


def test_trajectory_csv_bytes_round_trip(tmp_path):
    src = os.path.join(GOLDEN_DIR, "traj_two_way_12.csv")
    logs = read_trajectories(src)
    assert len(logs) == G["short_run"]["frames"] and logs[0].frame == 1
    assert logs[0].classes.dtype == np.int8 and logs[0].positions.shape[1] == 2
    out = tmp_path / "t.csv"
    write_trajectories(logs, out)
    assert out.read_bytes() == open(src, "rb").read()          # the reference's bytes, CRLF rows and all
    again = read_trajectories(out)
    assert again == logs
    with open(tmp_path / "bad.csv", "w") as f:
        f.write("frame,time\r\n")
    with pytest.raises(ValueError):
        read_trajectories(tmp_path / "bad.csv")


def test_metrics_summary_file(tmp_path):
    s = RunSummary(total_collisions=3, min_separation=0.125, mean_frame_ms=1.5, p95_frame_ms=2.25, agents=12,
                   seed=9, frames=12, terminated=False, arrived=0, total_fallbacks=0, mean_travel_time={})
    write_metrics_summary(s, tmp_path / "m.csv")
    lines = (tmp_path / "m.csv").read_bytes().split(b"\r\n")
    assert lines[0].decode() == G["short_run"]["metrics_csv_head"]
    assert lines[1] == b"3,0.125,1.5,2.25,12,9" and lines[2] == b""


def test_cli_exit_codes_without_touching_the_gpu(tmp_path, capsys):
    bad = tmp_path / "bad.yaml"
    bad.write_text("format_version: 1\nregions: 5\n")
    assert cli.main(["run", "--scenario", str(bad), "--out", str(tmp_path / "o")]) == cli.EXIT_VALIDATION
    assert "regions: expected a list of regions" in capsys.readouterr().err
    assert cli.main(["run", "--scenario", str(tmp_path / "missing.yaml"), "--out", str(tmp_path / "o")]) == cli.EXIT_IO
    with pytest.raises(SystemExit):
        cli.main(["crossing", "--kind", "roundabout", "--agents", "4", "--out", "x"])


def test_sha_fixture_is_well_formed():
    for name, rec in G["run_sha"].items():
        assert len(rec["trajectories"]) == 64 and len(rec["agents"]) == 64
        assert hashlib.sha256(b"").hexdigest() != rec["trajectories"]
    assert AgentClass.from_label("vehicle") == AgentClass.VEHICLE


def test_lp_object_api_matches_the_reference_schema():
    """LpStatus values, LpResult.feasible, HalfPlaneConstraint.satisfies and the LpProblem
    coercions of pkg/src/orcasim/lp.py:42-91; solve_batch validates worker_count (lp.py:268-269)."""
    import numpy as np
    import pytest
    from paper_2008_11578_b200 import HalfPlaneConstraint, LpProblem, LpResult, LpStatus, solve_batch
    assert LpStatus.FEASIBLE.value == "feasible" and LpStatus.FALLBACK_USED.value == "fallback_used"
    assert LpResult(np.zeros(2), LpStatus.FEASIBLE).feasible
    assert not LpResult(np.zeros(2), LpStatus.FALLBACK_USED, 3).feasible
    c = HalfPlaneConstraint((1, 0), (1, 0))
    assert c.point.dtype == float and c.satisfies((1.5, 9.0)) and not c.satisfies((0.5, 0.0))
    assert c.satisfies((0.9, 0.0), slack=0.2)
    p = LpProblem([c], (3, 4), "2", shuffle_seed=-1)
    assert p.target.dtype == float and p.speed_cap == 2.0 and p.shuffle_seed == (1 << 64) - 1
    with pytest.raises(ValueError, match="worker_count must be >= 1"):
        solve_batch([p], worker_count=0)
    assert solve_batch([]) == []


def test_agent_state_validation():
    import pytest
    from paper_2008_11578_b200 import AgentClass, AgentState
    a = AgentState(id=1, position=(0, 0), velocity=(1, 0), radius=0.3, pref_speed=1, max_speed=2, goal=(5, 5),
                   agent_class=1)
    assert a.agent_class is AgentClass.VEHICLE and a.position.dtype == float
    with pytest.raises(ValueError, match="radius must be positive"):
        AgentState(id=2, position=(0, 0), velocity=(0, 0), radius=0.0, pref_speed=1, max_speed=2, goal=(1, 1))
    with pytest.raises(ValueError, match="pref_speed <= max_speed"):
        AgentState(id=3, position=(0, 0), velocity=(0, 0), radius=0.3, pref_speed=3, max_speed=2, goal=(1, 1))


def test_max_neighbors_above_the_device_limit_is_a_scenario_error():
    import pytest
    from paper_2008_11578_b200 import ScenarioError, scenario_from_dict, two_way_dict
    doc = two_way_dict(4)
    doc["max_neighbors"] = 32
    scenario_from_dict(doc)
    doc["max_neighbors"] = 33
    with pytest.raises(ScenarioError, match="max_neighbors: 33 exceeds"):
        scenario_from_dict(doc)
