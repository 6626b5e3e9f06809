"""GPU: search() / dp_search() return the reference's plan bit for bit
(stage boundaries, submeshes, launch counts, K bounds, T*, eta, search_stats)
on the benchmark configs and on the reference tests' own seeded instances."""

import math

import pytest

import oracle as O
from helpers import assert_plan_equal, build, expected, load_json, plan_dict, seeded

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["A", "B", "C", "D1", "D2", "D3", "D4"])
def test_search_configs_equal_reference(name):
    from paper_2509_24859_b200.planner import search, validate_plan

    inst, exp = load_json(name), expected(name)
    store, costs, cluster, B, eps = build(inst)
    plan = search(store, costs, B, epsilon=eps, workers=8, batch_size=4)
    assert_plan_equal(plan_dict(plan), exp["plan"])
    assert plan.search_stats["backend"] == "cuda"
    assert validate_plan(plan, store, costs, cluster) == []


def _runs():
    for rec in seeded()["search"]:
        if "instance" not in rec:
            continue
        for run in rec["runs"]:
            yield rec, run


def test_seeded_searches_equal_reference():
    from paper_2509_24859_b200.planner import InfeasiblePlanError, PlannerError, search

    n = 0
    for rec, run in _runs():
        store, costs, cluster, B, eps = build(rec["instance"])
        assert store.stats.as_dict() == rec["stats"], rec["tag"]
        assert store.feasible_t_values() == rec["pool"], rec["tag"]
        kw = dict(run["kw"])
        if "error" in run:
            exc = InfeasiblePlanError if run["error"] == "InfeasiblePlanError" else PlannerError
            with pytest.raises(exc):
                search(store, costs, B, **kw)
            continue
        plan = search(store, costs, B, **kw)
        assert_plan_equal(plan_dict(plan), run["plan"])
        n += 1
    assert n > 200


def test_dp_search_single_candidate_equals_oracle():
    from paper_2509_24859_b200.planner import DpTables, dp_search

    inst = load_json("C")
    store, costs, cluster, B, eps = build(inst)
    tables = DpTables(store, costs)
    tb = O.tables(inst)
    pool = store.feasible_t_values()
    for t in pool[1100::97]:
        got = dp_search(store, costs, B, t, eps, tables)
        want = O.evaluate(inst, tb, t)
        if want is None:
            assert got is None
            continue
        d = plan_dict(got)
        for k in ("t_max", "predicted_latency", "eta_pct", "stages", "boundaries"):
            assert d[k] == want[k], k
        assert d["search_stats"]["dp_states"] == want["search_stats"]["dp_states"]


def test_infeasible_and_errors():
    from paper_2509_24859_b200.cluster import ClusterSpec, DeviceMesh
    from paper_2509_24859_b200.model_graph import uniform_layers
    from paper_2509_24859_b200.planner import InfeasiblePlanError, PlannerError, dp_search, search
    from paper_2509_24859_b200.profiling import (NoFeasibleCandidateError, boundary_costs,
                                                 build_store)

    layers = uniform_layers(2, 1e12, 100e9, 1e6)
    cl = ClusterSpec([DeviceMesh("m", 1, 2, 1e12, 60e9, 1e9, 1e9)], cross_bw=1e9)
    store = build_store(layers, cl, imbalance_ratio=math.inf)
    costs = boundary_costs(layers, cl)
    with pytest.raises(InfeasiblePlanError):
        search(store, costs, 4)
    with pytest.raises(PlannerError):
        dp_search(store, costs, 4, 0.0)
    tiny = ClusterSpec([DeviceMesh("m", 1, 1, 1e12, 1e3, 1e9, 1e9)], cross_bw=1e9)
    with pytest.raises(NoFeasibleCandidateError, match="tightest violation: span"):
        build_store(uniform_layers(2, 1e12, 1e9, 1e6), tiny)


def test_overrides_update_aliases_and_plans():
    from paper_2509_24859_b200.cluster import ClusterSpec, DeviceMesh
    from paper_2509_24859_b200.model_graph import uniform_layers
    from paper_2509_24859_b200.profiling import ProfilingError, build_store, import_profiles

    v = DeviceMesh("v", 1, 2, 125e12, 32e9, 150e9, 25e9)
    a = DeviceMesh("a", 2, 2, 312e12, 40e9, 300e9, 25e9)
    store = build_store(uniform_layers(3, 1e12, 1e9, 1e6), ClusterSpec([v, a], cross_bw=6.25e8),
                        imbalance_ratio=math.inf)
    before = store.lookup(1, 2, "v", (1, 2))
    assert store.apply_overrides(import_profiles({})) == 0
    assert store.lookup(1, 2, "v", (1, 2)) is before
    sig = store.signature_text(1, 2)
    assert store.apply_overrides(
        [{"signature": sig, "mesh": "v", "submesh": [1, 2], "t_fwd": 0.5, "t_bwd": 1.0}]) == 1
    assert store.lookup(1, 2, "v", (1, 2)).t == 1.5
    assert store.lookup(2, 3, "v", (1, 2)).t == 1.5
    assert store.lookup(1, 2, "a", (1, 2)).t != 1.5
    assert 1.5 in store.feasible_t_values()
    with pytest.raises(ProfilingError, match="positive"):
        store.apply_overrides([{"signature": sig, "mesh": "v", "submesh": [1, 1], "t_fwd": -1.0}])
    with pytest.raises(ProfilingError, match="unknown mesh"):
        store.apply_overrides([{"signature": "x", "mesh": "nope", "submesh": [1, 1]}])
