"""GPU: search_batches() -- one set of DP sweeps scored for many microbatch
counts -- returns, for every B, the reference's
search(store, costs, B) plan and search_stats (goldens:
tests/golden/make_golden_batches.py), and agrees with per-B search()."""

import gzip
import json
import os

import pytest

from helpers import assert_plan_equal, build, load_json, plan_dict

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def golden():
    with gzip.open(os.path.join(HERE, "golden", "batches.json.gz"), "rt") as fh:
        return json.load(fh)


@pytest.mark.parametrize("name", ["A", "B", "C", "D1"])
def test_search_batches_equal_reference(name):
    from paper_2509_24859_b200.planner import InfeasiblePlanError, search_batches

    recs = golden()[name]
    store, costs, cluster, _, eps = build(load_json(name))
    Bs = [r["B"] for r in recs]
    ok = [r for r in recs if "plan" in r]
    if len(ok) < len(recs):  # an infeasible B raises like search() would
        with pytest.raises(InfeasiblePlanError):
            search_batches(store, costs, Bs, epsilon=eps, batch_size=4)
    plans = search_batches(store, costs, [r["B"] for r in ok], epsilon=eps, batch_size=4)
    for r in ok:
        assert_plan_equal(plan_dict(plans[r["B"]]), r["plan"])


def test_search_batches_matches_search_unoptimized():
    from paper_2509_24859_b200.planner import search, search_batches

    store, costs, cluster, B, eps = build(load_json("A"))
    Bs = [1, 5, B, 77]
    plans = search_batches(store, costs, Bs, epsilon=eps, optimized=False)
    for b in Bs:
        one = search(store, costs, b, epsilon=eps, optimized=False)
        assert_plan_equal(plan_dict(plans[b]), plan_dict(one))
