"""GPU: the microbatch-configuration sweep (config D's "full microbatch-config
sweep") returns, for every (mb_size, B) point, the
layer aggregates of the reference front end and the reference search() plan
(goldens: tests/golden/make_golden_mbsweep.py)."""

import gzip
import json
import os

import pytest

from helpers import assert_plan_equal, load_json, plan_dict, to_types

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def golden():
    with gzip.open(os.path.join(HERE, "golden", "mbsweep.json.gz"), "rt") as fh:
        return json.load(fh)


def ops_builder(name):
    from paper_2509_24859_b200.model_graph import GptConfig, generate_gpt_sequence
    from paper_2509_24859_b200.workloads import llama_like_ops

    if name == "A":
        return lambda mb: generate_gpt_sequence(GptConfig(12, 768, 1024, mb, 50257))
    return lambda mb: llama_like_ops(b=mb)


@pytest.mark.parametrize("concurrent", [True, False])
@pytest.mark.parametrize("name", ["A", "D1"])
def test_microbatch_sweep_equals_reference(name, concurrent):
    from paper_2509_24859_b200.sweep import best_point, microbatch_sweep

    recs = golden()[name]
    _, cluster, model, rho, _, eps = to_types(load_json(name))
    points = [(r["mb"], r["B"]) for r in recs]
    res = microbatch_sweep(ops_builder(name), cluster, points, model=model,
                           imbalance_ratio=rho, epsilon=eps, batch_size=4,
                           concurrent=concurrent)
    for pt, r in zip(res, recs):
        assert (pt.mb_size, pt.num_microbatches) == (r["mb"], r["B"])
        assert [l.flops for l in pt.layers.layers] == r["flops"]
        assert [l.boundary_bytes for l in pt.layers.layers] == r["boundary_bytes"]
        assert_plan_equal(plan_dict(pt.plan), r["plan"])
    best = best_point(res)
    want = min(recs, key=lambda r: (r["plan"]["predicted_latency"] / (r["mb"] * r["B"]), r["mb"]))
    assert (best.mb_size, best.num_microbatches) == (want["mb"], want["B"])
