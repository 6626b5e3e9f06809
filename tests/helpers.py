"""Shared test helpers: golden instances -> package types, plan comparison."""

from __future__ import annotations

import gzip
import json
import math
import os

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")
INSTANCES = os.path.join(GOLDEN, "instances")

_seeded = None


def load_json(name: str) -> dict:
    with open(os.path.join(INSTANCES, f"{name}.json")) as fh:
        return json.load(fh)


def expected(name: str) -> dict:
    with open(os.path.join(INSTANCES, f"{name}_expected.json")) as fh:
        return json.load(fh)


def expected_arrays(name: str):
    import numpy as np

    return np.load(os.path.join(INSTANCES, f"{name}_expected.npz"))


def seeded() -> dict:
    global _seeded
    if _seeded is None:
        with gzip.open(os.path.join(GOLDEN, "seeded.json.gz"), "rt") as fh:
            _seeded = json.load(fh)
    return _seeded


def to_types(inst: dict):
    """Golden dict -> (LayerSequence, ClusterSpec, CostModel, rho, B, eps)."""
    from paper_2509_24859_b200.cluster import ClusterSpec, DeviceMesh
    from paper_2509_24859_b200.model_graph import layers_from_arrays
    from paper_2509_24859_b200.profiling import CostModel

    lay = inst["layers"]
    layers = layers_from_arrays(lay["flops"], lay["param_bytes"], lay["boundary_bytes"],
                                [tuple(s) for s in lay["signature"]])
    meshes = [DeviceMesh(m["id"], m["hosts"], m["devices_per_host"], m["peak_flops"],
                         m["mem_device"], m["intra_host_bw"], m["inter_host_bw"])
              for m in inst["cluster"]["meshes"]]
    cb = inst["cluster"]["cross_bw"]
    if isinstance(cb, list):
        cb = {(a, b): v for a, b, v in cb}
    cluster = ClusterSpec(meshes, cross_bw=cb, cross_latency=inst["cluster"]["cross_latency"])
    model = CostModel(**inst["model"])
    rho = float(inst["imbalance_ratio"])
    return layers, cluster, model, rho, inst["num_microbatches"], inst["epsilon"]


def build(inst: dict):
    from paper_2509_24859_b200.profiling import boundary_costs, build_store

    layers, cluster, model, rho, B, eps = to_types(inst)
    store = build_store(layers, cluster, model, imbalance_ratio=rho, dedup=inst.get("dedup", True))
    costs = boundary_costs(layers, cluster)
    return store, costs, cluster, B, eps


def plan_dict(plan) -> dict:
    from paper_2509_24859_b200.planner import plan_to_dict

    d = plan_to_dict(plan)
    d["search_stats"].pop("wall_time_s", None)
    return d


def assert_plan_equal(got: dict, ref: dict, stats: bool = True) -> None:
    """Bit-exact plan parity: every field of plan_to_dict, floats compared
    with ==, plus the search_stats the reference reports."""
    for key in ("num_microbatches", "t_max", "predicted_latency", "eta_pct", "epsilon"):
        assert got[key] == ref[key], (key, got[key], ref[key])
    assert got["stages"] == ref["stages"]
    assert got["boundaries"] == ref["boundaries"]
    if stats:
        for key, val in ref["search_stats"].items():
            if key in ("backend", "wall_time_s"):
                continue
            assert got["search_stats"].get(key) == val, (key, got["search_stats"].get(key), val)


def isinf(x) -> bool:
    return isinstance(x, float) and math.isinf(x)


REF = os.path.join(os.path.dirname(HERE), "oracle", "_ref")


def reference_meshpipe():
    """The unmodified reference package (oracle/_ref, built by oracle/Makefile)
    or None when it is not built.  Test infrastructure only."""
    import sys

    if not os.path.isdir(os.path.join(REF, "meshpipe")):
        return None
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import meshpipe  # noqa: F401
    import meshpipe.planner  # noqa: F401

    return meshpipe


def ref_types(inst: dict):
    """Golden dict -> the reference's own (store, costs, B, eps): reference
    LayerSequence / ClusterSpec / CostModel, reference build_store."""
    from meshpipe.cluster import ClusterSpec as RC, DeviceMesh as RM
    from meshpipe.model_graph import Layer as RL, LayerSequence as RS
    from meshpipe.profiling import CostModel as RCM, boundary_costs as rbc, build_store as rbs

    lay = inst["layers"]
    layers = RS(tuple(RL(i, i + 1, lay["flops"][i], lay["param_bytes"][i],
                         lay["boundary_bytes"][i], tuple(lay["signature"][i]))
                      for i in range(len(lay["flops"]))), ())
    meshes = [RM(m["id"], m["hosts"], m["devices_per_host"], m["peak_flops"], m["mem_device"],
                 m["intra_host_bw"], m["inter_host_bw"]) for m in inst["cluster"]["meshes"]]
    cb = inst["cluster"]["cross_bw"]
    if isinstance(cb, list):
        cb = {(a, b): v for a, b, v in cb}
    cl = RC(meshes, cross_bw=cb, cross_latency=inst["cluster"]["cross_latency"])
    store = rbs(layers, cl, RCM(**inst["model"]), imbalance_ratio=float(inst["imbalance_ratio"]),
                dedup=inst.get("dedup", True))
    return store, rbc(layers, cl), inst["num_microbatches"], inst["epsilon"]
