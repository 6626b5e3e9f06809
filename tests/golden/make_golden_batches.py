"""Golden plans for the microbatch-count sweep.

Runs the unmodified reference (oracle/_ref/meshpipe) search() on configs A, B,
C and D1 for several microbatch counts B and writes plan_to_dict of each
(wall_time_s dropped) to tests/golden/batches.json.gz.

    python tests/golden/make_golden_batches.py
"""

from __future__ import annotations

import gzip
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))
sys.path.insert(0, os.path.join(REPO, "tests"))

from meshpipe.cluster import ClusterSpec, DeviceMesh  # noqa: E402
from meshpipe.model_graph import Layer, LayerSequence  # noqa: E402
from meshpipe.planner import InfeasiblePlanError, plan_to_dict, search  # noqa: E402
from meshpipe.profiling import CostModel, boundary_costs, build_store  # noqa: E402

from helpers import load_json  # noqa: E402


def to_reference_types(inst):
    lay = inst["layers"]
    layers = LayerSequence(tuple(
        Layer(i, i + 1, lay["flops"][i], lay["param_bytes"][i], lay["boundary_bytes"][i],
              tuple(lay["signature"][i])) for i in range(len(lay["flops"]))), ())
    meshes = [DeviceMesh(m["id"], m["hosts"], m["devices_per_host"], m["peak_flops"],
                         m["mem_device"], m["intra_host_bw"], m["inter_host_bw"])
              for m in inst["cluster"]["meshes"]]
    cb = inst["cluster"]["cross_bw"]
    if isinstance(cb, list):
        cb = {(a, b): v for a, b, v in cb}
    cluster = ClusterSpec(meshes, cross_bw=cb, cross_latency=inst["cluster"]["cross_latency"])
    return (layers, cluster, CostModel(**inst["model"]), float(inst["imbalance_ratio"]),
            inst["num_microbatches"], inst["epsilon"])

BATCHES = {"A": [1, 2, 3, 8, 32, 128, 1024], "B": [1, 4, 16, 64, 256],
           "C": [1, 8, 48, 256], "D1": [16, 512]}


def main() -> None:
    out = {}
    for name, Bs in BATCHES.items():
        inst = load_json(name)
        layers, cluster, model, rho, _, eps = to_reference_types(inst)
        store = build_store(layers, cluster, model, imbalance_ratio=rho)
        costs = boundary_costs(layers, cluster)
        recs = []
        for B in Bs:
            try:
                d = plan_to_dict(search(store, costs, B, epsilon=eps, workers=8, batch_size=4))
                d["search_stats"].pop("wall_time_s", None)
                recs.append({"B": B, "plan": d})
            except InfeasiblePlanError as exc:
                recs.append({"B": B, "error": str(exc)})
        out[name] = recs
        print(name, [r["B"] for r in recs])
    with gzip.open(os.path.join(HERE, "batches.json.gz"), "wt") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
