"""Golden plans for the microbatch-configuration sweep (SURVEY.md §8(d)
config D "full microbatch-config sweep", §8(f)3).

For every (mb_size, B) point the unmodified reference (oracle/_ref/meshpipe)
runs its whole front end on the operator graph of that microbatch size
(detect_modules -> cluster_layers), builds the store and runs search();
the layer aggregates and plan_to_dict (wall_time_s dropped) go to
tests/golden/mbsweep.json.gz.  Configs: A (GPT-2 small ops, points (1,8),
(2,4), (4,2), (8,1)) and D1 (Llama-2 70B proxy, 2,006 ops, u=1, points (1,128),
(2,64), (4,32), (8,16)).

    python tests/golden/make_golden_mbsweep.py
"""

from __future__ import annotations

import gzip
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as MG  # noqa: E402  (reference types, oracle/_ref on sys.path)
from meshpipe.cluster import ClusterSpec  # noqa: E402
from meshpipe.model_graph import (  # noqa: E402
    GptConfig, cluster_layers, detect_modules, generate_gpt_sequence,
)
from meshpipe.planner import plan_to_dict, search  # noqa: E402
from meshpipe.profiling import CostModel, boundary_costs, build_store  # noqa: E402


def cluster_of(name):
    if name == "A":
        return ClusterSpec([MG.mesh("a100", "a100", 1, 4), MG.mesh("v100", "v100", 1, 4)],
                           cross_bw=MG.gbps(25))
    ids, kinds = ["s0", "s1", "s2", "s3"], ["h100", "a100", "a100", "v100"]
    adj = {("s0", "s1"): 100, ("s1", "s2"): 50, ("s2", "s3"): 25}
    cross = {(ids[a], ids[b]): MG.gbps(adj.get((ids[a], ids[b]), 1))
             for a in range(4) for b in range(a + 1, 4)}
    return ClusterSpec([MG.mesh(i, k, 8, 8) for i, k in zip(ids, kinds)], cross_bw=cross)


def ops_of(name, mb):
    if name == "A":
        return generate_gpt_sequence(GptConfig(12, 768, 1024, mb, 50257))
    return MG.llama_like_ops(8192, 4096, 28672, 32000, 80, b=mb)


POINTS = {"A": [(1, 8), (2, 4), (4, 2), (8, 1)], "D1": [(1, 128), (2, 64), (4, 32), (8, 16)]}


def main() -> None:
    out = {}
    for name, points in POINTS.items():
        cl = cluster_of(name)
        recs = []
        for mb, B in points:
            ops = ops_of(name, mb)
            layers = cluster_layers(detect_modules(ops), ops, 1)
            store = build_store(layers, cl, CostModel(), imbalance_ratio=3.0)
            plan = plan_to_dict(search(store, boundary_costs(layers, cl), B, epsilon=0.05,
                                       workers=8, batch_size=4))
            plan["search_stats"].pop("wall_time_s", None)
            recs.append({"mb": mb, "B": B, "plan": plan,
                         "flops": [l.flops for l in layers.layers],
                         "boundary_bytes": [l.boundary_bytes for l in layers.layers]})
            print(name, mb, B, plan["predicted_latency"], flush=True)
        out[name] = recs
    with gzip.open(os.path.join(HERE, "mbsweep.json.gz"), "wt") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
