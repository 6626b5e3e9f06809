"""Golden vectors from the reference tests' OWN seeded instances.

Runs the unmodified reference (oracle/_ref/meshpipe) on the instance
generators of pkg/tests/test_planner.py (uniform_instance, varied_instance,
random_cluster: seeds 4321, 1234, 99, 777), pkg/tests/test_acceptance.py
(_random_search_instance: seeds 20260808, 31337, 555; case_study_setup) and
pkg/tests/test_integration.py, plus random 1F1B plans for the simulator, and
writes each instance (plain dict, same format as instances/*.json) with the
reference outputs to tests/golden/seeded.json.gz.

    python tests/golden/make_golden_seeded.py
"""

from __future__ import annotations

import gzip
import hashlib
import json
import math
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))
sys.path.insert(0, HERE)

from meshpipe._core import dp_sweep  # noqa: E402
from meshpipe.cluster import ClusterSpec, DeviceMesh  # noqa: E402
from meshpipe.model_graph import (  # noqa: E402
    HEAVY, GptConfig, OperatorNode, cluster_layers, detect_modules, generate_gpt_sequence,
)
from meshpipe.planner import (  # noqa: E402
    DpTables, InfeasiblePlanError, PlannerError, candidate_tmax, plan_to_dict, search,
)
from meshpipe.profiling import CostModel, boundary_costs, build_store  # noqa: E402
from meshpipe.scheduling import (  # noqa: E402
    LaunchCounts, adaptive_counts, build_program, classic_counts, eager_counts,
)
from meshpipe.simulation import build_dag, simulate  # noqa: E402

from make_golden import instance_json  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# -- the reference tests' instance builders (test_planner.py:40-85,
#    test_acceptance.py:275-307), re-declared here to drive the same RNG calls
def uniform_instance(n_layers=8, flops=1e12, params=1e9, act=1e6):
    ops = [OperatorNode(i, HEAVY, flops, params, act, "blk") for i in range(n_layers)]
    return cluster_layers(detect_modules(ops), ops, 1)


def varied_instance(rng, n_layers):
    ops = [
        OperatorNode(i, HEAVY, rng.uniform(0.5, 3.0) * 1e12, rng.uniform(0.2, 2.0) * 1e9,
                     rng.uniform(0.1, 4.0) * 1e6, f"op{i}")
        for i in range(n_layers)
    ]
    return cluster_layers(detect_modules(ops), ops, n_layers)


def random_cluster(rng, cap_devices=True):
    meshes = []
    for idx in range(2):
        hosts = rng.choice([1, 2])
        per_host = rng.choice([1, 2])
        if cap_devices and hosts * per_host > 4:
            per_host = 1
        meshes.append(DeviceMesh(f"m{idx}", hosts, per_host, rng.uniform(50, 400) * 1e12,
                                 rng.uniform(8, 64) * 1e9, rng.uniform(50, 400) * 1e9,
                                 rng.uniform(10, 50) * 1e9))
    return ClusterSpec(meshes, cross_bw=rng.uniform(0.2, 20) * 1e9)


def random_search_instance(rng):
    layers = varied_instance(rng, rng.randint(3, 6))
    return layers, random_cluster(rng, cap_devices=False)


def plan_rec(plan):
    if plan is None:
        return None
    d = plan_to_dict(plan)
    d["search_stats"].pop("wall_time_s", None)
    return d


def search_rec(store, costs, B, **kw):
    try:
        return {"plan": plan_rec(search(store, costs, B, **kw))}
    except InfeasiblePlanError as e:
        return {"error": "InfeasiblePlanError", "msg": str(e)}
    except PlannerError as e:
        return {"error": "PlannerError", "msg": str(e)}


def inst_of(name, layers, cluster, rho, B, model=None):
    return instance_json(name, layers, cluster, model or CostModel(), rho, B, 0.05, name)


def main():
    out = {"parity": [], "search": [], "sim": []}

    # operator-level parity: TestBackends.test_parity_bitwise (seed 4321)
    rng = random.Random(4321)
    for trial in range(10):
        layers = varied_instance(rng, rng.randint(3, 6))
        cluster = random_cluster(rng)
        try:
            store = build_store(layers, cluster, CostModel(), imbalance_ratio=math.inf)
            costs = boundary_costs(layers, cluster)
        except Exception:
            continue
        tables = DpTables(store, costs)
        rec = {"instance": inst_of(f"parity{trial}", layers, cluster, math.inf, 8),
               "candidates": []}
        for t in candidate_tmax(store)[::3]:
            F, N, bi, bo = dp_sweep(t, tables.t_tab, tables.mp_tab, tables.ma_tab,
                                    tables.opt_cap, tables.opt_mesh, tables.opt_devs,
                                    tables.opt_off, tables.cb_same, tables.cb_next,
                                    tables.g_mesh, tables.g_avail, tables.s_max,
                                    tables.span_off, tables.span_items)
            rec["candidates"].append({"t_max": t, "F": sha(F), "N": sha(N), "bp_i": sha(bi),
                                      "bp_o": sha(bo)})
        out["parity"].append(rec)

    # search-level: brute force (1234), pruning (99), imbalance (777)
    def add_search(tag, layers, cluster, B, rho, kw_list, model=None):
        try:
            store = build_store(layers, cluster, model or CostModel(), imbalance_ratio=rho)
            costs = boundary_costs(layers, cluster)
        except Exception as e:  # noqa: BLE001
            out["search"].append({"tag": tag, "build_error": type(e).__name__})
            return
        rec = {"tag": tag, "instance": inst_of(tag, layers, cluster, rho, B, model),
               "stats": store.stats.as_dict(), "pool": candidate_tmax(store), "runs": []}
        for kw in kw_list:
            rec["runs"].append({"kw": kw, **search_rec(store, costs, B, **kw)})
        out["search"].append(rec)

    rng = random.Random(1234)
    for trial in range(50):
        layers = varied_instance(rng, rng.randint(3, 6))
        cluster = random_cluster(rng)
        B = rng.randint(4, 16)
        add_search(f"bf1234_{trial}", layers, cluster, B, math.inf, [{"optimized": False}])
    rng = random.Random(99)
    for trial in range(12):
        layers = varied_instance(rng, rng.randint(3, 6))
        cluster = random_cluster(rng)
        B = rng.randint(4, 12)
        add_search(f"prune99_{trial}", layers, cluster, B, math.inf,
                   [{"optimized": False}, {"optimized": True}])
    rng = random.Random(777)
    for trial in range(30):
        layers = varied_instance(rng, rng.randint(3, 6))
        cluster = random_cluster(rng)
        add_search(f"rho777_{trial}", layers, cluster, 8, 3.0, [{"optimized": False}])
    for seed, n, kws in ((20260808, 60, [{"optimized": False}]),
                         (31337, 60, [{"optimized": False},
                                      {"optimized": True, "workers": 2, "batch_size": 3}]),
                         (555, 15, [{}])):
        rng = random.Random(seed)
        for trial in range(n):
            layers, cluster = random_search_instance(rng)
            B = rng.randint(4, 16) if seed != 555 else 8
            add_search(f"acc{seed}_{trial}", layers, cluster, B, math.inf, kws)

    # fixed instances from test_planner.py / test_acceptance.py / test_integration.py
    two = ClusterSpec([DeviceMesh("a", 1, 2, 1e12, 1e12, 1e9, 1e9),
                       DeviceMesh("b", 1, 2, 2e12, 1e12, 1e9, 1e9)], cross_bw=1e9)
    add_search("uniform6_two", uniform_instance(6), two, 8, math.inf,
               [{}, {"batch_size": 1}, {"batch_size": 4, "workers": 2}, {"optimized": False}])
    add_search("forced_split", uniform_instance(4),
               ClusterSpec([DeviceMesh("slow", 1, 1, 1e12, 1e12, 1e9, 1e9),
                            DeviceMesh("fast", 1, 1, 3e12, 1e12, 1e9, 1e9)], cross_bw=1e9),
               8, math.inf, [{}])
    add_search("mem_infeasible", uniform_instance(2, params=100e9),
               ClusterSpec([DeviceMesh("m", 1, 2, 1e12, 60e9, 1e9, 1e9)], cross_bw=1e9),
               4, math.inf, [{}])
    add_search("launch_bound", uniform_instance(8, act=5e8),
               ClusterSpec([DeviceMesh("a", 1, 2, 1e12, 1e12, 1e9, 25e9),
                            DeviceMesh("b", 1, 2, 2e12, 1e12, 1e9, 25e9)], cross_bw=2e9),
               16, math.inf, [{}])
    add_search("mem_bound", uniform_instance(6, params=8e9, act=2e8),
               ClusterSpec([DeviceMesh("m", 2, 2, 1e12, 20e9, 1e9, 10e9)], cross_bw=1e9),
               12, math.inf, [{}])
    layers16 = uniform_instance(16, act=5e7)
    vv = DeviceMesh("v", 1, 2, 125e12, 1e12, 150e9, 25e9)
    aa = DeviceMesh("a", 2, 2, 312e12, 1e12, 300e9, 25e9)
    cl = ClusterSpec([vv, aa], cross_bw=6.25e8)
    add_search("alpha0", layers16, cl, 32, math.inf, [{}], CostModel(alpha=0.0))
    add_search("alpha1", layers16, cl, 32, math.inf, [{}], CostModel(alpha=1.0))
    ops = [OperatorNode(i, HEAVY, 6.25e11, 1.5e9, 2.0 * 512 * 256, "layer") for i in range(128)]
    cs_layers = cluster_layers(detect_modules(ops), ops, 1)
    cs_cluster = ClusterSpec(
        [DeviceMesh("v100", 1, 2, 125e12, 32e9, 150e9, 2.5e10),
         DeviceMesh("a100_h1", 1, 2, 312e12, 40e9, 300e9, 2.5e10),
         DeviceMesh("a100_h2", 1, 2, 312e12, 40e9, 300e9, 2.5e10)],
        cross_bw={("v100", "a100_h1"): 6.25e8, ("v100", "a100_h2"): 6.25e8,
                  ("a100_h1", "a100_h2"): 2.5e10})
    add_search("case_study", cs_layers, cs_cluster, 128, 3.0, [{}])
    ops = [OperatorNode(i, HEAVY, 6.25e11, 6.1e8, 2.0 * 512 * 256, "layer") for i in range(128)]
    bl = cluster_layers(detect_modules(ops), ops, 1)
    add_search("bench_dp128", bl, cs_cluster, 64, math.inf, [{}])
    gops = generate_gpt_sequence(GptConfig(num_blocks=48, hidden_dim=4096, seq_len=1024,
                                           vocab=32000))
    gl = cluster_layers(detect_modules(gops), gops, 3)
    add_search("integration150", gl, cs_cluster, 64, 3.0, [{"workers": 2}])
    for r in (2, 4, 8, 16):
        gops = generate_gpt_sequence(GptConfig(r, 256, 128, vocab=512))
        glr = cluster_layers(detect_modules(gops), gops, 2)
        c2 = ClusterSpec([DeviceMesh("a", 1, 2, 100e12, 1e12, 1e11, 2.5e10),
                          DeviceMesh("b", 1, 2, 300e12, 1e12, 1e11, 2.5e10)], cross_bw=5e9)
        add_search(f"dedup_r{r}", glr, c2, 8, math.inf, [{}])

    # simulator: random plans (classic / eager / adaptive counts)
    rng = random.Random(9)
    for trial in range(40):
        S = rng.randint(1, 6)
        f = [rng.uniform(0.2, 2.0) for _ in range(S)]
        b = [rng.uniform(0.2, 2.0) for _ in range(S)]
        c = [rng.uniform(0.0, 1.5) for _ in range(S - 1)]
        kind = rng.choice(["classic", "eager", "adaptive"])
        if kind == "classic":
            counts = classic_counts(S)
        elif kind == "eager":
            counts = eager_counts(S)
        else:
            try:
                counts = adaptive_counts([x + y for x, y in zip(f, b)], c)
            except Exception:  # noqa: BLE001
                counts = classic_counts(S)
        B = max(counts.counts[0], rng.choice([1, 3, 8, 16, 32]))
        trace = simulate(build_dag(f, b, c, build_program(counts, B)))
        out["sim"].append({"t_fwd": f, "t_bwd": b, "comm": c, "counts": list(counts.counts),
                           "B": B, "makespan": trace.makespan, "start": sha(np.array(trace.start)),
                           "end": sha(np.array(trace.end))})

    with gzip.open(os.path.join(HERE, "seeded.json.gz"), "wt") as fh:
        json.dump(out, fh)
    print({k: len(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
