"""GPU: shapes the benchmark configs never reach, against the oracle (which is
pinned to the reference on the goldens): meshes with more than 32 submesh
options (the kernels' 32-option chunks), one-device meshes, many layers with
few devices, a single layer, and alpha > 0 (the activation-transfer term)."""

import random

import numpy as np
import pytest

import oracle as O
from helpers import build

pytestmark = pytest.mark.gpu


def instance(seed, L, meshes, B=16, rho=3.0, alpha=0.0, rep_every=0):
    rng = random.Random(seed)
    flops = [rng.uniform(0.5, 4.0) * 1e12 for _ in range(L)]
    params = [rng.uniform(1, 8) * 1e8 for _ in range(L)]
    bb = [rng.uniform(1, 8) * 1e7 for _ in range(L)]
    if rep_every:  # repeated structure: equal signatures and aggregates
        for i in range(L):
            j = i % rep_every
            flops[i], params[i], bb[i] = flops[j], params[j], bb[j]
    sig = [i % rep_every if rep_every else i for i in range(L)]
    cluster_meshes = []
    for k, (hosts, dph) in enumerate(meshes):
        cluster_meshes.append({
            "id": f"m{k}", "hosts": hosts, "devices_per_host": dph,
            "peak_flops": rng.choice([312e12, 125e12, 65e12]),
            "mem_device": rng.choice([16e9, 40e9, 80e9]),
            "intra_host_bw": 300e9, "inter_host_bw": rng.choice([12.5e9, 25e9])})
    return {
        "name": f"edge{seed}",
        "layers": {"flops": flops, "param_bytes": params, "boundary_bytes": bb, "sig": sig,
                   "signature": [["rep", s, 0] if rep_every else ["solo", s, 0] for s in sig]},
        "cluster": {"meshes": cluster_meshes, "cross_bw": 3.125e9, "cross_latency": 1e-4},
        "model": {"beta": 2.0, "efficiency": 0.5, "alpha": alpha, "replication": 1.0,
                  "act_factor": 2.0},
        "imbalance_ratio": rho, "dedup": True, "num_microbatches": B, "epsilon": 0.05,
    }


CASES = [
    # (seed, L, meshes [(hosts, devices_per_host)], kwargs)
    (1, 20, [(40, 1), (3, 2)], {}),           # 40 + 3 options: two 32-option chunks
    (2, 24, [(36, 2), (1, 8)], {"rep_every": 4}),
    (3, 60, [(2, 2), (1, 2)], {}),            # many layers, 6 devices
    (4, 1, [(1, 4), (2, 4)], {}),             # a single layer
    (5, 16, [(1, 1), (1, 1), (1, 1)], {}),    # three one-device meshes
    (6, 18, [(4, 8), (8, 4)], {"alpha": 1.0, "rho": 1e9}),
]


@pytest.mark.parametrize("seed,L,meshes,kw", CASES)
def test_edge_pool_equals_oracle(seed, L, meshes, kw):
    from paper_2509_24859_b200.planner import InfeasiblePlanError, search, sweep_pool

    inst = instance(seed, L, meshes, **kw)
    store, costs, cluster, B, eps = build(inst)
    tb = O.tables(inst)
    if not tb["pool"]:
        pytest.skip("no feasible candidate on this draw")
    pool, tstar, best_s, states, winner = sweep_pool(store, costs, B)
    assert list(pool) == tb["pool"]
    rng = np.random.default_rng(seed)
    idx = sorted(set(rng.choice(len(pool), size=min(len(pool), 40), replace=False).tolist())
                 | {0, len(pool) - 1})
    ref = O.full_pool(inst, tb, pool=[tb["pool"][i] for i in idx])
    for k, i in enumerate(idx):
        tot, s, st = ref[0][k], ref[1][k], ref[2][k]
        assert best_s[i] == s, (i, best_s[i], s)
        assert states[i] == st, (i, states[i], st)
        if s >= 0:
            assert tstar[i] == tot, (i, tstar[i], tot)
    # the search driver agrees with the oracle's restatement of search()
    try:
        plan = search(store, costs, B, epsilon=eps)
    except InfeasiblePlanError:
        with pytest.raises(Exception):
            O.search(inst)
        return
    want = O.search(inst)
    assert plan.t_max == want["t_max"] and plan.predicted_latency == want["predicted_latency"]
    assert [(s.layer_start, s.layer_end) for s in plan.stages] == \
        [tuple(x["layers"]) for x in want["stages"]]
