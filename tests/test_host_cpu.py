"""CPU: host-side logic of the planner replica and the input/program types."""

import math
import random

import numpy as np
import pytest

from paper_2509_24859_b200.cluster import ClusterError, ClusterSpec, DeviceMesh, enumerate_submeshes
from paper_2509_24859_b200.planner import (
    InfeasiblePlanError,
    PlannerError,
    _count_batches,
    _probe_tree,
    bidirectional_prune,
    bidirectional_prune_replay,
    end_to_end_latency,
    load_balance_eta,
)
from paper_2509_24859_b200.scheduling import (
    LaunchCounts,
    ScheduleError,
    analytic_delta,
    build_program,
    classic_counts,
    eager_counts,
    program_to_text,
)
from paper_2509_24859_b200.simulation import NODE_B, NODE_CF, NODE_F, SimulationError, build_dag


class FakeEvaluator:
    """CandidateEvaluator stand-in with a scripted feasibility pattern."""

    def __init__(self, feas, tstar, tables=None):
        self.pool = np.arange(1.0, len(feas) + 1.0)
        self.feas = feas
        self.tstar = np.asarray(tstar, dtype=float)
        self.best_s = np.full(len(feas), -2)
        self.tables = tables or type("T", (), {"L": 64, "G": 64})()
        self.batches = []

    def known(self, i):
        return self.best_s[i] != -2

    def ensure(self, idx, keep_bp=True):
        todo = [i for i in idx if not self.known(i)]
        if todo:
            self.batches.append(sorted(todo))
        for i in todo:
            self.best_s[i] = 1 if self.feas[i] else -1

    def feasible(self, i):
        self.ensure([i])
        return self.best_s[i] >= 0


def reference_prune(feas, tstar, B):
    """The reference bidirectional_prune on the same pattern, via the
    reference-signature implementation."""
    pool = [float(i + 1) for i in range(len(feas))]
    calls = []

    class P:
        def __init__(self, i):
            self.predicted_latency = tstar[i]

    def dp(t):
        i = int(t) - 1
        calls.append(i)
        return P(i) if feas[i] else None

    t_s, t_e, surv, cache = bidirectional_prune(pool, dp, B)
    return pool.index(t_s), t_e, [pool.index(t) for t in surv], set(calls)


@pytest.mark.parametrize("seed", range(40))
def test_prune_replay_matches_sequential_binary_search(seed):
    rng = random.Random(seed)
    n = rng.randint(1, 300)
    first = rng.randint(0, n - 1)
    feas = [i >= first for i in range(n)]
    tstar = [rng.uniform(1, 2) * (n - i) for i in range(n)]
    B = rng.choice([1, 2, 8, 64])
    lo, t_e, surv, calls = reference_prune(feas, tstar, B)
    ev = FakeEvaluator(feas, tstar)
    got_lo, got_te, got_surv, probed = bidirectional_prune_replay(ev, B)
    assert (got_lo, got_surv) == (lo, surv)
    assert got_te == t_e or (math.isinf(got_te) and math.isinf(t_e))
    assert set(probed) == calls
    # speculation never needs more than a handful of device batches
    assert len(ev.batches) <= 1 + math.ceil(math.log2(n + 1) / 5) + 1


def test_prune_replay_non_monotone_and_infeasible():
    # lo only moves past an infeasible probe, so the reference's lo-1 check
    # (planner.py:468) re-reads a cached infeasible candidate; replay agrees
    feas = [False, True, False, True, True, True, True, True]
    assert reference_prune(feas, [1.0] * 8, 4)[0] == bidirectional_prune_replay(
        FakeEvaluator(feas, [1.0] * 8), 4)[0]
    with pytest.raises(InfeasiblePlanError):
        bidirectional_prune_replay(FakeEvaluator([False] * 5, [1.0] * 5), 4)


def test_probe_tree_covers_binary_search_paths():
    out = set()
    _probe_tree(0, 99, 3, out)
    assert out == {49, 24, 74, 12, 37, 62, 87}


def test_count_batches_matches_reference_grouping():
    assert _count_batches(list(range(10)), [7] * 10, 4) == 3
    assert _count_batches(list(range(6)), [1, 1, 2, 2, 2, 3], None) == 3
    assert _count_batches(list(range(6)), [1, 1, 2, 2, 2, 3], 2) == 4
    assert _count_batches(list(range(6)), None, None) == 1


def test_closed_forms():
    assert end_to_end_latency([2.0], [], 10) == 20.0
    with pytest.raises(PlannerError):
        end_to_end_latency([1.0, 1.0], [1.5], 4)
    assert load_balance_eta([2, 2], [1, 1]) == 100.0
    assert load_balance_eta([2, 1], [1, 1]) == pytest.approx(75.0)
    with pytest.raises(PlannerError):
        load_balance_eta([0, 0], [1, 1])


def test_submesh_order_and_cluster_checks():
    m = DeviceMesh("a", 4, 8, 1e12, 1e9, 1e9, 1e9)
    shapes = [s.shape for s in enumerate_submeshes(m)]
    assert shapes == [(1, 1), (1, 2), (1, 4), (1, 8), (2, 8), (3, 8), (4, 8)]
    with pytest.raises(ClusterError):
        DeviceMesh("b", 1, 3, 1e12, 1e9, 1e9, 1e9)
    cl = ClusterSpec([m, DeviceMesh("c", 1, 2, 1e12, 1e9, 1e9, 1e9)], cross_bw={("c", "a"): 5.0})
    assert cl.cross_bandwidth("a", "c") == 5.0 and cl.mesh_order("c") == 1


def test_launch_counts_and_programs():
    assert classic_counts(3).counts == (3, 2, 1)
    assert eager_counts(3).counts == (5, 3, 1)
    with pytest.raises(ScheduleError):
        LaunchCounts((2, 2), (0,), "classic")
    prog = build_program(LaunchCounts((3, 1), (2,), "adaptive"), 5)
    assert prog.stages[0].ops[:5] == (("F", 1), ("F", 2), ("F", 3), ("B", 1), ("F", 4))
    assert "stage 1 (N=3): F1 F2 F3 | B1 F4 B2 F5 | B3 B4 B5" in program_to_text(prog)
    with pytest.raises(ScheduleError):
        build_program(eager_counts(3), 4)
    assert analytic_delta(1.0, 2.0) == 2


def test_dag_structure_lazy_edges():
    prog = build_program(classic_counts(2), 3)
    dag = build_dag([1, 1], [1, 1], [0.2], prog)
    assert not dag.edges_materialised
    assert dag.num_nodes == 3 * (2 * 2 + 2 * 1) + 1
    c1, c2 = dag.node_id(NODE_CF, 1, 1), dag.node_id(NODE_CF, 2, 1)
    assert c2 in dag.succ[c1]
    f, b = dag.node_id(NODE_F, 1, 1), dag.node_id(NODE_B, 3, 1)
    assert dag.sink in dag.succ[b]
    assert dag.node_name(f) == "F[1,1]"
    with pytest.raises(SimulationError):
        build_dag([1.0], [1.0], [0.1], build_program(classic_counts(1), 2))


@pytest.mark.parametrize("n,W", [(1786, 2), (1786, 4), (15925, 4), (124, 2), (7019, 8)])
def test_pool_deal_blocks(n, W):
    """PoolSharding's deal: every candidate on exactly one rank, in contiguous
    group-aligned blocks (64 or 128), equal block counts +-1."""
    import numpy as np

    from paper_2509_24859_b200.distributed import PoolSharding

    sh = object.__new__(PoolSharding)
    sh.world = W
    parts = [sh._positions(n, r) for r in range(W)]
    allp = np.sort(np.concatenate(parts))
    assert np.array_equal(allp, np.arange(n))
    blk = 128 if n >= 1024 * W else 64
    for p in parts:
        blocks = set(int(x) // blk for x in p)
        for b in blocks:  # whole blocks only
            lo, hi = b * blk, min(n, (b + 1) * blk)
            assert np.isin(np.arange(lo, hi), p).all()
    counts = [len(set(int(x) // blk for x in p)) for p in parts]
    assert max(counts) - min(counts) <= 1
