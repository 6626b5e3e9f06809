"""GPU: K3 launch counts and 1F1B simulation, bit-exact against the
reference's simulate(build_dag(...)) goldens and the oracle's explicit-DAG
Kahn sweep."""

import hashlib
import math
import random

import numpy as np
import pytest

import oracle as O
from helpers import seeded

pytestmark = pytest.mark.gpu


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_simulate_equals_reference_goldens():
    from paper_2509_24859_b200.scheduling import LaunchCounts, build_program
    from paper_2509_24859_b200.simulation import build_dag, simulate

    for rec in seeded()["sim"]:
        c = rec["counts"]
        counts = LaunchCounts(tuple(c), tuple(c[i] - c[i + 1] for i in range(len(c) - 1)), "x")
        trace = simulate(build_dag(rec["t_fwd"], rec["t_bwd"], rec["comm"],
                                   build_program(counts, rec["B"])))
        assert trace.makespan == rec["makespan"]
        assert sha(np.array(trace.start)) == rec["start"]
        assert sha(np.array(trace.end)) == rec["end"]


def test_general_dag_path_and_cycle_error():
    from paper_2509_24859_b200.scheduling import build_program, classic_counts
    from paper_2509_24859_b200.simulation import NODE_B, NODE_F, CycleError, build_dag, simulate

    prog = build_program(classic_counts(2), 8)
    dag = build_dag([1, 1], [1, 1], [0.0], prog)
    fast = simulate(dag)
    _ = dag.succ  # materialised edges -> generic frontier kernel
    slow = simulate(dag)
    assert fast.start == slow.start and fast.makespan == slow.makespan == 18.0
    dag2 = build_dag([1, 1], [1, 1], [0.1], build_program(classic_counts(2), 2))
    f, b = dag2.node_id(NODE_F, 1, 1), dag2.node_id(NODE_B, 2, 1)
    dag2.succ[b].append(f)
    dag2.pred[f].append(b)
    with pytest.raises(CycleError) as err:
        simulate(dag2)
    assert "F[1,1]" in str(err.value)


def test_round_trip_and_lemma_values():
    from paper_2509_24859_b200.scheduling import LaunchCounts, build_program
    from paper_2509_24859_b200.simulation import NODE_B, NODE_F, build_dag, simulate

    trace = simulate(build_dag([1.0, 1.0], [1.0, 1.0], [0.5],
                               build_program(LaunchCounts((1, 1), (0,), "classic"), 1)))
    assert trace.makespan == 1 + 0.5 + 1 + 1 + 0.5 + 1
    # acceptance 01 of the reference: steady gap max{Kf+(K-1)b, 2f+b+2c}
    for K in range(1, 6):
        for c in (0.0, 0.3, 1.0):
            tr = simulate(build_dag([1.0, 1.0], [2.0, 2.0], [c],
                                    build_program(LaunchCounts((K, 1), (K - 1,), "a"), 32)))
            gap = tr.node_interval(NODE_B, 16, 1)[0] - tr.node_interval(NODE_F, 16, 1)[0]
            assert math.isclose(gap, max(K * 1 + (K - 1) * 2, 2 + 2 + 2 * c), rel_tol=1e-12)


def test_simulate_batch_config_e_equals_oracle():
    """Config E sample: adaptive counts + makespan for ragged plans in one
    launch each, compared with the oracle's explicit DAG per plan."""
    from paper_2509_24859_b200.scheduling import launch_counts_batch
    from paper_2509_24859_b200.simulation import simulate_batch
    from paper_2509_24859_b200.workloads import config_e

    f, b, c, S = config_e(3000)
    of, ob, oc, oS = O.config_e_plans(3000)
    assert np.array_equal(f, of) and np.array_equal(c, oc) and np.array_equal(S, oS)
    counts, status = launch_counts_batch(f, b, c, epsilon=0.05, kind="adaptive", stage_counts=S)
    assert (status == 0).all()
    dense = np.zeros((3000, 8), dtype=np.int32)
    off = np.concatenate([[0], np.cumsum(S)])
    for p in range(3000):
        dense[p, : S[p]] = counts[off[p]: off[p + 1]]
    mk, st = simulate_batch(f, b, c, dense, 128, stage_counts=S)
    mk = mk.cpu().numpy()
    assert (st.cpu().numpy() == 0).all()
    for p in range(0, 3000, 7):
        s = int(S[p])
        oc_ = O.adaptive_counts(list(f[p, :s] + b[p, :s]), list(c[p, : s - 1]), 0.05)
        assert list(dense[p, :s]) == oc_
        want, _, _ = O.simulate(f[p, :s], b[p, :s], c[p, : s - 1], oc_, 128)
        assert mk[p] == want, p


@pytest.mark.parametrize("B", [4, 17, 64])
def test_simulate_batch_many_stages_equals_oracle(B):
    """7- and 8-stage plans (one lane per stage, k_sim_l) and 5-6-stage ones
    (k_sim_s), with non-increasing launch counts from B down to 1 --
    including steps between neighbouring stages deeper than the transfer
    FIFOs, which hand the plan to the generic kernel -- against the
    oracle's explicit DAG."""
    from paper_2509_24859_b200.simulation import simulate_batch

    rng = np.random.default_rng(1000 + B)
    P = 600
    S = rng.choice(np.array([5, 6, 7, 8]), size=P).astype(np.int32)
    f = rng.uniform(0.5, 2.0, size=(P, 8)) * 1e-2
    b = f * rng.uniform(1.5, 2.5, size=(P, 8))
    c = rng.uniform(0.0, 1e-2, size=(P, 8))
    dense = np.zeros((P, 8), dtype=np.int32)
    for p in range(P):
        s_ = int(S[p])
        n = np.sort(rng.integers(1, B + 1, size=s_))[::-1].copy()  # non-increasing
        if p % 3 == 0:  # the reference's small steps (delta in 1..3)
            n = 1 + np.concatenate([np.cumsum(rng.integers(1, 4, size=s_ - 1)[::-1])[::-1], [0]])
            n = np.minimum(n, B)
        n[-1] = 1
        dense[p, :s_] = n
        f[p, s_:] = b[p, s_:] = 0.0
        c[p, s_ - 1:] = 0.0
    mk, st = simulate_batch(f, b, c, dense, B, stage_counts=S)
    mk, st = mk.cpu().numpy(), st.cpu().numpy()
    assert (st == 0).all()
    for p in range(P):
        s_ = int(S[p])
        want, _, _ = O.simulate(f[p, :s_], b[p, :s_], c[p, : s_ - 1], list(dense[p, :s_]), B)
        assert mk[p] == want, (p, s_, list(dense[p, :s_]))


def test_launch_counts_kinds_and_errors():
    from paper_2509_24859_b200.scheduling import (CommTooLargeError, ScheduleError,
                                                  adaptive_counts, launch_counts_batch)

    assert adaptive_counts([2.0, 2.0, 2.0], [1.5, 0.05]).counts == (5, 2, 1)
    assert adaptive_counts([1.0, 1.0], [0.0]).counts == (2, 1)
    with pytest.raises(CommTooLargeError):
        adaptive_counts([1.0, 1.0], [1.5])
    with pytest.raises(ScheduleError):
        adaptive_counts([1.0, 1.0], [0.5], t_max=0.5)
    assert adaptive_counts([1.0, 2.0], [1.5], t_max=3.0).deltas == (2,)
    assert adaptive_counts([1.0, 2.0], [1.6], t_max=3.0).deltas == (3,)
    rng = random.Random(7)
    P, S = 200, 5
    t = np.array([[rng.uniform(0.5, 2) for _ in range(S)] for _ in range(P)])
    c = np.array([[rng.uniform(0, 2.5) for _ in range(S)] for _ in range(P)])
    counts, status = launch_counts_batch(t, np.zeros_like(t), c, kind="adaptive")
    for p in range(P):
        try:
            want = O.adaptive_counts(list(t[p]), list(c[p, : S - 1]), 0.05)
            assert status[p] == 0 and list(counts[p]) == want
        except ValueError:
            assert status[p] == 4  # HAPT_ECOMM
    cl, _ = launch_counts_batch(t, np.zeros_like(t), c, kind="classic")
    assert (cl[:, 0] == S).all()
    eg, _ = launch_counts_batch(t, np.zeros_like(t), c, kind="eager")
    assert (eg[:, 0] == 2 * S - 1).all()


def test_config_e_benchmark_scale_equals_oracle():
    """The bench's config E workload at full size: all 10^6 plans through
    the same PlanBatch.counts + PlanBatch.simulate calls bench.py times
    (adaptive counts, B = 128), every launch count and every makespan
    compared bit for bit with the oracle's explicit-DAG Kahn simulator
    (oracle_config_e_batch: adaptive_counts + build_dag + simulate per plan)."""
    import torch

    from paper_2509_24859_b200.simulation import PlanBatch
    from paper_2509_24859_b200.workloads import config_e

    n = 1_000_000
    f, b, c, S = config_e(n)
    batch = PlanBatch(f, b, c, stage_counts=S, device=torch.device("cuda", 0))
    counts, status = batch.counts(0.05, "adaptive")
    mk, st = batch.simulate(counts, 128, ring_depth=3 * 8 + 2)
    assert (status == 0).all().item() and (st == 0).all().item()
    ocounts, ostatus, omk = O.config_e_batch(f, b, c, S, B=128, epsilon=0.05)
    assert (ostatus == 0).all()
    dense = np.zeros((n, 8), dtype=np.int32)
    mask = np.arange(8)[None, :] < S[:, None]
    dense[mask] = counts.cpu().numpy()
    assert np.array_equal(dense, ocounts)
    got = mk.cpu().numpy()
    bad = np.flatnonzero(got != omk)
    assert bad.size == 0, (bad[:10], got[bad[:10]], omk[bad[:10]])
