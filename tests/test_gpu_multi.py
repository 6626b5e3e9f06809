"""GPU, 2 ranks over NCCL (skipped on a 1-GPU box): search(dist=PoolSharding)
and sweep_pool(dist=...) shard the candidate pool across GPUs and still return
the reference's plan / full-pool results (goldens)."""

import os
import socket
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, names, out_q):
    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, HERE)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import numpy as np
    import torch
    import torch.distributed as dist

    from helpers import assert_plan_equal, build, expected, expected_arrays, load_json, plan_dict
    from paper_2509_24859_b200.distributed import PoolSharding
    from paper_2509_24859_b200.planner import search, search_batches, sweep_pool

    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    errors = []
    try:
        sh = PoolSharding()
        for name in names:
            inst = load_json(name)
            store, costs, cluster, B, eps = build(inst)
            try:
                plan = search(store, costs, B, epsilon=eps, batch_size=4, dist=sh)
                assert_plan_equal(plan_dict(plan), expected(name)["plan"])
                pool, tstar, best_s, states, winner = sweep_pool(store, costs, B, dist=sh)
                arr = expected_arrays(name)
                feas = np.where(arr["best_s"] >= 0)[0]
                want = int(feas[np.lexsort((arr["pool"][feas], arr["tstar"][feas]))[0]])
                assert winner == want, (winner, want)
                # sharded microbatch-count sweep == per-B sharded search
                many = search_batches(store, costs, [B, 2 * B], epsilon=eps, batch_size=4,
                                      dist=sh)
                assert_plan_equal(plan_dict(many[B]), expected(name)["plan"])
                one = search(store, costs, 2 * B, epsilon=eps, batch_size=4, dist=sh)
                assert_plan_equal(plan_dict(many[2 * B]), plan_dict(one))
            except AssertionError as exc:
                errors.append(f"{name}: {exc}")
    finally:
        dist.destroy_process_group()
    out_q.put((rank, errors))


def test_two_rank_search_and_pool_equal_reference():
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    names = ["A", "C", "D1"]
    procs = [ctx.Process(target=_worker, args=(r, 2, port, names, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, errors in results:
        assert not errors, (rank, errors)
