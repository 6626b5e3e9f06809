"""CPU, world_size 2 over gloo: the candidate sharding of
paper_2509_24859_b200.distributed (strided batches, all_gather of results,
allreduce-argmin) reproduces the single-process answers.  The per-rank DP is
a stand-in sweeper backed by the oracle (no GPU here)."""

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


class OracleSweeper:
    """Sweeper stand-in: evaluate(t_values, B) via the oracle C DP."""

    def __init__(self, inst, tb):
        self.inst, self.tb = inst, tb
        self.calls = []

    BP_BUDGET = 0  # keeps no backpointers (plans are not built here)

    def bp_bytes(self, n):
        return 1

    def evaluate(self, tmax_values, B, keep_bp=False, keep_ftop=False, cpl=0):  # (no lanes on CPU)
        import oracle as O
        from paper_2509_24859_b200.engine import SweepResult

        t = np.asarray(tmax_values, dtype=np.float64)
        self.calls.append(len(t))
        ts, bs, st = O.full_pool(self.inst, self.tb, pool=list(t))
        order = np.lexsort((t, ts))
        winner = int(order[0]) if bs[order[0]] >= 0 else -1
        return SweepResult(t, ts, bs.astype(np.int64), st, winner)


def _worker(rank, world, port, name, out_q, min_shard):
    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))
    sys.path.insert(0, HERE)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch.distributed as dist

    import oracle as O
    from helpers import load_json
    from paper_2509_24859_b200 import planner as P
    from paper_2509_24859_b200.distributed import PoolSharding

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        inst = load_json(name)
        tb = O.tables(inst)
        pool = tb["pool"]
        B = inst["num_microbatches"]
        sh = PoolSharding(min_shard=min_shard)
        sw = OracleSweeper(inst, tb)

        class Tables:
            L, G = tb["L"], tb["G"]
            sweeper = sw

        ev = P.CandidateEvaluator(Tables, pool, B, dist=sh)
        lo, t_e, surv, probed = P.bidirectional_prune_replay(ev, B)
        ev.ensure(surv)
        feas = [i for i in surv if ev.best_s[i] >= 0]
        best = min(feas, key=lambda i: (ev.tstar[i], pool[i]))
        # allreduce-argmin over a rank-local shard of the whole pool
        mine = [int(i) for i in sh.shard_positions(len(pool))]
        res = sw.evaluate([pool[i] for i in mine], B)
        w = res.winner
        g_t, g_i = sh.allreduce_argmin(float(res.tstar[w]) if w >= 0 else float("inf"),
                                       mine[w] if w >= 0 else -1)
        # the device-tensor variant bench.py uses (no host sync; CPU tensors on gloo)
        import torch

        d_bits, d_idx = sh.allreduce_argmin_device(
            torch.from_numpy(np.ascontiguousarray(res.tstar, dtype=np.float64)),
            torch.tensor([w], dtype=torch.int32), torch.tensor(mine, dtype=torch.int64))
        d_t = float(np.array([int(d_bits)], dtype=np.int64).view(np.float64)[0])
        # sweep_pool(dist)'s device-to-device gather of the per-candidate rows
        local = torch.from_numpy(np.stack([np.ascontiguousarray(res.tstar).view(np.int64),
                                           res.best_s, res.states], axis=1))
        full = sh.gather_positions(local, len(pool)).numpy()
        out_q.put((rank, lo, surv, best, float(ev.tstar[best]), g_t, g_i, sum(sw.calls),
                   sh.collective_calls, d_t, int(d_idx), full))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name,min_shard", [("A", 1), ("B", 1), ("B", 10 ** 6)])
def test_two_rank_search_and_argmin(name, min_shard):
    """min_shard=1 shards every batch; 10**6 replicates them all (only the
    full-pool argmin exchanges data)."""
    import oracle as O
    from helpers import expected, expected_arrays, load_json

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q, min_shard))
             for r in range(2)]
    for p in procs:
        p.start()
    results = sorted((q.get(timeout=300) for _ in procs), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    exp = expected(name)
    arr = expected_arrays(name)
    pool = arr["pool"]
    ref_plan = exp["plan"]
    for rank, lo, surv, best, tstar, g_t, g_i, n_eval, n_coll, d_t, d_i, full in results:
        assert np.array_equal(full[:, 0].view(np.float64), arr["tstar"])
        assert np.array_equal(full[:, 1], arr["best_s"])
        assert np.array_equal(full[:, 2], arr["states"])
        assert tstar == ref_plan["predicted_latency"]
        assert pool[best] == ref_plan["t_max"]
        assert lo == ref_plan["search_stats"]["pruned_below_ts"]
        assert len(surv) == ref_plan["search_stats"]["evaluated"]
        feas = np.where(arr["best_s"] >= 0)[0]
        win = feas[np.lexsort((pool[feas], arr["tstar"][feas]))[0]]
        assert (g_t, g_i) == (float(arr["tstar"][win]), int(win))
        assert (d_t, d_i) == (g_t, g_i)
        assert n_coll >= (4 if min_shard == 1 else 3)
    # every pool candidate evaluated exactly once across the two ranks
    assert results[0][7] + results[1][7] >= len(O.tables(load_json(name))["pool"])
    assert results[0][1:7] == results[1][1:7]
