"""One-GPU time of every 64-candidate block of a pool swept alone, and of
each rank's share under PoolSharding's deal: how balanced the multi-GPU
deal is.

    python tools/gpu/block_costs.py D1 8
"""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)


def main(name="D1", W="8", blk="64"):
    import numpy as np
    import torch

    from paper_2509_24859_b200.distributed import PoolSharding
    from paper_2509_24859_b200.planner import DpTables
    from paper_2509_24859_b200.profiling import boundary_costs, build_store
    from paper_2509_24859_b200.workloads import instance

    W, blk = int(W), int(blk)
    layers, cluster, model, rho, B, eps = instance(name)
    store = build_store(layers, cluster, model, imbalance_ratio=rho)
    tables = DpTables(store, boundary_costs(layers, cluster))
    pool = np.asarray(store.feasible_t_values())
    sw = tables.sweeper

    def timed(tm, reps=5):
        t = torch.from_numpy(np.ascontiguousarray(tm)).cuda()
        sw.sweep_device(t)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            sw.sweep_device(t)
        e.record()
        e.synchronize()
        return s.elapsed_time(e) / reps

    nb = (len(pool) + blk - 1) // blk
    costs = [timed(pool[b * blk:(b + 1) * blk]) for b in range(nb)]
    print(f"{name}: {nb} blocks of {blk}: " + " ".join(f"{c:.2f}" for c in costs), flush=True)
    ps = PoolSharding.__new__(PoolSharding)
    ps.world = W
    per = [timed(pool[ps._positions(len(pool), r)]) for r in range(W)]
    print(f"  deal W={W}: per-rank ms " + " ".join(f"{x:.3f}" for x in per) + f"  max {max(per):.3f}")


if __name__ == "__main__":
    main(*sys.argv[1:])
