"""Per-rank one-GPU times of an N-rank deal of a pool, for block sizes and
candidates-per-lane choices (balance of the multi-GPU deal).

    python tools/gpu/deal_w8.py D1 8
"""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)


def main(name="D1", W="8"):
    import numpy as np
    import torch

    from paper_2509_24859_b200.planner import DpTables
    from paper_2509_24859_b200.profiling import boundary_costs, build_store
    from paper_2509_24859_b200.workloads import instance

    W = int(W)
    layers, cluster, model, rho, B, eps = instance(name)
    store = build_store(layers, cluster, model, imbalance_ratio=rho)
    tables = DpTables(store, boundary_costs(layers, cluster))
    pool = np.asarray(store.feasible_t_values())
    sw = tables.sweeper

    def timed(tm, cpl, reps=5):
        t = torch.from_numpy(np.ascontiguousarray(tm)).cuda()
        sw.sweep_device(t, cpl=cpl)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            sw.sweep_device(t, cpl=cpl)
        e.record()
        e.synchronize()
        return s.elapsed_time(e) / reps

    def positions(n, r, blk):
        pos = np.arange(n)
        b = pos // blk
        owner = np.where((b // W) % 2 == 0, b % W, W - 1 - b % W)
        return pos[owner == r]

    for blk in (32, 64, 128):
        for cpl in (0, 1, 2):
            per = [timed(pool[positions(len(pool), r, blk)], cpl) for r in range(W)]
            print(f"{name} W={W} blk={blk} cpl={cpl}: " + " ".join(f"{x:.2f}" for x in per)
                  + f"  max {max(per):.3f}", flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
