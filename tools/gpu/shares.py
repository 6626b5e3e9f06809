"""Device time of every rank's share of a pool (PoolSharding's block deal)
swept alone on this GPU, for W = 2, 4, 8: shows the per-rank balance.

    python tools/gpu/shares.py [--config D1]
"""
import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="D1")
    ap.add_argument("--worlds", default="1,2,4,8")
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2509_24859_b200.distributed import PoolSharding
    from paper_2509_24859_b200.planner import DpTables
    from paper_2509_24859_b200.profiling import boundary_costs, build_store
    from paper_2509_24859_b200.workloads import instance

    layers, cluster, model, rho, B, eps = instance(args.config)
    store = build_store(layers, cluster, model, imbalance_ratio=rho)
    tables = DpTables(store, boundary_costs(layers, cluster))
    pool = np.asarray(store.feasible_t_values())
    sw = tables.sweeper
    for W in [int(w) for w in args.worlds.split(",")]:
        sh = object.__new__(PoolSharding)
        sh.world = W
        row = []
        for r in range(W):
            mine = pool[sh._positions(len(pool), r)]
            tm = torch.from_numpy(mine).cuda()
            for _ in range(2):
                sw.sweep_device(tm)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(5):
                ftop, st = sw.sweep_device(tm)
                sw.select_device(ftop, tm, B)
            e.record()
            e.synchronize()
            row.append(f"{len(mine)}:{s.elapsed_time(e) / 5:.3f}")
        print(f"{args.config} W={W}  " + "  ".join(row), flush=True)


if __name__ == "__main__":
    main()
