"""Device time of rank 0's share (blocks of 128 dealt round-robin) of a pool
for W in 1,2,4,8, at each candidates-per-lane setting.

    python tools/gpu/cpl.py [--config D1] [--cpl auto,1,2,4]
"""
import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="D1")
    ap.add_argument("--cpl", default="auto,1,2,4")
    ap.add_argument("--worlds", default="1,2,4,8")
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2509_24859_b200.planner import DpTables
    from paper_2509_24859_b200.profiling import boundary_costs, build_store
    from paper_2509_24859_b200.workloads import instance

    layers, cluster, model, rho, B, eps = instance(args.config)
    store = build_store(layers, cluster, model, imbalance_ratio=rho)
    tables = DpTables(store, boundary_costs(layers, cluster))
    pool = np.asarray(store.feasible_t_values())
    sw = tables.sweeper
    for W in [int(w) for w in args.worlds.split(",")]:
        blk = 128 if len(pool) >= 1024 * W else 64
        b = np.arange(len(pool)) // blk
        owner = np.where((b // W) % 2 == 0, b % W, W - 1 - b % W)
        mine = pool[owner == W - 1]  # the rank with the heaviest first block
        tm = torch.from_numpy(mine).cuda()
        row = []
        for c in args.cpl.split(","):
            if c == "auto":
                os.environ.pop("HAPT_CPL", None)
            else:
                os.environ["HAPT_CPL"] = c
            for _ in range(2):
                sw.sweep_device(tm)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(5):
                sw.sweep_device(tm)
            e.record()
            e.synchronize()
            row.append(f"cpl {c}: {s.elapsed_time(e) / 5:.3f} ms")
        print(f"{args.config} W={W} n={len(mine)}  " + "  ".join(row), flush=True)


if __name__ == "__main__":
    main()
