"""One small candidate batch swept a few times (driver for ncu launch lists
of the search's unit of work).

    python tools/one_batch.py [--config D1] [--n 38]
"""
import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="D1")
    ap.add_argument("--n", type=int, default=38)
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
    idx = np.linspace(len(pool) // 3, len(pool) - 1, args.n).astype(int)
    tm = torch.from_numpy(pool[idx]).cuda()
    for _ in range(3):
        tables.sweeper.sweep_device(tm)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
