"""Phase breakdown of the bench's e2e path (host inputs -> full-pool result).

    python tools/time_e2e.py [--config D1]
"""
import argparse
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="D1")
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2509_24859_b200 import planner as P
    from paper_2509_24859_b200.profiling import boundary_costs, build_store
    from paper_2509_24859_b200.workloads import instance

    layers, cluster, model, rho, B, eps = instance(args.config)
    for rep in range(6):
        torch.cuda.synchronize()
        t = [time.perf_counter()]
        st = build_store(layers, cluster, model, imbalance_ratio=rho)
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        costs = boundary_costs(layers, cluster)
        t.append(time.perf_counter())
        tables = P.DpTables(st, costs)
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        pool_dev = st.dev.pool()
        ftop, states = tables.sweeper.sweep_device(pool_dev)
        t.append(time.perf_counter())
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        res = P.sweep_pool(st, costs, B)
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        names = ["build_store", "boundary_costs", "DpTables", "sweep enqueue", "sweep wait",
                 "sweep_pool (again)"]
        print(f"{args.config} rep{rep}: " + " | ".join(
            f"{n} {1e3 * (t[i + 1] - t[i]):.2f}" for i, n in enumerate(names)), flush=True)


if __name__ == "__main__":
    main()
