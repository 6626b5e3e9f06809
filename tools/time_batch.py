"""Device time vs wall time of one candidate batch (the search's unit of work).

    python tools/time_batch.py [--config D1] [--sizes 1,38,117,256]
    python tools/time_batch.py --shards 1,2,4,8   # rank 0's share pool[0::W]
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
    ap.add_argument("--sizes", default="1,38,117,256")
    ap.add_argument("--shards", default="", help="time pool[0::W] for each W instead")
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
    if args.shards:
        batches = [np.arange(0, len(pool), int(w)) for w in args.shards.split(",")]
    else:
        batches = [np.linspace(len(pool) // 3, len(pool) - 1, int(n)).astype(int)
                   for n in args.sizes.split(",")]
    for idx in batches:
        n = len(idx)
        tm = torch.from_numpy(pool[idx]).cuda()
        for _ in range(3):
            sw.sweep_device(tm)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        t0 = time.perf_counter()
        s.record()
        for _ in range(reps):
            sw.sweep_device(tm)
        e.record()
        e.synchronize()
        wall = (time.perf_counter() - t0) / reps
        dev = s.elapsed_time(e) * 1e-3 / reps
        t0 = time.perf_counter()
        for _ in range(reps):
            sw.evaluate(pool[idx], B, keep_bp=True)
        ev = (time.perf_counter() - t0) / reps
        print(f"{args.config} n={n:5d}: sweep device {dev * 1e3:7.3f} ms  wall {wall * 1e3:7.3f} ms"
              f"  evaluate(keep_bp) {ev * 1e3:7.3f} ms")


if __name__ == "__main__":
    main()
