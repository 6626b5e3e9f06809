"""One full-pool DP sweep of a config (driver for ncu captures of dp_relax).

    python tools/profile_dp.py [--config D1] [--repeat 1]
"""
import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="D1")
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--time", type=int, default=0, help="timed sweeps after warm-up")
    ap.add_argument("--ws-mb", type=int, default=0, help="cap the DP workspace (MB) -> chunking")
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2509_24859_b200.planner import DpTables
    from paper_2509_24859_b200.profiling import boundary_costs, build_store
    from paper_2509_24859_b200.workloads import instance

    layers, cluster, model, rho, B, eps = instance(args.config)
    store = build_store(layers, cluster, model, imbalance_ratio=rho)
    tables = DpTables(store, boundary_costs(layers, cluster))
    if args.ws_mb:
        tables.sweeper.max_ws_bytes = args.ws_mb << 20
    tmax = torch.from_numpy(np.asarray(store.feasible_t_values())).cuda()
    for _ in range(args.repeat):
        ftop, states = tables.sweeper.sweep_device(tmax)
    torch.cuda.synchronize()
    if args.time:
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.time):
            ftop, states = tables.sweeper.sweep_device(tmax)
        e.record()
        e.synchronize()
        ms = s.elapsed_time(e) / args.time
        trans = tables.transitions_per_sweep()
        print(f"{args.config} lib={os.environ.get('HAPT_LIB', 'default')} pool={len(tmax)} "
              f"sweep={ms:.3f} ms  cand/s={len(tmax) / ms * 1e3:.0f}  "
              f"transitions/s={trans * len(tmax) / ms * 1e3:.3e}")
    print("ok", int(states.sum()))


if __name__ == "__main__":
    main()
