"""Quick kernel iteration on the GPU box: full-pool parity of B, C, D1 (and
the D2 sample) against the reference goldens, then full-pool sweep timings.

    python tools/gpu/iter.py [--configs D1,D2,C] [--no-parity]
"""
import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="D1,C,D2")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import numpy as np
    import torch

    from helpers import build, expected_arrays, load_json
    from paper_2509_24859_b200.planner import DpTables, sweep_pool

    if not args.no_parity:
        for name in ("A", "B", "C", "D1", "D2"):
            inst = load_json(name)
            store, costs, cluster, B, eps = build(inst)
            pool, tstar, best_s, states, winner = sweep_pool(store, costs, B)
            if name == "D2":
                smp = np.load(os.path.join(REPO, "tests/golden/instances/D2_sample.npz"))
                i = smp["idx"]
                ok = (np.array_equal(tstar[i], smp["tstar"]) and np.array_equal(best_s[i], smp["best_s"])
                      and np.array_equal(states[i], smp["states"]))
            else:
                arr = expected_arrays(name)
                ok = (np.array_equal(tstar, arr["tstar"]) and np.array_equal(best_s, arr["best_s"])
                      and np.array_equal(states, arr["states"]))
            print(f"parity {name}: {'OK' if ok else 'MISMATCH'}", flush=True)
    for name in args.configs.split(","):
        inst = load_json(name)
        store, costs, cluster, B, eps = build(inst)
        tables = DpTables(store, costs)
        tm = torch.from_numpy(np.asarray(store.feasible_t_values())).cuda()
        sw = tables.sweeper
        for _ in range(2):
            sw.sweep_device(tm)
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            sw.sweep_device(tm)
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e))
        ts.sort()
        print(f"time {name}: pool={len(tm)} median {ts[len(ts)//2]:.3f} ms min {ts[0]:.3f} ms "
              f"-> {len(tm) / ts[len(ts)//2] * 1e3:.0f} cand/s", flush=True)


if __name__ == "__main__":
    main()
