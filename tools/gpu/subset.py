"""Per-rank share of a full-pool sweep on ONE GPU: times sweep_device on the
candidates rank 0 of W ranks gets (PoolSharding's block deal), plus the
library's per-kind kernel times (relax / window / other, hapt_prof, no PDL).

    python tools/gpu/subset.py D1 1,2,4,8
"""
import ctypes
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def main(name="D1", worlds="1,2,4,8", reps=10):
    import numpy as np
    import torch

    from helpers import build, load_json
    from paper_2509_24859_b200 import _lib
    from paper_2509_24859_b200.distributed import PoolSharding
    from paper_2509_24859_b200.planner import DpTables

    lib = _lib.lib()
    inst = load_json(name)
    store, costs, cluster, B, eps = build(inst)
    tables = DpTables(store, costs)
    pool = np.asarray(store.feasible_t_values())
    sw = tables.sweeper
    for W in [int(x) for x in worlds.split(",")]:
        ps = PoolSharding.__new__(PoolSharding)
        ps.world = W
        if os.environ.get("SUBSET_ALL_RANKS") and W > 1:
            per = []
            for r in range(W):
                t = torch.from_numpy(pool[ps._positions(len(pool), r)]).cuda()
                for _ in range(3):
                    sw.sweep_device(t)
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                for _ in range(reps):
                    sw.sweep_device(t)
                e.record()
                e.synchronize()
                per.append(s.elapsed_time(e) / reps)
            print(f"{name} W={W}: per-rank ms " + " ".join(f"{x:.3f}" for x in per), flush=True)
        pos = ps._positions(len(pool), 0)
        tm = torch.from_numpy(pool[pos]).cuda()
        for _ in range(3):
            sw.sweep_device(tm)
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            sw.sweep_device(tm)
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e))
        ts.sort()
        ms = np.zeros(3)
        cnt = np.zeros(3, dtype=np.int64)
        lib.hapt_prof_enable(1)
        for _ in range(reps):
            sw.sweep_device(tm)
        torch.cuda.synchronize()
        lib.hapt_prof_enable(0)
        lib.hapt_prof_read(ms.ctypes.data_as(ctypes.c_void_p), cnt.ctypes.data_as(ctypes.c_void_p), 3)
        ms /= reps
        cnt = cnt // reps
        print(f"{name} W={W}: {len(pos)} cand  median {ts[len(ts)//2]:.3f} ms  "
              f"[prof, no PDL: relax {ms[0]:.3f} ms/{cnt[0]}  window {ms[1]:.3f} ms/{cnt[1]}  "
              f"other {ms[2]:.3f} ms/{cnt[2]}  sum {ms.sum():.3f}]", flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
