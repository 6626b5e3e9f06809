"""Executed vs admissible DP transitions of one full-pool sweep, from an
instrumented build (every lane-entry of the transition loop counted):

    python -m paper_2509_24859_b200.build -DHAPT_COUNT_WORK --out=libv_work.so
    HAPT_LIB=paper_2509_24859_b200/libv_work.so python tools/work_counts.py D1 C

writes profiles/dp_relax_work.json (read by bench.py).  The counts are a
property of the algorithm (deterministic), not of timing.
"""
import ctypes
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main(names):
    import numpy as np
    import torch

    from paper_2509_24859_b200 import _lib
    from paper_2509_24859_b200.planner import DpTables
    from paper_2509_24859_b200.profiling import boundary_costs, build_store
    from paper_2509_24859_b200.workloads import instance

    lib = _lib.lib()
    lib.hapt_debug_work.argtypes = [ctypes.c_void_p]
    out = {}
    for name in names:
        layers, cluster, model, rho, B, eps = instance(name)
        store = build_store(layers, cluster, model, imbalance_ratio=rho)
        tables = DpTables(store, boundary_costs(layers, cluster))
        pool = np.asarray(store.feasible_t_values())
        before = np.zeros(8, dtype=np.uint64)
        lib.hapt_debug_work(before.ctypes.data)
        tables.sweeper.sweep_device(torch.from_numpy(pool).cuda())
        torch.cuda.synchronize()
        after = np.zeros(8, dtype=np.uint64)
        lib.hapt_debug_work(after.ctypes.data)
        w = (after - before).astype(np.int64)
        ref = tables.transitions_per_sweep() * len(pool)
        out[name] = {"pool_candidates": len(pool), "reference_transitions": int(ref),
                     "executed_lane_transitions": int(w[0]),
                     "admissible_lane_transitions": int(w[1]),
                     "improving_lane_transitions": int(w[2]),
                     "cell_tasks": int(w[4]), "empty_cell_tasks": int(w[5]),
                     "infinite_cell_tasks": int(w[6]), "staged_chunks": int(w[7])}
        print(name, out[name])
    out["source"] = "tools/work_counts.py (HAPT_COUNT_WORK build), one full-pool sweep each"
    dst = "gpurun_out" if os.path.isdir(os.path.join(REPO, "gpurun_out")) else "profiles"
    with open(os.path.join(REPO, dst, "dp_relax_work.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or ["D1"])
