"""Per-layer work of one full-pool sweep from the instrumented build:

    python -m paper_2509_24859_b200.build -DHAPT_COUNT_WORK --out=libv_work.so
    HAPT_LIB=paper_2509_24859_b200/libv_work.so python tools/layer_counts.py D1

prints per layer s: (cell, group) tasks, tasks with no admissible entry,
staged 32-entry chunks, staged entries, entries kept by the lane bound,
entries kept after the probe (executed), tasks with a finite cell.
"""
import ctypes
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main(name="D1"):
    import numpy as np
    import torch

    from paper_2509_24859_b200 import _lib
    from paper_2509_24859_b200.planner import DpTables
    from paper_2509_24859_b200.profiling import boundary_costs, build_store
    from paper_2509_24859_b200.workloads import instance

    lib = _lib.lib()
    lib.hapt_debug_layers.argtypes = [ctypes.c_void_p]
    layers, cluster, model, rho, B, eps = instance(name)
    store = build_store(layers, cluster, model, imbalance_ratio=rho)
    tables = DpTables(store, boundary_costs(layers, cluster))
    pool = np.asarray(store.feasible_t_values())
    a = np.zeros(4096 * 8, dtype=np.uint64)
    lib.hapt_debug_layers(a.ctypes.data)
    tables.sweeper.sweep_device(torch.from_numpy(pool).cuda())
    torch.cuda.synchronize()
    b = np.zeros(4096 * 8, dtype=np.uint64)
    lib.hapt_debug_layers(b.ctypes.data)
    d = (b - a).astype(np.int64).reshape(4096, 8)
    print("s tasks empty chunks staged bound probe finite")
    for s in range(1, tables.s_max + 1):
        if d[s, 0]:
            print(s, *d[s, :7])
    print("total", *d.sum(0)[:7])


if __name__ == "__main__":
    main(*sys.argv[1:])
