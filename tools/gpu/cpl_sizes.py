"""Device time of a contiguous slice of n pool candidates (from the pool's
middle) at each candidates-per-lane setting: the CPL thresholds of cpl_for.

    python tools/gpu/cpl_sizes.py D1,C,B 16,38,64,128,192,256,448,890
"""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)


def main(configs="D1,C,B", sizes="16,38,64,128,192,256,448,890", cpls="auto,1,2,4"):
    import numpy as np
    import torch

    from paper_2509_24859_b200.planner import DpTables
    from paper_2509_24859_b200.profiling import boundary_costs, build_store
    from paper_2509_24859_b200.workloads import instance

    for cfg in configs.split(","):
        layers, cluster, model, rho, B, eps = instance(cfg)
        store = build_store(layers, cluster, model, imbalance_ratio=rho)
        tables = DpTables(store, boundary_costs(layers, cluster))
        pool = np.asarray(store.feasible_t_values())
        sw = tables.sweeper
        for n in [int(x) for x in sizes.split(",")]:
            if n > len(pool):
                continue
            a = (len(pool) - n) // 2
            tm = torch.from_numpy(pool[a:a + n].copy()).cuda()
            row = []
            for c in cpls.split(","):
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
                row.append(f"{c}: {s.elapsed_time(e) / 5:.3f}")
            os.environ.pop("HAPT_CPL", None)
            print(f"{cfg} n={n:5d}  " + "  ".join(row), flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
