"""search() latency per config (plan = reference's), e.g. to compare
HAPT_SEARCH_DEPTH settings:

    HAPT_SEARCH_DEPTH=6 python tools/time_search.py D1 D3
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(names):
    import torch

    from paper_2509_24859_b200.planner import search
    from paper_2509_24859_b200.profiling import boundary_costs, build_store
    from paper_2509_24859_b200.workloads import instance

    for name in names:
        layers, cluster, model, rho, B, eps = instance(name)
        ts = []
        for i in range(6):
            st = build_store(layers, cluster, model, imbalance_ratio=rho)
            c = boundary_costs(layers, cluster)
            torch.cuda.synchronize()
            t = time.perf_counter()
            plan = search(st, c, B, epsilon=eps)
            ts.append(time.perf_counter() - t)
        print(f"{name}: search {min(ts[1:]) * 1e3:.2f} ms (median {sorted(ts[1:])[2] * 1e3:.2f}), "
              f"evaluated {plan.search_stats['evaluated']} of {plan.search_stats['candidates_total']}")


if __name__ == "__main__":
    main(sys.argv[1:] or ["D1"])
