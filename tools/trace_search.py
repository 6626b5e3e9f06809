"""Batches a search() runs (sizes, device time each) -- where its latency goes.

    python tools/trace_search.py D1 C D3
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(names):
    import torch

    from paper_2509_24859_b200 import engine
    from paper_2509_24859_b200.planner import search
    from paper_2509_24859_b200.profiling import boundary_costs, build_store
    from paper_2509_24859_b200.workloads import instance

    log = []
    orig = engine.Sweeper.evaluate

    def traced(self, tmax_values, B, keep_bp=False, keep_ftop=False, cpl=0):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = orig(self, tmax_values, B, keep_bp=keep_bp, keep_ftop=keep_ftop, cpl=cpl)
        torch.cuda.synchronize()
        log.append((len(tmax_values), keep_bp, (time.perf_counter() - t0) * 1e3, cpl))
        return r

    engine.Sweeper.evaluate = traced
    for name in names:
        layers, cluster, model, rho, B, eps = instance(name)
        for i in range(3):
            log.clear()
            st = build_store(layers, cluster, model, imbalance_ratio=rho)
            c = boundary_costs(layers, cluster)
            torch.cuda.synchronize()
            t = time.perf_counter()
            plan = search(st, c, B, epsilon=eps)
            torch.cuda.synchronize()
            tot = (time.perf_counter() - t) * 1e3
        print(f"{name}: search {tot:.2f} ms; batches " +
              ", ".join(f"{n}{'+bp' if bp else ''}(cpl {c}): {ms:.2f} ms" for n, bp, ms, c in log), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["D1"])
