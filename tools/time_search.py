"""Phase breakdown of planner.search() on one config (GPU)."""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main(name):
    import torch

    from paper_2509_24859_b200 import planner as P
    from paper_2509_24859_b200.profiling import boundary_costs, build_store
    from paper_2509_24859_b200.workloads import instance

    layers, cluster, model, rho, B, eps = instance(name)
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        store = build_store(layers, cluster, model, imbalance_ratio=rho)
        costs = boundary_costs(layers, cluster)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        tables = P.DpTables(store, costs)
        pool = P.candidate_tmax(store)
        ev = P.CandidateEvaluator(tables, pool, B)
        lo, t_e, surv, probed = P.bidirectional_prune_replay(ev, B)
        t2 = time.perf_counter()
        nb1 = ev.batches
        ev.ensure(surv)
        t3 = time.perf_counter()
        best = min((i for i in surv if ev.best_s[i] >= 0), key=lambda i: (ev.tstar[i], pool[i]))
        plan = ev.plan(best, eps)
        t4 = time.perf_counter()
        P._activated_pairs(tables, [pool[i] for i in surv])
        tables.transitions_per_sweep()
        t5 = time.perf_counter()
        print(f"{name} rep{rep}: build {1e3*(t1-t0):.2f} ms | prune {1e3*(t2-t1):.2f} ms "
              f"({nb1} batches, {ev.evaluated} cand) | survivors {1e3*(t3-t2):.2f} ms "
              f"({len(surv)}) | backtrack+plan {1e3*(t4-t3):.2f} ms | stats {1e3*(t5-t4):.2f} ms")
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P.search(build_store(layers, cluster, model, imbalance_ratio=rho), boundary_costs(layers, cluster), B, epsilon=eps)
        print(f"{name} search() total {1e3*(time.perf_counter()-t0):.2f} ms")


if __name__ == "__main__":
    for n in sys.argv[1:] or ["D1"]:
        main(n)
