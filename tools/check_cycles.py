"""Allocated HBM across repeated e2e planning passes with the cyclic GC off:
growth means some object graph is only freed by the GC (a reference cycle)."""
import gc
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    import torch

    from paper_2509_24859_b200.planner import search, sweep_pool
    from paper_2509_24859_b200.profiling import boundary_costs, build_store
    from paper_2509_24859_b200.workloads import instance

    layers, cluster, model, rho, B, eps = instance("D1")
    gc.collect()
    gc.disable()
    for i in range(6):
        st = build_store(layers, cluster, model, imbalance_ratio=rho)
        sweep_pool(st, boundary_costs(layers, cluster), B)
        search(build_store(layers, cluster, model, imbalance_ratio=rho),
               boundary_costs(layers, cluster), B, epsilon=eps)
        del st
        torch.cuda.synchronize()
        print(f"pass {i}: allocated {torch.cuda.memory_allocated() / 1e6:.1f} MB, "
              f"gc-tracked garbage {len(gc.garbage)}")


if __name__ == "__main__":
    main()
