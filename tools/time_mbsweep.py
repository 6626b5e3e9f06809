"""Config D's four-point microbatch sweep, concurrent vs one size after the
other (sweep.microbatch_sweep):

    python tools/time_mbsweep.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2509_24859_b200.sweep import microbatch_sweep
    from paper_2509_24859_b200.workloads import instance, llama_like_ops

    _, cluster, model, rho, _, eps = instance("D1")
    for conc in (False, True, False, True):
        f = lambda: microbatch_sweep(lambda mb: llama_like_ops(b=mb), cluster, model=model,  # noqa: E731
                                     imbalance_ratio=rho, epsilon=eps, concurrent=conc)
        f()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            t = time.perf_counter()
            f()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t)
        print(f"concurrent={conc}: best {min(ts) * 1e3:.1f} ms, median {sorted(ts)[2] * 1e3:.1f} ms")


if __name__ == "__main__":
    main()
