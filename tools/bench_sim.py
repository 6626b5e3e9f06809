"""Config E timing: adaptive launch counts + 1F1B makespans for N synthetic
plans (device-resident inputs), plus a parity spot check against the oracle.

    python tools/bench_sim.py [--plans 1000000] [--check 2000]
"""
import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--plans", type=int, default=1_000_000)
    ap.add_argument("--check", type=int, default=2000)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2509_24859_b200.simulation import PlanBatch
    from paper_2509_24859_b200.workloads import config_e

    n = args.plans
    f, b, c, S = config_e(n)
    dev = torch.device("cuda", 0)
    batch = PlanBatch(f, b, c, stage_counts=S, device=dev)
    off = np.concatenate([[0], np.cumsum(S)])

    def step():
        counts, status = batch.counts(0.05, "adaptive")
        step.counts = counts
        return batch.simulate(counts, 128, ring_depth=26)

    for _ in range(2):
        mk, st = step()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.reps):
        mk, st = step()
    e.record()
    e.synchronize()
    dt = s.elapsed_time(e) / args.reps * 1e-3
    print(f"config E: {n} plans in {dt * 1e3:.2f} ms -> {n / dt:.3e} plans/s; "
          f"status ok: {bool((st == 0).all())}")
    if args.check:
        import oracle as O

        mkh = mk.cpu().numpy()
        ch = step.counts.cpu().numpy()
        bad = 0
        for p in range(0, n, max(1, n // args.check)):
            s_ = int(S[p])
            cnt = list(ch[off[p]: off[p + 1]])
            assert cnt == O.adaptive_counts(list(f[p, :s_] + b[p, :s_]), list(c[p, : s_ - 1]), 0.05)
            want, _, _ = O.simulate(f[p, :s_], b[p, :s_], c[p, : s_ - 1], cnt, 128)
            bad += mkh[p] != want
        print(f"parity: {args.check} sampled plans, {bad} mismatches")


if __name__ == "__main__":
    main()
