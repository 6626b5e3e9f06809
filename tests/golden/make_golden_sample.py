"""Strided full-pool goldens for the configs whose whole pool is too slow to
sweep on the reference here (D2: 7,019 candidates x ~4 s, D3: 15,925 x
~12 s).  Runs the UNMODIFIED reference (oracle/_ref, Cython backend): for a
strided sample of the t_max pool plus the neighbourhoods of the first
feasible candidate and of the search() winner, per candidate the reference's
own dp_sweep + _extract_plan (planner.py:385-421) -> T* (inf if infeasible),
best stage count, dp_states = isfinite(F[1:]).sum().

    python tests/golden/make_golden_sample.py [--only D2,D3] [--n 320]

Writes tests/golden/instances/<name>_sample.npz (idx, tmax, tstar, best_s,
states).  Build container only; the GPU tests read the committed npz.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as MG  # noqa: E402  (puts oracle/_ref on sys.path)
from meshpipe.planner import DpTables, candidate_tmax  # noqa: E402
from meshpipe.profiling import boundary_costs, build_store  # noqa: E402


def sample_indices(pool, t_win, first_feasible, n):
    P = len(pool)
    idx = {int(i * P / n) for i in range(n)}
    w = int(np.searchsorted(pool, t_win))
    for c in (w, first_feasible):
        idx.update(j for j in range(c - 4, c + 5) if 0 <= j < P)
    idx.add(P - 1)
    return np.array(sorted(idx), dtype=np.int64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="D2,D3")
    ap.add_argument("--n", type=int, default=320)
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    args = ap.parse_args()
    out_dir = os.path.join(HERE, "instances")
    for name in args.only.split(","):
        t0 = time.time()
        layers, cl, model, rho, B, eps, _ = MG.config(name)
        store = build_store(layers, cl, model, imbalance_ratio=rho)
        costs = boundary_costs(layers, cl)
        tables = DpTables(store, costs)
        pool = np.asarray(candidate_tmax(store))
        with open(os.path.join(out_dir, f"{name}_expected.json")) as fh:
            exp = json.load(fh)
        assert np.array_equal(pool, np.load(os.path.join(out_dir, f"{name}_expected.npz"))["pool"])
        t_win = exp["plan"]["t_max"]
        # first feasible candidate: the reference's binary search boundary is
        # not recorded, so locate it with the reference operator itself
        lo, hi = 0, len(pool) - 1
        while lo < hi:
            mid = (lo + hi) // 2
            ts, _, _ = MG.full_pool(tables, [pool[mid]], B, eps, 1)
            if np.isfinite(ts[0]):
                hi = mid
            else:
                lo = mid + 1
        idx = sample_indices(pool, t_win, lo, args.n)
        tstar, best_s, states = MG.full_pool(tables, list(pool[idx]), B, eps, args.workers)
        np.savez_compressed(os.path.join(out_dir, f"{name}_sample.npz"), idx=idx, tmax=pool[idx],
                            tstar=tstar, best_s=best_s, states=states,
                            first_feasible=np.int64(lo))
        print(f"{name}: {len(idx)} candidates, first feasible {lo}, "
              f"{int(np.isfinite(tstar).sum())} feasible, min T* {np.min(tstar)!r} "
              f"({time.time() - t0:.0f} s)", flush=True)


if __name__ == "__main__":
    main()
