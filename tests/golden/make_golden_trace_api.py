"""Golden vectors for the single-trace API (simulation.py:374-424):
steady_state_rate(trace, stage) at EVERY stage, steady_block_span(trace,
stage, i) and asap_tight(trace) -- the latter also on traces with one node's
start moved (inside and outside the isclose tolerance).  Runs the
unmodified reference (oracle/_ref) on the first 160 plans of
tests/golden/analyze.json.gz and writes tests/golden/trace_api.json.gz.

    python tests/golden/make_golden_trace_api.py
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))

from meshpipe.scheduling import LaunchCounts, build_program  # noqa: E402
from meshpipe.simulation import (  # noqa: E402
    ScheduleTrace, SimulationError, asap_tight, build_dag, simulate, steady_block_span,
    steady_state_rate,
)


def main() -> None:
    with gzip.open(os.path.join(HERE, "analyze.json.gz"), "rt") as fh:
        plans = json.load(fh)[:160]
    rng = random.Random(424)
    out = []
    for p in plans:
        S = len(p["t_fwd"])
        deltas = tuple(p["counts"][s] - p["counts"][s + 1] for s in range(S - 1))
        lc = LaunchCounts(tuple(p["counts"]), deltas, "golden")
        trace = simulate(build_dag(p["t_fwd"], p["t_bwd"], p["comm"], build_program(lc, p["B"])))
        rates, spans = [], []
        for s in range(1, S + 1):
            try:
                rates.append(steady_state_rate(trace, s).hex())
            except SimulationError:
                rates.append(None)
            K = p["counts"][s - 1]
            i = min(2 * K + 1, p["B"] - K)
            spans.append([i, steady_block_span(trace, s, i).hex()] if i >= 1 else None)
        rec = {"rates": rates, "spans": spans, "tight": asap_tight(trace), "moved": []}
        n = trace.dag.num_nodes
        for scale in (1e-13, 1e-6):
            v = rng.randrange(n - 1)
            start = list(trace.start)
            start[v] = start[v] * (1.0 + scale) + (scale if start[v] == 0.0 else 0.0)
            moved = ScheduleTrace(trace.dag, start, trace.end, trace.makespan)
            rec["moved"].append([v, start[v].hex(), asap_tight(moved)])
        out.append(rec)
    path = os.path.join(HERE, "trace_api.json.gz")
    with gzip.open(path, "wt") as fh:
        json.dump(out, fh)
    print(f"wrote {len(out)} traces to {path}")


if __name__ == "__main__":
    main()
