"""Golden vectors for the batched schedule analysis.

Runs the unmodified reference (oracle/_ref/meshpipe) on seeded random 1F1B
plans: launch counts (adaptive / classic / eager), build_program, build_dag,
simulate, analyze(trace, mem_act) and steady_state_rate(trace, 1), and writes
inputs + every report float (as float.hex) to tests/golden/analyze.json.gz.
Covers S = 1..12, B from N_1 (no steady phase) to 96, zero transfer times,
zero-length stages, and traces too short for steady_state_rate.

    python tests/golden/make_golden_analyze.py
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

from meshpipe.scheduling import (  # noqa: E402
    adaptive_counts, build_program, classic_counts, eager_counts,
)
from meshpipe.simulation import (  # noqa: E402
    SimulationError, analyze, build_dag, simulate, steady_state_rate,
)


def plan(rng: random.Random, idx: int) -> dict:
    S = rng.choice([1, 2, 2, 3, 4, 4, 5, 6, 8, 8, 12])
    t = [rng.uniform(0.5, 2.0) * 1e-2 for _ in range(S)]
    share = [rng.uniform(0.25, 0.45) for _ in range(S)]
    tf = [a * b for a, b in zip(t, share)]
    tb = [a - f for a, f in zip(t, tf)]
    tmax = max(a + b for a, b in zip(tf, tb))
    mode = idx % 5
    if mode == 0:
        comm = [0.0] * (S - 1)
    elif mode == 1:  # transfers up to t_max (adaptive δ = 1, 2, 3)
        comm = [rng.uniform(0.0, 1.0) * tmax for _ in range(S - 1)]
    else:
        comm = [rng.choice([0.0, rng.uniform(0.0, 0.6) * tmax]) for _ in range(S - 1)]
    kind = ["adaptive", "classic", "eager"][idx % 3]
    if kind != "adaptive" and idx % 7 == 0:  # zero-length ops (allowed off the adaptive path)
        tf[rng.randrange(S)] = 0.0
        tb[rng.randrange(S)] = 0.0
    if kind == "adaptive":
        lc = adaptive_counts([a + b for a, b in zip(tf, tb)], comm, 0.05)
    elif kind == "classic":
        lc = classic_counts(S)
    else:
        lc = eager_counts(S)
    counts = lc.counts
    n1 = counts[0]
    B = rng.choice([n1, n1 + 1, n1 + 3, 2 * n1 + 5, 32, 64, 96])
    B = max(B, n1)
    mem = [rng.uniform(1e8, 4e9) for _ in range(S)] if idx % 4 else None
    return {"t_fwd": tf, "t_bwd": tb, "comm": comm, "counts": list(counts), "B": B,
            "kind": kind, "mem_act": mem}, lc


def main() -> None:
    rng = random.Random(2509)
    out = []
    for idx in range(400):
        p, lc = plan(rng, idx)
        prog = build_program(lc, p["B"])
        dag = build_dag(p["t_fwd"], p["t_bwd"], p["comm"], prog)
        trace = simulate(dag)
        rep = analyze(trace, p["mem_act"])
        try:
            rate = steady_state_rate(trace, 1).hex()
        except SimulationError:
            rate = None
        p["makespan"] = trace.makespan.hex()
        p["stages"] = [[r.busy.hex(), r.window.hex(), r.bubble.hex(), r.bubble_fraction.hex(),
                        r.steady_bubble.hex(), float(r.peak_inflight_bytes).hex(),
                        r.peak_inflight] for r in rep.stages]
        p["links"] = [[float(l.fwd_time).hex(), float(l.bwd_time).hex(),
                       float(l.overlap_ratio).hex()] for l in rep.links]
        p["steady_rate"] = rate
        out.append(p)
    path = os.path.join(HERE, "analyze.json.gz")
    with gzip.open(path, "wt") as fh:
        json.dump(out, fh)
    print(f"wrote {len(out)} plans to {path}")


if __name__ == "__main__":
    main()
