"""Golden vectors for the plan / trace artifacts.

Runs the unmodified reference (oracle/_ref/meshpipe) on
  * the expected plans of configs A-D3 (tests/golden/instances/*_expected.json)
    plus hand-made variants (colocated boundary, missing optional fields,
    malformed files): plan_from_dict -> plan_report text and plan_to_dict
    round trip, or the PlannerError message;
  * small 1F1B plans: program_to_text, trace_to_text, trace_events and the
    analyze() report text;
and writes tests/golden/artifacts.json.gz.

    python tests/golden/make_golden_artifacts.py
"""

from __future__ import annotations

import copy
import gzip
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))

from meshpipe.planner import PlannerError, plan_from_dict, plan_report, plan_to_dict  # noqa: E402
from meshpipe.scheduling import adaptive_counts, build_program, program_to_text  # noqa: E402
from meshpipe.simulation import (  # noqa: E402
    analyze, build_dag, simulate, trace_events, trace_to_text,
)


def plan_cases():
    cases = []
    for name in ("A", "B", "C", "D1", "D2", "D3"):
        with open(os.path.join(HERE, "instances", f"{name}_expected.json")) as fh:
            cases.append((name, json.load(fh)["plan"]))
    base = cases[0][1]
    v = copy.deepcopy(base)
    if v["boundaries"]:
        v["boundaries"][0]["link"] = "colocated"
    cases.append(("colocated", v))
    v = copy.deepcopy(base)
    for s in v["stages"]:
        for k in ("mem_params", "mem_act", "launch_count", "dp_launch_bound"):
            s.pop(k, None)
    for k in ("t_max", "predicted_latency", "eta_pct", "epsilon", "search_stats"):
        v.pop(k, None)
    cases.append(("minimal", v))
    v = copy.deepcopy(base)
    v["search_stats"]["wall_time_s"] = 1.25
    cases.append(("wall_time", v))
    v = copy.deepcopy(base)
    del v["stages"][0]["mesh"]
    cases.append(("missing_mesh", v))
    v = copy.deepcopy(base)
    v["boundaries"] = v["boundaries"][1:]
    cases.append(("boundary_count", v))
    v = copy.deepcopy(base)
    v["stages"][0]["layers"] = [1]
    cases.append(("short_layers", v))
    return cases


def main() -> None:
    out = {"plans": [], "traces": []}
    for name, d in plan_cases():
        rec = {"name": name, "input": d}
        try:
            p = plan_from_dict(d)
            rec["report"] = plan_report(p)
            rec["to_dict"] = plan_to_dict(p)
        except PlannerError as exc:
            rec["error"] = str(exc)
        out["plans"].append(rec)
    for tf, tb, comm, B in [([0.010, 0.012], [0.020, 0.022], [0.004], 6),
                            ([0.01, 0.02, 0.015], [0.02, 0.03, 0.025], [0.005, 0.0], 8),
                            ([0.004, 0.004, 0.004, 0.004], [0.008] * 4, [0.009, 0.001, 0.002], 12)]:
        lc = adaptive_counts([a + b for a, b in zip(tf, tb)], comm, 0.05)
        prog = build_program(lc, B)
        trace = simulate(build_dag(tf, tb, comm, prog))
        labels = [f"stage-{i + 1} m({i},1)" for i in range(len(tf))]
        out["traces"].append({
            "t_fwd": tf, "t_bwd": tb, "comm": comm, "B": B, "counts": list(lc.counts),
            "program_text": program_to_text(prog), "trace_text": trace_to_text(trace),
            "events": trace_events(trace), "events_labeled": trace_events(trace, labels),
            "labels": labels, "report_text": analyze(trace, [1e9] * len(tf)).to_text()})
    path = os.path.join(HERE, "artifacts.json.gz")
    with gzip.open(path, "wt") as fh:
        json.dump(out, fh)
    print(f"wrote {len(out['plans'])} plans, {len(out['traces'])} traces to {path}")


if __name__ == "__main__":
    main()
