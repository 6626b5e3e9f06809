"""Plan / trace artifacts equal the reference's text and
dicts (goldens: tests/golden/make_golden_artifacts.py, produced by the
unmodified reference).  The plan-file half is host code (CPU); the trace half
needs the simulation kernel (GPU)."""

import gzip
import json
import os

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def golden():
    with gzip.open(os.path.join(HERE, "golden", "artifacts.json.gz"), "rt") as fh:
        return json.load(fh)


def test_plan_files_round_trip_and_report():
    from paper_2509_24859_b200.planner import (
        PlannerError, plan_from_dict, plan_report, plan_to_dict,
    )

    for rec in golden()["plans"]:
        if "error" in rec:
            with pytest.raises(PlannerError) as exc:
                plan_from_dict(rec["input"])
            assert str(exc.value) == rec["error"], rec["name"]
            continue
        plan = plan_from_dict(rec["input"])
        assert plan_report(plan) == rec["report"], rec["name"]
        # JSON round trip of the golden turns tuples into lists; compare likewise
        assert json.loads(json.dumps(plan_to_dict(plan))) == rec["to_dict"], rec["name"]


@pytest.mark.gpu
def test_trace_artifacts():
    from paper_2509_24859_b200.scheduling import adaptive_counts, build_program, program_to_text
    from paper_2509_24859_b200.simulation import (
        analyze, build_dag, simulate, trace_events, trace_to_text,
    )

    for rec in golden()["traces"]:
        tf, tb, comm, B = rec["t_fwd"], rec["t_bwd"], rec["comm"], rec["B"]
        lc = adaptive_counts([a + b for a, b in zip(tf, tb)], comm, 0.05)
        assert list(lc.counts) == rec["counts"]
        prog = build_program(lc, B)
        assert program_to_text(prog) == rec["program_text"]
        trace = simulate(build_dag(tf, tb, comm, prog))
        assert trace_to_text(trace) == rec["trace_text"]
        assert json.loads(json.dumps(trace_events(trace))) == rec["events"]
        assert json.loads(json.dumps(trace_events(trace, rec["labels"]))) == rec["events_labeled"]
        assert analyze(trace, [1e9] * len(tf)).to_text() == rec["report_text"]
