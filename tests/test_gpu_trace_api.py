"""GPU: the single-trace API of meshpipe.simulation (simulation.py:310-424)
-- analyze(trace, mem_act), steady_state_rate(trace, stage) at every stage,
steady_block_span and asap_tight (also on traces with a moved node) -- runs
on the device and equals the unmodified reference's floats bit for bit
(goldens: tests/golden/make_golden_analyze.py, make_golden_trace_api.py)."""

import gzip
import json
import os

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _load(name):
    with gzip.open(os.path.join(HERE, "golden", name), "rt") as fh:
        return json.load(fh)


def _trace(p):
    from paper_2509_24859_b200.scheduling import LaunchCounts, build_program
    from paper_2509_24859_b200.simulation import build_dag, simulate

    S = len(p["t_fwd"])
    deltas = tuple(p["counts"][s] - p["counts"][s + 1] for s in range(S - 1))
    lc = LaunchCounts(tuple(p["counts"]), deltas, "golden")
    return simulate(build_dag(p["t_fwd"], p["t_bwd"], p["comm"], build_program(lc, p["B"])))


def test_analyze_single_trace_equals_reference():
    from paper_2509_24859_b200.simulation import analyze

    for i, p in enumerate(_load("analyze.json.gz")):
        trace = _trace(p)
        assert trace.makespan.hex() == p["makespan"], i
        rep = analyze(trace, p["mem_act"])
        got = [[r.busy.hex(), r.window.hex(), r.bubble.hex(), r.bubble_fraction.hex(),
                r.steady_bubble.hex(), float(r.peak_inflight_bytes).hex(), r.peak_inflight]
               for r in rep.stages]
        assert got == p["stages"], i
        assert [[float(l.fwd_time).hex(), float(l.bwd_time).hex(), float(l.overlap_ratio).hex()]
                for l in rep.links] == p["links"], i


def test_steady_rate_spans_and_asap_equal_reference():
    from paper_2509_24859_b200.simulation import (
        ScheduleTrace, SimulationError, asap_tight, steady_block_span, steady_state_rate,
    )

    plans = _load("analyze.json.gz")
    for i, rec in enumerate(_load("trace_api.json.gz")):
        trace = _trace(plans[i])
        for s, want in enumerate(rec["rates"], start=1):
            if want is None:
                with pytest.raises(SimulationError):
                    steady_state_rate(trace, s)
            else:
                assert steady_state_rate(trace, s).hex() == want, (i, s)
        for s, sp in enumerate(rec["spans"], start=1):
            if sp is not None:
                assert steady_block_span(trace, s, sp[0]).hex() == sp[1], (i, s)
        assert asap_tight(trace) == rec["tight"], i
        for v, val, want in rec["moved"]:
            start = list(trace.start)
            start[v] = float.fromhex(val)
            moved = ScheduleTrace(trace.dag, start, trace.end, trace.makespan)
            assert asap_tight(moved) == want, (i, v)
