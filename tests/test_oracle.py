"""CPU: the oracle (oracle/hapt_oracle.c + oracle/oracle.py) is pinned against
the golden vectors the unmodified reference produced (tests/golden/)."""

import hashlib
import math

import numpy as np
import pytest

import oracle as O
from helpers import expected, expected_arrays, load_json, seeded


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


STAT_KEYS = ["candidates", "canonical", "canonical_feasible", "aliased", "pruned_oom",
             "pruned_imbalance"]


@pytest.mark.parametrize("name", ["A", "B", "C", "D1", "D2", "D3"])
def test_tables_match_reference(name):
    inst, exp = load_json(name), expected(name)
    tb = O.tables(inst)
    for key, want in exp["tables"]["sha"].items():
        got = sha(np.asarray(tb[key], dtype=np.float64)) if key == "pool" else sha(tb[key])
        assert got == want, key
    assert dict(zip(STAT_KEYS, tb["stats"].tolist())) == exp["tables"]["stats"]
    assert O.transitions_per_sweep(tb) == exp["tables"]["transitions_per_sweep"]
    assert len(tb["pool"]) == exp["tables"]["pool_len"]


@pytest.mark.parametrize("name", ["A", "B"])
def test_search_and_full_pool_match_reference(name):
    inst, exp, arr = load_json(name), expected(name), expected_arrays(name)
    plan = O.search(inst)
    ref = exp["plan"]
    for k in ("t_max", "predicted_latency", "eta_pct", "stages", "boundaries"):
        assert plan[k] == ref[k], k
    st = {k: v for k, v in ref["search_stats"].items() if k not in ("backend",)}
    assert plan["search_stats"] == st
    ts, bs, states = O.full_pool(inst)
    assert np.array_equal(ts, arr["tstar"])
    assert np.array_equal(bs, arr["best_s"])
    assert np.array_equal(states, arr["states"])


def test_full_pool_sample_C():
    """Every 40th candidate of config C through the oracle DP."""
    inst, arr = load_json("C"), expected_arrays("C")
    tb = O.tables(inst)
    pool = np.asarray(tb["pool"])
    pick = np.arange(0, len(pool), 40)
    ts, bs, st = O.full_pool(inst, tb, workers=4, pool=list(pool[pick]))
    assert np.array_equal(ts, arr["tstar"][pick])
    assert np.array_equal(bs, arr["best_s"][pick])
    assert np.array_equal(st, arr["states"][pick])


def test_dp_parity_hashes():
    """Operator-level golden: F/N/bp of the reference Cython kernel on the
    instances of test_planner.py::TestBackends (seed 4321)."""
    n = 0
    for rec in seeded()["parity"]:
        tb = O.tables(rec["instance"])
        for c in rec["candidates"]:
            F, N, bi, bo = O.dp_sweep(tb, c["t_max"])
            assert (sha(F), sha(N), sha(bi), sha(bo)) == (c["F"], c["N"], c["bp_i"], c["bp_o"])
            n += 1
    assert n > 10


def _oracle_search_matches(rec):
    inst = rec["instance"]
    for run in rec["runs"]:
        kw = run["kw"]
        try:
            plan = O.search(inst, optimized=kw.get("optimized", True),
                            batch_size=kw.get("batch_size"))
        except ValueError as e:
            assert "error" in run, (rec["tag"], str(e))
            continue
        assert "plan" in run and run["plan"] is not None, rec["tag"]
        ref = run["plan"]
        for k in ("t_max", "predicted_latency", "eta_pct", "stages", "boundaries"):
            assert plan[k] == ref[k], (rec["tag"], k)
        for k, v in ref["search_stats"].items():
            if k != "backend":
                assert plan["search_stats"][k] == v, (rec["tag"], k)


def test_seeded_search_plans():
    recs = [r for r in seeded()["search"] if "instance" in r and r["tag"] not in
            ("integration150", "bench_dp128", "case_study")]
    assert len(recs) > 150
    for rec in recs:
        _oracle_search_matches(rec)


def test_simulator_golden():
    for rec in seeded()["sim"]:
        mk, start, end = O.simulate(rec["t_fwd"], rec["t_bwd"], rec["comm"], rec["counts"], rec["B"])
        assert mk == rec["makespan"]
        assert sha(start) == rec["start"] and sha(end) == rec["end"]


def test_config_e_generator_bounds():
    f, b, c, S = O.config_e_plans(1000)
    t = f + b
    for p in range(1000):
        s = int(S[p])
        assert s in (2, 3, 4, 6, 8)
        tm = t[p, :s].max()
        assert (c[p, : s - 1] <= tm).all() and (c[p, s - 1 :] == 0).all()
        assert math.isfinite(tm)


def test_schedule_report_oracle_equals_reference_goldens():
    """Oracle restatement of analyze()/steady_state_rate() on its own DAG
    trace == the reference's reports (tests/golden/analyze.json.gz)."""
    import gzip
    import json

    from helpers import GOLDEN

    with gzip.open(GOLDEN + "/analyze.json.gz", "rt") as fh:
        plans = json.load(fh)
    for p in plans:
        mk, stages, links, rate = O.schedule_report(p["t_fwd"], p["t_bwd"], p["comm"],
                                                    p["counts"], p["B"], p["mem_act"])
        assert mk.hex() == p["makespan"]
        for got, want in zip(stages, p["stages"]):
            assert [float(x).hex() for x in got[:6]] + [got[6]] == want
        for got, want in zip(links, p["links"]):
            assert [float(x).hex() for x in got] == want
        assert (rate is None and p["steady_rate"] is None) or rate.hex() == p["steady_rate"]
