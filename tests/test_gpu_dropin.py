"""GPU: the operator-level drop-in exercised the way the
reference itself calls it.

* concurrent dp_sweep calls from a ThreadPoolExecutor (the reference's
  batched_search, planner.py:529-531) over interleaved table sets, against
  the Cython kernel's F/N/bp hashes (seed 4321, test_planner.py:339-377);
* the UNMODIFIED reference planner (oracle/_ref, Cython build) with
  `meshpipe.planner.dp_sweep` rebound to `paper_2509_24859_b200._core.dp_sweep`
  (the binding _core/__init__.py:6-18 would select), running its own
  `search()` with workers=4 on configs A/B/C and on the seeded instances of
  the reference's tests, against the plans the reference produced with its
  own kernel.
"""

import hashlib
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle as O
from helpers import assert_plan_equal, expected, load_json, ref_types, reference_meshpipe, seeded

pytestmark = pytest.mark.gpu


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _args(tb, t):
    return (t, tb["t_tab"], tb["mp_tab"], tb["ma_tab"], tb["opt_cap"], tb["opt_mesh"],
            tb["opt_devs"], tb["opt_off"], tb["cb_same"], tb["cb_next"], tb["g_mesh"],
            tb["g_avail"], tb["s_max"], tb["span_off"], tb["span_items"])


def test_dropin_is_reentrant_under_threadpool():
    """Interleaved calls over 10 table sets from 4 threads (more table sets
    than the drop-in's cache holds) equal the Cython kernel bit for bit."""
    from paper_2509_24859_b200._core import dp_sweep

    jobs = []
    for rec in seeded()["parity"]:
        tb = O.tables(rec["instance"])
        for c in rec["candidates"]:
            jobs.append((tb, c))
    # round-robin over instances so consecutive calls switch table sets
    order = sorted(range(len(jobs)), key=lambda j: (j % 7, j))

    def run(j):
        tb, c = jobs[j]
        F, N, bi, bo = dp_sweep(*_args(tb, c["t_max"]))
        return (sha(F), sha(N), sha(bi), sha(bo)) == (c["F"], c["N"], c["bp_i"], c["bp_o"])

    with ThreadPoolExecutor(4) as ex:
        ok = list(ex.map(run, order * 2))
    assert len(ok) > 20 and all(ok)


def test_dropin_encodings():
    """Encodings other than DpTables': meshes consumed in the reverse order
    (the boundary row is still a function of the successor state) equal the
    oracle's restatement of _dp.pyx; an interleaved encoding whose row
    depends on the caller, or an option with no device, is refused with
    ValueError -- never answered with different tables."""
    from paper_2509_24859_b200._core import dp_sweep

    tb = O.tables(load_json("A"))
    G = tb["G"]
    rev = dict(tb)
    rev["g_mesh"] = np.ascontiguousarray(
        np.concatenate([[0], np.asarray(tb["g_mesh"])[1:][::-1]]), dtype=np.int32)
    assert not np.array_equal(rev["g_mesh"], tb["g_mesh"])
    for t in tb["pool"][::9]:
        got = dp_sweep(*_args(rev, float(t)))
        want = O.dp_sweep(rev, float(t))
        for g, w in zip(got, want):
            assert np.array_equal(g, w)
    mixed = dict(tb)
    mixed["g_mesh"] = np.array([0] + [(g + 1) % 2 for g in range(1, G + 1)], dtype=np.int32)
    mixed["g_avail"] = np.array([0] + [(g + 1) // 2 for g in range(1, G + 1)], dtype=np.int32)
    with pytest.raises(ValueError):
        dp_sweep(*_args(mixed, float(tb["pool"][-1])))
    bad = dict(tb)
    bad["opt_devs"] = np.array(tb["opt_devs"], dtype=np.int32).copy()
    bad["opt_devs"][0] = 0
    with pytest.raises(ValueError):
        dp_sweep(*_args(bad, float(tb["pool"][-1])))


def _rebound():
    mp = reference_meshpipe()
    if mp is None:
        pytest.skip("oracle/_ref (the reference build) is not present")
    from paper_2509_24859_b200._core import dp_sweep

    assert mp.BACKEND == "cython"
    return mp, dp_sweep


@pytest.mark.parametrize("name", ["A", "B", "C"])
def test_reference_search_runs_on_the_dropin(name, monkeypatch):
    mp, ours = _rebound()
    calls = []

    def counted(*a):
        calls.append(a[0])
        return ours(*a)

    monkeypatch.setattr(mp.planner, "dp_sweep", counted)
    store, costs, B, eps = ref_types(load_json(name))
    plan = mp.planner.search(store, costs, B, epsilon=eps, workers=4, batch_size=4)
    d = mp.planner.plan_to_dict(plan)
    d["search_stats"].pop("wall_time_s", None)
    assert_plan_equal(d, expected(name)["plan"])
    assert mp.planner.validate_plan(plan, store, costs, store.cluster) == []
    assert len(calls) >= plan.search_stats["evaluated"]


def test_reference_seeded_searches_run_on_the_dropin(monkeypatch):
    """The seeded instances of the reference's own tests (test_planner.py,
    test_acceptance.py 08/09/10, ...), every recorded search() variant
    (optimized / full sweep, batch sizes, workers)."""
    mp, ours = _rebound()
    monkeypatch.setattr(mp.planner, "dp_sweep", ours)
    n = 0
    for rec in seeded()["search"]:
        if "instance" not in rec:
            continue
        store, costs, B, eps = ref_types(rec["instance"])
        for run in rec["runs"]:
            kw = dict(run["kw"])
            kw.setdefault("workers", 4)
            if "error" in run:
                with pytest.raises(mp.planner.PlannerError):
                    mp.planner.search(store, costs, B, **kw)
                continue
            plan = mp.planner.search(store, costs, B, **kw)
            d = mp.planner.plan_to_dict(plan)
            d["search_stats"].pop("wall_time_s", None)
            assert_plan_equal(d, run["plan"])
            n += 1
    assert n > 200
