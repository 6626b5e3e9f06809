"""GPU: K1 tables and the K2 DP operator, bit-exact against the reference
goldens and the oracle."""

import hashlib
import os

import numpy as np
import pytest

import oracle as O
from conftest import REPO
from helpers import build, expected, expected_arrays, load_json, seeded

pytestmark = pytest.mark.gpu

STAT_KEYS = ["candidates", "canonical", "canonical_feasible", "aliased", "pruned_oom",
             "pruned_imbalance"]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", ["A", "B", "C", "D1", "D2", "D3", "D4"])
def test_device_tables_equal_reference(name):
    """(D4: 320 layers, n_opts * L(L+1)/2 = 2.26 M span-option cells, past
    the 2^21 packing limit of round 1.)"""
    """hapt_tables_build reproduces DpTables + the t_max pool + StoreStats."""
    from paper_2509_24859_b200.planner import DpTables

    inst, exp = load_json(name), expected(name)
    store, costs, cluster, B, eps = build(inst)
    tables = DpTables(store, costs)
    for key, want in exp["tables"]["sha"].items():
        if key == "pool":
            got = sha(np.asarray(store.feasible_t_values(), dtype=np.float64))
        else:
            got = sha(getattr(tables, key))
        assert got == want, key
    assert store.stats.as_dict() == exp["tables"]["stats"]
    assert tables.transitions_per_sweep() == exp["tables"]["transitions_per_sweep"]


@pytest.mark.parametrize("name", ["A", "C"])
def test_store_lookup_equals_oracle(name):
    """Every (option, span) profile incl. pruned ones (ProfileStore.lookup)."""
    inst = load_json(name)
    store, *_ = build(inst)
    tb = O.tables(inst)
    for key in ("tf", "tb", "mp", "ma"):
        dev = store.dev.host(f"{key}_raw")
        L = store.num_layers
        for o in range(tb["n_opts"]):
            for q in range(1, L + 1):
                assert np.array_equal(dev[o, q, q:L + 1], tb[key][o, q, q:L + 1]), (key, o, q)
    st = store.dev.host("cell_state")
    assert np.array_equal(st & 1, tb["state"] & 1)
    mesh, sub = store.options[0]
    prof = store.lookup(1, 2, mesh.id, sub.shape)
    assert prof is store.lookup(1, 2, mesh.id, sub.shape)


def test_dp_sweep_dropin_matches_reference_kernel():
    """The 15-argument operator against the Cython kernel's outputs on the
    instances of test_planner.py::TestBackends (seed 4321)."""
    from paper_2509_24859_b200._core import dp_sweep

    n = 0
    for rec in seeded()["parity"]:
        tb = O.tables(rec["instance"])
        for c in rec["candidates"]:
            F, N, bi, bo = dp_sweep(c["t_max"], tb["t_tab"], tb["mp_tab"], tb["ma_tab"],
                                    tb["opt_cap"], tb["opt_mesh"], tb["opt_devs"], tb["opt_off"],
                                    tb["cb_same"], tb["cb_next"], tb["g_mesh"], tb["g_avail"],
                                    tb["s_max"], tb["span_off"], tb["span_items"])
            assert (sha(F), sha(N), sha(bi), sha(bo)) == (c["F"], c["N"], c["bp_i"], c["bp_o"])
            n += 1
    assert n > 10


def test_rows_with_split_gaps_equal_oracle():
    """K1 rows hold consecutive splits (the staging computes a successor
    from the entry's position); a CSR with gaps -- possible through the
    drop-in operator's caller-built span index -- takes the load-based path
    and still equals the reference algorithm."""
    from paper_2509_24859_b200._core import dp_sweep

    tb = dict(O.tables(load_json("B")))
    off, items = np.asarray(tb["span_off"]), np.asarray(tb["span_items"])
    keep = np.ones(len(items), dtype=bool)
    for r in range(len(off) - 1):
        if off[r + 1] - off[r] >= 3:
            keep[off[r] + 1] = False  # drop each long row's second split
    counts = np.diff(off)
    new_counts = np.array([keep[off[r]:off[r + 1]].sum() for r in range(len(counts))])
    tb["span_items"] = np.ascontiguousarray(items[keep], dtype=np.int32)
    tb["span_off"] = np.ascontiguousarray(np.concatenate([[0], np.cumsum(new_counts)]),
                                          dtype=np.int32)
    assert keep.sum() < len(items)
    for t in tb["pool"][::11]:
        got = dp_sweep(t, tb["t_tab"], tb["mp_tab"], tb["ma_tab"], tb["opt_cap"], tb["opt_mesh"],
                       tb["opt_devs"], tb["opt_off"], tb["cb_same"], tb["cb_next"], tb["g_mesh"],
                       tb["g_avail"], tb["s_max"], tb["span_off"], tb["span_items"])
        want = O.dp_sweep(tb, t)
        for g, w in zip(got, want):
            assert np.array_equal(g, w)


@pytest.mark.parametrize("name", ["A", "B"])
def test_dp_sweep_dropin_full_pool_equals_oracle(name):
    from paper_2509_24859_b200._core import dp_sweep

    tb = O.tables(load_json(name))
    for t in tb["pool"][::7]:
        got = dp_sweep(t, tb["t_tab"], tb["mp_tab"], tb["ma_tab"], tb["opt_cap"], tb["opt_mesh"],
                       tb["opt_devs"], tb["opt_off"], tb["cb_same"], tb["cb_next"], tb["g_mesh"],
                       tb["g_avail"], tb["s_max"], tb["span_off"], tb["span_items"])
        want = O.dp_sweep(tb, t)
        for g, w in zip(got, want):
            assert np.array_equal(g, w)


@pytest.mark.parametrize("name", ["A", "B", "C", "D1"])
def test_batched_full_pool_equals_reference(name):
    """Every candidate of the pool in batched sweeps: T*, best s and the
    finite-cell count equal the reference's per-candidate dp_search."""
    from paper_2509_24859_b200.planner import sweep_pool

    inst, arr = load_json(name), expected_arrays(name)
    store, costs, cluster, B, eps = build(inst)
    pool, tstar, best_s, states, winner = sweep_pool(store, costs, B)
    assert np.array_equal(pool, arr["pool"])
    assert np.array_equal(tstar, arr["tstar"])
    assert np.array_equal(best_s, arr["best_s"])
    assert np.array_equal(states, arr["states"])
    feas = np.where(best_s >= 0)[0]
    assert winner == feas[np.lexsort((pool[feas], tstar[feas]))[0]]


def test_batch_chunking_is_invisible():
    """Splitting a batch into workspace-sized chunks changes nothing."""
    from paper_2509_24859_b200.planner import DpTables

    inst = load_json("C")
    store, costs, cluster, B, eps = build(inst)
    tables = DpTables(store, costs)
    pool = store.feasible_t_values()
    a = tables.sweeper.evaluate(pool, B)
    tables.sweeper.max_ws_bytes = 1  # one 32-candidate group per chunk
    b = tables.sweeper.evaluate(pool, B)
    assert tables.sweeper.last_chunks == (len(pool) + 31) // 32
    assert np.array_equal(a.tstar, b.tstar) and np.array_equal(a.states, b.states)


def test_caller_chosen_cpl_equals_reference():
    """hapt_dp_sweep_batch_cpl: every candidates-per-lane choice, on the full
    pool and on a spread batch like the search's probe trees, gives the
    reference's per-candidate results."""
    import torch

    from paper_2509_24859_b200.planner import DpTables

    for name in ("B", "C", "D1"):
        inst, arr = load_json(name), expected_arrays(name)
        store, costs, cluster, B, eps = build(inst)
        tables = DpTables(store, costs)
        pool = np.asarray(store.feasible_t_values())
        for idx in (np.arange(len(pool)), np.arange(0, len(pool), 37)):
            for cpl in (0, 1, 2, 4):
                r = tables.sweeper.evaluate(pool[idx], B, cpl=cpl)
                assert np.array_equal(r.tstar, arr["tstar"][idx]), (name, cpl)
                assert np.array_equal(r.best_s, arr["best_s"][idx]), (name, cpl)
                assert np.array_equal(r.states, arr["states"][idx]), (name, cpl)
    torch.cuda.synchronize()


@pytest.mark.parametrize("env", [{"HAPT_CPL": "1"}, {"HAPT_CPL": "2"}, {"HAPT_CPL": "4"},
                                 {"HAPT_PROBE": "0"}])
def test_every_kernel_variant_equals_reference(env):
    """Each candidates-per-lane variant of dp_relax, and the sweep without the
    best-first probe, gives the reference's full-pool results (the library
    reads these knobs once per process, hence the subprocess)."""
    import subprocess
    import sys

    code = (
        "import sys, numpy as np; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "from helpers import build, load_json, expected_arrays\n"
        "from paper_2509_24859_b200.planner import sweep_pool\n"
        "for name in ('B', 'C', 'D1'):\n"
        "    inst, arr = load_json(name), expected_arrays(name)\n"
        "    store, costs, cluster, B, eps = build(inst)\n"
        "    pool, tstar, best_s, states, winner = sweep_pool(store, costs, B)\n"
        "    assert np.array_equal(tstar, arr['tstar']), name\n"
        "    assert np.array_equal(best_s, arr['best_s']), name\n"
        "    assert np.array_equal(states, arr['states']), name\n"
        "print('ok')\n" % (REPO, os.path.dirname(os.path.abspath(__file__))))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                       env={**os.environ, **env}, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


@pytest.mark.parametrize("name", ["D2", "D3"])
def test_full_pool_strided_sample_equals_reference(name):
    """D2 / D3 full pools (7,019 / 15,925 candidates, the bench's per_config
    lines): the batched sweep of the WHOLE pool, checked at a strided sample
    of >= 300 candidates plus the neighbourhoods of the first feasible
    candidate and of search()'s winner, against the reference's own
    per-candidate dp_sweep + _extract_plan (tests/golden/make_golden_sample.py)."""
    from paper_2509_24859_b200.planner import sweep_pool

    inst = load_json(name)
    smp = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "instances",
                               f"{name}_sample.npz"))
    store, costs, cluster, B, eps = build(inst)
    pool, tstar, best_s, states, winner = sweep_pool(store, costs, B)
    idx = smp["idx"]
    assert len(idx) >= 300
    assert np.array_equal(pool[idx], smp["tmax"])
    assert np.array_equal(tstar[idx], smp["tstar"])
    assert np.array_equal(best_s[idx], smp["best_s"])
    assert np.array_equal(states[idx], smp["states"])
    ff = int(smp["first_feasible"])
    assert np.isfinite(tstar[ff]) and not np.isfinite(tstar[ff - 1])
    assert pool[winner] == expected(name)["plan"]["t_max"]
