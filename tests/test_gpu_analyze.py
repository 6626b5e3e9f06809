"""GPU: batched schedule analysis equals the reference's
analyze(simulate(build_dag(...)), mem_act) and steady_state_rate(trace, 1)
float for float (goldens: tests/golden/make_golden_analyze.py, produced by the
unmodified reference)."""

import gzip
import json
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def load():
    with gzip.open(os.path.join(HERE, "golden", "analyze.json.gz"), "rt") as fh:
        return json.load(fh)


def dense(plans):
    P, W = len(plans), max(len(p["t_fwd"]) for p in plans)
    tf, tb, cm, mem = (np.zeros((P, W)) for _ in range(4))
    cn = np.ones((P, W), dtype=np.int32)
    sc = np.zeros(P, dtype=np.int32)
    for i, p in enumerate(plans):
        S = len(p["t_fwd"])
        sc[i] = S
        tf[i, :S], tb[i, :S], cn[i, :S] = p["t_fwd"], p["t_bwd"], p["counts"]
        cm[i, :S - 1] = p["comm"]
        if p["mem_act"] is not None:
            mem[i, :S] = p["mem_act"]
    B = np.array([p["B"] for p in plans], dtype=np.int32)
    return tf, tb, cm, cn, B, mem, sc


def check_against_goldens(rep, plans):
    so = rep.stage_off.cpu().numpy()
    st = rep.stage.cpu().numpy()
    pk = rep.peak_inflight.cpu().numpy()
    ln = rep.link.cpu().numpy()
    mk = rep.makespan.cpu().numpy()
    rate = rep.steady_rate.cpu().numpy()
    assert (rep.status.cpu().numpy() == 0).all()
    for i, p in enumerate(plans):
        a = so[i]
        assert float(mk[i]).hex() == p["makespan"], i
        for s, row in enumerate(p["stages"]):
            got = [float(x).hex() for x in st[a + s]] + [int(pk[a + s])]
            assert got == row, (i, s, got, row)
        for s, row in enumerate(p["links"]):
            assert [float(x).hex() for x in ln[a + s]] == row, (i, s)
        if p["steady_rate"] is None:
            assert math.isnan(rate[i])
        else:
            assert float(rate[i]).hex() == p["steady_rate"], i


def test_analyze_batch_equals_reference_goldens():
    from paper_2509_24859_b200.simulation import analyze_batch

    plans = load()
    tf, tb, cm, cn, B, mem, sc = dense(plans)
    rep = analyze_batch(tf, tb, cm, cn, B, mem_act=mem, stage_counts=sc)
    check_against_goldens(rep, plans)


def test_analyze_chunked_and_report_objects():
    """Tiny trace budget forces one plan per chunk; report(p) matches the host
    analyze() of this package on the kernel's own trace."""
    import torch

    from paper_2509_24859_b200.scheduling import build_program
    from paper_2509_24859_b200.simulation import (
        PlanBatch, analyze, build_dag, simulate, steady_state_rate,
    )

    plans = load()[:60]
    tf, tb, cm, cn, B, mem, sc = dense(plans)
    pb = PlanBatch(tf, tb, cm, stage_counts=sc)
    mask = np.arange(tf.shape[1])[None, :] < sc[:, None]
    rep = pb.analyze(torch.as_tensor(cn[mask]), torch.as_tensor(B), mem_act=mem[mask],
                     max_node_bytes=1)
    check_against_goldens(rep, plans)
    for i, p in enumerate(plans[:12]):
        prog = build_program(_counts(p), p["B"])
        trace = simulate(build_dag(p["t_fwd"], p["t_bwd"], p["comm"], prog))
        host = analyze(trace, p["mem_act"])
        assert rep.report(i) == host
        if p["steady_rate"] is not None:
            assert rep.steady_state_rate(i) == steady_state_rate(trace, 1)


def _counts(p):
    from paper_2509_24859_b200.scheduling import adaptive_counts, classic_counts, eager_counts

    S = len(p["t_fwd"])
    if p["kind"] == "classic":
        return classic_counts(S)
    if p["kind"] == "eager":
        return eager_counts(S)
    return adaptive_counts([a + b for a, b in zip(p["t_fwd"], p["t_bwd"])], p["comm"], 0.05)


def test_analyze_failed_plans_are_marked():
    """A plan whose program is invalid (B below the warm-up count) gets
    status != 0 and NaN rows; its neighbours are unaffected."""
    from paper_2509_24859_b200.simulation import analyze_batch

    plans = load()[:3]
    tf, tb, cm, cn, B, mem, sc = dense(plans)
    B = B.copy()
    B[1] = 0
    rep = analyze_batch(tf, tb, cm, cn, B, mem_act=mem, stage_counts=sc)
    status = rep.status.cpu().numpy()
    assert status[1] != 0 and status[0] == 0 and status[2] == 0
    a, b = int(rep.stage_off[1]), int(rep.stage_off[2])
    assert np.isnan(rep.stage[a:b].cpu().numpy()).all()
    with pytest.raises(Exception):
        rep.report(1)
    check_against_goldens_subset(rep, plans, [0, 2])


def check_against_goldens_subset(rep, plans, idx):
    st = rep.stage.cpu().numpy()
    so = rep.stage_off.cpu().numpy()
    for i in idx:
        for s, row in enumerate(plans[i]["stages"]):
            assert [float(x).hex() for x in st[so[i] + s]] == row[:6]


def test_analyze_large_batch_fast_path():
    """A batch large enough for the bucketed per-S simulation kernels (which
    then also write the node times) gives the same reports."""
    from paper_2509_24859_b200.simulation import analyze_batch

    plans = load() * 11  # 4,400 plans: past the generic-walk threshold
    tf, tb, cm, cn, B, mem, sc = dense(plans)
    rep = analyze_batch(tf, tb, cm, cn, B, mem_act=mem, stage_counts=sc)
    check_against_goldens(rep, plans)


@pytest.mark.parametrize("copies", [1, 11])  # generic walk / bucketed per-S kernels
def test_both_node_layouts_through_the_abi(copies):
    """hapt_sim_1f1b (reference node numbering) + hapt_analyze_1f1b give the
    goldens too, and hapt_sim_1f1b_trace's pairs are the same node times in
    the trace order the header documents."""
    import torch

    from paper_2509_24859_b200 import _lib
    from paper_2509_24859_b200._lib import check, ptr, stream_ptr
    from paper_2509_24859_b200.simulation import BatchReport, PlanBatch, _sim_ws

    plans = load() * copies
    tf, tb, cm, cn, B, mem, sc = dense(plans)
    pb = PlanBatch(tf, tb, cm, stage_counts=sc)
    dev = pb.device
    mask = np.arange(tf.shape[1])[None, :] < sc[:, None]
    counts = torch.as_tensor(cn[mask], dtype=torch.int32, device=dev)
    memd = torch.as_tensor(mem[mask], dtype=torch.float64, device=dev)
    mb = torch.as_tensor(B, dtype=torch.int32, device=dev)
    P, TS = pb.n_plans, pb.total_stages
    ref_nodes = B.astype(np.int64) * (4 * sc - 2) + 1
    tr_pairs = B.astype(np.int64) * (4 * sc - 2)
    roff = torch.as_tensor(np.concatenate([[0], np.cumsum(ref_nodes)[:-1]]), device=dev)
    toff = torch.as_tensor(np.concatenate([[0], np.cumsum(tr_pairs)[:-1]]), device=dev)
    start = torch.empty(int(ref_nodes.sum()), dtype=torch.float64, device=dev)
    end = torch.empty_like(start)
    trace = torch.empty(2 * int(tr_pairs.sum()), dtype=torch.float64, device=dev)
    ring = int(counts.max().item()) + 2
    lib = _lib.lib()
    nb = lib.hapt_sim_workspace_bytes(TS, ring)
    ws = _sim_ws(dev, nb)

    def report():
        return BatchReport(
            stage_off=pb.stage_off,
            makespan=torch.empty(P, dtype=torch.float64, device=dev),
            status=torch.empty(P, dtype=torch.int32, device=dev),
            stage=torch.empty(TS, 6, dtype=torch.float64, device=dev),
            peak_inflight=torch.empty(TS, dtype=torch.int32, device=dev),
            link=torch.empty(TS, 3, dtype=torch.float64, device=dev),
            steady_rate=torch.empty(P, dtype=torch.float64, device=dev))

    common = (pb.stage_off.data_ptr(), ptr(pb.t_fwd), ptr(pb.t_bwd), ptr(pb.comm), ptr(counts),
              ptr(mb))
    ra, rb = report(), report()
    check(lib.hapt_sim_1f1b(P, *common, ptr(ra.makespan), ptr(start), ptr(end), ptr(roff), ring,
                            ptr(ra.status), ws.data_ptr(), nb, stream_ptr()))
    check(lib.hapt_analyze_1f1b(P, TS, *common, ptr(memd), ptr(start), ptr(end), ptr(roff),
                                ptr(ra.status), ptr(ra.stage), ptr(ra.peak_inflight),
                                ptr(ra.link), ptr(ra.steady_rate), stream_ptr()))
    check(lib.hapt_sim_1f1b_trace(P, *common, ptr(rb.makespan), ptr(trace), ptr(toff), ring,
                                  ptr(rb.status), ws.data_ptr(), nb, stream_ptr()))
    check(lib.hapt_analyze_1f1b_trace(P, TS, *common, ptr(memd), ptr(trace), ptr(toff),
                                      ptr(rb.status), ptr(rb.stage), ptr(rb.peak_inflight),
                                      ptr(rb.link), ptr(rb.steady_rate), stream_ptr()))
    check_against_goldens(ra, plans)
    check_against_goldens(rb, plans)
    # trace pairs vs reference-numbered nodes, for a few plans
    from paper_2509_24859_b200.scheduling import FWD, build_program

    st_h, en_h, tr_h = start.cpu().numpy(), end.cpu().numpy(), trace.cpu().numpy()
    for i in range(0, len(plans), max(1, len(plans) // 25)):
        p, S, Bi = plans[i], int(sc[i]), int(B[i])
        prog = build_program(_counts(p), Bi)
        r0, t0 = int(roff[i]), 2 * int(toff[i])
        want = []
        for s in range(S):
            for kind, m in prog.stages[s].ops:
                j = r0 + 2 * (s * Bi + m - 1) + (0 if kind == FWD else 1)
                want.append((st_h[j], en_h[j]))
        for l in range(S - 1):
            for d in (0, 1):
                for m in range(1, Bi + 1):
                    j = r0 + 2 * S * Bi + 2 * (l * Bi + m - 1) + d
                    want.append((st_h[j], en_h[j]))
        got = tr_h[t0:t0 + 2 * len(want)].reshape(-1, 2)
        assert np.array_equal(got, np.array(want)), i
