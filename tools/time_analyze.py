"""Split of PlanBatch.analyze time: simulation with node times vs the report
kernel, on config-E plans (B = 128), in both node layouts (reference
numbering; trace layout, which PlanBatch.analyze uses).

    python tools/time_analyze.py [--plans 100000]
"""
import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--plans", type=int, default=100_000)
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2509_24859_b200 import _lib
    from paper_2509_24859_b200._lib import check, ptr, stream_ptr
    from paper_2509_24859_b200.simulation import PlanBatch, _sim_ws
    from paper_2509_24859_b200.workloads import config_e

    f, b, c, S = config_e(args.plans, seed=7)
    pb = PlanBatch(f, b, c, stage_counts=S)
    counts, _ = pb.counts(0.05, "adaptive")
    lib = _lib.lib()
    dev = pb.device
    P, TS = pb.n_plans, pb.total_stages
    B = 128
    mb = torch.full((P,), B, dtype=torch.int32, device=dev)
    sc = np.diff(pb.stage_off_host)
    nodes = B * (4 * sc - 2) + 1
    noff = torch.zeros(P, dtype=torch.int64, device=dev)
    noff[1:] = torch.from_numpy(np.cumsum(nodes[:-1])).to(dev)
    n = int(nodes.sum())
    start = torch.empty(n, dtype=torch.float64, device=dev)
    end = torch.empty(n, dtype=torch.float64, device=dev)
    tpairs = B * (4 * sc - 2)
    toff = torch.zeros(P, dtype=torch.int64, device=dev)
    toff[1:] = torch.from_numpy(np.cumsum(tpairs[:-1])).to(dev)
    trace = torch.empty(2 * int(tpairs.sum()), dtype=torch.float64, device=dev)
    ring = int(counts.max().item()) + 2
    nb = lib.hapt_sim_workspace_bytes(TS, ring)
    ws = _sim_ws(dev, nb)
    mk = torch.empty(P, dtype=torch.float64, device=dev)
    status = torch.empty(P, dtype=torch.int32, device=dev)
    stage = torch.empty(TS, 6, dtype=torch.float64, device=dev)
    peak = torch.empty(TS, dtype=torch.int32, device=dev)
    link = torch.empty(TS, 3, dtype=torch.float64, device=dev)
    rate = torch.empty(P, dtype=torch.float64, device=dev)

    def sim():
        check(lib.hapt_sim_1f1b(P, pb.stage_off.data_ptr(), ptr(pb.t_fwd), ptr(pb.t_bwd),
                                ptr(pb.comm), ptr(counts), ptr(mb), ptr(mk), ptr(start),
                                ptr(end), ptr(noff), ring, ptr(status), ws.data_ptr(), nb,
                                stream_ptr()))

    def rep():
        check(lib.hapt_analyze_1f1b(P, TS, pb.stage_off.data_ptr(), ptr(pb.t_fwd),
                                    ptr(pb.t_bwd), ptr(pb.comm), ptr(counts), ptr(mb), 0,
                                    ptr(start), ptr(end), ptr(noff), ptr(status), ptr(stage),
                                    ptr(peak), ptr(link), ptr(rate), stream_ptr()))

    def sim_t():
        check(lib.hapt_sim_1f1b_trace(P, pb.stage_off.data_ptr(), ptr(pb.t_fwd), ptr(pb.t_bwd),
                                      ptr(pb.comm), ptr(counts), ptr(mb), ptr(mk), ptr(trace),
                                      ptr(toff), ring, ptr(status), ws.data_ptr(), nb,
                                      stream_ptr()))

    def rep_t():
        check(lib.hapt_analyze_1f1b_trace(P, TS, pb.stage_off.data_ptr(), ptr(pb.t_fwd),
                                          ptr(pb.t_bwd), ptr(pb.comm), ptr(counts), ptr(mb), 0,
                                          ptr(trace), ptr(toff), ptr(status), ptr(stage),
                                          ptr(peak), ptr(link), ptr(rate), stream_ptr()))

    for name, fn in (("sim+nodes", sim), ("analyze", rep), ("sim+trace", sim_t),
                     ("analyze/tr", rep_t)):
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            fn()
        e.record()
        e.synchronize()
        dt = s.elapsed_time(e) / 5
        print(f"{name:10s} {dt:8.3f} ms  ({P / dt * 1e3:.3e} plans/s, {n * 16 / 1e9:.2f} GB of node times)")


if __name__ == "__main__":
    main()
