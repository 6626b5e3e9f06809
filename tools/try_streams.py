"""Experiment: the full pool as k independent batches on k CUDA streams (each
its own workspace), so one batch's per-layer tails and launch gaps overlap
another's work.  Prints device time per pool for k = 1, 2, 3, 4.

    python tools/try_streams.py [--config D1]
"""
import argparse
import ctypes
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="D1")
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2509_24859_b200._lib import check
    from paper_2509_24859_b200.planner import DpTables
    from paper_2509_24859_b200.profiling import boundary_costs, build_store
    from paper_2509_24859_b200.workloads import instance

    layers, cluster, model, rho, B, eps = instance(args.config)
    store = build_store(layers, cluster, model, imbalance_ratio=rho)
    tables = DpTables(store, boundary_costs(layers, cluster))
    sw = tables.sweeper
    lib, t = sw.lib, sw.tables
    pool = torch.from_numpy(np.asarray(store.feasible_t_values())).cuda()
    n = pool.numel()
    s1 = t.s_max + 1
    for k in (1, 2, 3, 4):
        # contiguous 128-candidate blocks dealt back and forth (as across GPUs)
        b = np.arange(n) // 128
        owner = np.where((b // k) % 2 == 0, b % k, k - 1 - b % k)
        parts = [torch.from_numpy(np.flatnonzero(owner == j)).cuda() for j in range(k)]
        tm = [pool[p].contiguous() for p in parts]
        streams = [torch.cuda.Stream() for _ in range(k)]
        ws = [torch.empty(lib.hapt_dp_workspace_bytes(ctypes.byref(t.t), x.numel()),
                          dtype=torch.uint8, device="cuda") for x in tm]
        ftop = [torch.empty((x.numel(), s1), dtype=torch.float64, device="cuda") for x in tm]
        states = [torch.empty(x.numel(), dtype=torch.int64, device="cuda") for x in tm]

        def run():
            main_s = torch.cuda.current_stream()
            for j in range(k):
                streams[j].wait_stream(main_s)
                check(lib.hapt_dp_sweep_batch(ctypes.byref(t.t), tm[j].data_ptr(), tm[j].numel(),
                                              ftop[j].data_ptr(), states[j].data_ptr(), None,
                                              ws[j].data_ptr(), ws[j].numel(),
                                              streams[j].cuda_stream))
            for j in range(k):
                main_s.wait_stream(streams[j])

        for _ in range(2):
            run()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            run()
        e.record()
        e.synchronize()
        total = sum(int(x.sum()) for x in states)
        print(f"{args.config} k={k}: {s.elapsed_time(e) / 10:.3f} ms per pool  states {total}")


if __name__ == "__main__":
    main()
