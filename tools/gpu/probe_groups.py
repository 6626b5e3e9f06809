"""The search's first speculative batch (top candidate + binary-search probe
tree) swept as one warp group vs split into k t_max-contiguous groups, each
padded to 32 lanes by repeating its last candidate.

    python tools/gpu/probe_groups.py D2 D3
"""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)


def main(names):
    import numpy as np
    import torch

    from paper_2509_24859_b200.planner import DpTables, _batch_depth, _probe_tree
    from paper_2509_24859_b200.profiling import boundary_costs, build_store
    from paper_2509_24859_b200.workloads import instance

    def timed(sw, tm, cpl, reps=3):
        t = torch.from_numpy(np.ascontiguousarray(tm)).cuda()
        sw.sweep_device(t, cpl=cpl)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            out = sw.sweep_device(t, cpl=cpl)
        e.record()
        e.synchronize()
        return s.elapsed_time(e) / reps, out

    for name in names:
        layers, cluster, model, rho, B, eps = instance(name)
        store = build_store(layers, cluster, model, imbalance_ratio=rho)
        tables = DpTables(store, boundary_costs(layers, cluster))
        pool = np.asarray(store.feasible_t_values())
        n = len(pool)
        spec = {n - 1}
        _probe_tree(0, n - 1, _batch_depth(tables, n), spec)
        idx = np.array(sorted(spec))
        tm = pool[idx]
        sw = tables.sweeper
        ms, ref = timed(sw, tm, 1)
        print(f"{name}: {len(idx)} probes, one group: {ms:.2f} ms", flush=True)
        print(f"  top alone {timed(sw, tm[-1:], 1)[0]:.2f} ms, without top {timed(sw, tm[:-1], 1)[0]:.2f} ms")
        for k in (2, 4, 8, 16, 32):
            parts = np.array_split(np.arange(len(tm)), k)
            padded = np.concatenate([np.resize(tm[p], 32) if len(p) else [] for p in parts])
            padded = np.concatenate([np.pad(tm[p], (0, 32 - len(p)), mode="edge") for p in parts])
            ms, out = timed(sw, padded, 1)
            pos = np.concatenate([np.arange(len(p)) + 32 * j for j, p in enumerate(parts)])
            same = torch.equal(out[0][torch.from_numpy(pos).cuda()], ref[0])
            print(f"  {k} groups: {ms:.2f} ms (ftop identical: {same})", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["D2"])
