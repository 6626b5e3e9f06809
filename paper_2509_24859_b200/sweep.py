"""Microbatch-configuration sweep.

The reference plans one (microbatch size, microbatch count) point per
`meshpipe plan` run; config D's "full microbatch-config sweep" is the outer
loop over the points (mb_size, B) in {(1,128), (2,64), (4,32), (8,16)}, one
search() each.  Here the loop shares what does not change:

  * module detection depends only on the operators' shape tags and kinds
    (model_graph.py:169-208), which a microbatch size does not alter, so
    `detect_modules` runs once per distinct tag sequence;
  * every mb_size gets its own layer aggregates and cost tables (K1, one
    launch chain per point);
  * points that share an mb_size share their DP sweeps (F does not depend
    on B): `planner.search_batches`;
  * distinct microbatch sizes are independent searches, each a chain of
    small latency-bound launches with host decisions in between, so they run
    concurrently: one host thread and one CUDA stream each (ctypes and the
    stream synchronisations release the GIL; scratch buffers are per stream).

Every point's plan and search_stats equal what `search()` returns for that
point alone (tests/test_gpu_sweep.py, against reference goldens).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

from .model_graph import cluster_layers, detect_modules
from .planner import ParallelPlan, search, search_batches
from .profiling import CostModel, boundary_costs, build_store

DEFAULT_POINTS = ((1, 128), (2, 64), (4, 32), (8, 16))


@dataclass
class SweepPoint:
    mb_size: int
    num_microbatches: int
    layers: object          # LayerSequence of this microbatch size
    plan: ParallelPlan

    @property
    def samples(self) -> int:
        return self.mb_size * self.num_microbatches

    @property
    def seconds_per_sample(self) -> float:
        return self.plan.predicted_latency / self.samples


def microbatch_sweep(build_ops: Callable[[int], list], cluster,
                     points: Sequence[tuple] = DEFAULT_POINTS, model: CostModel | None = None,
                     layers_per_module_unit: int = 1, imbalance_ratio: float = 3.0,
                     epsilon: float = 0.05, z: int = 1, batch_size=None, dist=None,
                     concurrent: bool = True) -> list:
    """Plan every (mb_size, B) point.  `build_ops(mb_size)` returns the
    operator sequence of one microbatch of that size (e.g.
    workloads.llama_like_ops(b=mb_size) or generate_gpt_sequence(GptConfig(...,
    mb_size=...))).  Returns SweepPoints in the order of `points`.  `dist`
    (PoolSharding) shards every candidate batch across ranks (the sizes are
    then planned one after another, so every rank issues the same
    collectives in the same order); otherwise `concurrent` plans the
    microbatch sizes on parallel streams."""
    by_mb: dict = {}
    for mb, B in points:
        by_mb.setdefault(int(mb), []).append(int(B))
    jobs = []
    spans, tags_seen = None, None
    for mb, Bs in by_mb.items():
        ops = build_ops(mb)
        tags = [(op.shape_tag, op.kind) for op in ops]
        if spans is None or tags != tags_seen:
            spans, tags_seen = detect_modules(ops, z), tags
        jobs.append((mb, Bs, ops, spans))

    def plan_size(mb, Bs, ops, spans):
        layers = cluster_layers(spans, ops, layers_per_module_unit)
        store = build_store(layers, cluster, model, imbalance_ratio=imbalance_ratio)
        costs = boundary_costs(layers, cluster)
        if len(set(Bs)) > 1:
            plans = search_batches(store, costs, sorted(set(Bs)), epsilon=epsilon,
                                   batch_size=batch_size, dist=dist)
        else:
            plans = {Bs[0]: search(store, costs, Bs[0], epsilon=epsilon, batch_size=batch_size,
                                   dist=dist)}
        return mb, Bs, layers, plans

    if concurrent and dist is None and len(jobs) > 1:
        results = _on_streams(plan_size, jobs)
    else:
        results = [plan_size(*j) for j in jobs]
    done: dict = {}
    for mb, Bs, layers, plans in results:
        for B in Bs:
            done[(mb, B)] = SweepPoint(mb, B, layers, plans[B])
    return [done[(int(mb), int(B))] for mb, B in points]


_STREAMS: dict = {}  # device -> side streams reused across calls


def _on_streams(fn, jobs):
    """fn(*job) for every job, each on its own host thread and CUDA stream;
    results in job order (exceptions propagate)."""
    from concurrent.futures import ThreadPoolExecutor

    import torch

    dev = torch.device("cuda", torch.cuda.current_device())
    pool = _STREAMS.setdefault(dev, [])
    while len(pool) < len(jobs):
        pool.append(torch.cuda.Stream(dev))
    # side streams start after everything already queued on the caller's
    origin = torch.cuda.current_stream(dev)
    for st in pool[:len(jobs)]:
        st.wait_stream(origin)

    def run(i):
        torch.cuda.set_device(dev)
        with torch.cuda.stream(pool[i]):
            out = fn(*jobs[i])
        pool[i].synchronize()
        return out

    with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
        return list(ex.map(run, range(len(jobs))))


def best_point(points: Sequence[SweepPoint]) -> SweepPoint:
    """The point with the least predicted time per sample (ties: smaller
    microbatch size); for a fixed global batch this is the least T*."""
    return min(points, key=lambda p: (p.seconds_per_sample, p.mb_size, p.num_microbatches))
