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
    on B): `planner.search_batches`.

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
                     epsilon: float = 0.05, z: int = 1, batch_size=None, dist=None) -> list:
    """Plan every (mb_size, B) point.  `build_ops(mb_size)` returns the
    operator sequence of one microbatch of that size (e.g.
    workloads.llama_like_ops(b=mb_size) or generate_gpt_sequence(GptConfig(...,
    mb_size=...))).  Returns SweepPoints in the order of `points`.  `dist`
    (PoolSharding) shards every candidate batch across ranks."""
    by_mb: dict = {}
    for mb, B in points:
        by_mb.setdefault(int(mb), []).append(int(B))
    spans, tags_seen = None, None
    done: dict = {}
    for mb, Bs in by_mb.items():
        ops = build_ops(mb)
        tags = [(op.shape_tag, op.kind) for op in ops]
        if spans is None or tags != tags_seen:
            spans, tags_seen = detect_modules(ops, z), tags
        layers = cluster_layers(spans, ops, layers_per_module_unit)
        store = build_store(layers, cluster, model, imbalance_ratio=imbalance_ratio)
        costs = boundary_costs(layers, cluster)
        if len(set(Bs)) > 1:
            plans = search_batches(store, costs, sorted(set(Bs)), epsilon=epsilon,
                                   batch_size=batch_size, dist=dist)
        else:
            plans = {Bs[0]: search(store, costs, Bs[0], epsilon=epsilon, batch_size=batch_size,
                                   dist=dist)}
        for B in Bs:
            done[(mb, B)] = SweepPoint(mb, B, layers, plans[B])
    return [done[(int(mb), int(B))] for mb, B in points]


def best_point(points: Sequence[SweepPoint]) -> SweepPoint:
    """The point with the least predicted time per sample (ties: smaller
    microbatch size); for a fixed global batch this is the least T*."""
    return min(points, key=lambda p: (p.seconds_per_sample, p.mb_size, p.num_microbatches))
