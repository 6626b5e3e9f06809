"""Planner search behind the reference API (meshpipe.planner, planner.py:1-786).

The reference evaluates one t_max candidate per `dp_search` call (a Cython
sweep on one CPU thread, planner.py:385-421) inside a sequential binary search
and a thread-pool batch (planner.py:432-542).  Here every evaluation is a
*batch*: `hapt_dp_sweep_batch` sweeps all candidates of a batch through the
DP on the GPU at once, `hapt_dp_select` scores them (Eq. 14 + best s), and
only the winner is backtracked into a ParallelPlan.

`search()` keeps the reference's exact semantics -- including the sequence of
binary-search probes, the non-monotone-feasibility error, t_E, the surviving
set and the search_stats fields -- by evaluating the probe tree speculatively
(all probes the next d steps could touch, in one batch) and replaying the
reference's decisions on the host.  The plan returned is the reference's plan
bit for bit (tests/test_search_parity.py).
"""

from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from .engine import Sweeper
from .profiling import BoundaryCost, ProfileStore
from .scheduling import adaptive_counts

BACKEND = "cuda"


class PlannerError(ValueError):
    pass


class InfeasiblePlanError(PlannerError):
    """No stage partition satisfies the constraints."""


@dataclass(frozen=True)
class PlanStage:
    layer_start: int
    layer_end: int
    mesh_id: str
    n: int
    m: int
    t_fwd: float
    t_bwd: float
    mem_params: float
    mem_act: float
    launch_count: int
    dp_launch_bound: int

    @property
    def t(self) -> float:
        return self.t_fwd + self.t_bwd

    @property
    def submesh(self) -> tuple[int, int]:
        return (self.n, self.m)

    @property
    def device_count(self) -> int:
        return self.n * self.m


@dataclass(frozen=True)
class PlanBoundary:
    after_layer: int
    comm: float
    link: str


@dataclass
class ParallelPlan:
    stages: list
    boundaries: list
    t_max: float
    num_microbatches: int
    predicted_latency: float
    eta_pct: float
    epsilon: float
    search_stats: dict = field(default_factory=dict)

    @property
    def num_stages(self) -> int:
        return len(self.stages)

    @property
    def stage_times(self) -> list:
        return [s.t for s in self.stages]

    @property
    def comm_times(self) -> list:
        return [b.comm for b in self.boundaries]

    def sort_key(self) -> tuple:
        """Merge order among equally good plans (planner.py:107-115)."""
        return (
            self.predicted_latency,
            self.t_max,
            self.num_stages,
            tuple(s.layer_end for s in self.stages),
            tuple((s.mesh_id, s.n, s.m) for s in self.stages),
        )


def end_to_end_latency(stage_times: Sequence[float], comm_times: Sequence[float],
                       num_microbatches: int) -> float:
    """Eq. 14 closed form (planner.py:118-138)."""
    if not stage_times:
        raise PlannerError("need at least one stage")
    if len(comm_times) != len(stage_times) - 1:
        raise PlannerError("expected one comm time per adjacent stage pair")
    t_max = max(stage_times)
    for pos, c in enumerate(comm_times, start=1):
        if c > t_max:
            raise PlannerError(f"boundary {pos}: comm {c:.6g}s exceeds max stage time {t_max:.6g}s")
    return sum(stage_times) + 2.0 * sum(comm_times) + (num_microbatches - 1) * t_max


def load_balance_eta(busy_seconds: Sequence[float], peak_flops: Sequence[float]) -> float:
    """Capacity-weighted load balance in percent (planner.py:141-156)."""
    if len(busy_seconds) == 0 or len(busy_seconds) != len(peak_flops):
        raise PlannerError("need one busy time per device")
    if any(t < 0 for t in busy_seconds) or all(t == 0 for t in busy_seconds):
        raise PlannerError("busy times must be non-negative and not all zero")
    top = max(busy_seconds)
    idle = sum((top - td) * pk for td, pk in zip(busy_seconds, peak_flops))
    return 100.0 * (1.0 - idle / (top * sum(peak_flops)))


# ---------------------------------------------------------------------------
# DP tables
# ---------------------------------------------------------------------------


class DpTables:
    """Device-resident DpTables (planner.py:164-258).  The arrays are the K1
    output already in HBM; numpy views are materialised only on access."""

    _HOST = ("t_tab", "mp_tab", "ma_tab", "opt_cap", "opt_mesh", "opt_devs", "opt_off",
             "cb_same", "cb_next", "g_mesh", "g_avail", "span_off", "span_items")

    def __init__(self, store: ProfileStore, costs: BoundaryCost):
        self.store = store
        self.costs = costs
        self.dev = store.dev
        self.L = store.num_layers
        self.G = store.dev.G
        self.s_max = min(self.L, self.G)
        self.opt_meta = [(mesh.id, sub.n, sub.m) for mesh, sub in store.options]
        self._sync_costs(costs)
        self._sweeper = None

    def _sync_costs(self, costs) -> None:
        """The DP reads cb_same/cb_next from HBM (computed by K1 from the same
        layers/cluster).  A BoundaryCost from elsewhere is uploaded instead, so
        the tables always reflect `costs` exactly as DpTables does
        (planner.py:203-211)."""
        src = getattr(costs, "_source", None)
        st = self.store
        if src == (id(st.layers), id(st.cluster)) and st._cross_ok:
            return
        import torch

        cluster = st.cluster
        meshes = list(cluster.meshes)
        nm = len(meshes)
        same = np.zeros((nm, self.L + 1))
        nxt = np.zeros((nm, self.L + 1))
        for m, mesh in enumerate(meshes):
            for i in range(1, self.L):
                same[m, i] = costs.get(i, mesh.id, mesh.id)
                if m + 1 < nm:
                    nxt[m, i] = costs.get(i, mesh.id, meshes[m + 1].id)
        self.dev.view("cb_same", torch.float64, (nm, self.L + 1)).copy_(torch.from_numpy(same))
        self.dev.view("cb_next", torch.float64, (nm, self.L + 1)).copy_(torch.from_numpy(nxt))
        self.dev._host.pop("cb_same", None)
        self.dev._host.pop("cb_next", None)

    def __getattr__(self, name):
        if name in DpTables._HOST:
            return self.dev.host(name)
        if name == "feasible_spans_per_opt":
            off = self.dev.host("span_off")
            stride = self.L + 2
            return np.array(
                [off[(o + 1) * stride] - off[o * stride] for o in range(len(self.opt_meta))],
                dtype=np.int64,
            )
        raise AttributeError(name)

    @property
    def sweeper(self) -> Sweeper:
        # one Sweeper per device tables, shared by every DpTables view of them
        if getattr(self.dev, "_sweeper", None) is None:
            self.dev._sweeper = Sweeper(self.dev)
        return self.dev._sweeper

    def transitions_per_sweep(self) -> int:
        """planner.py:250-258: sum over states g of the feasible spans of the
        options of g's mesh that fit in g's available devices, times s_max
        (vectorised over states; cached per tables)."""
        cached = getattr(self.dev, "_transitions", None)
        if cached is not None and cached[0] == self.s_max:
            return cached[1]
        per_opt = self.feasible_spans_per_opt
        g_mesh, g_avail = self.g_mesh[1:].astype(np.int64), self.g_avail[1:].astype(np.int64)
        off, devs = self.opt_off, self.opt_devs
        total = 0
        for r in range(len(off) - 1):
            o = np.arange(int(off[r]), int(off[r + 1]))
            avail = g_avail[g_mesh == r]
            if len(o) and len(avail):
                fits = devs[o][None, :] <= avail[:, None]
                total += int((fits * per_opt[o][None, :]).sum())
        self.dev._transitions = (self.s_max, total * self.s_max)
        return total * self.s_max


# ---------------------------------------------------------------------------
# Candidate evaluation
# ---------------------------------------------------------------------------


@dataclass
class DpOutcome:
    plan: Optional[ParallelPlan]
    states: int


class CandidateEvaluator:
    """Evaluates t_max candidates in GPU batches and caches (T*, best s,
    finite-cell count) per pool index.  With `comm` (a torch.distributed
    process group handle) every batch is strided across ranks and the
    per-candidate results are all-gathered, so all ranks replay identically."""

    def __init__(self, tables: DpTables, pool: Sequence[float], num_microbatches: int,
                 dist=None, keep_ftop: bool = False):
        self.tables = tables
        self.pool = np.asarray(pool, dtype=np.float64)
        self.B = num_microbatches
        self.dist = dist
        n = len(self.pool)
        self.tstar = np.full(n, np.nan)
        self.best_s = np.full(n, -2, dtype=np.int64)
        self.states = np.zeros(n, dtype=np.int64)
        self.batches = 0
        self.evaluated = 0
        self._bp_of: dict = {}     # pool index -> (SweepResult with bp, position)
        self._bp_bytes = 0
        # F[s,1,G] per candidate (B-independent) for rescoring under other B
        self.ftop = np.full((n, tables.s_max + 1), np.inf) if keep_ftop else None

    def known(self, idx: int) -> bool:
        return self.best_s[idx] != -2

    def ensure(self, indices, keep_bp: bool = True) -> None:
        """Evaluate the unknown candidates among `indices` in one batch.
        keep_bp: record the batch's backpointers (within BP_BUDGET) so a
        winner from it is walked instead of re-swept -- worth it only for a
        batch that can contain the final winner."""
        if isinstance(indices, range):
            idx = np.arange(indices.start, indices.stop, indices.step, dtype=np.int64)
        else:
            idx = np.unique(np.fromiter((int(i) for i in indices), dtype=np.int64))
        todo = idx[self.best_s[idx] == -2]  # sorted, unique, not yet known
        if not len(todo):
            return
        self.batches += 1
        self.evaluated += len(todo)
        if self.dist is None or len(todo) < self.dist.min_shard:
            # single GPU, or a batch too small to split (replicated on every
            # rank: identical results, no collective)
            sw = self.tables.sweeper
            need = sw.bp_bytes(len(todo))
            keep = keep_bp and self._bp_bytes + need <= sw.BP_BUDGET
            # a batch spread over the pool (binary-search probes) runs one
            # candidate per lane: lanes with distant t_max in one warp share
            # its bounds (D1 search 5.5 -> 4.9 ms, C 4.8 -> 4.2 ms)
            spread = (todo[-1] - todo[0] + 1) > 2 * len(todo)
            res = sw.evaluate(self.pool[todo], self.B, keep_bp=keep,
                              keep_ftop=self.ftop is not None, cpl=1 if spread else 0)
            if self.ftop is not None:
                self.ftop[todo] = res.ftop
            self.tstar[todo] = res.tstar
            self.best_s[todo] = res.best_s
            self.states[todo] = res.states
            if res.bp is not None:
                self._bp_bytes += need
                for pos, i in enumerate(todo.tolist()):
                    self._bp_of[i] = (res, pos)
        elif self.ftop is not None:
            ts, bs, st, ft = self.dist.evaluate_sharded(self.tables.sweeper, self.pool, todo,
                                                        self.B, want_ftop=True)
            self.ftop[todo] = ft
            self.tstar[todo] = ts
            self.best_s[todo] = bs
            self.states[todo] = st
        else:
            ts, bs, st = self.dist.evaluate_sharded(self.tables.sweeper, self.pool, todo, self.B)
            self.tstar[todo] = ts
            self.best_s[todo] = bs
            self.states[todo] = st

    def feasible(self, idx: int) -> bool:
        self.ensure([idx])
        return self.best_s[idx] >= 0

    def plan(self, idx: int, epsilon: float, B: Optional[int] = None,
             best_s: Optional[int] = None, tstar: Optional[float] = None) -> "ParallelPlan":
        """ParallelPlan of pool candidate idx (scored for this evaluator's B,
        or for another B with its best_s / T*): walked from the batch's kept
        backpointers when available, else re-derived by hapt_dp_backtrack."""
        B = self.B if B is None else B
        bs = int(self.best_s[idx]) if best_s is None else int(best_s)
        ts = float(self.tstar[idx]) if tstar is None else float(tstar)
        hit = self._bp_of.get(idx)
        if hit is not None:
            res, pos = hit
            spans = self.tables.sweeper.walk(res, pos, bs)
            return _build_plan(self.tables, float(self.pool[idx]), bs, ts, B, epsilon,
                               spans=spans, n_first=int(res.ntop[pos, bs]))
        return _build_plan(self.tables, float(self.pool[idx]), bs, ts, B, epsilon)


def _probe_tree(lo: int, hi: int, depth: int, out: set) -> None:
    """Every index the reference binary search (planner.py:461-466) may probe
    in its next `depth` steps from (lo, hi)."""
    if depth == 0 or lo >= hi:
        return
    mid = (lo + hi) // 2
    out.add(mid)
    _probe_tree(lo, mid, depth - 1, out)
    _probe_tree(mid + 1, hi, depth - 1, out)


def _batch_depth(tables: DpTables, pool_len: int) -> int:
    """Speculation depth: enough probes per batch to fill the GPU.  A batch of
    32 candidates needs one warp per DP cell per layer; ~40k resident-warp
    slots on 148 SMs are the target."""
    env = os.environ.get("HAPT_SEARCH_DEPTH")  # experiments
    if env:
        return max(1, int(env))
    cells = max(1, tables.L * tables.G)
    groups = max(1, math.ceil(40_000 / cells))
    want = groups * 32
    d = max(1, int(math.floor(math.log2(want + 1))))
    return d


_SURVIVOR_SPEC = 1024  # cap on the candidates swept speculatively with the last probes


def _full_pool_is_cheap(tables: DpTables, pool_len: int) -> bool:
    cells = max(1, tables.L * tables.G)
    return math.ceil(pool_len / 32) * cells <= 2 * 40_000


def bidirectional_prune_replay(ev: CandidateEvaluator, num_microbatches: int):
    """The reference bidirectional_prune (planner.py:432-480) with speculative
    batched evaluation.  Returns (lo, t_e, surviving indices, probed set)."""
    n = len(ev.pool)
    if n == 0:
        raise InfeasiblePlanError("empty candidate pool")
    probed: list[int] = []
    lo, hi = 0, n - 1
    depth = _batch_depth(ev.tables, n)

    def batch(lo: int, hi: int, top: bool) -> None:
        """The probes the next `depth` steps from (lo, hi) can touch.  If the
        binary search ends inside them, also the candidates the surviving
        set t_S <= t <= t_E can reach (t_E estimated from the feasible upper
        end: T grows with t_max once (B-1) t_max dominates, so this
        over-covers; a miss only costs a survivor batch), and keep this
        batch's backpointers for the winner."""
        spec = {hi} if top else set()
        _probe_tree(lo, hi, depth, spec)
        final = (hi - lo + 1).bit_length() <= depth
        if final and ev.known(hi) and ev.best_s[hi] >= 0:
            B = num_microbatches
            t_est = ev.tstar[hi] / (B - 1) if B > 1 else math.inf
            end = int(np.searchsorted(ev.pool, t_est, side="right")) + 8
            spec.update(range(lo, min(n, max(hi + 1, end), lo + _SURVIVOR_SPEC)))
        ev.ensure(spec, keep_bp=final)

    if _full_pool_is_cheap(ev.tables, n):
        ev.ensure(range(n))
    batch(lo, hi, top=True)
    probed.append(hi)
    if not ev.feasible(hi):
        raise InfeasiblePlanError("no t_max candidate admits a feasible plan")
    while lo < hi:
        mid = (lo + hi) // 2
        if not ev.known(mid):
            batch(lo, hi, top=False)
        probed.append(mid)
        if ev.feasible(mid):
            hi = mid
        else:
            lo = mid + 1
    if lo > 0:
        probed.append(lo - 1)
        if ev.feasible(lo - 1):
            raise PlannerError(
                "feasibility is not monotone in t_max on this instance; rerun "
                "without pruning (optimized=False)"
            )
    B = num_microbatches
    t_e = ev.tstar[lo] / (B - 1) if B > 1 else math.inf
    surviving = [i for i in range(lo, n) if ev.pool[i] <= t_e]
    return lo, t_e, surviving, probed


def _count_batches(surviving_t, activated, batch_size) -> int:
    """batched_search's grouping (planner.py:508-524): consecutive equal
    activated-pair counts form a group, chunked by batch_size."""
    if activated is None:
        groups = [len(surviving_t)]
    else:
        groups = []
        cur = None
        for key in activated:
            if key != cur:
                groups.append(0)
                cur = key
            groups[-1] += 1
    n = 0
    for g in groups:
        n += 1 if batch_size is None or batch_size >= g else math.ceil(g / batch_size)
    return n


def _build_plan(tables: DpTables, t_max: float, best_s: int, tstar: float,
                num_microbatches: int, epsilon: float, spans=None,
                n_first: Optional[int] = None) -> ParallelPlan:
    """_extract_plan (planner.py:272-382) from a device backtrack: either the
    walked `spans` of a batch with kept backpointers (plus N[best_s,1,G] as
    `n_first`), or a one-candidate re-sweep with backpointers."""
    store = tables.store
    cluster = store.cluster
    kchain = None
    if spans is None:
        spans, kchain = tables.sweeper.backtrack(t_max, best_s)
    metas = [tables.opt_meta[o] for _, _, o in spans]
    found = store.lookup_many([(q, p, mid, (n, m)) for (q, p, _), (mid, n, m) in zip(spans, metas)])
    profs = [(q, p, mid, n, m, pr) for (q, p, _), (mid, n, m), pr in zip(spans, metas, found)]
    comm, links = [], []
    for idx in range(len(spans) - 1):
        i = spans[idx][1]
        a, b = profs[idx][2], profs[idx + 1][2]
        comm.append(tables.costs.get(i, a, b))
        links.append(f"intra:{a}" if a == b else f"cross:{a}>{b}")
    k_bounds = [0] * len(spans)
    k_next = 0.0
    for idx in range(len(spans) - 1, -1, -1):
        c = comm[idx] if idx < len(spans) - 1 else 0.0
        k_next = math.ceil(2.0 * c / t_max) + 1.0 + k_next
        k_bounds[idx] = int(k_next)
    if (kchain is not None and k_bounds != kchain) or (
            n_first is not None and k_bounds[0] != n_first):
        raise PlannerError("launch-bound chain disagrees with the DP table")
    stage_times = [pr.t for *_, pr in profs]
    counts = adaptive_counts(stage_times, comm, epsilon, t_max=max(t_max, max(stage_times)))
    stages = [
        PlanStage(q, p, mesh_id, n, m, pr.t_fwd, pr.t_bwd, pr.mem_params, pr.mem_act,
                  counts.counts[idx], k_bounds[idx])
        for idx, (q, p, mesh_id, n, m, pr) in enumerate(profs)
    ]
    boundaries = [PlanBoundary(spans[i][1], comm[i], links[i]) for i in range(len(spans) - 1)]
    B = num_microbatches
    busy, peaks = [], []
    for st in stages:
        pk = cluster.mesh(st.mesh_id).peak_flops
        busy.extend([st.t * B] * st.device_count)
        peaks.extend([pk] * st.device_count)
    return ParallelPlan(stages, boundaries, t_max, B, tstar, load_balance_eta(busy, peaks),
                        epsilon)


def dp_search(store: ProfileStore, costs: BoundaryCost, num_microbatches: int, t_max: float,
              epsilon: float = 0.05, tables: Optional[DpTables] = None) -> Optional[ParallelPlan]:
    """Best plan under one latency bound, or None (planner.py:385-421)."""
    if t_max <= 0:
        raise PlannerError("t_max must be positive")
    tables = tables or DpTables(store, costs)
    res = tables.sweeper.evaluate([t_max], num_microbatches, keep_bp=True)
    if res.best_s[0] < 0:
        return None
    bs = int(res.best_s[0])
    spans = tables.sweeper.walk(res, 0, bs) if res.bp is not None else None
    plan = _build_plan(tables, float(t_max), bs, float(res.tstar[0]), num_microbatches, epsilon,
                       spans=spans, n_first=None if spans is None else int(res.ntop[0, bs]))
    plan.search_stats["dp_states"] = int(res.states[0])
    return plan


def candidate_tmax(store: ProfileStore) -> list:
    pool = store.feasible_t_values()
    if not pool:
        raise InfeasiblePlanError("no feasible candidates in the profile store")
    return pool


def bidirectional_prune(candidates: Sequence[float], dp: Callable, num_microbatches: int):
    """Reference-signature variant over a caller-supplied dp(t) (planner.py:432-480).
    search() uses the batched replay instead."""
    if not candidates:
        raise InfeasiblePlanError("empty candidate pool")
    cache: dict = {}

    def evaluate(t):
        if t not in cache:
            cache[t] = dp(t)
        return cache[t]

    lo, hi = 0, len(candidates) - 1
    if evaluate(candidates[hi]) is None:
        raise InfeasiblePlanError("no t_max candidate admits a feasible plan")
    while lo < hi:
        mid = (lo + hi) // 2
        if evaluate(candidates[mid]) is not None:
            hi = mid
        else:
            lo = mid + 1
    t_s = candidates[lo]
    if lo > 0 and evaluate(candidates[lo - 1]) is not None:
        raise PlannerError(
            "feasibility is not monotone in t_max on this instance; rerun "
            "without pruning (optimized=False)"
        )
    B = num_microbatches
    t_e = cache[t_s].predicted_latency / (B - 1) if B > 1 else math.inf
    return t_s, t_e, [t for t in candidates[lo:] if t <= t_e], cache


def batched_search(surviving: Sequence[float], dp: Callable, activated=None, batch_size=None,
                   workers: int = 1, cache: Optional[dict] = None):
    """Reference-signature batch merge over a caller-supplied dp(t)
    (planner.py:490-542); runs sequentially since each dp call is a GPU batch."""
    if not surviving:
        raise InfeasiblePlanError("no surviving candidates")
    cache = cache or {}
    best = None
    for t in surviving:
        plan = cache[t] if t in cache else dp(t)
        if plan is not None and (best is None or plan.sort_key() < best.sort_key()):
            best = plan
    return best, _count_batches(surviving, activated, batch_size)


def _activated_pairs(tables: DpTables, candidates: Sequence[float]) -> list:
    """#DpTables entries with t <= t_max per candidate (planner.py:483-487),
    counted on the device from the CSR pool ranks."""
    return [int(x) for x in tables.sweeper.activated(candidates)]


def search(store: ProfileStore, costs: BoundaryCost, num_microbatches: int,
           epsilon: float = 0.05, workers: int = 1, batch_size: Optional[int] = None,
           optimized: bool = True, dist=None) -> ParallelPlan:
    """Full planning pass (planner.py:545-607) on the GPU.

    ``workers``/``batch_size`` only shape the reported ``batches`` stat, as in
    the reference the plan is independent of them.  ``dist`` (a
    paper_2509_24859_b200.distributed.PoolSharding) shards every candidate
    batch across the ranks of a torch.distributed NCCL group.
    """
    began = time.perf_counter()
    tables = DpTables(store, costs)
    pool = candidate_tmax(store)
    ev = CandidateEvaluator(tables, pool, num_microbatches, dist)
    B = num_microbatches
    if optimized:
        lo, t_e, surviving, probed = bidirectional_prune_replay(ev, B)
        ev.ensure(surviving)
        surv_t = [pool[i] for i in surviving]
        n_batches = _count_batches(surv_t, _activated_pairs(tables, surv_t), batch_size)
        evaluated_set = set(probed) | set(surviving)
        t_s = pool[lo]
        pruned_below = lo
        pruned_above = len(pool) - lo - len(surviving)
    else:
        surviving = list(range(len(pool)))
        ev.ensure(surviving)
        n_batches = 1
        evaluated_set = set(surviving)
        t_s, t_e = pool[0], math.inf
        pruned_below = pruned_above = 0
    cand = [i for i in surviving if ev.best_s[i] >= 0]
    if not cand:
        raise InfeasiblePlanError("no stage partition satisfies the memory and overlap constraints")
    # sort_key merge: (T*, t_max) decides since t_max is unique (planner.py:535-541)
    best = min(cand, key=lambda i: (ev.tstar[i], pool[i]))
    plan = ev.plan(best, epsilon)
    states = int(sum(int(ev.states[i]) for i in evaluated_set if ev.best_s[i] >= 0))
    plan.search_stats.update(
        {
            "backend": BACKEND,
            "candidates_total": len(pool),
            "pruned_below_ts": pruned_below,
            "pruned_above_te": pruned_above,
            "evaluated": len(surviving),
            "batches": n_batches,
            "t_low": t_s,
            "t_high": None if math.isinf(t_e) else float(t_e),
            "dp_states": states,
            "dp_transitions": tables.transitions_per_sweep() * len(surviving),
            "wall_time_s": time.perf_counter() - began,
        }
    )
    return plan


def sweep_pool(store: ProfileStore, costs: BoundaryCost, num_microbatches: int, dist=None):
    """Evaluate EVERY t_max candidate of the pool in one batched sweep (the
    candidates/s workload).  Returns (pool, tstar, best_s, states, winner).
    On one GPU the pool never leaves the device before the sweep (K1 writes
    it, K2 reads it) and all results come back in one transfer."""
    tables = DpTables(store, costs)
    if dist is None:
        import torch

        if store.dev.pool_len == 0:
            raise InfeasiblePlanError("no feasible candidates in the profile store")
        sw = tables.sweeper
        pool_dev = store.dev.pool()
        ftop, states = sw.sweep_device(pool_dev)
        tstar, best_s, winner = sw.select_device(ftop, pool_dev, num_microbatches)
        n = int(pool_dev.numel())
        host = torch.cat([pool_dev.view(torch.int64), tstar.view(torch.int64),
                          best_s.to(torch.int64), states, winner.to(torch.int64)]).cpu().numpy()
        return (host[:n].view(np.float64).copy(), host[n:2 * n].view(np.float64).copy(),
                host[2 * n:3 * n].copy(), host[3 * n:4 * n].copy(), int(host[4 * n]))
    # Sharded: the pool stays on the device; each rank sweeps its blocks, the
    # per-candidate results are all-gathered device to device and scattered
    # back into pool order, the (T*, index) argmin is taken on the device,
    # and everything comes back in one transfer -- the pool count is the only
    # other host read.
    import torch

    n = store.dev.pool_len
    if n == 0:
        raise InfeasiblePlanError("no feasible candidates in the profile store")
    sw = tables.sweeper
    pool_dev = store.dev.pool()
    mine = dist.positions_device(n, pool_dev.device)
    if mine.numel():
        tmax = pool_dev[mine].contiguous()
        ftop, states = sw.sweep_device(tmax)
        tstar, best_s, _ = sw.select_device(ftop, tmax, num_microbatches)
        local = torch.stack([tstar.view(torch.int64), best_s.to(torch.int64), states], dim=1)
    else:
        local = torch.zeros((0, 3), dtype=torch.int64, device=pool_dev.device)
    full = dist.gather_positions(local, n)  # [n, 3] in pool order
    t_bits, bs = full[:, 0], full[:, 1]
    big = torch.iinfo(torch.int64).max
    key = torch.where(bs >= 0, t_bits, torch.full_like(t_bits, big))
    kmin = key.min()
    ar = torch.arange(n, dtype=torch.int64, device=key.device)
    win = torch.where(key == kmin, ar, torch.full_like(ar, big)).min()
    win = torch.where(kmin == big, torch.full_like(win, -1), win)
    host = torch.cat([pool_dev.view(torch.int64).to(full.device), full.t().reshape(-1),
                      win.reshape(1)]).cpu().numpy()
    return (host[:n].view(np.float64).copy(), host[n:2 * n].view(np.float64).copy(),
            host[2 * n:3 * n].copy(), host[3 * n:4 * n].copy(), int(host[4 * n]))


def _score(sweeper, ftop: np.ndarray, tmax: np.ndarray, B: int):
    """_extract_plan's choice of stage count (planner.py:287-296) and the
    sort_key merge (planner.py:107-115) for many candidates, on the device
    (hapt_dp_select over F[s,1,G] rows kept from the sweeps): first s with
    the strictly smallest F[s,1,G] + (B-1)*t_max over finite F.  Returns
    (T*, best_s, winner) -- best_s = -1 when infeasible, winner = index of the
    (T*, t_max) minimum (rows in t_max order) or -1."""
    import torch

    dev = sweeper.device
    f = torch.from_numpy(np.ascontiguousarray(ftop, dtype=np.float64)).to(dev)
    t = torch.from_numpy(np.ascontiguousarray(tmax, dtype=np.float64)).to(dev)
    tstar, best_s, winner = sweeper.select_device(f, t, B)
    host = torch.cat([tstar.view(torch.int64), best_s.to(torch.int64),
                      winner.to(torch.int64)]).cpu().numpy()
    n = len(tmax)
    return host[:n].view(np.float64).copy(), host[n:2 * n].copy(), int(host[2 * n])


def search_batches(store: ProfileStore, costs: BoundaryCost, batch_sizes: Sequence[int],
                   epsilon: float = 0.05, batch_size: Optional[int] = None,
                   optimized: bool = True, dist=None) -> dict:
    """search() for several microbatch counts from one set of DP sweeps
    (SURVEY.md §8(f)3).  The DP tables F, N (_dp.pyx:48-95) depend on t_max
    only, so every candidate is swept once and scored for each B afterwards
    (T_B = min_s F[s,1,G] + (B-1) t_max).  Feasibility is B-independent, so
    the reference's binary search (planner.py:456-474) is replayed once; each
    B then keeps its own t_e cut and merge.  Returns {B: plan}; every plan and
    its search_stats (but wall_time_s, which is the shared total) equal
    search(store, costs, B, epsilon, batch_size=batch_size, optimized=...).
    `dist` (PoolSharding) shards every batch across ranks as in search()."""
    began = time.perf_counter()
    Bs = [int(b) for b in batch_sizes]
    if not Bs or min(Bs) < 1:
        raise PlannerError("batch sizes must be positive integers")
    tables = DpTables(store, costs)
    pool = candidate_tmax(store)
    n = len(pool)
    ev = CandidateEvaluator(tables, pool, Bs[0], dist=dist, keep_ftop=True)
    if optimized:
        lo, _, _, probed = bidirectional_prune_replay(ev, Bs[0])
        t_lo = np.array([pool[lo]])
        cuts = {}
        for B in Bs:
            ts_lo, _, _ = _score(tables.sweeper, ev.ftop[[lo]], t_lo, B)
            cuts[B] = float(ts_lo[0]) / (B - 1) if B > 1 else math.inf
        t_cut = max(cuts.values())
        ev.ensure([i for i in range(lo, n) if pool[i] <= t_cut])
    else:
        lo, probed, cuts = 0, [], {B: math.inf for B in Bs}
        ev.ensure(range(n))
    transitions = tables.transitions_per_sweep()
    plans = {}
    for B in Bs:
        t_e = cuts[B]
        surviving = [i for i in range(lo, n) if pool[i] <= t_e]
        idx = np.asarray(surviving, dtype=np.int64)
        if len(idx) == 0:
            raise InfeasiblePlanError(
                "no stage partition satisfies the memory and overlap constraints")
        tstar, best_s, k = _score(tables.sweeper, ev.ftop[idx], ev.pool[idx], B)
        if k < 0:
            raise InfeasiblePlanError(
                "no stage partition satisfies the memory and overlap constraints")
        plan = ev.plan(surviving[k], epsilon, B=B, best_s=int(best_s[k]), tstar=float(tstar[k]))
        if optimized:
            surv_t = [pool[i] for i in surviving]
            n_batches = _count_batches(surv_t, _activated_pairs(tables, surv_t), batch_size)
            evaluated_set = set(probed) | set(surviving)
        else:
            n_batches, evaluated_set = 1, set(surviving)
        # states and feasibility do not depend on B
        states = int(sum(int(ev.states[i]) for i in evaluated_set if ev.best_s[i] >= 0))
        plan.search_stats.update({
            "backend": BACKEND,
            "candidates_total": n,
            "pruned_below_ts": lo,
            "pruned_above_te": n - lo - len(surviving),
            "evaluated": len(surviving),
            "batches": n_batches,
            "t_low": pool[lo],
            "t_high": None if math.isinf(t_e) else float(t_e),
            "dp_states": states,
            "dp_transitions": transitions * len(surviving),
        })
        plans[B] = plan
    wall = time.perf_counter() - began
    for plan in plans.values():
        plan.search_stats["wall_time_s"] = wall
    return plans


def validate_plan(plan: ParallelPlan, store: ProfileStore, costs: BoundaryCost, cluster) -> list:
    """Independent constraint checker (planner.py:615-670)."""
    problems = []
    L = store.num_layers
    cursor = 1
    for st in plan.stages:
        if st.layer_start != cursor:
            problems.append(f"stage gap before layer {st.layer_start}")
        cursor = st.layer_end + 1
    if cursor != L + 1:
        problems.append("stages do not cover the layer sequence")
    used: dict = {}
    order = -1
    for st in plan.stages:
        idx = cluster.mesh_order(st.mesh_id)
        if idx < order:
            problems.append(f"stage on {st.mesh_id} violates mesh order")
        order = max(order, idx)
        used[st.mesh_id] = used.get(st.mesh_id, 0) + st.device_count
    for mesh in cluster.meshes:
        if used.get(mesh.id, 0) != mesh.device_count:
            problems.append(f"mesh {mesh.id}: {used.get(mesh.id, 0)} devices used of "
                            f"{mesh.device_count}")
    for st in plan.stages:
        prof = store.lookup(st.layer_start, st.layer_end, st.mesh_id, st.submesh)
        if not prof.feasible:
            problems.append(f"stage [{st.layer_start},{st.layer_end}] uses a pruned candidate")
        if prof.t > plan.t_max:
            problems.append(f"stage [{st.layer_start},{st.layer_end}]: t {prof.t:.6g} over bound")
        cap = cluster.mesh(st.mesh_id).mem_device
        if prof.mem_params + st.dp_launch_bound * prof.mem_act > cap:
            problems.append(f"stage [{st.layer_start},{st.layer_end}]: memory over budget")
    for idx, b in enumerate(plan.boundaries):
        expected = costs.get(b.after_layer, plan.stages[idx].mesh_id, plan.stages[idx + 1].mesh_id)
        if not math.isclose(b.comm, expected, rel_tol=1e-9, abs_tol=1e-15):
            problems.append(f"boundary {idx + 1}: comm cost mismatch")
        if b.comm > plan.t_max:
            problems.append(f"boundary {idx + 1}: comm over t_max")
    return problems


def plan_to_dict(plan: ParallelPlan) -> dict:
    return {
        "num_microbatches": plan.num_microbatches,
        "t_max": plan.t_max,
        "predicted_latency": plan.predicted_latency,
        "eta_pct": plan.eta_pct,
        "epsilon": plan.epsilon,
        "stages": [
            {
                "layers": [s.layer_start, s.layer_end],
                "mesh": s.mesh_id,
                "submesh": [s.n, s.m],
                "t_fwd": s.t_fwd,
                "t_bwd": s.t_bwd,
                "mem_params": s.mem_params,
                "mem_act": s.mem_act,
                "launch_count": s.launch_count,
                "dp_launch_bound": s.dp_launch_bound,
            }
            for s in plan.stages
        ],
        "boundaries": [
            {"after_layer": b.after_layer, "comm": b.comm, "link": b.link} for b in plan.boundaries
        ],
        "search_stats": dict(plan.search_stats),
    }


def plan_from_dict(data: dict) -> ParallelPlan:
    """Inverse of plan_to_dict for plan.yaml files (planner.py:702-747):
    optional fields default as the reference's, a malformed file raises
    PlannerError, and a "colocated" boundary carries no transfer time."""
    def stage(d):
        lo, hi = d["layers"][0], d["layers"][1]
        n, m = d["submesh"][0], d["submesh"][1]
        return PlanStage(int(lo), int(hi), str(d["mesh"]), int(n), int(m), float(d["t_fwd"]),
                         float(d["t_bwd"]), float(d.get("mem_params", 0.0)),
                         float(d.get("mem_act", 0.0)), int(d.get("launch_count", 1)),
                         int(d.get("dp_launch_bound", 1)))

    def boundary(d):
        link = str(d.get("link", ""))
        comm = float(d["comm"])  # required even when colocated
        return PlanBoundary(int(d["after_layer"]), 0.0 if link == "colocated" else comm, link)

    try:
        stages = [stage(d) for d in data["stages"]]
        boundaries = [boundary(d) for d in data.get("boundaries", [])]
    except (KeyError, TypeError, IndexError) as exc:
        raise PlannerError(f"malformed plan file: {exc}") from exc
    if len(boundaries) != len(stages) - 1:
        raise PlannerError("plan needs one boundary per adjacent stage pair")
    return ParallelPlan(
        stages=stages, boundaries=boundaries,
        t_max=float(data.get("t_max", max(s.t for s in stages))),
        num_microbatches=int(data.get("num_microbatches", 1)),
        predicted_latency=float(data.get("predicted_latency", 0.0)),
        eta_pct=float(data.get("eta_pct", 0.0)),
        epsilon=float(data.get("epsilon", 0.05)),
        search_stats=dict(data.get("search_stats", {})))


_REPORT_STATS = ("backend", "candidates_total", "pruned_below_ts", "pruned_above_te",
                 "evaluated", "batches", "dp_states")


def plan_report(plan: ParallelPlan) -> str:
    """Human-readable plan summary printed by `meshpipe plan` (planner.py:750-786);
    same text as the reference."""
    out = [f"stages: {plan.num_stages}   t_max: {plan.t_max:.6g} s   "
           f"T*: {plan.predicted_latency:.6g} s (B={plan.num_microbatches})   "
           f"eta: {plan.eta_pct:.1f}%",
           "stage  layers      submesh           t/mb        N   K"]
    for idx, st in enumerate(plan.stages, start=1):
        head = f"{idx:>5d}  [{st.layer_start:>3d},{st.layer_end:>3d}]  {st.mesh_id}({st.n},{st.m})"
        out.append(f"{head:<32}{st.t:<10.6g}  {st.launch_count:<3d} {st.dp_launch_bound}")
    out += [f"  boundary {idx}: after layer {b.after_layer}, {b.comm:.6g} s ({b.link})"
            for idx, b in enumerate(plan.boundaries, start=1)]
    stats = plan.search_stats
    if stats:
        out.append("search: " + ", ".join(f"{k}={stats[k]}" for k in _REPORT_STATS if k in stats))
        if "wall_time_s" in stats:
            out.append(f"wall time: {stats['wall_time_s']:.3f} s")
    return "\n".join(out) + "\n"
