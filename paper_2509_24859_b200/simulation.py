"""Exact 1F1B schedule evaluation on the GPU (meshpipe.simulation, simulation.py:1-479).

`simulate(build_dag(...))` returns the reference's ScheduleTrace, but the
start times come from the hapt_sim_1f1b kernel, which walks each stage's
program with per-link FIFOs instead of materialising the DAG (the reference's
dominant per-plan cost).  The DAG's successor/predecessor
lists are only built if a caller reads them; if they were read (and possibly
edited, as the reference's cycle test does), simulate() runs the generic
frontier kernel hapt_dag_longest_path over the current lists instead, with
the reference's CycleError diagnosis.

`simulate_batch` is the config-E workload: makespans of many plans in one
launch.  `analyze` / `steady_state_rate` / `asap_tight` of a trace run on the
device over the trace's node times (hapt_analyze_1f1b, hapt_steady_rate_1f1b,
hapt_dag_asap_check), as do the batched reports (`analyze_batch`,
`PlanBatch.analyze`); trace export (`trace_events`, `trace_to_text`) is
host-side formatting of the wire formats.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from .scheduling import FWD, StageProgram

NODE_F = 0
NODE_B = 1
NODE_CF = 2
NODE_CB = 3
NODE_SINK = 4

_KIND_NAMES = {NODE_F: "F", NODE_B: "B", NODE_CF: "CF", NODE_CB: "CB", NODE_SINK: "sink"}


class SimulationError(ValueError):
    pass


class CycleError(SimulationError):
    def __init__(self, cycle: list):
        self.cycle = cycle
        super().__init__("dependency cycle: " + " -> ".join(cycle))


def _node_id(kind: int, mb: int, stage: int, S: int, B: int) -> int:
    """Reference node numbering (simulation.py:103-111)."""
    if kind == NODE_F or kind == NODE_B:
        return 2 * ((stage - 1) * B + (mb - 1)) + (kind == NODE_B)
    if kind == NODE_CF or kind == NODE_CB:
        return 2 * S * B + 2 * ((stage - 1) * B + (mb - 1)) + (kind == NODE_CB)
    return 2 * S * B + 2 * (S - 1) * B


class PipelineDag:
    """Execution DAG of a 1F1B pipeline with lazily materialised edges."""

    def __init__(self, t_fwd, t_bwd, comm, program: StageProgram):
        self.num_stages = len(t_fwd)
        self.num_microbatches = program.num_microbatches
        self.program = program
        self.t_fwd = [float(x) for x in t_fwd]
        self.t_bwd = [float(x) for x in t_bwd]
        self.comm = [float(x) for x in comm]
        self._succ = None
        self._pred = None
        self._duration = None
        self._meta = None

    # -- structure ------------------------------------------------------------
    @property
    def num_nodes(self) -> int:
        S, B = self.num_stages, self.num_microbatches
        return B * (2 * S + 2 * (S - 1)) + 1

    @property
    def sink(self) -> int:
        return self.num_nodes - 1

    def node_id(self, kind: int, mb: int, stage: int) -> int:
        S, B = self.num_stages, self.num_microbatches
        if kind == NODE_SINK:
            return self.sink
        top = S if kind in (NODE_F, NODE_B) else S - 1
        if not (1 <= stage <= top and 1 <= mb <= B):
            raise KeyError((kind, mb, stage))
        return _node_id(kind, mb, stage, S, B)

    @property
    def meta(self) -> list:
        if self._meta is None:
            S, B = self.num_stages, self.num_microbatches
            meta = []
            for s in range(1, S + 1):
                for i in range(1, B + 1):
                    meta += [(NODE_F, i, s), (NODE_B, i, s)]
            for s in range(1, S):
                for i in range(1, B + 1):
                    meta += [(NODE_CF, i, s), (NODE_CB, i, s)]
            meta.append((NODE_SINK, 0, 0))
            self._meta = meta
        return self._meta

    @property
    def duration(self) -> list:
        if self._duration is None:
            S, B = self.num_stages, self.num_microbatches
            d = []
            for s in range(S):
                d += [self.t_fwd[s], self.t_bwd[s]] * B
            for s in range(S - 1):
                d += [self.comm[s], self.comm[s]] * B
            d.append(0.0)
            self._duration = d
        return self._duration

    def node_name(self, node: int) -> str:
        kind, mb, stage = self.meta[node]
        if kind == NODE_SINK:
            return "sink"
        return f"{_KIND_NAMES[kind]}[{mb},{stage}]"

    def _materialise(self) -> None:
        S, B = self.num_stages, self.num_microbatches
        n = self.num_nodes
        succ = [[] for _ in range(n)]
        pred = [[] for _ in range(n)]

        def link(u, v):
            succ[u].append(v)
            pred[v].append(u)

        nid = lambda k, i, s: _node_id(k, i, s, S, B)  # noqa: E731
        for s in range(1, S + 1):  # program order per stage (simulation.py:121-127)
            prev = None
            for kind, mb in self.program.stages[s - 1].ops:
                v = nid(NODE_F if kind == FWD else NODE_B, mb, s)
                if prev is not None:
                    link(prev, v)
                prev = v
        for s in range(1, S):  # serial transfers per direction (130-133)
            for i in range(1, B):
                link(nid(NODE_CF, i, s), nid(NODE_CF, i + 1, s))
                link(nid(NODE_CB, i, s), nid(NODE_CB, i + 1, s))
        for s in range(1, S):  # cross-stage dependencies (136-141)
            for i in range(1, B + 1):
                link(nid(NODE_F, i, s), nid(NODE_CF, i, s))
                link(nid(NODE_CF, i, s), nid(NODE_F, i, s + 1))
                link(nid(NODE_B, i, s + 1), nid(NODE_CB, i, s))
                link(nid(NODE_CB, i, s), nid(NODE_B, i, s))
        for v in range(n - 1):
            if not succ[v]:
                link(v, n - 1)
        self._succ, self._pred = succ, pred

    @property
    def succ(self) -> list:
        if self._succ is None:
            self._materialise()
        return self._succ

    @property
    def pred(self) -> list:
        if self._pred is None:
            self._materialise()
        return self._pred

    @property
    def edges_materialised(self) -> bool:
        return self._succ is not None


def build_dag(t_fwd: Sequence[float], t_bwd: Sequence[float], comm: Sequence[float],
              program: StageProgram) -> PipelineDag:
    """Validate and describe the pipeline DAG (simulation.py:73-149); edges
    are not built unless read."""
    S = len(t_fwd)
    if len(t_bwd) != S or len(comm) != S - 1 or len(program.stages) != S:
        raise SimulationError("inconsistent stage/boundary dimensions")
    if any(d < 0 for d in list(t_fwd) + list(t_bwd) + list(comm)):
        raise SimulationError("durations must be non-negative")
    return PipelineDag(t_fwd, t_bwd, comm, program)


@dataclass
class ScheduleTrace:
    dag: PipelineDag
    start: list
    end: list
    makespan: float

    @property
    def num_stages(self) -> int:
        return self.dag.num_stages

    def node_interval(self, kind: int, mb: int, stage: int) -> tuple:
        v = self.dag.node_id(kind, mb, stage)
        return self.start[v], self.end[v]

    def stage_op_nodes(self, stage: int) -> list:
        return [
            self.dag.node_id(NODE_F if kind == FWD else NODE_B, mb, stage)
            for kind, mb in self.dag.program.stages[stage - 1].ops
        ]


def _find_cycle(dag: PipelineDag, remaining: set) -> list:
    """Error-path diagnosis, same walk as simulation.py:176-201."""
    state = {v: 0 for v in remaining}
    stack: list = []

    def dfs(v):
        state[v] = 1
        stack.append(v)
        for w in dag.succ[v]:
            if w not in state:
                continue
            if state[w] == 1:
                return stack[stack.index(w):] + [w]
            if state[w] == 0:
                got = dfs(w)
                if got:
                    return got
        state[v] = 2
        stack.pop()
        return None

    for v in remaining:
        if state[v] == 0:
            got = dfs(v)
            if got:
                return [dag.node_name(x) for x in got]
    return []


def _simulate_general(dag: PipelineDag) -> ScheduleTrace:
    import torch

    from . import _lib
    from ._lib import check, stream_ptr

    lib = _lib.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    n = dag.num_nodes
    succ = dag.succ
    off = np.zeros(n + 1, dtype=np.int32)
    off[1:] = np.cumsum([len(s) for s in succ])
    idx = np.fromiter((v for s in succ for v in s), dtype=np.int32, count=int(off[-1]))
    indeg = np.array([len(p) for p in dag.pred], dtype=np.int32)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    d_off, d_idx, d_indeg = T(off), T(idx if len(idx) else np.zeros(1, np.int32)), T(indeg)
    d_dur = T(np.asarray(dag.duration, dtype=np.float64))
    start = torch.empty(n, dtype=torch.float64, device=dev)
    end = torch.empty(n, dtype=torch.float64, device=dev)
    mk = torch.empty(1, dtype=torch.float64, device=dev)
    processed = torch.empty(1, dtype=torch.int32, device=dev)
    ws = torch.empty(lib.hapt_dag_workspace_bytes(n), dtype=torch.uint8, device=dev)
    check(lib.hapt_dag_longest_path(n, d_off.data_ptr(), d_idx.data_ptr(), d_indeg.data_ptr(),
                                    d_dur.data_ptr(), start.data_ptr(), end.data_ptr(),
                                    mk.data_ptr(), processed.data_ptr(), ws.data_ptr(),
                                    ws.numel(), stream_ptr()))
    if int(processed.item()) != n:
        left = ws[: n * 4].view(torch.int32).cpu().numpy()
        raise CycleError(_find_cycle(dag, {v for v in range(n) if left[v] > 0}))
    return ScheduleTrace(dag, start.cpu().tolist(), end.cpu().tolist(), float(mk.item()))


def simulate(dag: PipelineDag) -> ScheduleTrace:
    """Earliest start times of every node (simulation.py:204-228), on the GPU."""
    if dag.edges_materialised:
        return _simulate_general(dag)
    S, B = dag.num_stages, dag.num_microbatches
    counts = dag.program.counts.counts
    mk, start, end, status = _sim_call(
        np.asarray([dag.t_fwd]), np.asarray([dag.t_bwd]),
        np.asarray([list(dag.comm) + [0.0]]), np.asarray([counts], dtype=np.int32),
        np.asarray([B], dtype=np.int32), want_nodes=True,
    )
    if int(status[0]) == 7:  # deadlocking program: let the generic kernel diagnose
        return _simulate_general(dag)
    if int(status[0]) != 0:
        raise SimulationError(f"simulation kernel rejected the program (status {int(status[0])})")
    return ScheduleTrace(dag, start.tolist(), end.tolist(), float(mk[0]))


def _sim_call(t_fwd, t_bwd, comm, counts, num_mb, want_nodes=False, stage_counts=None):
    import torch

    from . import _lib
    from ._lib import check, stream_ptr

    lib = _lib.lib()
    dev = (t_fwd.device if isinstance(t_fwd, torch.Tensor) and t_fwd.is_cuda
           else torch.device("cuda", torch.cuda.current_device()))
    T = lambda a, dt=torch.float64: torch.as_tensor(a, dtype=dt).to(dev).contiguous()  # noqa: E731
    tf, tb, cm = T(t_fwd), T(t_bwd), T(comm)
    cn = T(counts, torch.int32)
    P, S = tf.shape
    mb = T(num_mb, torch.int32).reshape(-1)
    if mb.numel() == 1 and P > 1:
        mb = mb.expand(P).contiguous()
    if stage_counts is None:
        off = torch.arange(0, (P + 1) * S, S, dtype=torch.int32, device=dev)
        ftf, ftb, fcm, fcn = tf.reshape(-1), tb.reshape(-1), cm.reshape(-1), cn.reshape(-1)
        total = P * S
    else:
        sc = T(stage_counts, torch.int32)
        off = torch.zeros(P + 1, dtype=torch.int32, device=dev)
        off[1:] = torch.cumsum(sc, 0)
        mask = torch.arange(S, device=dev)[None, :] < sc[:, None].long()
        ftf, ftb, fcm, fcn = (x[mask].contiguous() for x in (tf, tb, cm, cn))
        total = int(off[-1])
    ring = int(cn.max().item()) + 2
    ws = torch.empty(lib.hapt_sim_workspace_bytes(total, ring), dtype=torch.uint8, device=dev)
    mk = torch.empty(P, dtype=torch.float64, device=dev)
    status = torch.empty(P, dtype=torch.int32, device=dev)
    start = end = node_off = None
    if want_nodes:
        Sv = (off[1:] - off[:-1]).long()
        nodes = mb.long() * (4 * Sv - 2) + 1
        node_off = torch.zeros(P, dtype=torch.int64, device=dev)
        node_off[1:] = torch.cumsum(nodes, 0)[:-1]
        n_all = int(nodes.sum())
        start = torch.empty(n_all, dtype=torch.float64, device=dev)
        end = torch.empty(n_all, dtype=torch.float64, device=dev)
    check(lib.hapt_sim_1f1b(P, off.data_ptr(), ftf.data_ptr(), ftb.data_ptr(), fcm.data_ptr(),
                            fcn.data_ptr(), mb.data_ptr(), mk.data_ptr(),
                            0 if start is None else start.data_ptr(),
                            0 if end is None else end.data_ptr(),
                            0 if node_off is None else node_off.data_ptr(), ring,
                            status.data_ptr(), ws.data_ptr(), ws.numel(), stream_ptr()))
    if want_nodes:
        return mk.cpu().numpy(), start.cpu().numpy(), end.cpu().numpy(), status.cpu().numpy()
    return mk, status


class PlanBatch:
    """Many plans packed once on the device (plan p owns stages
    [stage_off[p], stage_off[p+1]); comm[stage_off[p] + j] is boundary j).
    Built from dense [P, S] arrays (+ optional per-plan stage counts)."""

    def __init__(self, t_fwd, t_bwd, comm, stage_counts=None, device=None):
        import torch

        dev = device or (t_fwd.device if isinstance(t_fwd, torch.Tensor) and t_fwd.is_cuda
                         else torch.device("cuda", torch.cuda.current_device()))
        T = lambda a, dt=torch.float64: torch.as_tensor(a, dtype=dt).to(dev).contiguous()  # noqa: E731
        tf, tb, cm = T(t_fwd), T(t_bwd), T(comm)
        P, S = tf.shape
        self.n_plans, self.width, self.device = P, S, dev
        if stage_counts is None:
            self.stage_off = torch.arange(0, (P + 1) * S, S, dtype=torch.int32, device=dev)
            self.t_fwd, self.t_bwd, self.comm = tf.reshape(-1), tb.reshape(-1), cm.reshape(-1)
            self.max_stages = S
        else:
            sc = T(stage_counts, torch.int32)
            self.stage_off = torch.zeros(P + 1, dtype=torch.int32, device=dev)
            self.stage_off[1:] = torch.cumsum(sc, 0)
            mask = torch.arange(S, device=dev)[None, :] < sc[:, None].long()
            self.t_fwd, self.t_bwd, self.comm = (x[mask].contiguous() for x in (tf, tb, cm))
            self.max_stages = int(sc.max().item())
        self.total_stages = int(self.t_fwd.numel())
        self.stage_off_host = self.stage_off.cpu().numpy().astype(np.int64)

    def counts(self, epsilon: float = 0.05, kind: str = "adaptive", tmax=None):
        """Packed launch counts (hapt_launch_counts) and per-plan status."""
        import torch

        from . import _lib
        from ._lib import check, stream_ptr

        counts = torch.empty(self.total_stages, dtype=torch.int32, device=self.device)
        status = torch.empty(self.n_plans, dtype=torch.int32, device=self.device)
        kind_id = {"classic": _lib.COUNTS_CLASSIC, "eager": _lib.COUNTS_EAGER,
                   "adaptive": _lib.COUNTS_ADAPTIVE}[kind]
        tm = None if tmax is None else torch.as_tensor(tmax, dtype=torch.float64).to(self.device)
        check(_lib.lib().hapt_launch_counts(
            self.n_plans, self.stage_off.data_ptr(), self.t_fwd.data_ptr(),
            self.t_bwd.data_ptr(), self.comm.data_ptr(), 0 if tm is None else tm.data_ptr(),
            float(epsilon), kind_id, counts.data_ptr(), status.data_ptr(), stream_ptr()))
        return counts, status

    def simulate(self, counts, num_microbatches, ring_depth: int | None = None):
        """Makespans (hapt_sim_1f1b) for packed counts; returns (makespan,
        status) CUDA tensors."""
        import torch

        from . import _lib
        from ._lib import check, stream_ptr

        lib = _lib.lib()
        mb = torch.as_tensor(num_microbatches, dtype=torch.int32).to(self.device).reshape(-1)
        if mb.numel() == 1 and self.n_plans > 1:
            mb = mb.expand(self.n_plans).contiguous()
        if ring_depth is None:  # generic-kernel FIFO depth >= N_1 + 1
            ring_depth = int(counts.max().item()) + 2
        nb = lib.hapt_sim_workspace_bytes(self.total_stages, ring_depth)
        ws = _sim_ws(self.device, nb)
        mk = torch.empty(self.n_plans, dtype=torch.float64, device=self.device)
        status = torch.empty(self.n_plans, dtype=torch.int32, device=self.device)
        check(lib.hapt_sim_1f1b(self.n_plans, self.stage_off.data_ptr(), self.t_fwd.data_ptr(),
                                self.t_bwd.data_ptr(), self.comm.data_ptr(), counts.data_ptr(),
                                mb.data_ptr(), mk.data_ptr(), 0, 0, 0, ring_depth,
                                status.data_ptr(), ws.data_ptr(), nb, stream_ptr()))
        return mk, status

    def analyze(self, counts, num_microbatches, mem_act=None,
                max_node_bytes: int = 4 << 30) -> "BatchReport":
        """simulate + analyze + steady_state_rate(stage=1) of every plan
        (SURVEY.md §8(f)2): per plan the reference's SimulationReport, as
        packed device arrays.  Plans are processed in chunks whose traces
        (16 B per DAG node: start and end) fit `max_node_bytes`; each chunk is
        one hapt_sim_1f1b_trace launch writing node times (trace layout: each
        stage's ops in program order, so stores fill whole sectors) and one
        hapt_analyze_1f1b_trace launch reading them back."""
        import torch

        from . import _lib
        from ._lib import check, ptr, stream_ptr

        lib = _lib.lib()
        dev = self.device
        P, TS = self.n_plans, self.total_stages
        mb = torch.as_tensor(num_microbatches, dtype=torch.int32).to(dev).reshape(-1)
        if mb.numel() == 1 and P > 1:
            mb = mb.expand(P).contiguous()
        mb_host = mb.cpu().numpy().astype(np.int64)
        counts = torch.as_tensor(counts, dtype=torch.int32).to(dev).reshape(-1).contiguous()
        if counts.numel() != TS:
            raise SimulationError("counts must hold one launch count per packed stage")
        mem = None
        if mem_act is not None:
            mem = torch.as_tensor(mem_act, dtype=torch.float64).to(dev).reshape(-1).contiguous()
            if mem.numel() != TS:
                raise SimulationError("mem_act must hold one value per packed stage")
        so = self.stage_off_host
        sc = np.diff(so)
        nodes = mb_host * (4 * sc - 2)  # B(4S-2) per plan + the sink (simulation.py:103-111)
        rep = BatchReport(
            stage_off=self.stage_off,
            makespan=torch.empty(P, dtype=torch.float64, device=dev),
            status=torch.empty(P, dtype=torch.int32, device=dev),
            stage=torch.empty(TS, 6, dtype=torch.float64, device=dev),
            peak_inflight=torch.empty(TS, dtype=torch.int32, device=dev),
            link=torch.empty(TS, 3, dtype=torch.float64, device=dev),
            steady_rate=torch.empty(P, dtype=torch.float64, device=dev))
        ring = int(counts.max().item()) + 2
        cap = max(1, int(max_node_bytes) // 16)
        cum = np.concatenate([[0], np.cumsum(nodes)])  # chunk = longest run within cap
        p0 = 0
        while p0 < P:
            p1 = max(p0 + 1, int(np.searchsorted(cum, cum[p0] + cap, side="right")) - 1)
            n = int(cum[p1] - cum[p0])
            s0, s1 = int(so[p0]), int(so[p1])
            off = (self.stage_off[p0:p1 + 1] - s0).contiguous()
            noff = torch.zeros(p1 - p0, dtype=torch.int64, device=dev)
            if p1 - p0 > 1:
                noff[1:] = torch.from_numpy(np.cumsum(nodes[p0:p1 - 1])).to(dev)
            trace = torch.empty(2 * max(n, 1), dtype=torch.float64, device=dev)
            nb = lib.hapt_sim_workspace_bytes(s1 - s0, ring)
            ws = _sim_ws(dev, nb)
            sl = lambda t: t[s0:s1]  # noqa: E731
            check(lib.hapt_sim_1f1b_trace(
                p1 - p0, off.data_ptr(), ptr(sl(self.t_fwd)), ptr(sl(self.t_bwd)),
                ptr(sl(self.comm)), ptr(sl(counts)), ptr(mb[p0:p1]), ptr(rep.makespan[p0:p1]),
                trace.data_ptr(), noff.data_ptr(), ring, ptr(rep.status[p0:p1]),
                ws.data_ptr(), nb, stream_ptr()))
            check(lib.hapt_analyze_1f1b_trace(
                p1 - p0, s1 - s0, off.data_ptr(), ptr(sl(self.t_fwd)), ptr(sl(self.t_bwd)),
                ptr(sl(self.comm)), ptr(sl(counts)), ptr(mb[p0:p1]),
                0 if mem is None else ptr(sl(mem)), trace.data_ptr(),
                noff.data_ptr(), ptr(rep.status[p0:p1]), ptr(rep.stage[s0:s1]),
                ptr(rep.peak_inflight[s0:s1]), ptr(rep.link[s0:s1]),
                ptr(rep.steady_rate[p0:p1]), stream_ptr()))
            p0 = p1
        return rep


@dataclass
class BatchReport:
    """Packed per-plan schedule reports (device tensors).  Plan p owns rows
    [stage_off[p], stage_off[p+1]) of `stage` (busy, window, bubble,
    bubble_fraction, steady_bubble, peak_inflight_bytes), `peak_inflight`
    and `link` (fwd_time, bwd_time, overlap_ratio of the boundary after the
    stage; NaN on the last stage).  steady_rate[p] is steady_state_rate(trace,
    1), NaN where the reference raises.  status[p] != 0: simulation failed."""

    stage_off: object
    makespan: object
    status: object
    stage: object
    peak_inflight: object
    link: object
    steady_rate: object

    def report(self, p: int) -> "SimulationReport":
        """Plan p as the reference's SimulationReport (analyze() output)."""
        a, b = int(self.stage_off[p]), int(self.stage_off[p + 1])
        if int(self.status[p]) != 0:
            raise SimulationError(f"plan {p}: simulation failed (status {int(self.status[p])})")
        st = self.stage[a:b].cpu().numpy()
        pk = self.peak_inflight[a:b].cpu().numpy()
        ln = self.link[a:b].cpu().numpy()
        stages = [StageReport(s + 1, float(st[s, 0]), float(st[s, 1]), float(st[s, 2]),
                              float(st[s, 3]), float(st[s, 4]), int(pk[s]), float(st[s, 5]))
                  for s in range(b - a)]
        links = [LinkReport(s + 1, float(ln[s, 0]), float(ln[s, 1]), float(ln[s, 2]))
                 for s in range(b - a - 1)]
        return SimulationReport(float(self.makespan[p]), stages, links)

    def steady_state_rate(self, p: int) -> float:
        v = float(self.steady_rate[p])
        if math.isnan(v):
            raise SimulationError("steady window too short: need >= 3 blocks of microbatches")
        return v


_SIM_WS: dict = {}


def _sim_ws(device, nbytes):
    import torch

    key = (device, torch.cuda.current_stream(device).cuda_stream)  # one per stream
    buf = _SIM_WS.get(key)
    if buf is None or buf.numel() < nbytes:
        _SIM_WS.pop(key, None)
        buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        _SIM_WS[key] = buf
    return buf


def simulate_batch(t_fwd, t_bwd, comm, counts, num_microbatches, stage_counts=None):
    """Makespans of many 1F1B plans in one launch (config E).

    t_fwd, t_bwd, comm, counts: [P, S] (comm[:, S-1] and entries past a plan's
    own stage count are ignored; ragged plans give `stage_counts` [P]).
    num_microbatches: scalar or [P].  Each makespan equals
    simulate(build_dag(...)).makespan bit for bit.  Returns (makespan, status)
    as CUDA tensors.
    """
    return _sim_call(t_fwd, t_bwd, comm, counts, num_microbatches, stage_counts=stage_counts)


def analyze_batch(t_fwd, t_bwd, comm, counts, num_microbatches, mem_act=None,
                  stage_counts=None) -> BatchReport:
    """analyze(simulate(build_dag(...)), mem_act) and steady_state_rate(...,
    stage=1) of many plans on the device (dense [P, S] inputs as
    simulate_batch; mem_act [P, S] or None).  BatchReport.report(p) equals the
    reference's SimulationReport for plan p, float for float."""
    import torch

    pb = PlanBatch(t_fwd, t_bwd, comm, stage_counts=stage_counts)
    dev = pb.device
    cn = torch.as_tensor(counts, dtype=torch.int32).to(dev)
    mem = None if mem_act is None else torch.as_tensor(mem_act, dtype=torch.float64).to(dev)
    if stage_counts is None:
        cn = cn.reshape(-1)
        mem = None if mem is None else mem.reshape(-1)
    else:
        sc = torch.as_tensor(stage_counts, dtype=torch.int32).to(dev)
        mask = torch.arange(cn.shape[1], device=dev)[None, :] < sc[:, None].long()
        cn = cn[mask]
        mem = None if mem is None else mem[mask]
    return pb.analyze(cn, num_microbatches, mem_act=mem)


# ---------------------------------------------------------------------------
# Analysis of one trace (simulation.py:268-424): the report dataclasses are
# the reference's API types; every figure comes from the device kernels
# (hapt_analyze_1f1b / hapt_steady_rate_1f1b / hapt_dag_asap_check) over the
# trace's own node times.
# ---------------------------------------------------------------------------


@dataclass
class StageReport:
    stage: int
    busy: float
    window: float
    bubble: float
    bubble_fraction: float
    steady_bubble: float
    peak_inflight: int
    peak_inflight_bytes: float


@dataclass
class LinkReport:
    boundary: int
    fwd_time: float
    bwd_time: float
    overlap_ratio: float


@dataclass
class SimulationReport:
    makespan: float
    stages: list
    links: list

    def to_text(self) -> str:
        lines = [f"makespan: {self.makespan:.6g} s",
                 "stage  busy        bubble      steady-bubble  peak-inflight"]
        for r in self.stages:
            lines.append(f"{r.stage:>5d}  {r.busy:<10.6g}  {r.bubble:<10.6g}  "
                         f"{r.steady_bubble:<13.6g}  {r.peak_inflight}")
        if self.links:
            lines.append("link   comm-fwd    comm-bwd    overlap")
            for l in self.links:
                lines.append(f"{l.boundary:>4d}>  {l.fwd_time:<10.6g}  {l.bwd_time:<10.6g}  "
                             f"{l.overlap_ratio:.3f}")
        return "\n".join(lines) + "\n"


class _TraceDev:
    """One trace on the device: the plan's stage arrays and the trace's node
    times in the reference numbering (plan count 1, node_off 0)."""

    def __init__(self, trace: ScheduleTrace, with_end: bool = True):
        import torch

        dag = trace.dag
        dev = torch.device("cuda", torch.cuda.current_device())
        T = lambda a, dt=torch.float64: torch.as_tensor(np.asarray(a), dtype=dt).to(dev)  # noqa: E731
        S = dag.num_stages
        self.S, self.B, self.dev = S, dag.num_microbatches, dev
        self.off = T([0, S], torch.int32)
        self.t_fwd, self.t_bwd = T(dag.t_fwd), T(dag.t_bwd)
        self.comm = T(list(dag.comm) + [0.0])
        self.counts = T(dag.program.counts.counts, torch.int32)
        self.mb = T([self.B], torch.int32)
        self.node_off = T([0], torch.int64)
        self.start = T(trace.start)
        self.end = T(trace.end) if with_end else None


def analyze(trace: ScheduleTrace, mem_act_per_stage=None) -> SimulationReport:
    """Per-stage busy / bubble / steady bubble / peak in-flight and per-link
    overlap of one trace (simulation.py:310-371): hapt_analyze_1f1b over the
    trace's node times, one plan."""
    import torch

    from . import _lib
    from ._lib import check, stream_ptr

    td = _TraceDev(trace)
    S, dev = td.S, td.dev
    mem = None
    if mem_act_per_stage:  # the reference's `if mem_act_per_stage` (else bytes 0.0)
        mem = torch.as_tensor([float(x) for x in mem_act_per_stage[:S]], dtype=torch.float64,
                              device=dev)
    out = torch.empty(S * 6 + S * 3 + 1, dtype=torch.float64, device=dev)
    peak = torch.empty(S, dtype=torch.int32, device=dev)
    check(_lib.lib().hapt_analyze_1f1b(
        1, S, td.off.data_ptr(), td.t_fwd.data_ptr(), td.t_bwd.data_ptr(), td.comm.data_ptr(),
        td.counts.data_ptr(), td.mb.data_ptr(), 0 if mem is None else mem.data_ptr(),
        td.start.data_ptr(), td.end.data_ptr(), td.node_off.data_ptr(), None,
        out.data_ptr(), peak.data_ptr(), out[S * 6:].data_ptr(), out[S * 9:].data_ptr(),
        stream_ptr()))
    h = out.cpu().numpy()
    pk = peak.cpu().numpy()
    st = h[: S * 6].reshape(S, 6)
    ln = h[S * 6: S * 9].reshape(S, 3)
    stages = [StageReport(s + 1, float(st[s, 0]), float(st[s, 1]), float(st[s, 2]),
                          float(st[s, 3]), float(st[s, 4]), int(pk[s]), float(st[s, 5]))
              for s in range(S)]
    links = [LinkReport(s + 1, float(ln[s, 0]), float(ln[s, 1]), float(ln[s, 2]))
             for s in range(S - 1)]
    return SimulationReport(trace.makespan, stages, links)


def steady_state_rate(trace: ScheduleTrace, stage: int = 1) -> float:
    """Least-squares time per microbatch of the steady block starts of one
    stage (simulation.py:374-395), on the device (hapt_steady_rate_1f1b)."""
    import torch

    from . import _lib
    from ._lib import check, stream_ptr

    dag = trace.dag
    K = dag.program.counts.counts[stage - 1]  # IndexError past the last stage, as the reference
    if len(range(2 * K + 1, dag.num_microbatches + 1, K)) < 4:
        raise SimulationError(f"steady window too short: need >= 3 blocks of {K} microbatches")
    if not 1 <= int(stage) <= dag.num_stages:
        raise KeyError((NODE_F, 2 * K + 1, stage))  # the reference's node-id lookup
    td = _TraceDev(trace, with_end=False)
    rs = torch.tensor([int(stage)], dtype=torch.int32, device=td.dev)
    out = torch.empty(1, dtype=torch.float64, device=td.dev)
    check(_lib.lib().hapt_steady_rate_1f1b(
        1, td.off.data_ptr(), td.counts.data_ptr(), td.mb.data_ptr(), td.start.data_ptr(),
        td.node_off.data_ptr(), rs.data_ptr(), None, out.data_ptr(), stream_ptr()))
    return float(out.item())


def steady_block_span(trace: ScheduleTrace, stage: int, i: int) -> float:
    """start(F[i+K]) - start(F[i]) on a stage (simulation.py:398-404), K its
    launch count; the subtraction runs on the device like every other
    figure of a trace."""
    import torch

    dag = trace.dag
    K = dag.program.counts.counts[stage - 1]
    a, b = dag.node_id(NODE_F, i + K, stage), dag.node_id(NODE_F, i, stage)
    t = torch.tensor([trace.start[a], trace.start[b]], dtype=torch.float64,
                     device=torch.device("cuda", torch.cuda.current_device()))
    return float((t[0] - t[1]).item())


def asap_tight(trace: ScheduleTrace, rel_tol: float = 1e-9) -> bool:
    """Every node starts as soon as its predecessors allow (simulation.py:
    407-424), checked on the device over the DAG's edges
    (hapt_dag_asap_check)."""
    import torch

    from . import _lib
    from ._lib import check, stream_ptr

    lib = _lib.lib()
    dag = trace.dag
    dev = torch.device("cuda", torch.cuda.current_device())
    n = dag.num_nodes
    succ = dag.succ
    off = np.zeros(n + 1, dtype=np.int32)
    off[1:] = np.cumsum([len(x) for x in succ])
    idx = np.fromiter((v for x in succ for v in x), dtype=np.int32, count=int(off[-1]))
    indeg = np.array([len(x) for x in dag.pred], dtype=np.int32)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    d_off, d_idx, d_indeg = T(off), T(idx if len(idx) else np.zeros(1, np.int32)), T(indeg)
    d_dur = T(np.asarray(dag.duration, dtype=np.float64))
    d_start = T(np.asarray(trace.start, dtype=np.float64))
    bad = torch.empty(1, dtype=torch.int32, device=dev)
    ws = torch.empty(lib.hapt_asap_workspace_bytes(n), dtype=torch.uint8, device=dev)
    check(lib.hapt_dag_asap_check(n, d_off.data_ptr(), d_idx.data_ptr(), d_indeg.data_ptr(),
                                  d_dur.data_ptr(), d_start.data_ptr(), float(rel_tol),
                                  bad.data_ptr(), ws.data_ptr(), ws.numel(), stream_ptr()))
    return int(bad.item()) >= n


def trace_events(trace: ScheduleTrace, labels=None) -> list:
    dag = trace.dag
    S = dag.num_stages
    dur = dag.duration
    events = []
    for v, (kind, mb, stage) in enumerate(dag.meta):
        if kind == NODE_SINK or dur[v] <= 0.0:
            continue
        if kind in (NODE_F, NODE_B):
            pid, tid = (labels[stage - 1] if labels else f"stage-{stage}"), stage
        elif kind == NODE_CF:
            pid, tid = f"link-{stage}>{stage + 1} fwd", S + 2 * stage - 1
        else:
            pid, tid = f"link-{stage}>{stage + 1} bwd", S + 2 * stage
        events.append({"name": f"{_KIND_NAMES[kind]}{mb}", "cat": _KIND_NAMES[kind], "ph": "X",
                       "pid": pid, "tid": tid, "ts": trace.start[v] * 1e6,
                       "dur": dur[v] * 1e6})
    return events


def write_trace_events(trace: ScheduleTrace, path, labels=None) -> None:
    with open(path, "w") as fh:
        json.dump({"traceEvents": trace_events(trace, labels)}, fh, indent=1)


def trace_to_text(trace: ScheduleTrace) -> str:
    dag = trace.dag
    lines = ["# node         start        end          duration"]
    for v in sorted(range(dag.num_nodes), key=lambda v: (trace.start[v], v)):
        if dag.meta[v][0] == NODE_SINK:
            continue
        lines.append(f"{dag.node_name(v):<12s}  {trace.start[v]:<11.6g}  {trace.end[v]:<11.6g}"
                     f"  {dag.duration[v]:.6g}")
    lines.append(f"makespan {trace.makespan:.6g}")
    return "\n".join(lines) + "\n"
