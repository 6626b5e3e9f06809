"""Launch counts and 1F1B stage programs (meshpipe.scheduling, scheduling.py:1-262).

The counts themselves are computed by the hapt_launch_counts kernel -- one
thread per plan -- both for single plans (`adaptive_counts`, used by the
planner for its winner) and for millions of plans at once
(`launch_counts_batch`, config E).  Argument validation and error messages
follow the reference; programs (`build_program`) are host data structures of
the reference type consumed by `simulation.build_dag`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np

KINDS = ("classic", "eager", "adaptive")
FWD = "F"
BWD = "B"


class ScheduleError(ValueError):
    pass


class CommTooLargeError(ScheduleError):
    """Some boundary cost exceeds the slowest stage time."""

    def __init__(self, boundary: int, c: float, t_max: float):
        self.boundary = boundary
        self.c = c
        self.t_max = t_max
        super().__init__(
            f"boundary {boundary}: comm cost {c:.6g}s exceeds max stage time "
            f"{t_max:.6g}s; full overlap impossible"
        )


@dataclass(frozen=True)
class LaunchCounts:
    counts: tuple
    deltas: tuple
    kind: str

    @property
    def num_stages(self) -> int:
        return len(self.counts)

    def __post_init__(self):
        if not self.counts or self.counts[-1] != 1:
            raise ScheduleError("last stage must launch exactly one forward")
        for i in range(len(self.counts) - 1):
            if self.counts[i] != self.counts[i + 1] + self.deltas[i]:
                raise ScheduleError("counts and deltas are inconsistent")


def _from_deltas(deltas: Sequence[int], kind: str) -> LaunchCounts:
    counts = [1]
    for d in reversed(list(deltas)):
        counts.append(counts[-1] + d)
    return LaunchCounts(tuple(reversed(counts)), tuple(deltas), kind)


def classic_counts(num_stages: int) -> LaunchCounts:
    if num_stages < 1:
        raise ScheduleError("need at least one stage")
    return _from_deltas([1] * (num_stages - 1), "classic")


def eager_counts(num_stages: int) -> LaunchCounts:
    if num_stages < 1:
        raise ScheduleError("need at least one stage")
    return _from_deltas([2] * (num_stages - 1), "eager")


def _validate_adaptive(stage_times, comm_times, t_max):
    if len(stage_times) < 1:
        raise ScheduleError("need at least one stage")
    if len(comm_times) != len(stage_times) - 1:
        raise ScheduleError("expected one comm time per stage boundary")
    if any(t <= 0 for t in stage_times):
        raise ScheduleError("stage times must be positive")
    if any(c < 0 for c in comm_times):
        raise ScheduleError("comm times must be non-negative")
    slowest = max(stage_times)
    if t_max is None:
        return slowest
    if t_max < slowest:
        raise ScheduleError("t_max override below the slowest stage time")
    return t_max


def adaptive_counts(stage_times: Sequence[float], comm_times: Sequence[float],
                    epsilon: float = 0.05, t_max: float | None = None) -> LaunchCounts:
    """Communication-aware (H-1F1B) launch counts (scheduling.py:89-124),
    evaluated by the hapt_launch_counts kernel."""
    tm = _validate_adaptive(stage_times, comm_times, t_max)
    for i, c in enumerate(comm_times):
        if c > tm:
            raise CommTooLargeError(i + 1, c, tm)
    S = len(stage_times)
    # one plan: stage_times carried as t_fwd with t_bwd = 0 gives the same
    # t = t_fwd + 0.0 the kernel maxes over
    counts, status = launch_counts_batch(
        np.asarray(stage_times, dtype=np.float64)[None, :],
        np.zeros((1, S)),
        np.asarray(list(comm_times) + [0.0], dtype=np.float64)[None, :],
        epsilon=epsilon,
        tmax=None if t_max is None else np.array([t_max], dtype=np.float64),
        kind="adaptive",
    )
    if int(status[0]) != 0:
        raise ScheduleError(f"launch-count kernel rejected the plan (status {int(status[0])})")
    c = [int(x) for x in counts[0]]
    return LaunchCounts(tuple(c), tuple(c[i] - c[i + 1] for i in range(S - 1)), "adaptive")


def launch_counts_batch(t_fwd, t_bwd, comm, epsilon: float = 0.05, tmax=None,
                        kind: str = "adaptive", stage_counts=None, device=None):
    """Counts for many plans on the GPU.

    Dense form: t_fwd, t_bwd, comm are [P, S] (comm[:, S-1] unused) numpy or
    torch arrays; with `stage_counts` [P] plans may be ragged (entries past a
    plan's S are ignored).  Returns (counts [P, S] int32, status [P] int32)
    as numpy arrays, or torch CUDA tensors when the inputs are CUDA tensors.
    """
    import torch

    from . import _lib
    from ._lib import check, stream_ptr

    lib = _lib.lib()
    as_torch = isinstance(t_fwd, torch.Tensor) and t_fwd.is_cuda
    dev = t_fwd.device if as_torch else torch.device("cuda", torch.cuda.current_device())

    def T(x, dt=torch.float64):
        return torch.as_tensor(x, dtype=dt).to(dev).contiguous()

    tf, tb, cm = T(t_fwd), T(t_bwd), T(comm)
    P, S = tf.shape
    if stage_counts is None:
        off = torch.arange(0, (P + 1) * S, S, dtype=torch.int32, device=dev)
        flat = lambda x: x.reshape(-1)  # noqa: E731
    else:
        sc = T(stage_counts, torch.int32)
        off = torch.zeros(P + 1, dtype=torch.int32, device=dev)
        off[1:] = torch.cumsum(sc, 0)
        mask = torch.arange(S, device=dev)[None, :] < sc[:, None].long()
        flat = lambda x: x[mask]  # noqa: E731
    counts = torch.zeros(int(off[-1]) if stage_counts is not None else P * S,
                         dtype=torch.int32, device=dev)
    status = torch.empty(P, dtype=torch.int32, device=dev)
    tmx = None if tmax is None else T(tmax)
    kind_id = {"classic": _lib.COUNTS_CLASSIC, "eager": _lib.COUNTS_EAGER,
               "adaptive": _lib.COUNTS_ADAPTIVE}[kind]
    ftf, ftb, fcm = flat(tf).contiguous(), flat(tb).contiguous(), flat(cm).contiguous()
    check(lib.hapt_launch_counts(P, off.data_ptr(), ftf.data_ptr(), ftb.data_ptr(),
                                 fcm.data_ptr(), 0 if tmx is None else tmx.data_ptr(),
                                 float(epsilon), kind_id, counts.data_ptr(), status.data_ptr(),
                                 stream_ptr()))
    if stage_counts is None:
        counts = counts.view(P, S)
    if as_torch:
        return counts, status
    return counts.cpu().numpy(), status.cpu().numpy()


def analytic_delta(comm: float, stage_time: float) -> int:
    if stage_time <= 0:
        raise ScheduleError("stage time must be positive")
    return math.ceil(1.0 + 2.0 * comm / stage_time)


def delta_diagnostics(stage_times, comm_times, epsilon: float = 0.05, t_max=None) -> list:
    counts = adaptive_counts(stage_times, comm_times, epsilon, t_max=t_max)
    if t_max is None:
        t_max = max(stage_times)
    rows = []
    for i, c in enumerate(comm_times):
        applied = counts.deltas[i]
        analytic = analytic_delta(c, t_max) if c > 0 else 1
        rows.append({"boundary": i + 1, "comm": c, "applied_delta": applied,
                     "analytic_delta": analytic, "agrees": applied >= analytic})
    return rows


def memory_dominance_report(stage_times, comm_times, epsilon: float = 0.05) -> list:
    adaptive = adaptive_counts(stage_times, comm_times, epsilon)
    eager = eager_counts(len(stage_times))
    return [i + 1 for i, (a, e) in enumerate(zip(adaptive.counts, eager.counts)) if a > e]


@dataclass(frozen=True)
class StageOps:
    ops: tuple
    warmup: int
    steady: int


@dataclass(frozen=True)
class StageProgram:
    stages: tuple
    counts: LaunchCounts
    num_microbatches: int

    def validate(self) -> None:
        B = self.num_microbatches
        full = set(range(1, B + 1))
        for s, stage in enumerate(self.stages):
            fwd, bwd = set(), set()
            for kind, mb in stage.ops:
                if kind == FWD:
                    fwd.add(mb)
                else:
                    if mb not in fwd:
                        raise ScheduleError(f"stage {s + 1}: backward {mb} before its forward")
                    bwd.add(mb)
            if fwd != full or bwd != fwd:
                raise ScheduleError(f"stage {s + 1}: microbatch coverage broken")


def _stage_ops(n: int, B: int) -> tuple:
    """N warm-up forwards, (B_j, F_{N+j}) pairs, then the B drain
    (scheduling.py:241-249); the same order hapt_sim.cu:decode_op walks."""
    ops = [(FWD, j) for j in range(1, n + 1)]
    for j in range(1, B - n + 1):
        ops += [(BWD, j), (FWD, n + j)]
    ops += [(BWD, j) for j in range(B - n + 1, B + 1)]
    return tuple(ops)


def build_program(counts: LaunchCounts, num_microbatches: int) -> StageProgram:
    B = num_microbatches
    if B < counts.counts[0]:
        raise ScheduleError(
            f"batch of {B} microbatches smaller than warm-up launch count "
            f"{counts.counts[0]} of stage 1"
        )
    stages = tuple(StageOps(_stage_ops(n, B), warmup=n, steady=2 * (B - n)) for n in counts.counts)
    program = StageProgram(stages, counts, B)
    program.validate()
    return program


def program_to_text(program: StageProgram) -> str:
    out = []
    for s, stage in enumerate(program.stages, start=1):
        toks = [f"{kind}{mb}" for kind, mb in stage.ops]
        w, t = stage.warmup, stage.warmup + stage.steady
        body = " ".join(toks[:w]) + " | " + " ".join(toks[w:t]) + " | " + " ".join(toks[t:])
        out.append(f"stage {s} (N={program.counts.counts[s - 1]}): {body.strip(' |')}")
    return "\n".join(out) + "\n"
