"""Operator sequences, repeated-module detection, layer clustering
(meshpipe.model_graph, model_graph.py:1-411).

The planner hot path only reads, per layer, `flops`, `param_bytes`,
`boundary_bytes` and `signature` (profiling.py:201-224, 135); reference
LayerSequence objects are accepted unchanged by the rest of this package.
This module also provides the front end that builds them -- SURVEY.md
§8(f)1, the next wall-clock bottleneck of `meshpipe plan` (16-26 s of pure
Python at 2,006 ops): `detect_modules` and `cluster_layers` run in native
C++ (csrc/hapt_frontend.cpp, host code) with results identical to the
reference (tests/test_frontend_cpu.py); types, validation, error messages
and the synthetic GPT generator are the reference's.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

HEAVY = "heavy"
LIGHT = "light"


class ModelGraphError(ValueError):
    pass


class GranularityError(ModelGraphError):
    """Requested more layers than a module has operators."""


@dataclass(frozen=True)
class OperatorNode:
    index: int
    kind: str
    flops: float
    param_bytes: float
    out_activation_bytes: float
    shape_tag: str

    def __post_init__(self):
        if self.kind not in (HEAVY, LIGHT):
            raise ModelGraphError(f"operator {self.index}: unknown kind {self.kind!r}")
        if self.flops < 0 or self.param_bytes < 0 or self.out_activation_bytes < 0:
            raise ModelGraphError(f"operator {self.index}: negative cost field")


OperatorSequence = Sequence[OperatorNode]


@dataclass(frozen=True)
class ModuleSpan:
    start: int
    end: int
    kind: str  # "repeated" or "non_repeated"
    group_id: int = -1
    occurrence: int = 0

    def __len__(self):
        return self.end - self.start


@dataclass(frozen=True)
class Layer:
    op_start: int
    op_end: int
    flops: float
    param_bytes: float
    boundary_bytes: float
    signature: tuple

    def __len__(self):
        return self.op_end - self.op_start


@dataclass(frozen=True)
class LayerSequence:
    layers: tuple
    module_spans: tuple = ()

    def __len__(self):
        return len(self.layers)

    def validate(self, ops: OperatorSequence) -> None:
        cursor = 0
        for layer in self.layers:
            if layer.op_start != cursor:
                raise ModelGraphError("layers do not partition the operator sequence")
            cursor = layer.op_end
        if cursor != len(ops):
            raise ModelGraphError("layers do not cover the operator sequence")
        seen: dict = {}
        for layer in self.layers:
            agg = (layer.flops, layer.param_bytes, layer.boundary_bytes)
            if seen.setdefault(layer.signature, agg) != agg:
                raise ModelGraphError(
                    f"layers with signature {layer.signature} disagree on aggregates")


def validate_operator_sequence(ops: OperatorSequence) -> None:
    if not ops:
        raise ModelGraphError("empty operator sequence")
    for pos, op in enumerate(ops):
        if op.index != pos:
            raise ModelGraphError(f"operator indices not contiguous at position {pos}")


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def detect_modules(ops: OperatorSequence, z: int = 1) -> list:
    """Repeated / non-repeated module partition (model_graph.py:169-208),
    computed by the native front end."""
    from ._lib import check_host, host_lib

    validate_operator_sequence(ops)
    if z < 1:
        raise ModelGraphError("z must be >= 1")
    ids: dict = {}
    tags = np.array([ids.setdefault(op.shape_tag, len(ids)) for op in ops], dtype=np.int32)
    heavy = np.array([op.kind == HEAVY for op in ops], dtype=np.uint8)
    n = len(ops)
    out = np.zeros((4, n), dtype=np.int32)
    cnt = np.zeros(1, dtype=np.int32)
    check_host(host_lib().hapt_detect_modules(n, _p(tags), _p(heavy), int(z), _p(out[0]),
                                              _p(out[1]), _p(out[2]), _p(out[3]), _p(cnt)))
    spans = []
    for j in range(int(cnt[0])):
        s, e, grp, occ = (int(x) for x in out[:, j])
        spans.append(ModuleSpan(s, e, "repeated", grp, occ) if grp >= 0
                     else ModuleSpan(s, e, "non_repeated"))
    return spans


def validate_module_spans(spans: Iterable[ModuleSpan], ops: OperatorSequence) -> None:
    cursor = 0
    groups: dict = {}
    for span in spans:
        if span.start != cursor:
            raise ModelGraphError("module spans do not partition the sequence")
        cursor = span.end
        if span.kind == "repeated":
            groups.setdefault(span.group_id, []).append(span)
    if cursor != len(ops):
        raise ModelGraphError("module spans do not cover the sequence")
    for gid, members in groups.items():
        ref = [ops[i].shape_tag for i in range(members[0].start, members[0].end)]
        for span in members[1:]:
            if [ops[i].shape_tag for i in range(span.start, span.end)] != ref:
                raise ModelGraphError(f"group {gid} occurrences differ in shape tags")


def cluster_layers(spans: Sequence[ModuleSpan], ops: OperatorSequence,
                   layers_per_module_unit: int = 1) -> LayerSequence:
    """u layers per module by min-max flops partition; occurrences of a
    repeated group share the first occurrence's cuts (model_graph.py:269-333),
    computed by the native front end."""
    from ._lib import check_host, host_lib

    if layers_per_module_unit < 1:
        raise ModelGraphError("layers_per_module_unit must be >= 1")
    validate_module_spans(spans, ops)
    u = layers_per_module_unit
    for span in spans:
        if u > len(span):
            name = (f"repeated module g{span.group_id}#{span.occurrence}"
                    if span.kind == "repeated" else "non-repeated module")
            raise GranularityError(
                f"{name} at ops [{span.start},{span.end}) has {len(span)} operators,"
                f" cannot form {u} layers")
    n = len(ops)
    f = np.array([op.flops for op in ops], dtype=np.float64)
    pb = np.array([op.param_bytes for op in ops], dtype=np.float64)
    ob = np.array([op.out_activation_bytes for op in ops], dtype=np.float64)
    ss = np.array([s.start for s in spans], dtype=np.int32)
    se = np.array([s.end for s in spans], dtype=np.int32)
    sg = np.array([s.group_id if s.kind == "repeated" else -1 for s in spans], dtype=np.int32)
    cap = n
    li = np.zeros((2, cap), dtype=np.int32)
    ld = np.zeros((3, cap), dtype=np.float64)
    sig = np.zeros((cap, 3), dtype=np.int32)
    cnt = np.zeros(1, dtype=np.int32)
    check_host(host_lib().hapt_cluster_layers(
        n, _p(f), _p(pb), _p(ob), len(spans), _p(ss), _p(se), _p(sg), int(u), _p(li[0]),
        _p(li[1]), _p(ld[0]), _p(ld[1]), _p(ld[2]), _p(sig), _p(cnt)))
    layers = []
    for j in range(int(cnt[0])):
        kind = "rep" if sig[j, 0] == 0 else "solo"
        layers.append(Layer(int(li[0, j]), int(li[1, j]), float(ld[0, j]), float(ld[1, j]),
                            float(ld[2, j]), (kind, int(sig[j, 1]), int(sig[j, 2]))))
    seq = LayerSequence(tuple(layers), tuple(spans))
    seq.validate(ops)
    return seq


# ---------------------------------------------------------------------------
# Synthetic GPT-style workload generator (model_graph.py:341-400)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class GptConfig:
    num_blocks: int
    hidden_dim: int
    seq_len: int
    mb_size: int = 1
    vocab: int = 32000

    def __post_init__(self):
        for name in ("num_blocks", "hidden_dim", "seq_len", "mb_size", "vocab"):
            if getattr(self, name) <= 0:
                raise ModelGraphError(f"gpt config: {name} must be positive")


def generate_gpt_sequence(cfg: GptConfig) -> list:
    """Deterministic transformer operator sequence: embedding prologue,
    num_blocks identical 11-op blocks (attention + MLP GEMMs heavy, norms /
    softmax / residual light), head epilogue; fp16 boundary activations of
    mb_size x seq_len x hidden_dim."""
    b, s, h, v = cfg.mb_size, cfg.seq_len, cfg.hidden_dim, cfg.vocab
    act = 2.0 * b * s * h
    light = float(b * s * h)
    seq = [
        (f"embed[{v}x{h}]", LIGHT, light, 2.0 * v * h),
        (f"pos_embed[{s}x{h}]", LIGHT, light, 2.0 * s * h),
        (f"embed_drop[{h}]", LIGHT, light, 0.0),
    ]
    block = [
        (f"ln1[{h}]", LIGHT, light, 4.0 * h),
        (f"qkv_proj[{h}x{3 * h}]", HEAVY, 6.0 * b * s * h * h, 2.0 * 3 * h * h),
        (f"attn_score[{s}x{s}]", HEAVY, 2.0 * b * s * s * h, 0.0),
        (f"attn_softmax[{s}]", LIGHT, light, 0.0),
        (f"attn_ctx[{s}x{h}]", HEAVY, 2.0 * b * s * s * h, 0.0),
        (f"out_proj[{h}x{h}]", HEAVY, 2.0 * b * s * h * h, 2.0 * h * h),
        (f"ln2[{h}]", LIGHT, light, 4.0 * h),
        (f"mlp_fc1[{h}x{4 * h}]", HEAVY, 8.0 * b * s * h * h, 2.0 * 4 * h * h),
        (f"gelu[{4 * h}]", LIGHT, light, 0.0),
        (f"mlp_fc2[{4 * h}x{h}]", HEAVY, 8.0 * b * s * h * h, 2.0 * 4 * h * h),
        (f"residual[{h}]", LIGHT, light, 0.0),
    ]
    seq += block * cfg.num_blocks
    seq += [
        (f"final_ln[{h}]", LIGHT, light, 4.0 * h),
        (f"lm_head[{h}x{v}]", HEAVY, 2.0 * b * s * h * v, 2.0 * v * h),
        (f"loss[{v}]", LIGHT, light, 0.0),
    ]
    return [OperatorNode(i, kind, fl, pb, act, tag) for i, (tag, kind, fl, pb) in enumerate(seq)]


def gpt_param_bytes_estimate(cfg: GptConfig) -> float:
    h, v = cfg.hidden_dim, cfg.vocab
    return 2.0 * (12.0 * cfg.num_blocks * h * h + 2.0 * v * h)


def layers_to_text(seq: LayerSequence) -> str:
    rows = ["# layer  ops        flops          params_bytes   boundary_bytes  signature"]
    for idx, layer in enumerate(seq.layers, start=1):
        rows.append(f"{idx:>7d}  [{layer.op_start},{layer.op_end})  {layer.flops:.6e}  "
                    f"{layer.param_bytes:.6e}  {layer.boundary_bytes:.6e}  {layer.signature}")
    return "\n".join(rows) + "\n"


# ---------------------------------------------------------------------------
# Direct constructors (instances stored as per-layer arrays)
# ---------------------------------------------------------------------------


def layers_from_arrays(flops, param_bytes, boundary_bytes, signatures) -> LayerSequence:
    """A LayerSequence from per-layer arrays (one op per layer)."""
    n = len(flops)
    if not (len(param_bytes) == len(boundary_bytes) == len(signatures) == n) or n == 0:
        raise ModelGraphError("per-layer arrays must be non-empty and equally long")
    out = []
    for i in range(n):
        sig = signatures[i]
        sig = tuple(sig) if isinstance(sig, (list, tuple)) else (sig,)
        out.append(Layer(i, i + 1, float(flops[i]), float(param_bytes[i]),
                         float(boundary_bytes[i]), sig))
    return LayerSequence(tuple(out))


def uniform_layers(n: int, flops: float, params: float, act: float) -> LayerSequence:
    """n structurally identical layers: what detect_modules + cluster_layers
    give for n equal-tag heavy operators at one layer per module."""
    sig = ("rep", 0, 0)
    return LayerSequence(tuple(Layer(i, i + 1, flops, params, act, sig) for i in range(n)))
