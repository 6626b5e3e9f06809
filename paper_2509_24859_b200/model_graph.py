"""Layer-sequence input types of the planner hot path.

The reference builds a LayerSequence from an operator graph with
detect_modules / cluster_layers (model_graph.py:169-333) -- a front end that
SURVEY.md §8(f) ranks as the next row to port, not part of this path.  The
planner only reads, per layer, `flops`, `param_bytes`, `boundary_bytes` and
`signature` (profiling.py:201-224, 135); these types carry exactly that, and
reference LayerSequence objects are accepted unchanged (duck typing).
"""

from __future__ import annotations

from dataclasses import dataclass


class ModelGraphError(ValueError):
    pass


@dataclass(frozen=True)
class Layer:
    op_start: int
    op_end: int
    flops: float
    param_bytes: float
    boundary_bytes: float
    signature: tuple


@dataclass(frozen=True)
class LayerSequence:
    layers: tuple
    module_spans: tuple = ()

    def __len__(self):
        return len(self.layers)


def layers_from_arrays(flops, param_bytes, boundary_bytes, signatures) -> LayerSequence:
    """Build a LayerSequence from per-layer arrays (one op per layer)."""
    n = len(flops)
    if not (len(param_bytes) == len(boundary_bytes) == len(signatures) == n) or n == 0:
        raise ModelGraphError("per-layer arrays must be non-empty and equally long")
    out = []
    for i in range(n):
        sig = signatures[i]
        sig = tuple(sig) if isinstance(sig, (list, tuple)) else (sig,)
        out.append(
            Layer(i, i + 1, float(flops[i]), float(param_bytes[i]), float(boundary_bytes[i]), sig)
        )
    return LayerSequence(tuple(out))


def uniform_layers(n: int, flops: float, params: float, act: float) -> LayerSequence:
    """n structurally identical layers: what the reference produces for n
    equal-tag heavy operators at one layer per module (all one signature)."""
    sig = ("rep", 0, 0)
    return LayerSequence(tuple(Layer(i, i + 1, flops, params, act, sig) for i in range(n)))
