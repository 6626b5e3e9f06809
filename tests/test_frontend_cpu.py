"""CPU: the native model-graph front end (csrc/hapt_frontend.cpp) rebuilds
the reference's layer sequences exactly, and passes the reference's own
model_graph tests (pkg/tests/test_model_graph.py)."""

import itertools
import math
import random
import time

import pytest

from helpers import load_json
from paper_2509_24859_b200.model_graph import (
    HEAVY,
    LIGHT,
    GptConfig,
    GranularityError,
    Layer,
    ModelGraphError,
    OperatorNode,
    cluster_layers,
    detect_modules,
    generate_gpt_sequence,
    gpt_param_bytes_estimate,
    validate_module_spans,
)
from paper_2509_24859_b200.workloads import config_ops


@pytest.mark.parametrize("name", ["A", "B", "C", "D1", "D2", "D3"])
def test_config_layers_equal_reference(name):
    """The golden instances hold the reference front end's output for each
    config; ours must match field for field (float equality)."""
    ops, u = config_ops(name)
    t0 = time.perf_counter()
    seq = cluster_layers(detect_modules(ops), ops, u)
    dt = time.perf_counter() - t0
    lay = load_json(name)["layers"]
    assert len(seq) == len(lay["flops"])
    assert [l.flops for l in seq.layers] == lay["flops"]
    assert [l.param_bytes for l in seq.layers] == lay["param_bytes"]
    assert [l.boundary_bytes for l in seq.layers] == lay["boundary_bytes"]
    assert [list(l.signature) for l in seq.layers] == lay["signature"]
    if name.startswith("D"):
        assert dt < 5.0, dt  # reference: 16-26 s


def test_python_sum_semantics():
    """Layer aggregates are CPython sums (compensated on >= 3.12)."""
    import ctypes

    import numpy as np

    from paper_2509_24859_b200._lib import host_lib

    rng = random.Random(5)
    for _ in range(200):
        xs = [rng.choice([1e16, -1e16, 1.0, rng.uniform(-1e6, 1e6), rng.random() * 1e-8])
              for _ in range(rng.randint(1, 30))]
        a = np.array(xs, dtype=np.float64)
        assert host_lib().hapt_py_sum(a.ctypes.data, len(xs)) == sum(xs)


# -- the reference's own tests (pkg/tests/test_model_graph.py) ---------------


def make_ops(tags, kinds=None, flops=None):
    kinds = kinds or [HEAVY] * len(tags)
    flops = flops or [1.0] * len(tags)
    return [OperatorNode(i, kinds[i], flops[i], 1.0, 1.0, tags[i]) for i in range(len(tags))]


def census_best(tags, kinds, z=1):
    """Brute-force winner under most-frequent / longest / earliest (the
    reference's tests/oracles.py census, restated)."""
    n = len(tags)
    best = None
    seen = set()
    for length in range(1, n + 1):
        for start in range(n - length + 1):
            pat = tuple(tags[start:start + length])
            if pat in seen:
                continue
            seen.add(pat)
            if sum(1 for k in kinds[start:start + length] if k == HEAVY) < z:
                continue
            c = pos = 0
            while pos + length <= n:
                if tuple(tags[pos:pos + length]) == pat:
                    c, pos = c + 1, pos + length
                else:
                    pos += 1
            if c < 2:
                continue
            first = next(i for i in range(n - length + 1) if tuple(tags[i:i + length]) == pat)
            key = (c, length, -first)
            if best is None or key > best[0]:
                best = (key, pat)
    return None if best is None else best[1]


def min_max_partition_value(values, parts):
    n = len(values)
    best = math.inf
    for cuts in itertools.combinations(range(1, n), parts - 1):
        b = [0, *cuts, n]
        best = min(best, max(sum(values[b[i]:b[i + 1]]) for i in range(parts)))
    return best


def test_all_distinct_yields_single_span():
    spans = detect_modules(make_ops(["a", "b", "c", "d", "e"]), z=1)
    assert len(spans) == 1 and spans[0].kind == "non_repeated"
    assert (spans[0].start, spans[0].end) == (0, 5)


def test_gpt_like_blocks():
    block = ["ln", "qkv", "score", "softmax", "ctx", "proj"]
    tags = ["embed", "pos"] + block * 4 + ["head", "loss"]
    kinds = [LIGHT, LIGHT] + ([LIGHT, HEAVY, HEAVY, LIGHT, HEAVY, HEAVY] * 4) + [HEAVY, LIGHT]
    spans = detect_modules(make_ops(tags, kinds), z=1)
    rep = [s for s in spans if s.kind == "repeated"]
    assert len(rep) == 4 and len({s.group_id for s in rep}) == 1
    assert len([s for s in spans if s.kind == "non_repeated"]) == 2
    assert census_best(tags, kinds, z=1) == tuple(block)


def test_abab_prefers_longer_pattern():
    spans = detect_modules(make_ops(["a", "b", "a", "b"]), z=1)
    assert [(s.kind, s.start, s.end) for s in spans] == [("repeated", 0, 2), ("repeated", 2, 4)]


def test_partition_property_and_census_random():
    rng = random.Random(7)
    for _ in range(60):
        n = rng.randint(1, 40)
        tags = [rng.choice("abcd") for _ in range(n)]
        ops = make_ops(tags)
        spans = detect_modules(ops, z=1)
        validate_module_spans(spans, ops)
        rep = [s for s in spans if s.kind == "repeated" and s.group_id == 0]
        want = census_best(tags, [HEAVY] * n)
        if want is None:
            assert not rep
        else:
            assert tuple(tags[rep[0].start:rep[0].end]) == want


def test_z_rules():
    spans = detect_modules(make_ops(["x", "y"] * 3, kinds=[LIGHT] * 6), z=1)
    assert all(s.kind == "non_repeated" for s in spans)
    tags = ["h", "x", "h", "h", "x", "h"]
    spans = detect_modules(make_ops(tags, [HEAVY, LIGHT, HEAVY] * 2), z=2)
    assert [(s.start, s.end) for s in spans if s.kind == "repeated"] == [(0, 3), (3, 6)]


def test_cluster_layers_reference_cases():
    seq = cluster_layers(detect_modules(make_ops(["a", "b", "c", "d"])), make_ops(["a", "b", "c", "d"]), 2)
    assert [l.flops for l in seq.layers] == [2, 2]
    ops = make_ops(["a", "b", "c", "d"], flops=[3, 1, 1, 3])
    assert [l.flops for l in cluster_layers(detect_modules(ops), ops, 2).layers] == [4, 4]
    ops = generate_gpt_sequence(GptConfig(4, 512, 512))
    seq = cluster_layers(detect_modules(ops), ops, 2)
    blocks = [l for l in seq.layers if l.signature[0] == "rep"]
    assert len(blocks) == 8 and len({l.signature for l in blocks}) == 2
    rng = random.Random(11)
    for _ in range(30):
        n = rng.randint(2, 12)
        parts = rng.randint(1, n)
        fl = [rng.randint(1, 9) for _ in range(n)]
        ops = make_ops([f"u{i}" for i in range(n)], flops=fl)
        seq = cluster_layers(detect_modules(ops), ops, parts)
        assert max(l.flops for l in seq.layers) == min_max_partition_value(fl, parts)
    with pytest.raises(GranularityError, match="non-repeated module"):
        ops = make_ops(["a", "b"])
        cluster_layers(detect_modules(ops), ops, 3)


def test_generator_and_invariants():
    ops = generate_gpt_sequence(GptConfig(2, 128, 64))
    spans = detect_modules(ops)
    assert len({s.group_id for s in spans if s.kind == "repeated"}) == 1
    cfg = GptConfig(8, 1024, 1024, vocab=32000)
    total = sum(op.param_bytes for op in generate_gpt_sequence(cfg))
    assert math.isclose(total, gpt_param_bytes_estimate(cfg), rel_tol=0.01)
    with pytest.raises(ModelGraphError):
        GptConfig(0, 64, 64)
    with pytest.raises(ModelGraphError):
        OperatorNode(0, "medium", 1.0, 1.0, 1.0, "x")
    with pytest.raises(ModelGraphError):
        detect_modules([OperatorNode(1, HEAVY, 1.0, 1.0, 1.0, "x")])
    assert len(Layer(2, 5, 1.0, 1.0, 1.0, ("solo", 0, 0))) == 3
