"""Benchmark workloads of BASELINE.json as concrete synthetic inputs.

Configs A-D are planning instances: their layer sequences were produced once
by the reference front end (detect_modules + cluster_layers, out of scope for
this path) and stored with the cluster/model description in
tests/golden/instances/<name>.json (tests/golden/make_golden.py, SURVEY.md
Appendix B).  Config E is the seeded synthetic 1F1B plan generator.
"""

from __future__ import annotations

import json
import os

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INSTANCES = os.path.join(REPO, "tests", "golden", "instances")

CONFIGS = {
    "A": "GPT-2 small (12 layers), 4xA100 + 4xV100, 25 Gbps cross link, 8 microbatches",
    "B": "GPT-3 1.3B (24 layers), 8xA100 + 8xV100 + 8xT4, 10 Gbps, 32 microbatches",
    "C": "Llama-2 7B proxy (op-level, 102 layers), 4 subclusters x 16 GPUs, 25/10/5 Gbps, "
         "64 microbatches",
    "D1": "Llama-2 70B proxy (2,006-op graph, 82 layers), 4 subclusters x 64 GPUs, "
          "100/50/25 Gbps, 128 microbatches",
    "D2": "Llama-2 70B proxy (2,006-op graph, 164 layers), 4 subclusters x 64 GPUs, "
          "100/50/25 Gbps, 128 microbatches",
    "D3": "Llama-2 70B proxy (2,006-op graph, 246 layers), 4 subclusters x 64 GPUs, "
          "100/50/25 Gbps, 128 microbatches",
    "D4": "Llama-2 70B proxy blocks (2,000 ops, 320 layers: 2.26 M span-option cells), "
          "4 subclusters x 64 GPUs, 100/50/25 Gbps, 128 microbatches",
    "E": "1F1B schedule-simulation sweep: synthetic plans x 128 microbatches, "
         "S in {2,3,4,6,8}, cross bandwidth log-uniform 1-200 Gbps",
}


def instance_dict(name: str) -> dict:
    with open(os.path.join(INSTANCES, f"{name}.json")) as fh:
        return json.load(fh)


def instance(name: str):
    """(layers, cluster, model, imbalance_ratio, num_microbatches, epsilon)."""
    from .cluster import ClusterSpec, DeviceMesh
    from .model_graph import layers_from_arrays
    from .profiling import CostModel

    d = instance_dict(name)
    lay = d["layers"]
    layers = layers_from_arrays(lay["flops"], lay["param_bytes"], lay["boundary_bytes"],
                                [tuple(s) for s in lay["signature"]])
    meshes = [DeviceMesh(m["id"], m["hosts"], m["devices_per_host"], m["peak_flops"],
                         m["mem_device"], m["intra_host_bw"], m["inter_host_bw"])
              for m in d["cluster"]["meshes"]]
    cb = d["cluster"]["cross_bw"]
    if isinstance(cb, list):
        cb = {(a, b): v for a, b, v in cb}
    cluster = ClusterSpec(meshes, cross_bw=cb, cross_latency=d["cluster"]["cross_latency"])
    return (layers, cluster, CostModel(**d["model"]), float(d["imbalance_ratio"]),
            d["num_microbatches"], d["epsilon"])


def llama_like_ops(h=8192, s=4096, ffn=28672, vocab=32000, blocks=80, b=1) -> list:
    """Config D operator list: 3-op prologue, `blocks`
    x 25-op blocks, 3-op epilogue (2,006 ops); heavy ops carry 2*b*s*in*out
    flops.  Same recipe as tests/golden/make_golden.py (reference types)."""
    from .model_graph import HEAVY, LIGHT, OperatorNode

    act = 2.0 * b * s * h
    light = float(b * s * h)
    kv = h // 8
    ops = [(f"embed[{vocab}x{h}]", LIGHT, light, 2.0 * vocab * h),
           (f"scale[{h}]", LIGHT, light, 0.0),
           (f"embed_drop[{h}]", LIGHT, light, 0.0)]
    block = [
        (f"rms1[{h}]", LIGHT, light, 2.0 * h),
        (f"q[{h}x{h}]", HEAVY, 2.0 * b * s * h * h, 2.0 * h * h),
        (f"k[{h}x{kv}]", HEAVY, 2.0 * b * s * h * kv, 2.0 * h * kv),
        (f"v[{h}x{kv}]", HEAVY, 2.0 * b * s * h * kv, 2.0 * h * kv),
        (f"rope_q[{h}]", LIGHT, light, 0.0),
        (f"rope_k[{kv}]", LIGHT, float(b * s * kv), 0.0),
        (f"score[{s}x{s}]", HEAVY, 2.0 * b * s * s * h, 0.0),
        (f"mask[{s}]", LIGHT, light, 0.0),
        (f"softmax[{s}]", LIGHT, light, 0.0),
        (f"attn_drop[{s}]", LIGHT, light, 0.0),
        (f"ctx[{s}x{h}]", HEAVY, 2.0 * b * s * s * h, 0.0),
        (f"o[{h}x{h}]", HEAVY, 2.0 * b * s * h * h, 2.0 * h * h),
        (f"res1[{h}]", LIGHT, light, 0.0),
        (f"rms2[{h}]", LIGHT, light, 2.0 * h),
        (f"gate[{h}x{ffn}]", HEAVY, 2.0 * b * s * h * ffn, 2.0 * h * ffn),
        (f"up[{h}x{ffn}]", HEAVY, 2.0 * b * s * h * ffn, 2.0 * h * ffn),
        (f"silu[{ffn}]", LIGHT, float(b * s * ffn), 0.0),
        (f"mul[{ffn}]", LIGHT, float(b * s * ffn), 0.0),
        (f"down[{ffn}x{h}]", HEAVY, 2.0 * b * s * ffn * h, 2.0 * ffn * h),
        (f"res2[{h}]", LIGHT, light, 0.0),
        (f"cast[{h}]", LIGHT, light, 0.0),
        (f"drop[{h}]", LIGHT, light, 0.0),
        (f"stat[{h}]", LIGHT, light, 0.0),
        (f"id[{h}]", LIGHT, 0.0, 0.0),
        (f"id[{h}]", LIGHT, 0.0, 0.0),
    ]
    ops += block * blocks
    ops += [(f"final_rms[{h}]", LIGHT, light, 2.0 * h),
            (f"lm_head[{h}x{vocab}]", HEAVY, 2.0 * b * s * h * vocab, 2.0 * vocab * h),
            (f"loss[{vocab}]", LIGHT, light, 0.0)]
    return [OperatorNode(i, kind, fl, pb, act, tag) for i, (tag, kind, fl, pb) in enumerate(ops)]


def config_ops(name: str):
    """(operator list, layers per module unit) of configs A-D (SURVEY.md
    Appendix B)."""
    from .model_graph import GptConfig, generate_gpt_sequence

    if name == "A":
        return generate_gpt_sequence(GptConfig(12, 768, 1024, 1, 50257)), 1
    if name == "B":
        return generate_gpt_sequence(GptConfig(24, 2048, 2048, 1, 50257)), 1
    if name == "C":
        return generate_gpt_sequence(GptConfig(32, 4096, 4096, 1, 32000)), 3
    if name.startswith("D"):
        return llama_like_ops(), int(name[1:])
    raise KeyError(name)


def config_e(n_plans: int, seed: int = 24859):
    """Config E generator: S ~ {2,3,4,6,8}; stage time
    t ~ U(0.5, 2)e-2 s; forward share U(0.3, 0.4); boundary bandwidth
    log-uniform in [1, 200] Gbps; bytes ~ U(0,1) * t_max * 1.25e8 so every
    boundary satisfies c <= t_max.  Returns dense [P, 8] float64 t_fwd,
    t_bwd, comm (unused slots 0) and S [P] int32."""
    rng = np.random.default_rng(seed)
    S = rng.choice(np.array([2, 3, 4, 6, 8]), size=n_plans)
    t = rng.uniform(0.5, 2.0, size=(n_plans, 8)) * 1e-2
    f = t * rng.uniform(0.3, 0.4, size=(n_plans, 8))
    b = t - f
    live = np.arange(8)[None, :] < S[:, None]
    tm = np.where(live, f + b, 0.0).max(axis=1)
    bw = np.exp(rng.uniform(np.log(1.0), np.log(200.0), size=(n_plans, 8))) * 1.25e8
    nbytes = rng.uniform(0.0, 1.0, size=(n_plans, 8)) * tm[:, None] * 1.25e8
    comm = np.where(np.arange(8)[None, :] < (S[:, None] - 1), nbytes / bw, 0.0)
    return f, b, comm, S.astype(np.int32)
