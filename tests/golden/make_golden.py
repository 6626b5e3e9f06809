"""Golden-vector generator: runs the UNMODIFIED reference (meshpipe, built from
/root/reference into oracle/_ref by oracle/Makefile) on the benchmark configs
A-D of BASELINE.json and on the reference tests' own seeded instances, and
writes the instances plus the reference outputs under tests/golden/.

Runs only in the build container (it needs oracle/_ref/meshpipe).  Everything
it writes is committed; nothing on the GPU box imports the reference.

    python tests/golden/make_golden.py [--only A,B] [--skip-full-pool]

Instance recipes follow SURVEY.md Appendix B.  Config D's operator list is
defined here (25-op Llama-style blocks, 2,006 ops); detect_modules /
cluster_layers of the reference turn it into the layer sequence, which is
stored so the GPU side never needs the (out-of-scope) front end.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))

from meshpipe import BACKEND  # noqa: E402
from meshpipe._core import dp_sweep  # noqa: E402
from meshpipe.cluster import ClusterSpec, DeviceMesh  # noqa: E402
from meshpipe.model_graph import (  # noqa: E402
    HEAVY,
    LIGHT,
    GptConfig,
    OperatorNode,
    cluster_layers,
    detect_modules,
    generate_gpt_sequence,
)
from meshpipe.planner import (  # noqa: E402
    DpTables,
    _extract_plan,
    candidate_tmax,
    plan_to_dict,
    search,
)
from meshpipe.profiling import CostModel, boundary_costs, build_store  # noqa: E402

assert BACKEND == "cython", "build oracle/_ref first (make -C oracle ref)"

GB = 1e9


def gbps(x):
    return x * 1e9 / 8


def mesh(mid, kind, hosts, per_host):
    specs = {
        "a100": (312e12, 40 * GB, 300e9, gbps(200)),
        "v100": (125e12, 32 * GB, 150e9, gbps(200)),
        "t4": (65e12, 16 * GB, 32e9, gbps(100)),
        "h100": (989e12, 80 * GB, 900e9, gbps(400)),
    }
    peak, mem, intra, inter = specs[kind]
    return DeviceMesh(mid, hosts, per_host, peak, mem, intra, inter)


def llama_like_ops(h, s, ffn, vocab, blocks, b=1):
    """Config D operator list: 3-op prologue, `blocks` x 25-op blocks, 3-op
    epilogue.  Heavy ops carry 2*b*s*(in*out) flops."""
    act = 2.0 * b * s * h
    light = float(b * s * h)
    kv = h // 8
    ops = [
        (f"embed[{vocab}x{h}]", LIGHT, light, 2.0 * vocab * h),
        (f"scale[{h}]", LIGHT, light, 0.0),
        (f"embed_drop[{h}]", LIGHT, light, 0.0),
    ]
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
    for _ in range(blocks):
        ops.extend(block)
    ops += [
        (f"final_rms[{h}]", LIGHT, light, 2.0 * h),
        (f"lm_head[{h}x{vocab}]", HEAVY, 2.0 * b * s * h * vocab, 2.0 * vocab * h),
        (f"loss[{vocab}]", LIGHT, light, 0.0),
    ]
    return [
        OperatorNode(i, kind, fl, pb, act, tag)
        for i, (tag, kind, fl, pb) in enumerate(ops)
    ]


def config(name):
    """(layers, cluster, CostModel, rho, B, eps, description)"""
    model = CostModel()
    if name == "A":
        ops = generate_gpt_sequence(GptConfig(12, 768, 1024, 1, 50257))
        layers = cluster_layers(detect_modules(ops), ops, 1)
        cl = ClusterSpec([mesh("a100", "a100", 1, 4), mesh("v100", "v100", 1, 4)],
                         cross_bw=gbps(25))
        return layers, cl, model, 3.0, 8, 0.05, "GPT-2 small, 4xA100 + 4xV100, 25 Gbps, B=8"
    if name == "B":
        ops = generate_gpt_sequence(GptConfig(24, 2048, 2048, 1, 50257))
        layers = cluster_layers(detect_modules(ops), ops, 1)
        cl = ClusterSpec([mesh("a100", "a100", 1, 8), mesh("v100", "v100", 1, 8),
                          mesh("t4", "t4", 1, 8)], cross_bw=gbps(10))
        return layers, cl, model, 3.0, 32, 0.05, "GPT-3 1.3B, 8xA100 + 8xV100 + 8xT4, 10 Gbps, B=32"
    if name == "C":
        ops = generate_gpt_sequence(GptConfig(32, 4096, 4096, 1, 32000))
        layers = cluster_layers(detect_modules(ops), ops, 3)
        ids = ["s0", "s1", "s2", "s3"]
        kinds = ["a100", "a100", "v100", "v100"]
        meshes = [mesh(i, k, 2, 8) for i, k in zip(ids, kinds)]
        cross = {}
        adj = {("s0", "s1"): 25, ("s1", "s2"): 10, ("s2", "s3"): 5}
        for a in range(4):
            for b_ in range(a + 1, 4):
                cross[(ids[a], ids[b_])] = gbps(adj.get((ids[a], ids[b_]), 1))
        cl = ClusterSpec(meshes, cross_bw=cross)
        return layers, cl, model, 3.0, 64, 0.05, "Llama-2 7B proxy (u=3), 4 meshes x 16 GPUs, 25/10/5 Gbps, B=64"
    if name.startswith("D"):
        u = int(name[1:])
        ops = llama_like_ops(8192, 4096, 28672, 32000, 80)
        if u == 4:
            # the 3-op prologue/epilogue cannot form 4 layers (GranularityError):
            # the size-limit instance keeps the 80 blocks only -> 320 layers,
            # n_opts * L(L+1)/2 = 2.26 M (span, option) cells > 2^21
            ops = [OperatorNode(i, o.kind, o.flops, o.param_bytes, o.out_activation_bytes,
                                o.shape_tag)
                   for i, o in enumerate(ops[3:-3])]
        layers = cluster_layers(detect_modules(ops), ops, u)
        ids = ["s0", "s1", "s2", "s3"]
        kinds = ["h100", "a100", "a100", "v100"]
        meshes = [mesh(i, k, 8, 8) for i, k in zip(ids, kinds)]
        cross = {}
        adj = {("s0", "s1"): 100, ("s1", "s2"): 50, ("s2", "s3"): 25}
        for a in range(4):
            for b_ in range(a + 1, 4):
                cross[(ids[a], ids[b_])] = gbps(adj.get((ids[a], ids[b_]), 1))
        cl = ClusterSpec(meshes, cross_bw=cross)
        return (layers, cl, model, 3.0, 128, 0.05,
                f"Llama-2 70B proxy, {len(ops):,} ops, u={u}, 4 meshes x 64 GPUs, 100/50/25 Gbps, "
                f"B=128")
    raise KeyError(name)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def instance_json(name, layers, cl, model, rho, B, eps, desc):
    sig_ids: dict = {}
    sigs = []
    for l in layers.layers:
        sigs.append(sig_ids.setdefault(l.signature, len(sig_ids)))
    if isinstance(cl.cross_bw, dict):
        cross = [[a, b, v] for (a, b), v in sorted(cl.cross_bw.items())]
    else:
        cross = cl.cross_bw
    return {
        "name": name,
        "description": desc,
        "layers": {
            "flops": [l.flops for l in layers.layers],
            "param_bytes": [l.param_bytes for l in layers.layers],
            "boundary_bytes": [l.boundary_bytes for l in layers.layers],
            "sig": sigs,
            "signature": [list(l.signature) for l in layers.layers],
        },
        "cluster": {
            "meshes": [
                {
                    "id": m.id,
                    "hosts": m.hosts,
                    "devices_per_host": m.devices_per_host,
                    "peak_flops": m.peak_flops,
                    "mem_device": m.mem_device,
                    "intra_host_bw": m.intra_host_bw,
                    "inter_host_bw": m.inter_host_bw,
                }
                for m in cl.meshes
            ],
            "cross_bw": cross,
            "cross_latency": cl.cross_latency,
        },
        "model": {
            "beta": model.beta,
            "efficiency": model.efficiency,
            "alpha": model.alpha,
            "replication": model.replication,
            "act_factor": model.act_factor,
        },
        "imbalance_ratio": rho,
        "dedup": True,
        "num_microbatches": B,
        "epsilon": eps,
    }


def table_record(store, tables, pool):
    return {
        "stats": store.stats.as_dict(),
        "pool_len": len(pool),
        "L": tables.L,
        "G": tables.G,
        "s_max": tables.s_max,
        "n_opts": len(tables.opt_meta),
        "nnz": int(tables.span_off[-1]),
        "transitions_per_sweep": tables.transitions_per_sweep(),
        "sha": {
            "t_tab": sha(tables.t_tab),
            "mp_tab": sha(tables.mp_tab),
            "ma_tab": sha(tables.ma_tab),
            "cb_same": sha(tables.cb_same),
            "cb_next": sha(tables.cb_next),
            "span_off": sha(tables.span_off),
            "span_items": sha(tables.span_items),
            "g_mesh": sha(tables.g_mesh),
            "g_avail": sha(tables.g_avail),
            "pool": sha(np.asarray(pool, dtype=np.float64)),
        },
    }


def full_pool(tables, pool, B, eps, workers):
    """Reference per-candidate outcome over the whole pool: T* (inf when
    infeasible), best stage count, finite-cell count (dp_states)."""

    def one(t):
        F, N, bpi, bpo = dp_sweep(t, tables.t_tab, tables.mp_tab, tables.ma_tab,
                                  tables.opt_cap, tables.opt_mesh, tables.opt_devs,
                                  tables.opt_off, tables.cb_same, tables.cb_next,
                                  tables.g_mesh, tables.g_avail, tables.s_max,
                                  tables.span_off, tables.span_items)
        plan = _extract_plan(tables, F, N, bpi, bpo, t, B, eps)
        states = int(np.isfinite(F[1:]).sum())
        if plan is None:
            return math.inf, -1, states
        return plan.predicted_latency, plan.num_stages, states

    with ThreadPoolExecutor(workers) as ex:
        res = list(ex.map(one, pool))
    return (np.array([r[0] for r in res]), np.array([r[1] for r in res], dtype=np.int32),
            np.array([r[2] for r in res], dtype=np.int64))


def plan_record(plan):
    d = plan_to_dict(plan)
    d["search_stats"].pop("wall_time_s", None)
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="A,B,C,D1")
    ap.add_argument("--skip-full-pool", action="store_true")
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    args = ap.parse_args()
    out_dir = os.path.join(HERE, "instances")
    os.makedirs(out_dir, exist_ok=True)
    for name in args.only.split(","):
        t0 = time.time()
        layers, cl, model, rho, B, eps, desc = config(name)
        inst = instance_json(name, layers, cl, model, rho, B, eps, desc)
        with open(os.path.join(out_dir, f"{name}.json"), "w") as fh:
            json.dump(inst, fh)
        store = build_store(layers, cl, model, imbalance_ratio=rho)
        costs = boundary_costs(layers, cl)
        tables = DpTables(store, costs)
        pool = candidate_tmax(store)
        rec = {"name": name, "tables": table_record(store, tables, pool)}
        t1 = time.time()
        plan = search(store, costs, B, epsilon=eps, workers=args.workers, batch_size=4)
        rec["search_seconds_ref"] = time.time() - t1
        rec["plan"] = plan_record(plan)
        arrays = {"pool": np.asarray(pool)}
        if not args.skip_full_pool:
            t1 = time.time()
            tstar, best_s, states = full_pool(tables, pool, B, eps, args.workers)
            rec["full_pool_seconds_ref"] = time.time() - t1
            arrays.update(tstar=tstar, best_s=best_s, states=states)
        np.savez_compressed(os.path.join(out_dir, f"{name}_expected.npz"), **arrays)
        with open(os.path.join(out_dir, f"{name}_expected.json"), "w") as fh:
            json.dump(rec, fh, indent=1)
        print(f"{name}: L={tables.L} G={tables.G} pool={len(pool)} S={plan.num_stages} "
              f"T*={plan.predicted_latency!r} ({time.time() - t0:.1f}s)", flush=True)


if __name__ == "__main__":
    main()
