"""ORACLE -- TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference planner hot path (meshpipe; files under
/root/reference/pkg/src/meshpipe/), used ONLY by tests/, by
__graft_entry__.smoke() and by bench.py's cpu_baseline / `--impl reference`
leg, always as the checker or the CPU baseline -- never as the thing measured
or shipped.  The product package (paper_2509_24859_b200/) must not import it.

Numeric kernels are plain C (oracle/hapt_oracle.c, built by oracle/Makefile
into oracle/hapt_oracle.so); the search driver is restated here in Python.
Pinned against golden vectors the unmodified reference produced
(tests/golden/instances/*_expected.*, tests/test_oracle.py).

Instances are the plain-dict format of tests/golden/instances/<name>.json.
"""

from __future__ import annotations

import ctypes
import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "hapt_oracle.so")

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            import subprocess

            subprocess.run(["make", "-C", HERE, "hapt_oracle.so"], check=True,
                           capture_output=True)
        _lib = ctypes.CDLL(SO)
        P = ctypes.c_void_p
        i32, i64, d = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        _lib.oracle_dp_sweep.argtypes = [d] + [P] * 11 + [i32, P, P, i32, i32, P, P, P, P]
        _lib.oracle_dp_sweep.restype = None
        _lib.oracle_profile.argtypes = (
            [i32, P, P, P, P, i32, P, P, P, P, P, P, P] + [d] * 8 + [i32] + [P] * 7
        )
        _lib.oracle_profile.restype = None
        _lib.oracle_simulate.argtypes = [i32, i32, P, P, P, P, P, P, P]
        _lib.oracle_simulate.restype = ctypes.c_long
        _lib.oracle_adaptive_counts.argtypes = [i32, P, P, d, d, P]
        _lib.oracle_adaptive_counts.restype = i32
        _lib.oracle_config_e_batch.argtypes = [i64, i64, i32, P, P, P, P, d, P, P, P]
        _lib.oracle_config_e_batch.restype = None
    return _lib


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


# ---------------------------------------------------------------------------
# instance -> DpTables (profiling.py:88-286, planner.py:164-258, cluster.py:157-168)
# ---------------------------------------------------------------------------


def submeshes(mesh: dict) -> list:
    """enumerate_submeshes (cluster.py:157-168)."""
    shapes = []
    m = 1
    while m <= mesh["devices_per_host"]:
        shapes.append((1, m))
        m *= 2
    shapes += [(n, mesh["devices_per_host"]) for n in range(2, mesh["hosts"] + 1)]
    shapes.sort(key=lambda s: s[0] * s[1])
    return shapes


def cross_bw(inst: dict, a: str, b: str) -> float:
    cb = inst["cluster"]["cross_bw"]
    if isinstance(cb, list):
        key = tuple(sorted((a, b)))
        for x, y, v in cb:
            if tuple(sorted((x, y))) == key:
                return v
        raise KeyError(key)
    return cb


def comm_cost(inst: dict, i: int, a: str, b: str) -> float:
    """BoundaryCost.get over boundary_costs (profiling.py:120-147)."""
    lay = inst["layers"]
    L = len(lay["flops"])
    if i <= 0 or i >= L:
        return 0.0
    bb = lay["boundary_bytes"][i - 1]
    if a == b:
        mesh = next(m for m in inst["cluster"]["meshes"] if m["id"] == a)
        return bb / mesh["inter_host_bw"]
    return bb / cross_bw(inst, a, b) + inst["cluster"]["cross_latency"]


def tables(inst: dict) -> dict:
    lay = inst["layers"]
    meshes = inst["cluster"]["meshes"]
    model = inst["model"]
    L = len(lay["flops"])
    opts = [(mi, n, m) for mi, mesh in enumerate(meshes) for (n, m) in submeshes(mesh)]
    n_opts = len(opts)
    S = L + 2
    f64 = lambda x: np.ascontiguousarray(x, dtype=np.float64)  # noqa: E731
    i32 = lambda x: np.ascontiguousarray(x, dtype=np.int32)  # noqa: E731
    flops, params, bb = f64(lay["flops"]), f64(lay["param_bytes"]), f64(lay["boundary_bytes"])
    sig = i32(lay["sig"])
    opt_mesh = i32([o[0] for o in opts])
    opt_n = i32([o[1] for o in opts])
    opt_m = i32([o[2] for o in opts])
    peak = f64([m["peak_flops"] for m in meshes])
    mem = f64([m["mem_device"] for m in meshes])
    intra = f64([m["intra_host_bw"] for m in meshes])
    inter = f64([m["inter_host_bw"] for m in meshes])
    total_flops = sum(float(x) for x in lay["flops"])  # CPython sum, profiling.py:214
    total_peak = sum(m["hosts"] * m["devices_per_host"] * m["peak_flops"] for m in meshes)
    t = np.empty((n_opts, S, S))
    tf, tb, mp, ma = (np.empty((n_opts, S, S)) for _ in range(4))
    state = np.empty((n_opts, S, S), dtype=np.int8)
    stats = np.zeros(6, dtype=np.int64)
    lib().oracle_profile(
        L, _p(flops), _p(params), _p(bb), _p(sig), n_opts, _p(opt_mesh), _p(opt_n), _p(opt_m),
        _p(peak), _p(mem), _p(intra), _p(inter), model["beta"], model["efficiency"],
        model["alpha"], model["replication"], model["act_factor"],
        float(inst["imbalance_ratio"]), total_flops, total_peak, 1 if inst.get("dedup", True) else 0,
        _p(t), _p(tf), _p(tb), _p(mp), _p(ma), _p(state), _p(stats),
    )
    feasible = (state & 1).astype(bool)
    mp_tab = np.where(feasible, mp, np.inf)
    ma_tab = np.where(feasible, ma, np.inf)
    n_meshes = len(meshes)
    opt_off = np.zeros(n_meshes + 1, dtype=np.int32)
    for mi in range(n_meshes):
        opt_off[mi + 1] = opt_off[mi] + int((opt_mesh == mi).sum())
    cb_same = np.zeros((n_meshes, L + 1))
    cb_next = np.zeros((n_meshes, L + 1))
    for mi, mesh in enumerate(meshes):
        for i in range(1, L):
            cb_same[mi, i] = comm_cost(inst, i, mesh["id"], mesh["id"])
            if mi + 1 < n_meshes:
                cb_next[mi, i] = comm_cost(inst, i, mesh["id"], meshes[mi + 1]["id"])
    budgets = [m["hosts"] * m["devices_per_host"] for m in meshes]
    G = sum(budgets)
    suffix = [0] * (n_meshes + 1)
    for mi in range(n_meshes - 1, -1, -1):
        suffix[mi] = suffix[mi + 1] + budgets[mi]
    g_mesh = np.zeros(G + 1, dtype=np.int32)
    g_avail = np.zeros(G + 1, dtype=np.int32)
    for g in range(1, G + 1):
        for mi in range(n_meshes):
            if suffix[mi + 1] < g <= suffix[mi]:
                g_mesh[g], g_avail[g] = mi, g - suffix[mi + 1]
                break
    offs = np.zeros(n_opts * S + 1, dtype=np.int32)
    items = []
    for o in range(n_opts):
        for k in range(S):
            offs[o * S + k] = len(items)
            if 1 <= k <= L:
                items.extend(p for p in range(k, L + 1) if math.isfinite(t[o, k, p]))
    offs[n_opts * S] = len(items)
    canon_feasible = ((state & 3) == 3)
    pool = sorted({float(x) for x in t[canon_feasible]})
    return {
        "L": L, "G": G, "s_max": min(L, G), "n_opts": n_opts, "opts": opts,
        "opt_meta": [(meshes[o[0]]["id"], o[1], o[2]) for o in opts],
        "t_tab": t, "mp_tab": mp_tab, "ma_tab": ma_tab, "tf": tf, "tb": tb, "mp": mp, "ma": ma,
        "state": state, "stats": stats,
        "opt_cap": f64([mem[o[0]] for o in opts]), "opt_mesh": opt_mesh,
        "opt_devs": i32([o[1] * o[2] for o in opts]), "opt_off": opt_off,
        "cb_same": cb_same, "cb_next": cb_next, "g_mesh": g_mesh, "g_avail": g_avail,
        "span_off": offs,
        "span_items": np.array(items, dtype=np.int32) if items else np.zeros(1, dtype=np.int32),
        "pool": pool,
    }


def transitions_per_sweep(tb: dict) -> int:
    """DpTables.transitions_per_sweep (planner.py:250-258)."""
    S = tb["L"] + 2
    off = tb["span_off"]
    per = [int(off[(o + 1) * S] - off[o * S]) for o in range(tb["n_opts"])]
    tot = 0
    for g in range(1, tb["G"] + 1):
        r = int(tb["g_mesh"][g])
        for o in range(int(tb["opt_off"][r]), int(tb["opt_off"][r + 1])):
            if tb["opt_devs"][o] <= tb["g_avail"][g]:
                tot += per[o]
    return tot * tb["s_max"]


# ---------------------------------------------------------------------------
# DP + plan extraction (_dp.pyx, planner.py:272-421)
# ---------------------------------------------------------------------------


def dp_sweep(tb: dict, t_max: float):
    L, G, s_max = tb["L"], tb["G"], tb["s_max"]
    shape = (s_max + 1, L + 2, G + 1)
    F, N = np.empty(shape), np.empty(shape)
    bpi, bpo = np.empty(shape, dtype=np.int32), np.empty(shape, dtype=np.int32)
    lib().oracle_dp_sweep(
        float(t_max), _p(tb["t_tab"]), _p(tb["mp_tab"]), _p(tb["ma_tab"]), _p(tb["opt_cap"]),
        _p(tb["opt_mesh"]), _p(tb["opt_devs"]), _p(tb["opt_off"]), _p(tb["cb_same"]),
        _p(tb["cb_next"]), _p(tb["g_mesh"]), _p(tb["g_avail"]), s_max, _p(tb["span_off"]),
        _p(tb["span_items"]), L, G, _p(F), _p(N), _p(bpi), _p(bpo),
    )
    return F, N, bpi, bpo


def adaptive_counts(stage_t, comm, epsilon, t_max=None):
    S = len(stage_t)
    st = np.ascontiguousarray(stage_t, dtype=np.float64)
    cm = np.ascontiguousarray(list(comm) + [0.0], dtype=np.float64)
    out = np.zeros(S, dtype=np.int32)
    bad = lib().oracle_adaptive_counts(S, _p(st), _p(cm), float(epsilon),
                                       math.nan if t_max is None else float(t_max), _p(out))
    if bad:
        raise ValueError(f"comm of boundary {bad} exceeds t_max")
    return [int(x) for x in out]


def best_stage(F: np.ndarray, tb: dict, t_max: float, B: int):
    """best s and T* (planner.py:287-298)."""
    best_s, best_total = -1, math.inf
    for s in range(1, tb["s_max"] + 1):
        v = float(F[s, 1, tb["G"]])
        if not math.isfinite(v):
            continue
        total = v + (B - 1) * t_max
        if total < best_total:
            best_total, best_s = total, s
    return best_s, best_total


def extract(inst: dict, tb: dict, F, N, bpi, bpo, t_max: float, B: int, eps: float):
    """_extract_plan (planner.py:272-382) -> plan_to_dict layout, or None."""
    best_s, best_total = best_stage(F, tb, t_max, B)
    if best_s < 0:
        return None
    L, G = tb["L"], tb["G"]
    spans = []
    s, k, g = best_s, 1, G
    while s > 0:
        i, o = int(bpi[s, k, g]), int(bpo[s, k, g])
        assert i >= 0, "broken backpointer chain"
        spans.append((k, i, o))
        g -= int(tb["opt_devs"][o])
        k, s = i + 1, s - 1
    assert k == L + 1 and g == 0
    comm, links = [], []
    for idx in range(len(spans) - 1):
        a = tb["opt_meta"][spans[idx][2]][0]
        b = tb["opt_meta"][spans[idx + 1][2]][0]
        comm.append(comm_cost(inst, spans[idx][1], a, b))
        links.append(f"intra:{a}" if a == b else f"cross:{a}>{b}")
    kb, k_next = [0] * len(spans), 0.0
    for idx in range(len(spans) - 1, -1, -1):
        c = comm[idx] if idx < len(spans) - 1 else 0.0
        k_next = math.ceil(2.0 * c / t_max) + 1.0 + k_next
        kb[idx] = int(k_next)
    assert kb[0] == int(N[best_s, 1, G])
    st_t = [float(tb["tf"][o, q, p] + tb["tb"][o, q, p]) for q, p, o in spans]
    counts = adaptive_counts(st_t, comm, eps, t_max=max(t_max, max(st_t)))
    meshes = {m["id"]: m for m in inst["cluster"]["meshes"]}
    stages = []
    busy, peaks = [], []
    for idx, (q, p, o) in enumerate(spans):
        mid, n, m = tb["opt_meta"][o]
        stages.append({
            "layers": [q, p], "mesh": mid, "submesh": [n, m],
            "t_fwd": float(tb["tf"][o, q, p]), "t_bwd": float(tb["tb"][o, q, p]),
            "mem_params": float(tb["mp"][o, q, p]), "mem_act": float(tb["ma"][o, q, p]),
            "launch_count": counts[idx], "dp_launch_bound": kb[idx],
        })
        t = stages[-1]["t_fwd"] + stages[-1]["t_bwd"]
        for _ in range(n * m):
            busy.append(t * B)
            peaks.append(meshes[mid]["peak_flops"])
    top = max(busy)
    eta = 100.0 * (1.0 - sum((top - x) * pk for x, pk in zip(busy, peaks)) / (top * sum(peaks)))
    return {
        "num_microbatches": B, "t_max": t_max, "predicted_latency": best_total, "eta_pct": eta,
        "epsilon": eps, "stages": stages,
        "boundaries": [{"after_layer": spans[i][1], "comm": comm[i], "link": links[i]}
                       for i in range(len(spans) - 1)],
        "search_stats": {"dp_states": int(np.isfinite(F[1:]).sum())},
    }


def evaluate(inst: dict, tb: dict, t_max: float):
    B, eps = inst["num_microbatches"], inst["epsilon"]
    F, N, bpi, bpo = dp_sweep(tb, t_max)
    return extract(inst, tb, F, N, bpi, bpo, t_max, B, eps)


def full_pool(inst: dict, tb: dict | None = None, workers: int = 1, pool=None):
    """T*, best s and dp_states for every candidate (candidates/s workload)."""
    tb = tb or tables(inst)
    pool = tb["pool"] if pool is None else pool
    B = inst["num_microbatches"]

    def one(t):
        F, _, _, _ = dp_sweep(tb, t)
        s, tot = best_stage(F, tb, t, B)
        return tot, s, int(np.isfinite(F[1:]).sum())

    if workers > 1:
        with ThreadPoolExecutor(workers) as ex:
            res = list(ex.map(one, pool))
    else:
        res = [one(t) for t in pool]
    return (np.array([r[0] for r in res]), np.array([r[1] for r in res], dtype=np.int32),
            np.array([r[2] for r in res], dtype=np.int64))


def _sort_key(plan: dict):
    return (plan["predicted_latency"], plan["t_max"], len(plan["stages"]),
            tuple(s["layers"][1] for s in plan["stages"]),
            tuple((s["mesh"], *s["submesh"]) for s in plan["stages"]))


def search(inst: dict, optimized: bool = True, batch_size=None):
    """search() (planner.py:545-607) with bidirectional_prune (432-480) and the
    batched merge (490-542), evaluated sequentially."""
    tb = tables(inst)
    pool = tb["pool"]
    if not pool:
        raise ValueError("no feasible candidates in the profile store")
    B = inst["num_microbatches"]
    cache: dict = {}
    states = 0

    def dp(t):
        nonlocal states
        if t not in cache:
            cache[t] = evaluate(inst, tb, t)
            if cache[t] is not None:
                states += cache[t]["search_stats"]["dp_states"]
        return cache[t]

    if optimized:
        lo, hi = 0, len(pool) - 1
        if dp(pool[hi]) is None:
            raise ValueError("no t_max candidate admits a feasible plan")
        while lo < hi:
            mid = (lo + hi) // 2
            if dp(pool[mid]) is not None:
                hi = mid
            else:
                lo = mid + 1
        if lo > 0 and dp(pool[lo - 1]) is not None:
            raise ValueError("feasibility is not monotone in t_max")
        t_s = pool[lo]
        t_e = cache[t_s]["predicted_latency"] / (B - 1) if B > 1 else math.inf
        surviving = [t for t in pool[lo:] if t <= t_e]
        finite = np.sort(tb["t_tab"][np.isfinite(tb["t_tab"])])
        act = [int(np.searchsorted(finite, t, side="right")) for t in surviving]
        groups, cur = [], None
        for a in act:
            if a != cur:
                groups.append(0)
                cur = a
            groups[-1] += 1
        n_batches = sum(1 if batch_size is None or batch_size >= g else math.ceil(g / batch_size)
                        for g in groups)
        below, above = lo, len(pool) - lo - len(surviving)
    else:
        t_s, t_e, surviving = pool[0], math.inf, pool
        n_batches, below, above = 1, 0, 0
    plans = [p for p in (dp(t) for t in surviving) if p is not None]
    if not plans:
        raise ValueError("no stage partition satisfies the memory and overlap constraints")
    best = min(plans, key=_sort_key)
    best = dict(best)
    best["search_stats"] = {
        "candidates_total": len(pool), "pruned_below_ts": below, "pruned_above_te": above,
        "evaluated": len(surviving), "batches": n_batches, "t_low": t_s,
        "t_high": None if math.isinf(t_e) else t_e, "dp_states": states,
        "dp_transitions": transitions_per_sweep(tb) * len(surviving),
    }
    return best


# ---------------------------------------------------------------------------
# 1F1B simulation (simulation.py:73-228)
# ---------------------------------------------------------------------------


def simulate(t_fwd, t_bwd, comm, counts, B: int):
    """Explicit-DAG longest path for one plan -> (makespan, start, end)."""
    S = len(t_fwd)
    n = B * (4 * S - 2) + 1
    tf = np.ascontiguousarray(t_fwd, dtype=np.float64)
    tbw = np.ascontiguousarray(t_bwd, dtype=np.float64)
    cm = np.ascontiguousarray(list(comm) + [0.0], dtype=np.float64)
    cn = np.ascontiguousarray(counts, dtype=np.int32)
    start, end = np.empty(n), np.empty(n)
    mk = np.zeros(1)
    done = lib().oracle_simulate(S, B, _p(tf), _p(tbw), _p(cm), _p(cn), _p(start), _p(end), _p(mk))
    if done != n:
        raise ValueError("dependency cycle")
    return float(mk[0]), start, end


def _merge_busy(iv):
    """Disjoint busy intervals of a set of (lo, hi) (simulation.py:236-246):
    sort, drop empty ones, fuse overlapping or touching ones."""
    busy = []
    for lo, hi in sorted(iv):
        if not hi > lo:
            continue
        if busy and lo <= busy[-1][1]:
            busy[-1][1] = hi if hi > busy[-1][1] else busy[-1][1]
        else:
            busy.append([lo, hi])
    return [tuple(x) for x in busy]


def _overlap(a, b):
    """Pairwise intersection of two sorted disjoint lists (simulation.py:249-262)."""
    out, i, j = [], 0, 0
    while i < len(a) and j < len(b):
        lo, hi = max(a[i][0], b[j][0]), min(a[i][1], b[j][1])
        if hi > lo:
            out.append((lo, hi))
        if a[i][1] <= b[j][1]:
            i += 1
        else:
            j += 1
    return out


def schedule_report(t_fwd, t_bwd, comm, counts, B: int, mem_act=None):
    """analyze() + steady_state_rate(stage 1) of one plan (simulation.py:
    310-395), on the oracle's own explicit-DAG trace.  Reductions use the
    interpreter's builtin sum() on purpose: that IS the reference's
    arithmetic (compensated on CPython >= 3.12).  Returns (makespan, stage
    rows [busy, window, bubble, bubble_fraction, steady_bubble, peak_bytes,
    peak], link rows [fwd, bwd, overlap], rate or None)."""
    S = len(t_fwd)
    mk, start, end = simulate(t_fwd, t_bwd, comm, counts, B)
    # plain floats: builtin sum() compensates only exact float items
    start, end = start.tolist(), end.tolist()

    def fb(kind, mb, s):  # reference node numbering (simulation.py:103-111)
        return 2 * ((s - 1) * B + (mb - 1)) + kind

    def cfb(kind, mb, s):
        return 2 * S * B + 2 * ((s - 1) * B + (mb - 1)) + kind

    def program(n):  # scheduling.py:241-249
        ops = [(0, j) for j in range(1, n + 1)]
        for j in range(1, B - n + 1):
            ops += [(1, j), (0, n + j)]
        return ops + [(1, j) for j in range(B - n + 1, B + 1)]

    stages, busy_sets = [], []
    for s in range(1, S + 1):
        n = counts[s - 1]
        ops = program(n)
        ids = [fb(k, mb, s) for k, mb in ops]
        dur = [t_fwd[s - 1] if k == 0 else t_bwd[s - 1] for k, _ in ops]
        busy_sets.append(_merge_busy([(start[v], end[v]) for v in ids]))
        busy = sum(dur)
        window = end[ids[-1]] - start[ids[0]]
        w0, w1 = n, n + 2 * (B - n)
        sb = ((end[ids[w1 - 1]] - start[ids[w0]]) - sum(dur[w0:w1])) if w1 > w0 else 0.0
        level, peak = 0, 0
        for k, _ in ops:
            level += 1 if k == 0 else -1
            peak = max(peak, level)
        per = mem_act[s - 1] if mem_act else 0.0
        stages.append([busy, window, window - busy,
                       (window - busy) / window if window > 0 else 0.0, sb, peak * per, peak])
    links = []
    for s in range(1, S):
        ids = [cfb(k, mb, s) for mb in range(1, B + 1) for k in (0, 1)]
        u = _merge_busy([(start[v], end[v]) for v in ids])
        tot = sum(hi - lo for lo, hi in u)
        if tot <= 0.0:
            ratio = 1.0
        else:
            both = _overlap(_overlap(u, busy_sets[s - 1]), busy_sets[s])
            ratio = sum(hi - lo for lo, hi in both) / tot
        links.append([sum([comm[s - 1]] * B), sum([comm[s - 1]] * B), ratio])
    K = counts[0]
    xs = list(range(2 * K + 1, B + 1, K))
    rate = None
    if len(xs) >= 4:
        ys = [start[fb(0, i, 1)] for i in xs]
        n = float(len(xs))
        mx, my = sum(xs) / n, sum(ys) / n
        rate = (sum((x - mx) * (y - my) for x, y in zip(xs, ys))
                / sum((x - mx) ** 2 for x in xs))
    return mk, stages, links, rate


def config_e_batch(t_fwd, t_bwd, comm, S, B: int = 128, epsilon: float = 0.05,
                   threads: int | None = None):
    """Adaptive counts + explicit-DAG makespan of every plan of dense [P, 8]
    inputs (oracle_config_e_batch), split over host threads.  Returns
    (counts [P, 8] int32, status [P] int32, makespan [P] float64)."""
    f = np.ascontiguousarray(t_fwd, dtype=np.float64)
    b = np.ascontiguousarray(t_bwd, dtype=np.float64)
    c = np.ascontiguousarray(comm, dtype=np.float64)
    s = np.ascontiguousarray(S, dtype=np.int32)
    P = len(s)
    counts = np.zeros((P, 8), dtype=np.int32)
    status = np.zeros(P, dtype=np.int32)
    mk = np.full(P, np.nan)
    threads = threads or os.cpu_count() or 1
    step = (P + threads - 1) // threads

    def run(lo):
        lib().oracle_config_e_batch(lo, min(P, lo + step), B, _p(s), _p(f), _p(b), _p(c),
                                    float(epsilon), _p(counts), _p(status), _p(mk))

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(run, range(0, P, step)))
    return counts, status, mk


def config_e_plans(n_plans: int, seed: int = 24859, B: int = 128):
    """Config E synthetic plan generator: S in {2,3,4,6,8},
    t ~ U(0.5, 2)e-2, f = t*U(.3,.4), b = t - f, bw ~ logU(1, 200) Gbps,
    bytes ~ U(0,1) * t_max * 1.25e8 so that c <= t_max.  Returns dense
    [P, 8] arrays (t_fwd, t_bwd, comm) and S [P].  Same generator as
    paper_2509_24859_b200.workloads.config_e (kept separate on purpose)."""
    rng = np.random.default_rng(seed)
    S = rng.choice(np.array([2, 3, 4, 6, 8]), size=n_plans)
    t = rng.uniform(0.5, 2.0, size=(n_plans, 8)) * 1e-2
    f = t * rng.uniform(0.3, 0.4, size=(n_plans, 8))
    b = t - f
    mask = np.arange(8)[None, :] < S[:, None]
    tm = np.where(mask, f + b, 0.0).max(axis=1)
    bw = np.exp(rng.uniform(np.log(1.0), np.log(200.0), size=(n_plans, 8))) * 1.25e8
    nbytes = rng.uniform(0.0, 1.0, size=(n_plans, 8)) * tm[:, None] * 1.25e8
    comm = nbytes / bw
    comm = np.where(np.arange(8)[None, :] < (S[:, None] - 1), comm, 0.0)
    return f, b, comm, S.astype(np.int32)
