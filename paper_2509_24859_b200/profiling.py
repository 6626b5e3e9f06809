"""Cost-table evaluation (K1) behind the reference's profiling API.

Same names, arguments, return types and errors as meshpipe.profiling
(profiling.py:27-400), but ProfileStore is built by the hapt_tables_build
kernel chain on the GPU: one thread per (option, layer span), structural
dedup through a canonical-start table, OOM / imbalance masks, the CSR
feasible-span index and the sorted t_max pool all in HBM.  Host-side Python
only marshals inputs and answers point queries (lookup) from a cached copy.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace
from typing import Optional

import numpy as np

from .cluster import enumerate_submeshes
from .engine import DeviceTables


class ProfilingError(ValueError):
    pass


class NoFeasibleCandidateError(ProfilingError):
    pass


@dataclass(frozen=True)
class CostModel:
    """Analytic cost constants (profiling.py:35-59)."""

    beta: float = 2.0
    efficiency: float = 0.5
    alpha: float = 0.0
    replication: float = 1.0
    act_factor: float = 2.0

    def __post_init__(self):
        if self.beta <= 0 or self.efficiency <= 0 or self.efficiency > 1:
            raise ProfilingError("invalid cost model constants")
        if self.alpha < 0 or self.replication < 1 or self.act_factor <= 0:
            raise ProfilingError("invalid cost model constants")


@dataclass(frozen=True)
class StageCandidate:
    q: int
    p: int
    signature: tuple
    flops: float
    param_bytes: float
    act_bytes: float


@dataclass(frozen=True)
class StageMeshProfile:
    t_fwd: float
    t_bwd: float
    mem_params: float
    mem_act: float
    feasible: bool
    prune_reason: str = ""

    @property
    def t(self) -> float:
        return self.t_fwd + self.t_bwd


_REASONS = {0: "", 1: "oom", 2: "imbalance"}


@dataclass(frozen=True)
class BoundaryCost:
    """Per-boundary transfer seconds by link class (profiling.py:106-125)."""

    num_layers: int
    intra: dict
    cross: dict

    def get(self, i: int, mesh_a: str, mesh_b: str) -> float:
        if i <= 0 or i >= self.num_layers:
            return 0.0
        if mesh_a == mesh_b:
            return self.intra[mesh_a][i]
        return self.cross[tuple(sorted((mesh_a, mesh_b)))][i]


def boundary_costs(layers, cluster) -> BoundaryCost:
    """Transfer time of every layer boundary over every link class.

    Host-side data object for plan assembly / validation, with the reference
    semantics (profiling.py:128-147: intra-mesh boundaries use the mesh's
    inter-host bandwidth; cross links add cross_latency).  The DP itself reads
    the device copies cb_same / cb_next that K1 computes with the same
    expressions (hapt_tables.cu:k1_meta); DpTables checks the two agree by
    construction (same inputs) and otherwise uploads these rows.
    """
    L = len(layers)
    bb = [layers.layers[i].boundary_bytes for i in range(L)]
    intra = {}
    for mesh in cluster.meshes:
        row = [0.0] * (L + 1)
        for i in range(1, L):
            row[i] = bb[i - 1] / mesh.inter_host_bw
        intra[mesh.id] = tuple(row)
    cross = {}
    meshes = list(cluster.meshes)
    for a in range(len(meshes)):
        for b in range(a + 1, len(meshes)):
            bw = cluster.cross_bandwidth(meshes[a].id, meshes[b].id)
            row = [0.0] * (L + 1)
            for i in range(1, L):
                row[i] = bb[i - 1] / bw + cluster.cross_latency
            cross[tuple(sorted((meshes[a].id, meshes[b].id)))] = tuple(row)
    bc = BoundaryCost(L, intra, cross)
    object.__setattr__(bc, "_source", (id(layers), id(cluster)))
    return bc


@dataclass
class StoreStats:
    candidates: int = 0
    canonical: int = 0
    canonical_feasible: int = 0
    aliased: int = 0
    pruned_oom: int = 0
    pruned_imbalance: int = 0

    def as_dict(self) -> dict:
        return dict(self.__dict__)


class ProfileStore:
    """Profiles for every (layer span, submesh) pair, deduplicated by
    structural signature, computed on the GPU (K1).  Query interface of
    meshpipe.profiling.ProfileStore (profiling.py:168-368)."""

    def __init__(
        self,
        layers,
        cluster,
        model: Optional[CostModel] = None,
        imbalance_ratio: float = 3.0,
        dedup: bool = True,
        device=None,
    ):
        if imbalance_ratio < 1.0:
            raise ProfilingError("imbalance_ratio must be >= 1 (or inf to disable)")
        self.layers = layers
        self.cluster = cluster
        self.model = model or CostModel()
        self.imbalance_ratio = imbalance_ratio
        self.dedup = dedup
        self.options = [(mesh, sub) for mesh in cluster.meshes for sub in enumerate_submeshes(mesh)]
        self._opt_index = {
            (mesh.id, sub.shape): o for o, (mesh, sub) in enumerate(self.options)
        }
        self._sig_ids: dict = {}
        self._sig = np.array(
            [self._sig_ids.setdefault(l.signature, len(self._sig_ids)) for l in layers.layers],
            dtype=np.int32,
        )
        self._overrides: dict = {}  # (o, qc, pc) -> (t_fwd, t_bwd, mem_params, mem_act)
        self._profiles: dict = {}   # canonical (o, qc, pc) -> StageMeshProfile
        self._alias_key: dict = {}  # (o, q, p) -> canonical key
        L = len(layers)
        G = sum(m.hosts * m.devices_per_host for m in cluster.meshes)
        self.dev = DeviceTables(L, G, len(self.options), len(cluster.meshes), device)
        self._build()

    # -- construction (K1 on the device) -------------------------------------
    def _desc(self):
        layers, cluster, model = self.layers.layers, self.cluster, self.model
        meshes = list(cluster.meshes)
        nm = len(meshes)
        cross_next = np.zeros(nm)
        cross_ok = True
        for m in range(nm - 1):
            try:
                cross_next[m] = cluster.cross_bandwidth(meshes[m].id, meshes[m + 1].id)
            except ValueError:
                cross_next[m] = math.nan  # boundary_costs would raise; DpTables re-checks
                cross_ok = False
        self._cross_ok = cross_ok
        arrays = {
            "layer_flops": [l.flops for l in layers],
            "layer_params": [l.param_bytes for l in layers],
            "layer_bbytes": [l.boundary_bytes for l in layers],
            "layer_sig": self._sig,
            "mesh_hosts": [m.hosts for m in meshes],
            "mesh_dph": [m.devices_per_host for m in meshes],
            "mesh_peak": [m.peak_flops for m in meshes],
            "mesh_mem": [m.mem_device for m in meshes],
            "mesh_intra_bw": [m.intra_host_bw for m in meshes],
            "mesh_inter_bw": [m.inter_host_bw for m in meshes],
            "cross_bw_next": cross_next,
            "opt_n": [sub.n for _, sub in self.options],
            "opt_m": [sub.m for _, sub in self.options],
            "opt_mesh": [cluster.mesh_order(mesh.id) for mesh, _ in self.options],
            "ovr_index": None,
            "ovr_vals": None,
        }
        if self._overrides:
            S = len(layers) + 2
            idx = np.full((len(self.options), S, S), -1, dtype=np.int32)
            vals = np.zeros((len(self._overrides), 4))
            for row, (key, v) in enumerate(self._overrides.items()):
                idx[key] = row
                vals[row] = v
            arrays["ovr_index"] = idx
            arrays["ovr_vals"] = vals
        scalars = {
            "cross_latency": float(cluster.cross_latency),
            "beta": float(model.beta),
            "efficiency": float(model.efficiency),
            "alpha": float(model.alpha),
            "replication": float(model.replication),
            "act_factor": float(model.act_factor),
            "imbalance_ratio": float(self.imbalance_ratio),
            # CPython sums, exactly as profiling.py:214-215
            "total_flops": float(sum(l.flops for l in layers)),
            "total_peak": float(cluster.total_peak_flops),
            "dedup": 1 if self.dedup else 0,
        }
        return arrays, scalars

    def _build(self) -> None:
        arrays, scalars = self._desc()
        self.dev.build(arrays, scalars)
        self._profiles.clear()
        self._alias_key.clear()
        c = self.dev.counters()
        self.stats = StoreStats(*(int(x) for x in c[2:8]))
        if self.stats.canonical_feasible == 0:
            raise NoFeasibleCandidateError(
                f"no feasible stage-mesh candidate; tightest violation: {self._tightest()}"
            )

    def _tightest(self) -> str:
        """Least-violated prune among canonical entries, in the reference's
        iteration order (profiling.py:226-286).  Error path only."""
        L = len(self.layers)
        if L == 0:
            return "no candidates at all"
        state = self.dev.host("cell_state")
        mp, ma = self.dev.host("mp_raw"), self.dev.host("ma_raw")
        canon = self.dev.host("canon_q")
        lay = self.layers.layers
        pf = [0.0] * (L + 1)
        for i in range(1, L + 1):
            pf[i] = pf[i - 1] + lay[i - 1].flops
        total_flops = sum(l.flops for l in lay)
        total_peak = self.cluster.total_peak_flops
        rho = self.imbalance_ratio
        best = None
        for q in range(1, L + 1):
            for p in range(q, L + 1):
                for o, (mesh, sub) in enumerate(self.options):
                    st = int(state[o, q, p])
                    if not (st & 2):
                        continue
                    reason = (st >> 2) & 3
                    if reason == 1:
                        need = mp[o, q, p] + ma[o, q, p]
                        ratio = need / mesh.mem_device
                        text = (f"span [{q},{p}] on {mesh.id}{sub.shape}: needs "
                                f"{need:.3e} B vs {mesh.mem_device:.3e} B per device")
                    elif reason == 2:
                        qc = int(canon[q, p])
                        flops = pf[qc + (p - q)] - pf[qc - 1]
                        fs = flops / total_flops if total_flops > 0 else 0.0
                        cs = sub.device_count * mesh.peak_flops / total_peak
                        ratio = max(fs / cs, cs / fs) / rho
                        text = (f"span [{q},{p}] on {mesh.id}{sub.shape}: flops share "
                                f"{fs:.3f} vs capacity share {cs:.3f}")
                    else:
                        continue
                    if best is None or ratio < best[0]:
                        best = (ratio, text)
        return best[1] if best else "no candidates at all"

    # -- queries ---------------------------------------------------------------
    @property
    def num_layers(self) -> int:
        return len(self.layers)

    def _option(self, mesh_id: str, shape) -> int:
        o = self._opt_index.get((mesh_id, tuple(shape)))
        if o is None:
            raise KeyError((mesh_id, shape))
        return o

    def _canon(self, q: int, p: int) -> tuple[int, int]:
        qc = int(self.dev.host("canon_q")[q, p])
        return qc, qc + (p - q)

    def _signature_key(self, q: int, p: int) -> tuple:
        return tuple(int(x) for x in self._sig[q - 1 : p])

    def lookup(self, q: int, p: int, mesh_id: str, shape) -> StageMeshProfile:
        return self.lookup_many([(q, p, mesh_id, shape)])[0]

    def lookup_many(self, spans) -> list:
        """lookup() for several (q, p, mesh_id, shape) at once: the needed
        cells are gathered on the device (canonical span resolved there too)
        and copied back in one transfer; profiles are cached per canonical
        entry, so repeated lookups return the same object."""
        import torch

        L = self.num_layers
        S = L + 2
        req = []
        for q, p, mesh_id, shape in spans:
            try:
                if not (1 <= q <= p <= L):
                    raise KeyError
                o = self._option(mesh_id, shape)
            except KeyError:
                raise ProfilingError(
                    f"no profile for span [{q},{p}] on {mesh_id}{tuple(shape)}") from None
            req.append((o, q, p))
        miss = [r for r in req if r not in self._alias_key]
        if miss:
            dev = self.dev
            qp = torch.tensor([q * S + p for _, q, p in miss], dtype=torch.int64)
            lens = torch.tensor([p - q for _, q, p in miss], dtype=torch.int64)
            opt = torch.tensor([o for o, _, _ in miss], dtype=torch.int64)
            qp, lens, opt = (x.to(dev.device) for x in (qp, lens, opt))
            qc = dev.view("canon_q", torch.int32, (S * S,))[qp].to(torch.int64)
            cell = opt * (S * S) + qc * S + qc + lens
            flat = lambda n: dev.view(n, torch.float64, (dev.n_opts * S * S,))  # noqa: E731
            st = dev.view("cell_state", torch.int8, (dev.n_opts * S * S,))[cell]
            vals = torch.stack([flat("tf_raw")[cell], flat("tb_raw")[cell], flat("mp_raw")[cell],
                                flat("ma_raw")[cell], st.to(torch.float64),
                                qc.to(torch.float64)]).cpu().numpy()
            for j, (o, q, p) in enumerate(miss):
                qcj = int(vals[5, j])
                key = (o, qcj, qcj + (p - q))
                if key not in self._profiles:
                    sb = int(vals[4, j])
                    self._profiles[key] = StageMeshProfile(
                        float(vals[0, j]), float(vals[1, j]), float(vals[2, j]),
                        float(vals[3, j]), feasible=bool(sb & 1),
                        prune_reason=_REASONS[(sb >> 2) & 3])
                self._alias_key[(o, q, p)] = key
        return [self._profiles[self._alias_key[r]] for r in req]

    def canonical_key(self, q: int, p: int, mesh_id: str, shape) -> tuple:
        shape = tuple(shape)
        self._option(mesh_id, shape)
        if not self.dedup:
            return ((q, p), mesh_id, shape)
        qc, pc = self._canon(q, p)
        return (self._signature_key(qc, pc), mesh_id, shape)

    def candidate(self, q: int, p: int) -> StageCandidate:
        lay = self.layers.layers
        f = pp = a = 0.0
        pre = [(0.0, 0.0, 0.0)]
        for l in lay[:p]:
            f += l.flops
            pp += l.param_bytes
            a += l.boundary_bytes
            pre.append((f, pp, a))
        return StageCandidate(
            q, p, self._signature_key(q, p),
            pre[p][0] - pre[q - 1][0], pre[p][1] - pre[q - 1][1], pre[p][2] - pre[q - 1][2],
        )

    def feasible_t_values(self) -> list[float]:
        """Sorted, deduplicated t of feasible canonical entries -- the t_max
        pool, produced on the device (sort + unique of the CSR t values)."""
        return [float(x) for x in self.dev.host("pool")]

    def signature_text(self, q: int, p: int) -> str:
        return "+".join(
            "/".join(str(part) for part in layer.signature)
            for layer in self.layers.layers[q - 1 : p]
        )

    # -- measured overrides ------------------------------------------------------
    def apply_overrides(self, overrides: list) -> int:
        """Replace canonical entries with measured numbers (profiling.py:328-368);
        the tables are rebuilt on the device with the overrides folded in."""
        if not overrides:
            return 0
        L = self.num_layers
        by_text: dict = {}
        for q in range(1, L + 1):
            for p in range(q, L + 1):
                text = self.signature_text(q, p)
                qc, pc = self._canon(q, p) if self.dedup else (q, p)
                for o, (mesh, sub) in enumerate(self.options):
                    by_text.setdefault((text, mesh.id, sub.shape), (o, qc, pc))
        mesh_ids = {m.id for m in self.cluster.meshes}
        updated = 0
        error = None
        for entry in overrides:
            try:
                sig = str(entry["signature"])
                mesh_id = str(entry["mesh"])
                shape = tuple(int(x) for x in entry["submesh"])
            except (KeyError, TypeError) as exc:
                error = ProfilingError(f"malformed override entry {entry!r}")
                error.__cause__ = exc
                break
            if mesh_id not in mesh_ids:
                error = ProfilingError(f"override references unknown mesh {mesh_id!r}")
                break
            key = by_text.get((sig, mesh_id, shape))
            if key is None:
                error = ProfilingError(
                    f"override references unknown candidate {sig!r} on {mesh_id}{shape}"
                )
                break
            o, qc, pc = key
            cur = self._overrides.get(key)
            if cur is None:
                prof = self.lookup(qc, pc, self.options[o][0].id, self.options[o][1].shape)
                cur = (prof.t_fwd, prof.t_bwd, prof.mem_params, prof.mem_act)
            t_fwd = float(entry.get("t_fwd", cur[0]))
            t_bwd = float(entry.get("t_bwd", cur[1]))
            if t_fwd <= 0 or t_bwd <= 0:
                error = ProfilingError(f"override for {sig!r}: compute times must be positive")
                break
            mem_p = float(entry.get("mem_params", cur[2]))
            mem_a = float(entry.get("mem_act", cur[3]))
            if mem_p < 0 or mem_a < 0:
                error = ProfilingError(f"override for {sig!r}: memory must be >= 0")
                break
            self._overrides[key] = (t_fwd, t_bwd, mem_p, mem_a)
            updated += 1
        if updated:
            self._build()
        if error is not None:
            raise error
        return updated


def build_store(layers, cluster, model: Optional[CostModel] = None,
                imbalance_ratio: float = 3.0, dedup: bool = True, device=None) -> ProfileStore:
    return ProfileStore(layers, cluster, model, imbalance_ratio, dedup, device)


def import_profiles(data: dict) -> list:
    entries = data.get("overrides", [])
    if not isinstance(entries, list):
        raise ProfilingError("override file: 'overrides' must be a list")
    return entries


def store_dump(store: ProfileStore) -> str:
    s = store.stats
    rows = [
        ("candidates", s.candidates),
        ("canonical", s.canonical),
        ("canonical feasible", s.canonical_feasible),
        ("aliased", s.aliased),
        ("pruned (oom)", s.pruned_oom),
        ("pruned (imbalance)", s.pruned_imbalance),
    ]
    return "".join(f"{name:<20}{val}\n" for name, val in rows)


__all__ = [
    "BoundaryCost", "CostModel", "NoFeasibleCandidateError", "ProfileStore", "ProfilingError",
    "StageCandidate", "StageMeshProfile", "StoreStats", "boundary_costs", "build_store",
    "import_profiles", "store_dump", "replace",
]
