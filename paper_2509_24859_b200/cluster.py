"""Cluster description consumed by the planner hot path.

Input types only: the same fields and semantics as the reference's
`meshpipe.cluster` (cluster.py:69-179) so a reference ClusterSpec can be passed
in unchanged (duck-typed); YAML/unit parsing (cluster.py:17-66, 182-212) is
outside the hot path and not mirrored.
"""

from __future__ import annotations

from dataclasses import dataclass, field


class ClusterError(ValueError):
    pass


def _pow2(n: int) -> bool:
    return n >= 1 and n & (n - 1) == 0


@dataclass(frozen=True)
class DeviceMesh:
    """Homogeneous mesh of `hosts` x `devices_per_host` devices
    (reference cluster.py:69-90)."""

    id: str
    hosts: int
    devices_per_host: int
    peak_flops: float
    mem_device: float
    intra_host_bw: float
    inter_host_bw: float

    def __post_init__(self):
        if self.hosts < 1:
            raise ClusterError(f"mesh {self.id}: hosts must be >= 1")
        if not _pow2(self.devices_per_host):
            raise ClusterError(f"mesh {self.id}: devices_per_host must be a power of two")
        for attr in ("peak_flops", "mem_device", "intra_host_bw", "inter_host_bw"):
            if not getattr(self, attr) > 0:
                raise ClusterError(f"mesh {self.id}: {attr} must be positive")

    @property
    def device_count(self) -> int:
        return self.hosts * self.devices_per_host


@dataclass(frozen=True)
class Submesh:
    mesh_id: str
    n: int
    m: int

    @property
    def device_count(self) -> int:
        return self.n * self.m

    @property
    def shape(self) -> tuple[int, int]:
        return (self.n, self.m)


@dataclass
class ClusterSpec:
    """Ordered meshes plus the cross-mesh link model (cluster.py:108-154)."""

    meshes: list
    cross_bw: object = 0.0
    cross_latency: float = 0.0
    _index: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        if not self.meshes:
            raise ClusterError("cluster needs at least one mesh")
        ids = [m.id for m in self.meshes]
        if len(ids) != len(set(ids)):
            raise ClusterError("duplicate mesh ids")
        self._index = {mid: pos for pos, mid in enumerate(ids)}
        if isinstance(self.cross_bw, dict):
            self.cross_bw = {tuple(sorted(k)): v for k, v in self.cross_bw.items()}

    def mesh(self, mesh_id: str):
        pos = self._index.get(mesh_id)
        if pos is None:
            raise ClusterError(f"unknown mesh id {mesh_id!r}")
        return self.meshes[pos]

    def mesh_order(self, mesh_id: str) -> int:
        pos = self._index.get(mesh_id)
        if pos is None:
            raise ClusterError(f"unknown mesh id {mesh_id!r}")
        return pos

    @property
    def total_devices(self) -> int:
        return sum(m.device_count for m in self.meshes)

    @property
    def total_peak_flops(self) -> float:
        # CPython's sum() -- compensated on 3.12 -- exactly as the reference
        # (cluster.py:140-142); a host-side scalar input of the K1 kernel.
        return sum(m.device_count * m.peak_flops for m in self.meshes)

    def cross_bandwidth(self, a: str, b: str) -> float:
        if isinstance(self.cross_bw, dict):
            key = tuple(sorted((a, b)))
            if key not in self.cross_bw:
                raise ClusterError(f"no cross bandwidth configured for pair {key}")
            bw = self.cross_bw[key]
        else:
            bw = self.cross_bw
        if bw <= 0:
            raise ClusterError(f"cross bandwidth between {a} and {b} must be positive")
        return bw


def enumerate_submeshes(mesh) -> list[Submesh]:
    """Legal slices (1,1),(1,2),...,(1,M) then (2,M)..(N,M), ordered by device
    count (cluster.py:157-168).  The option order is a tie-break key of the
    DP, so it must match the reference exactly."""
    shapes = []
    width = 1
    while width <= mesh.devices_per_host:
        shapes.append(Submesh(mesh.id, 1, width))
        width *= 2
    shapes.extend(Submesh(mesh.id, n, mesh.devices_per_host) for n in range(2, mesh.hosts + 1))
    shapes.sort(key=lambda s: s.device_count)
    return shapes


def link_bandwidth(spec, a: Submesh, b: Submesh) -> float:
    """Stage-boundary link bandwidth (cluster.py:171-179)."""
    mesh_a = spec.mesh(a.mesh_id)
    spec.mesh(b.mesh_id)
    if a.mesh_id == b.mesh_id:
        return mesh_a.inter_host_bw
    return spec.cross_bandwidth(a.mesh_id, b.mesh_id)
