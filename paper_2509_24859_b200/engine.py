"""Device-side engine: one instance's tables in HBM plus the batched DP.

`DeviceTables` owns a single HBM buffer laid out by hapt_tables_init (the K1
output: dense DpTables arrays, CSR feasible-span index with per-entry DP
metadata, the t_max pool, StoreStats counters).  `Sweeper` evaluates batches
of t_max candidates through hapt_dp_sweep_batch + hapt_dp_select and
re-derives a winner's stage chain with hapt_dp_backtrack.

Everything numeric happens in the C-ABI library; this module only allocates,
copies and sequences calls.
"""

from __future__ import annotations

import ctypes
import weakref
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import DpFull, ModelDesc, Tables, check, ptr, stream_ptr

_F64 = torch.float64
_I32 = torch.int32


def default_device() -> torch.device:
    _lib.lib()  # raises without a GPU or without the built library
    return torch.device("cuda", torch.cuda.current_device())


class DeviceTables:
    """hapt_tables for one planning instance."""

    def __init__(self, L: int, G: int, n_opts: int, n_meshes: int, device=None):
        self.lib = _lib.lib()
        self.device = torch.device(device) if device is not None else default_device()
        self.dims = (L, G, n_opts, n_meshes)
        nbytes = self.lib.hapt_tables_bytes(L, G, n_opts, n_meshes)
        self.buf = torch.empty(nbytes + 512, dtype=torch.uint8, device=self.device)
        base = self.buf.data_ptr()
        self._shift = (-base) % 256
        self.t = Tables()
        check(
            self.lib.hapt_tables_init(
                ctypes.byref(self.t), base + self._shift, nbytes, L, G, n_opts, n_meshes
            )
        )
        self.L, self.G, self.n_opts, self.n_meshes = L, G, n_opts, n_meshes
        self._counters = None
        self._host = {}

    # -- typed views into the buffer ---------------------------------------
    def view(self, name: str, dtype, shape) -> torch.Tensor:
        addr = getattr(self.t, name)
        off = addr - self.buf.data_ptr()
        n = int(np.prod(shape)) if len(shape) else 1
        itemsize = torch.empty(0, dtype=dtype).element_size()
        return self.buf[off : off + n * itemsize].view(dtype).view(*shape)

    def dense(self, name: str) -> torch.Tensor:
        S = self.L + 2
        return self.view(name, _F64, (self.n_opts, S, S))

    @property
    def s_max(self) -> int:
        return self.t.s_max

    @s_max.setter
    def s_max(self, v: int) -> None:
        self.t.s_max = int(v)

    # -- construction ------------------------------------------------------
    def build(self, desc_arrays: dict, scalars: dict) -> "DeviceTables":
        """Run K1 from host description arrays (hapt_model_desc)."""
        dev = self.device
        d = ModelDesc()
        d.L, d.n_meshes, d.n_opts, d.G = self.L, self.n_meshes, self.n_opts, self.G
        f64 = ("layer_flops", "layer_params", "layer_bbytes", "mesh_peak", "mesh_mem",
               "mesh_intra_bw", "mesh_inter_bw", "cross_bw_next", "ovr_vals")
        # every description array in one host buffer and one H2D copy
        parts, offs, cur = [], {}, 0
        for name, arr in desc_arrays.items():
            if arr is None:
                continue
            a = np.ascontiguousarray(arr, dtype=np.float64 if name in f64 else np.int32)
            offs[name] = cur
            parts.append((cur, a.view(np.uint8).reshape(-1)))
            cur += (a.nbytes + 15) // 16 * 16
        host = np.zeros(max(cur, 16), dtype=np.uint8)
        for off, raw in parts:
            host[off : off + raw.size] = raw
        blob = torch.from_numpy(host).to(dev)
        self.h2d_bytes = int(host.nbytes)  # bench.py's e2e accounting
        base = blob.data_ptr()
        for name in desc_arrays:
            setattr(d, name, base + offs[name] if name in offs else None)
        keep = {"blob": blob}
        for name, val in scalars.items():
            setattr(d, name, val)
        check(self.lib.hapt_tables_build(ctypes.byref(self.t), ctypes.byref(d), stream_ptr()))
        self._keep = keep  # inputs must outlive the asynchronous build
        self._counters = None
        self._host.clear()
        self._transitions = None  # planner.DpTables.transitions_per_sweep cache
        return self

    def load_dense(self, arrays: dict, s_max: int) -> "DeviceTables":
        """Drop-in path: copy DpTables arrays in, then hapt_tables_finalize."""
        S = self.L + 2
        spec = {
            "t_tab": (_F64, (self.n_opts, S, S)),
            "mp_tab": (_F64, (self.n_opts, S, S)),
            "ma_tab": (_F64, (self.n_opts, S, S)),
            "opt_cap": (_F64, (self.n_opts,)),
            "opt_mesh": (_I32, (self.n_opts,)),
            "opt_devs": (_I32, (self.n_opts,)),
            "opt_off": (_I32, (self.n_meshes + 1,)),
            "cb_same": (_F64, (self.n_meshes, self.L + 1)),
            "cb_next": (_F64, (self.n_meshes, self.L + 1)),
            "g_mesh": (_I32, (self.G + 1,)),
            "g_avail": (_I32, (self.G + 1,)),
            "span_off": (_I32, (self.n_opts * S + 1,)),
        }
        for name, (dtype, shape) in spec.items():
            src = torch.as_tensor(np.ascontiguousarray(arrays[name]).reshape(shape))
            self.view(name, dtype, shape).copy_(src.to(dtype))
        items = np.ascontiguousarray(arrays["span_items"], dtype=np.int32)
        nnz = int(np.asarray(arrays["span_off"])[-1])
        if nnz > self.t.nnz_cap:
            raise ValueError("span index larger than n_opts*L*(L+1)/2")
        if nnz:
            self.view("span_items", _I32, (nnz,)).copy_(torch.from_numpy(items[:nnz]))
        self.s_max = s_max
        check(self.lib.hapt_tables_finalize(ctypes.byref(self.t), stream_ptr()))
        self._counters = None
        self._host.clear()
        self._transitions = None  # planner.DpTables.transitions_per_sweep cache
        return self

    # -- host-side reads -----------------------------------------------------
    def counters(self) -> np.ndarray:
        if self._counters is None:
            self._counters = self.view("counters", torch.int64, (16,)).cpu().numpy().copy()
        return self._counters

    @property
    def nnz(self) -> int:
        return int(self.counters()[0])

    @property
    def pool_len(self) -> int:
        return int(self.counters()[1])

    def pool(self) -> torch.Tensor:
        return self.view("pool", _F64, (self.t.pool_cap,))[: self.pool_len]

    def host(self, name: str) -> np.ndarray:
        """Cached host copy of a table (for API queries, not the hot path)."""
        if name not in self._host:
            S = self.L + 2
            shapes = {
                "t_tab": (_F64, (self.n_opts, S, S)),
                "mp_tab": (_F64, (self.n_opts, S, S)),
                "ma_tab": (_F64, (self.n_opts, S, S)),
                "tf_raw": (_F64, (self.n_opts, S, S)),
                "tb_raw": (_F64, (self.n_opts, S, S)),
                "mp_raw": (_F64, (self.n_opts, S, S)),
                "ma_raw": (_F64, (self.n_opts, S, S)),
                "cell_state": (torch.int8, (self.n_opts, S, S)),
                "canon_q": (_I32, (S, S)),
                "opt_cap": (_F64, (self.n_opts,)),
                "opt_mesh": (_I32, (self.n_opts,)),
                "opt_devs": (_I32, (self.n_opts,)),
                "opt_off": (_I32, (self.n_meshes + 1,)),
                "cb_same": (_F64, (self.n_meshes, self.L + 1)),
                "cb_next": (_F64, (self.n_meshes, self.L + 1)),
                "g_mesh": (_I32, (self.G + 1,)),
                "g_avail": (_I32, (self.G + 1,)),
                "g_crow": (_I32, (self.G + 1,)),
                "span_off": (_I32, (self.n_opts * S + 1,)),
            }
            if name == "span_items":
                arr = self.view("span_items", _I32, (max(self.nnz, 1),)).cpu().numpy().copy()
                if self.nnz == 0:
                    arr[:] = 0
            elif name == "pool":
                arr = self.pool().cpu().numpy().copy()
            else:
                dtype, shape = shapes[name]
                arr = self.view(name, dtype, shape).cpu().numpy().copy()
            self._host[name] = arr
        return self._host[name]


@dataclass
class SweepResult:
    tmax: np.ndarray
    tstar: np.ndarray     # T* per candidate (+inf: infeasible)
    best_s: np.ndarray    # stage count of the best plan (-1: infeasible)
    states: np.ndarray    # isfinite(F[1:]).sum()
    winner: int           # argmin (T*, index), -1 if none
    bp: torch.Tensor | None = None     # packed backpointers [n][s_max+1][L+2][G+1]
    ntop: np.ndarray | None = None     # N[s,1,G] per candidate [n][s_max+1]
    ftop: np.ndarray | None = None     # F[s,1,G] per candidate [n][s_max+1] (keep_ftop)


_WS_CACHE: dict = {}  # (device, stream) -> scratch tensor reused by every Sweeper
_FREE_MEM: dict = {}


def _scratch(device: torch.device, nbytes: int) -> torch.Tensor:
    """Scratch shared by every sweep issued on the current stream (work on one
    stream is ordered, so reuse is safe; other streams get their own)."""
    key = (device, torch.cuda.current_stream(device).cuda_stream)
    buf = _WS_CACHE.get(key)
    if buf is None or buf.numel() < nbytes:
        _WS_CACHE.pop(key, None)
        buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        _WS_CACHE[key] = buf
    return buf


class Sweeper:
    """Batched K2 over one DeviceTables.  Workspaces are shared per device and
    candidate batches are chunked so the successor tables stay within
    `max_ws_bytes`."""

    # bytes of packed backpointers kept for a batch: a quarter of the free HBM
    # at first use, at most 40 GB (a D3 survivor batch needs ~24 GB)
    BP_CAP = 40 * 2**30

    def __init__(self, tables: DeviceTables, max_ws_bytes: int | None = None):
        # weak: DeviceTables caches its Sweeper, and a strong back-reference
        # would make the pair a cycle that only the cyclic GC frees -- the
        # 100 MB tables buffer must go back to the allocator by refcount
        self._tables = weakref.ref(tables)
        self.lib = tables.lib
        self.device = tables.device
        if self.device not in _FREE_MEM:
            _FREE_MEM[self.device] = torch.cuda.mem_get_info(self.device)[0]
        if max_ws_bytes is None:
            max_ws_bytes = int(min(0.5 * _FREE_MEM[self.device], 48 * 2**30))
        self.max_ws_bytes = max_ws_bytes
        self.BP_BUDGET = int(min(self.BP_CAP, 0.25 * _FREE_MEM[self.device]))
        self._bt_ws = None
        self.last_chunks = 0

    @property
    def tables(self) -> "DeviceTables":
        t = self._tables()
        if t is None:
            raise RuntimeError("the device tables of this sweeper were released")
        return t

    def _chunk(self) -> int:
        per32 = self.lib.hapt_dp_workspace_bytes(ctypes.byref(self.tables.t), 32)
        groups = max(1, self.max_ws_bytes // max(per32, 1))
        return int(groups * 32)

    def _workspace(self, nbytes: int) -> torch.Tensor:
        return _scratch(self.device, nbytes)

    def bp_bytes(self, n: int) -> int:
        t = self.tables
        return 4 * n * (t.s_max + 1) * (t.L + 2) * (t.G + 1)

    def sweep_device(self, tmax: torch.Tensor, full: DpFull | None = None, cpl: int = 0):
        """tmax: float64 CUDA tensor [n].  Returns (ftop [n, s_max+1], states [n])
        as device tensors; no host synchronisation.  cpl: candidates per lane
        of the DP warps (0 = the library's choice; results never depend on it)."""
        t = self.tables
        n = int(tmax.numel())
        s1 = t.s_max + 1
        ftop = torch.empty((n, s1), dtype=_F64, device=self.device)
        states = torch.empty(n, dtype=torch.int64, device=self.device)
        chunk = self._chunk() if full is None else n
        self.last_chunks = 0
        for c0 in range(0, n, chunk):
            c1 = min(n, c0 + chunk)
            m = c1 - c0
            need = self.lib.hapt_dp_workspace_bytes(ctypes.byref(t.t), m)
            ws = self._workspace(need)
            check(
                self.lib.hapt_dp_sweep_batch_cpl(
                    ctypes.byref(t.t),
                    tmax[c0:c1].data_ptr(),
                    m,
                    ftop[c0:c1].data_ptr(),
                    states[c0:c1].data_ptr(),
                    ctypes.byref(full) if full is not None else None,
                    ws.data_ptr(),
                    ws.numel(),
                    int(cpl),
                    stream_ptr(),
                )
            )
            self.last_chunks += 1
        return ftop, states

    def select_device(self, ftop: torch.Tensor, tmax: torch.Tensor, num_microbatches: int):
        n = int(tmax.numel())
        tstar = torch.empty(n, dtype=_F64, device=self.device)
        best_s = torch.empty(n, dtype=_I32, device=self.device)
        winner = torch.empty(1, dtype=_I32, device=self.device)
        check(
            self.lib.hapt_dp_select(
                ftop.data_ptr(), tmax.data_ptr(), n, self.tables.s_max, int(num_microbatches),
                tstar.data_ptr(), best_s.data_ptr(), winner.data_ptr(), stream_ptr(),
            )
        )
        return tstar, best_s, winner

    def evaluate(self, tmax_values, num_microbatches: int, keep_bp: bool = False,
                 keep_ftop: bool = False, cpl: int = 0) -> SweepResult:
        """Sweep + select a batch; one host transfer for all per-candidate
        results.  keep_bp also records packed backpointers for every
        candidate (when they fit BP_BUDGET) so a winner can be walked without
        a re-sweep (hapt_dp_walk); keep_ftop also returns F[s,1,G] per
        candidate, which does not depend on B (rescoring for other B)."""
        tm = np.asarray(tmax_values, dtype=np.float64)
        n = len(tm)
        tmax = torch.from_numpy(tm).to(self.device)
        full = bp = ntop = None
        if keep_bp and self.bp_bytes(n) <= self.BP_BUDGET:
            t = self.tables
            bp = torch.empty((n, t.s_max + 1, t.L + 2, t.G + 1), dtype=_I32, device=self.device)
            ntop = torch.zeros((n, t.s_max + 1), dtype=_I32, device=self.device)
            full = DpFull(None, None, None, None, bp.data_ptr(), ntop.data_ptr())
        ftop, states = self.sweep_device(tmax, full=full, cpl=cpl)
        tstar, best_s, winner = self.select_device(ftop, tmax, num_microbatches)
        parts = [tstar.view(torch.int64), best_s.to(torch.int64), states,
                 winner.to(torch.int64)]
        if ntop is not None:
            parts.append(ntop.to(torch.int64).reshape(-1))
        n_ntop = 0 if ntop is None else ntop.numel()
        if keep_ftop:
            parts.append(ftop.reshape(-1).view(torch.int64))
        host = torch.cat(parts).cpu().numpy()
        ftop_host = None
        if keep_ftop:
            ftop_host = host[3 * n + 1 + n_ntop:].view(np.float64).reshape(n, -1).copy()
            host = host[:3 * n + 1 + n_ntop]
        return SweepResult(
            ftop=ftop_host,
            tmax=tm,
            tstar=host[:n].view(np.float64).copy(),
            best_s=host[n : 2 * n].copy(),
            states=host[2 * n : 3 * n].copy(),
            winner=int(host[3 * n]),
            bp=bp,
            ntop=None if ntop is None else host[3 * n + 1 :].reshape(n, -1).copy(),
        )

    def walk(self, res: SweepResult, idx: int, best_s: int):
        """Stage chain [(layer_start, layer_end, option)] of candidate idx of a
        keep_bp batch, walked on the device (planner.py:300-312)."""
        t = self.tables
        out = torch.empty(3 * t.s_max + 1, dtype=_I32, device=self.device)
        check(self.lib.hapt_dp_walk(ctypes.byref(t.t), res.bp[idx].data_ptr(), int(best_s),
                                    out.data_ptr(), out[3 * t.s_max :].data_ptr(), stream_ptr()))
        h = out.cpu().numpy()
        n = int(h[3 * t.s_max])
        if n < 0:
            from .planner import PlannerError

            raise PlannerError("broken backpointer chain" if n == -1
                               else "plan does not cover all layers and devices")
        return [tuple(int(x) for x in row) for row in h[: 3 * n].reshape(n, 3)]

    def full_tables(self, t_max: float):
        """Reference-layout F, N, bp_i, bp_o for one candidate (drop-in
        dp_sweep); returns device tensors."""
        t = self.tables
        shape = (t.s_max + 1, t.L + 2, t.G + 1)
        if not t_max > 0:  # no span fits: the reference's fresh arrays, untouched
            F = torch.full(shape, math.inf, dtype=_F64, device=self.device)
            F[0, t.L + 1, 0] = 0.0
            return (F, torch.zeros(shape, dtype=_F64, device=self.device),
                    torch.full(shape, -1, dtype=_I32, device=self.device),
                    torch.full(shape, -1, dtype=_I32, device=self.device))
        F = torch.empty(shape, dtype=_F64, device=self.device)
        N = torch.empty(shape, dtype=_F64, device=self.device)
        bpi = torch.empty(shape, dtype=_I32, device=self.device)
        bpo = torch.empty(shape, dtype=_I32, device=self.device)
        ws = self._workspace(self.lib.hapt_dp_sweep_workspace_bytes(ctypes.byref(t.t)))
        check(self.lib.hapt_dp_sweep(ctypes.byref(t.t), float(t_max), F.data_ptr(), N.data_ptr(),
                                     bpi.data_ptr(), bpo.data_ptr(), ws.data_ptr(), ws.numel(),
                                     stream_ptr()))
        return F, N, bpi, bpo

    def backtrack(self, t_max: float, best_s: int):
        """[(layer_start, layer_end, option)] from (best_s, 1, G) and the K chain."""
        t = self.tables
        need = self.lib.hapt_backtrack_workspace_bytes(ctypes.byref(t.t))
        if self._bt_ws is None or self._bt_ws.numel() < need:
            self._bt_ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        out = torch.empty(3 * t.s_max + t.s_max + 1, dtype=_I32, device=self.device)
        stages = out[: 3 * t.s_max]
        kchain = out[3 * t.s_max : 4 * t.s_max]
        n_st = out[4 * t.s_max :]
        code = self.lib.hapt_dp_backtrack(
            ctypes.byref(t.t), float(t_max), int(best_s), stages.data_ptr(), kchain.data_ptr(),
            n_st.data_ptr(), self._bt_ws.data_ptr(), self._bt_ws.numel(), stream_ptr(),
        )
        if code == _lib.HAPT_ECHAIN:
            from .planner import PlannerError

            raise PlannerError(self.lib.hapt_last_error().decode())
        check(code)
        h = out.cpu().numpy()
        n = int(h[4 * t.s_max])
        st = h[: 3 * n].reshape(n, 3)
        return [tuple(int(x) for x in row) for row in st], [int(x) for x in h[3 * t.s_max : 3 * t.s_max + n]]

    def activated(self, tmax_values) -> np.ndarray:
        tm = torch.as_tensor(np.asarray(tmax_values, dtype=np.float64)).to(self.device)
        out = torch.empty(int(tm.numel()), dtype=torch.int64, device=self.device)
        check(
            self.lib.hapt_activated_pairs(
                ctypes.byref(self.tables.t), tm.data_ptr(), int(tm.numel()), out.data_ptr(),
                stream_ptr(),
            )
        )
        return out.cpu().numpy()
