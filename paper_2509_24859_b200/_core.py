"""Drop-in replacement for `meshpipe._core` (reference _core/__init__.py:1-20).

`dp_sweep` keeps the exact 15-argument signature and return tuple of the
reference operator (_dp.pyx:14-28; dp_py.py:27-43): numpy inputs in the
DpTables layout, numpy outputs F, N (float64) and bp_i, bp_o (int32) of shape
[s_max+1, L+2, G+1].  The sweep runs on the GPU (hapt_tables_finalize +
hapt_dp_sweep with full outputs); a reference caller such as
planner.dp_search or benchmarks/bench_dp.py can be pointed at it unchanged
by rebinding the reference module attribute `planner.dp_sweep` to this
function (INTEGRATION.md shows the one-line binding; tests/test_gpu_dropin.py
runs the reference's own search() through it).

Encodings: any (g_mesh, g_avail) the DP's successor-table hoisting can
represent is accepted -- every option uses >= 1 device and the boundary row
of a transition is a function of its successor state (include/hapt_b200.h,
hapt_tables_finalize).  DpTables' encoding always qualifies; others raise
ValueError instead of returning different tables.

There is no CPU fallback: without the CUDA library this module raises.
"""

from __future__ import annotations

import threading
from collections import OrderedDict

import numpy as np

from .engine import DeviceTables, Sweeper

BACKEND = "cuda"

# The reference calls dp_sweep from ThreadPoolExecutor workers
# (planner.py:529-531), and the Cython kernel is reentrant.  Here one lock
# covers the whole call -- table lookup/upload, the ~2 launches per layer on
# the shared per-stream workspace, and the device-to-host copies -- so
# concurrent calls are serialised instead of interleaving their kernels on
# one scratch buffer.  Table sets are cached per call key (several DpTables
# may be in use at once), least recently used first out.
_lock = threading.Lock()
_cache: "OrderedDict[tuple, tuple]" = OrderedDict()
_CACHE_MAX = 4


def _entry(args: dict, s_max: int):
    """(DeviceTables, Sweeper) for these arrays.  Tables are cached on the
    identity of the caller's arrays (DpTables keeps them alive for a whole
    search), so repeated sweeps skip the upload; the entry also holds the
    arrays, so an id cannot be recycled while its entry lives."""
    key = tuple(id(args[k]) for k in sorted(args)) + (s_max,)
    hit = _cache.get(key)
    if hit is not None and all(hit[1][k] is args[k] for k in args):
        _cache.move_to_end(key)
        return hit[0], hit[2]
    L = args["t_tab"].shape[1] - 2
    G = args["g_mesh"].shape[0] - 1
    n_opts = args["t_tab"].shape[0]
    n_meshes = args["cb_same"].shape[0]
    opt_off = np.asarray(args["opt_off"])
    g_mesh = np.asarray(args["g_mesh"])
    if (len(opt_off) != n_meshes + 1 or int(opt_off[0]) != 0 or int(opt_off[-1]) != n_opts
            or np.any(np.diff(opt_off) < 0)):
        raise ValueError("dp_sweep: opt_off must partition the options by mesh")
    if G >= 1 and (np.any(g_mesh[1:] < 0) or np.any(g_mesh[1:] >= n_meshes)):
        raise ValueError("dp_sweep: g_mesh out of range")
    dt = DeviceTables(L, G, n_opts, n_meshes).load_dense(args, s_max)
    if int(dt.counters()[10]):
        raise ValueError(
            "dp_sweep: unsupported remaining-device encoding (an option with no "
            "device, or a successor state whose boundary row depends on the "
            "caller; see hapt_tables_finalize in include/hapt_b200.h)")
    _cache[key] = (dt, dict(args), Sweeper(dt))
    while len(_cache) > _CACHE_MAX:
        _cache.popitem(last=False)
    return dt, _cache[key][2]


def dp_sweep(t_max, t_tab, mp_tab, ma_tab, opt_cap, opt_mesh, opt_devs, opt_off, cb_same,
             cb_next, g_mesh, g_avail, s_max, span_off, span_items):
    """One t_max candidate through the stage-partition DP (_dp.pyx:48-95)."""
    t_tab = np.asarray(t_tab)
    for name, arr, dt, nd in (
        ("t_tab", t_tab, np.float64, 3), ("mp_tab", mp_tab, np.float64, 3),
        ("ma_tab", ma_tab, np.float64, 3), ("opt_cap", opt_cap, np.float64, 1),
        ("opt_mesh", opt_mesh, np.int32, 1), ("opt_devs", opt_devs, np.int32, 1),
        ("opt_off", opt_off, np.int32, 1), ("cb_same", cb_same, np.float64, 2),
        ("cb_next", cb_next, np.float64, 2), ("g_mesh", g_mesh, np.int32, 1),
        ("g_avail", g_avail, np.int32, 1), ("span_off", span_off, np.int32, 1),
        ("span_items", span_items, np.int32, 1),
    ):
        a = np.asarray(arr)
        if a.dtype != dt or a.ndim != nd:
            # the Cython memoryviews reject these the same way
            raise ValueError(f"Buffer dtype mismatch for {name}: expected {np.dtype(dt)} "
                             f"with {nd} dims, got {a.dtype} with {a.ndim}")
    s_max = int(s_max)
    args = dict(t_tab=t_tab, mp_tab=mp_tab, ma_tab=ma_tab, opt_cap=opt_cap, opt_mesh=opt_mesh,
                opt_devs=opt_devs, opt_off=opt_off, cb_same=cb_same, cb_next=cb_next,
                g_mesh=g_mesh, g_avail=g_avail, span_off=span_off, span_items=span_items)
    with _lock:
        _dt, sw = _entry(args, s_max)  # _dt keeps the tables alive for the call
        F, N, bpi, bpo = sw.full_tables(float(t_max))
        return F.cpu().numpy(), N.cpu().numpy(), bpi.cpu().numpy(), bpo.cpu().numpy()


__all__ = ["dp_sweep", "BACKEND"]
