"""ctypes binding of libhapt_b200.so (ABI: include/hapt_b200.h).

PyTorch is used only for device memory and the current stream; every kernel
lives in the C-ABI library.  There is no CPU fallback: if the library is not
built, or no CUDA device is present, `lib()` raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HAPT_LIB") or os.path.join(PKG, "libhapt_b200.so")

HAPT_OK = 0
HAPT_EINVAL = 1
HAPT_ECUDA = 2
HAPT_ENOSPACE = 3
HAPT_ECOMM = 4
HAPT_ESCHED = 5
HAPT_ECHAIN = 6
HAPT_ECYCLE = 7

COUNTS_CLASSIC = 0
COUNTS_EAGER = 1
COUNTS_ADAPTIVE = 2

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
c_sz = ctypes.c_size_t


class ModelDesc(ctypes.Structure):
    _fields_ = [
        ("L", c_i32),
        ("n_meshes", c_i32),
        ("n_opts", c_i32),
        ("G", c_i32),
        ("layer_flops", c_vp),
        ("layer_params", c_vp),
        ("layer_bbytes", c_vp),
        ("layer_sig", c_vp),
        ("mesh_hosts", c_vp),
        ("mesh_dph", c_vp),
        ("mesh_peak", c_vp),
        ("mesh_mem", c_vp),
        ("mesh_intra_bw", c_vp),
        ("mesh_inter_bw", c_vp),
        ("cross_bw_next", c_vp),
        ("opt_n", c_vp),
        ("opt_m", c_vp),
        ("opt_mesh", c_vp),
        ("ovr_index", c_vp),
        ("ovr_vals", c_vp),
        ("cross_latency", c_dbl),
        ("beta", c_dbl),
        ("efficiency", c_dbl),
        ("alpha", c_dbl),
        ("replication", c_dbl),
        ("act_factor", c_dbl),
        ("imbalance_ratio", c_dbl),
        ("total_flops", c_dbl),
        ("total_peak", c_dbl),
        ("dedup", c_i32),
    ]


class Tables(ctypes.Structure):
    _fields_ = [
        ("L", c_i32),
        ("G", c_i32),
        ("n_opts", c_i32),
        ("n_meshes", c_i32),
        ("s_max", c_i32),
        ("nnz_cap", c_i32),
        ("pool_cap", c_i32),
        ("t_tab", c_vp),
        ("mp_tab", c_vp),
        ("ma_tab", c_vp),
        ("tf_raw", c_vp),
        ("tb_raw", c_vp),
        ("mp_raw", c_vp),
        ("ma_raw", c_vp),
        ("cell_state", c_vp),
        ("canon_q", c_vp),
        ("opt_cap", c_vp),
        ("opt_mesh", c_vp),
        ("opt_devs", c_vp),
        ("opt_off", c_vp),
        ("cb_same", c_vp),
        ("cb_next", c_vp),
        ("g_mesh", c_vp),
        ("g_avail", c_vp),
        ("g_crow", c_vp),
        ("span_off", c_vp),
        ("span_items", c_vp),
        ("spans", c_vp),
        ("span_srank", c_vp),
        ("row_kmin", c_vp),
        ("row_pos", c_vp),
        ("pool", c_vp),
        ("counters", c_vp),
        ("scratch", c_vp),
        ("scratch_bytes", c_sz),
    ]


class DpFull(ctypes.Structure):
    _fields_ = [("F", c_vp), ("N", c_vp), ("bp_i", c_vp), ("bp_o", c_vp), ("bp_packed", c_vp),
                ("ntop", c_vp)]


_SIGNATURES = {
    "hapt_last_error": (ctypes.c_char_p, []),
    "hapt_version": (c_i32, []),
    "hapt_launches": (c_i64, []),
    "hapt_tables_bytes": (c_sz, [c_i32, c_i32, c_i32, c_i32]),
    "hapt_tables_init": (c_i32, [ctypes.POINTER(Tables), c_vp, c_sz, c_i32, c_i32, c_i32, c_i32]),
    "hapt_tables_build": (c_i32, [ctypes.POINTER(Tables), ctypes.POINTER(ModelDesc), c_vp]),
    "hapt_tables_finalize": (c_i32, [ctypes.POINTER(Tables), c_vp]),
    "hapt_dp_workspace_bytes": (c_sz, [ctypes.POINTER(Tables), c_i32]),
    "hapt_dp_sweep_batch": (
        c_i32,
        [ctypes.POINTER(Tables), c_vp, c_i32, c_vp, c_vp, ctypes.POINTER(DpFull), c_vp, c_sz, c_vp],
    ),
    "hapt_dp_sweep_batch_cpl": (
        c_i32,
        [ctypes.POINTER(Tables), c_vp, c_i32, c_vp, c_vp, ctypes.POINTER(DpFull), c_vp, c_sz,
         c_i32, c_vp],
    ),
    "hapt_dp_select": (c_i32, [c_vp, c_vp, c_i32, c_i32, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "hapt_dp_sweep_workspace_bytes": (c_sz, [ctypes.POINTER(Tables)]),
    "hapt_dp_sweep": (
        c_i32, [ctypes.POINTER(Tables), c_dbl, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp],
    ),
    "hapt_backtrack_workspace_bytes": (c_sz, [ctypes.POINTER(Tables)]),
    "hapt_dp_backtrack": (
        c_i32,
        [ctypes.POINTER(Tables), c_dbl, c_i32, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp],
    ),
    "hapt_dp_walk": (c_i32, [ctypes.POINTER(Tables), c_vp, c_i32, c_vp, c_vp, c_vp]),
    "hapt_activated_pairs": (c_i32, [ctypes.POINTER(Tables), c_vp, c_i32, c_vp, c_vp]),
    "hapt_launch_counts": (
        c_i32,
        [c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_dbl, c_i32, c_vp, c_vp, c_vp],
    ),
    "hapt_sim_workspace_bytes": (c_sz, [c_i64, c_i32]),
    "hapt_sim_1f1b": (
        c_i32,
        [c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp,
         c_sz, c_vp],
    ),
    "hapt_analyze_1f1b": (
        c_i32,
        [c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
         c_vp, c_vp, c_vp, c_vp],
    ),
    "hapt_sim_1f1b_trace": (
        c_i32,
        [c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_sz,
         c_vp],
    ),
    "hapt_analyze_1f1b_trace": (
        c_i32,
        [c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
         c_vp, c_vp, c_vp],
    ),
    "hapt_prof_enable": (c_i32, [c_i32]),
    "hapt_prof_read": (c_i32, [c_vp, c_vp, c_i32]),
    "hapt_steady_rate_1f1b": (c_i32, [c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "hapt_asap_workspace_bytes": (c_sz, [c_i32]),
    "hapt_dag_asap_check": (
        c_i32, [c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_dbl, c_vp, c_vp, c_sz, c_vp],
    ),
    "hapt_dag_workspace_bytes": (c_sz, [c_i32]),
    "hapt_dag_longest_path": (
        c_i32,
        [c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp],
    ),
    "hapt_fp64_probe": (c_i32, [c_vp, c_i32, c_i32, c_i32, c_vp]),
    "hapt_detect_modules": (c_i32, [c_i32, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "hapt_cluster_layers": (
        c_i32,
        [c_i32, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp,
         c_vp, c_vp],
    ),
    "hapt_py_sum": (c_dbl, [c_vp, c_i32]),
}

EXPORTED = tuple(_SIGNATURES)

_lock = threading.Lock()
_handle = None


class HaptError(RuntimeError):
    def __init__(self, code: int, message: str):
        self.code = code
        super().__init__(f"hapt error {code}: {message}")


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the shared library and declare every exported signature (no GPU
    needed; used by the CPU test that checks the ABI)."""
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is not built; run `python -m paper_2509_24859_b200.build` "
            "(no CPU fallback exists for the planner hot path)"
        )
    h = ctypes.CDLL(path)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(h, name)
        fn.restype = res
        fn.argtypes = args
    return h


def lib() -> ctypes.CDLL:
    """The library, checked to be usable: it must load and a CUDA device must
    be present.  Raises instead of falling back to a CPU path."""
    global _handle
    if _handle is None:
        with _lock:
            if _handle is None:
                import torch

                if not torch.cuda.is_available():
                    raise RuntimeError(
                        "paper_2509_24859_b200 needs a CUDA device (sm_100a); "
                        "the planner hot path has no CPU fallback"
                    )
                _handle = load()
    return _handle


_host_handle = None


def host_lib() -> ctypes.CDLL:
    """The library for its host-only entry points (the model-graph front end
    is native C++ host code, like the reference's front end is host Python);
    no CUDA device needed."""
    global _host_handle
    if _host_handle is None:
        with _lock:
            if _host_handle is None:
                _host_handle = _handle if _handle is not None else load()
    return _host_handle


def check(code: int) -> None:
    if code != HAPT_OK:
        msg = lib().hapt_last_error()
        raise HaptError(code, msg.decode() if msg else "")


def check_host(code: int) -> None:
    if code != HAPT_OK:
        msg = host_lib().hapt_last_error()
        raise HaptError(code, msg.decode() if msg else "")


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t) -> int:
    return 0 if t is None else t.data_ptr()
