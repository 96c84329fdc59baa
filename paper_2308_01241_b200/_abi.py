"""ctypes / numpy mirror of include/vxb.h (the C ABI of the CUDA engine).

The numpy structured dtypes are byte-identical to the C structs so tables of
any size can be built with vectorised numpy and handed to vxb_create without
per-record Python work.  The loader fails loudly: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libvxb.so"

VXB_OK, VXB_ECONFIG, VXB_ESIM = 0, 2, 3
RECEPTORS = 4

# ---------------------------------------------------------------- dtypes
SYN_DTYPE = np.dtype(
    {
        "names": ["src_local", "src_worker", "cls", "pad", "wq_fast", "wq_slow"],
        "formats": ["<u4", "<u2", "u1", "u1", "<i4", "<i4"],
        "offsets": [0, 4, 6, 7, 8, 12],
        "itemsize": 16,
    }
)

NEURON_DTYPE = np.dtype(
    {
        "names": [
            "gid", "dst_mask", "voxel", "unit", "row_len", "refractory_steps", "pop",
            "excitatory", "pad0", "capacitance", "g_leak", "e_leak", "v_threshold",
            "v_reset", "e_rev", "tau", "omega", "g", "ou_mean", "ou_sigma", "ou_tau",
            "v_init",
        ],
        "formats": [
            "<u8", "<u8", "<u4", "<u4", "<u4", "<u4", "<u2", "u1", "u1", "<f4", "<f4",
            "<f4", "<f4", "<f4", ("<f4", 4), ("<f4", 4), ("<f4", 4), ("<f4", 4), "<f4",
            "<f4", "<f4", "<f4",
        ],
        "offsets": [0, 8, 16, 20, 24, 28, 32, 34, 35, 36, 40, 44, 48, 52, 56, 72, 88,
                    104, 120, 124, 128, 132],
        "itemsize": 136,
    }
)

UNIT_DTYPE = np.dtype(
    {
        "names": ["gid_base", "voxel", "neurons", "pop", "excitatory", "pad0", "pad1"],
        "formats": ["<u8", "<u4", "<u4", "<u2", "u1", "u1", "<u4"],
        "offsets": [0, 8, 12, 16, 18, 19, 20],
        "itemsize": 24,
    }
)

RASTER_DTYPE = np.dtype(
    {
        "names": ["step", "worker", "pad0", "local", "pad1", "gid"],
        "formats": ["<u4", "<u2", "<u2", "<u4", "<u4", "<u8"],
        "offsets": [0, 4, 6, 8, 12, 16],
        "itemsize": 24,
    }
)

TIMINGS_DTYPE = np.dtype(
    {
        "names": [
            "step", "worker", "pad0", "t", "send_intra_ns", "send_inter_ns",
            "recv_intra_ns", "recv_inter_ns", "bytes_sent_intra", "bytes_sent_inter",
            "bytes_recv_intra", "bytes_recv_inter", "spikes", "pad1",
        ],
        "formats": [
            "<u4", "<u2", "<u2", ("<i8", 11), "<i8", "<i8", "<i8", "<i8", "<u8", "<u8",
            "<u8", "<u8", "<u4", "<u4",
        ],
        "offsets": [0, 4, 6, 8, 96, 104, 112, 120, 128, 136, 144, 152, 160, 164],
        "itemsize": 168,
    }
)

INJECTION_DTYPE = np.dtype([("from_step", "<u4"), ("to_step", "<u4"), ("voxel", "<u4"),
                            ("current_pa", "<f4")])
FORCED_DTYPE = np.dtype([("step", "<u4"), ("pad0", "<u4"), ("gid", "<u8")])


# ------------------------------------------------------- ctypes descriptors
class WorkerTable(C.Structure):
    _fields_ = [
        ("worker", C.c_uint16),
        ("worker_count", C.c_uint16),
        ("n_neurons", C.c_uint32),
        ("seed", C.c_uint64),
        ("n_synapses", C.c_uint64),
        ("neurons", C.c_void_p),
        ("synapses", C.c_void_p),
        ("row_base", C.c_void_p),
    ]


class Network(C.Structure):
    _fields_ = [
        ("n_workers", C.c_uint32),
        ("n_units", C.c_uint32),
        ("n_voxels", C.c_uint32),
        ("pad0", C.c_uint32),
        ("workers", C.POINTER(WorkerTable)),
        ("unit_worker", C.c_void_p),
        ("unit_local_base", C.c_void_p),
        ("units", C.c_void_p),
    ]


class Options(C.Structure):
    _fields_ = [
        ("dt_ms", C.c_double),
        ("scheduler", C.c_char_p),
        ("transport", C.c_char_p),
        ("workers_per_node", C.c_uint16),
        ("pad0", C.c_uint16),
        ("recv_timeout_ms", C.c_int32),
        ("record_raster", C.c_int32),
        ("record_timings", C.c_int32),
        ("probe_gids", C.c_void_p),
        ("n_probes", C.c_uint32),
        ("n_injections", C.c_uint32),
        ("injections", C.c_void_p),
        ("forced_spikes", C.c_void_p),
        ("n_forced", C.c_uint32),
        ("device", C.c_int32),
        ("n_devices", C.c_int32),
        ("pad1", C.c_int32),
    ]


class HemoParams(C.Structure):  # vxb_hemo_params == HemoParams (hemo.hpp:10-23)
    _fields_ = [(n, C.c_double) for n in ("kappa", "gamma", "tau", "alpha", "e0", "v0")]


class Flops(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in
                ("membrane", "gating_inner", "gating_outer", "gating_decay", "current")]


EXPORTS = [
    "vxb_create", "vxb_destroy", "vxb_last_error", "vxb_abi_version", "vxb_advance",
    "vxb_current_step", "vxb_result_steps_done", "vxb_result_total_spikes",
    "vxb_result_raster_size", "vxb_result_raster", "vxb_result_rates",
    "vxb_result_probes", "vxb_result_flops", "vxb_result_timings_size",
    "vxb_result_timings", "vxb_result_device_ms", "vxb_result_h2d_bytes",
    "vxb_result_d2h_bytes", "vxb_result_launches", "vxb_set_conductances",
    "vxb_membrane_snapshot", "vxb_worker_neurons", "vxb_workers", "vxb_units",
    "vxb_probes", "vxb_run_simulation", "vxb_debug_stream_normal", "vxb_debug_stream_xi",
    "vxb_create_generated",
    "vxb_generate_worker_table", "vxb_create_generated_rank", "vxb_mask_bytes",
    "vxb_mask_out", "vxb_mask_in", "vxb_ipc_handle", "vxb_connect_peers",
    "vxb_result_exchange_wait_ms", "vxb_fnv1a", "vxb_set_hemodynamics", "vxb_hemo_get_state",
    "vxb_result_bold_size", "vxb_result_bold", "vxb_debug_bold_from_drive",
    "vxb_result_voxel_counts", "vxb_hemo_feed_counts", "vxb_create_member",
    "vxb_schedule_info", "vxb_build_hash", "vxb_result_wire_bytes", "vxb_set_recv_wire_bytes",
    "vxb_crossing_matrix", "vxb_set_conductances_batch", "vxb_result_exchange_arrival_ms",
    "vxb_advance_members",
]

_lib = None


def _declare(lib):
    P = C.c_void_p
    sig = {
        "vxb_create": (C.c_int, [C.POINTER(Network), C.POINTER(Options), C.POINTER(P)]),
        "vxb_destroy": (None, [P]),
        "vxb_last_error": (C.c_char_p, [P]),
        "vxb_abi_version": (C.c_int, []),
        "vxb_advance": (C.c_int, [P, C.c_uint32]),
        "vxb_current_step": (C.c_uint32, [P]),
        "vxb_result_steps_done": (C.c_uint32, [P]),
        "vxb_result_total_spikes": (C.c_uint64, [P]),
        "vxb_result_raster_size": (C.c_uint64, [P]),
        "vxb_result_raster": (C.c_int, [P, P, C.c_uint64]),
        "vxb_result_rates": (C.c_int, [P, P, C.c_uint64]),
        "vxb_result_probes": (C.c_int, [P, P, P, C.c_uint64]),
        "vxb_result_flops": (C.c_int, [P, C.POINTER(Flops)]),
        "vxb_result_timings_size": (C.c_uint64, [P]),
        "vxb_result_timings": (C.c_int, [P, P, C.c_uint64]),
        "vxb_result_device_ms": (C.c_double, [P]),
        "vxb_result_h2d_bytes": (C.c_uint64, [P]),
        "vxb_result_exchange_wait_ms": (C.c_double, [P]),
        "vxb_result_exchange_arrival_ms": (C.c_double, [P]),
        "vxb_advance_members": (C.c_int, [P, C.c_uint32, C.c_uint32]),
        "vxb_fnv1a": (C.c_uint64, [P, C.c_uint64, C.c_uint64]),
        "vxb_result_d2h_bytes": (C.c_uint64, [P]),
        "vxb_result_launches": (C.c_uint64, [P]),
        "vxb_schedule_info": (C.c_int, [P, C.c_char_p, C.c_uint64]),
        "vxb_build_hash": (C.c_char_p, []),
        "vxb_result_wire_bytes": (C.c_int, [P, P, C.c_uint64]),
        "vxb_crossing_matrix": (C.c_int, [P, P, C.c_uint64]),
        "vxb_set_conductances_batch": (C.c_int, [P, C.c_uint32, P, P, P, P, P]),
        "vxb_set_recv_wire_bytes": (C.c_int, [P, P, C.c_uint32]),
        "vxb_set_conductances": (C.c_int, [P, C.c_uint32, C.c_int, P, C.c_uint32]),
        "vxb_membrane_snapshot": (C.c_int, [P, C.c_uint16, P, C.c_uint32]),
        "vxb_worker_neurons": (C.c_uint32, [P, C.c_uint16]),
        "vxb_workers": (C.c_uint16, [P]),
        "vxb_units": (C.c_uint32, [P]),
        "vxb_probes": (C.c_uint32, [P]),
        "vxb_debug_stream_normal": (C.c_int, [C.c_int, P, P, C.c_uint64, P]),
        "vxb_debug_stream_xi": (C.c_int, [C.c_int, P, P, C.c_uint64, P]),
        "vxb_create_generated": (C.c_int, [P, C.POINTER(Options), C.POINTER(P)]),
        "vxb_generate_worker_table": (C.c_int, [P, C.c_int, C.c_uint16, P, C.c_uint32, P,
                                                C.c_uint64, P]),
        "vxb_create_generated_rank": (C.c_int, [P, C.POINTER(Options), C.c_uint32, C.c_uint32,
                                                C.POINTER(P)]),
        "vxb_mask_bytes": (C.c_uint64, [P, C.c_uint32]),
        "vxb_mask_out": (C.c_int, [P, C.c_uint32, P, C.c_uint64]),
        "vxb_mask_in": (C.c_int, [P, C.c_uint32, P, C.c_uint64]),
        "vxb_ipc_handle": (C.c_int, [P, P, C.c_uint64]),
        "vxb_connect_peers": (C.c_int, [P, P, C.c_uint64]),
        "vxb_run_simulation": (C.c_int, [C.POINTER(Network), C.POINTER(Options), C.c_uint32,
                                         C.POINTER(P)]),
        "vxb_set_hemodynamics": (C.c_int, [P, C.POINTER(HemoParams), C.c_double, C.c_uint32, P]),
        "vxb_hemo_get_state": (C.c_int, [P, P, C.c_uint32]),
        "vxb_result_bold_size": (C.c_uint64, [P]),
        "vxb_result_bold": (C.c_int, [P, P, C.c_uint64]),
        "vxb_result_voxel_counts": (C.c_int, [P, P, C.c_uint64]),
        "vxb_hemo_feed_counts": (C.c_int, [P, P, C.c_uint32]),
        "vxb_create_member": (C.c_int, [P, P, P, C.POINTER(Options), C.POINTER(P)]),
        "vxb_debug_bold_from_drive": (C.c_int, [C.c_int, C.POINTER(HemoParams), P, C.c_uint32,
                                                C.c_uint32, C.c_double, C.c_uint32, P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args


def load_library(path: str | os.PathLike | None = None):
    """Load libvxb.so (the CUDA engine).  Raises if it has not been built."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else Path(os.environ.get("VXB_LIB", LIB_PATH))
    if not p.exists():
        raise RuntimeError(
            f"CUDA engine library {p} is missing: run `python -c 'import __graft_entry__ as g; "
            "g.build()'` (there is no CPU fallback)")
    lib = C.CDLL(str(p))
    _declare(lib)
    if path is None:
        _lib = lib
    return lib


def ptr(a: np.ndarray | None) -> int | None:
    if a is None or a.size == 0:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data
