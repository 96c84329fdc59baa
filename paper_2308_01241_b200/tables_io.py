"""VXTB v1 worker-table files + manifest.json (next-2 row of SURVEY.md §8(f)).

Byte-compatible with the reference's save_tables / load_tables
(/root/reference/proj/src/netgen.cpp:359-539): 36-byte LE header (magic
"VXTB", version 1, worker, worker_count, seed, n_neurons, n_synapses), 136-byte
neuron records, 16-byte synapse entries; manifest.json lists the files with
their FNV-1a hashes (util.hpp:39-46), unit_worker and unit_local_base.

The synapse block of a file is exactly the vxb_syn_entry array, so it is mapped
and handed to the engine without any per-synapse host work; FNV-1a runs in
native code (vxb_fnv1a).  The layout (units) is not stored in the tables: as in
cmd_simulate --tables (voxsim.cpp:149-156) it is rebuilt from the config
(config.json, written next to the tables by `generate`).
"""
from __future__ import annotations

import json
import mmap
import os
from pathlib import Path

import numpy as np

from . import _abi
from ._abi import NEURON_DTYPE, SYN_DTYPE, ptr
from .engine import NetworkTables, SimError, WorkerTable

MAGIC = 0x42545856  # "VXTB"
VERSION = 1
HEADER = np.dtype([("magic", "<u4"), ("version", "<u4"), ("worker", "<u2"),
                   ("worker_count", "<u2"), ("seed", "<u8"), ("n_neurons", "<u8"),
                   ("n_synapses", "<u8")])
DISK_NEURON = np.dtype([  # netgen.cpp:375-396 field order
    ("gid", "<u8"), ("voxel", "<u4"), ("pop", "<u2"), ("excitatory", "u1"), ("pad", "u1"),
    ("unit", "<u4"), ("row_len", "<u4"), ("dst_mask", "<u8"), ("capacitance", "<f4"),
    ("g_leak", "<f4"), ("e_leak", "<f4"), ("v_threshold", "<f4"), ("v_reset", "<f4"),
    ("refractory_steps", "<u4"), ("e_rev", "<f4", 4), ("tau", "<f4", 4), ("omega", "<f4", 4),
    ("g", "<f4", 4), ("ou_mean", "<f4"), ("ou_sigma", "<f4"), ("ou_tau", "<f4"),
    ("v_init", "<f4")])
assert HEADER.itemsize == 36 and DISK_NEURON.itemsize == 136
FNV_OFFSET = 0xCBF29CE484222325


def fnv1a(data, h: int = FNV_OFFSET) -> int:
    """FNV-1a 64 of a bytes-like object (native loop in libvxb)."""
    lib = _abi.load_library()
    arr = np.frombuffer(data, np.uint8)
    if arr.size == 0:
        return h
    return int(lib.vxb_fnv1a(arr.ctypes.data, arr.size, h))


def _to_disk(neurons: np.ndarray) -> np.ndarray:
    d = np.zeros(neurons.shape[0], DISK_NEURON)
    for f in DISK_NEURON.names:
        if f != "pad":
            d[f] = neurons[f]
    return d


def _from_disk(d: np.ndarray) -> np.ndarray:
    n = np.zeros(d.shape[0], NEURON_DTYPE)
    for f in DISK_NEURON.names:
        if f != "pad":
            n[f] = d[f]
    return n


def save_worker_table(t: WorkerTable, path) -> None:
    """netgen.cpp:362-406"""
    hdr = np.zeros(1, HEADER)
    hdr[0] = (MAGIC, VERSION, t.worker, t.worker_count, t.seed, t.neurons.shape[0],
              t.synapses.shape[0])
    with open(path, "wb") as f:
        f.write(hdr.tobytes())
        f.write(_to_disk(t.neurons).tobytes())
        f.write(np.ascontiguousarray(t.synapses).view(np.uint8).tobytes())


def load_worker_table(path) -> WorkerTable:
    """netgen.cpp:408-464: same validation and error messages."""
    path = str(path)
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        mm = mmap.mmap(f.fileno(), 0, access=mmap.ACCESS_READ) if size else b""
    buf = memoryview(mm) if size else memoryview(b"")
    if size < 8:
        raise SimError(f"truncated table file: {path}")
    magic, version = np.frombuffer(buf[:8], "<u4")
    if magic != MAGIC:
        raise SimError(f"not a worker table file: {path}")
    if version != VERSION:
        raise SimError(f"unsupported table version: {path}")
    if size < HEADER.itemsize:
        raise SimError(f"truncated table file: {path}")
    h = np.frombuffer(buf[:HEADER.itemsize], HEADER)[0]
    nn, ns = int(h["n_neurons"]), int(h["n_synapses"])
    off_n = HEADER.itemsize
    off_s = off_n + nn * DISK_NEURON.itemsize
    if off_s > size:
        raise SimError(f"truncated table file: {path}")
    neurons = _from_disk(np.frombuffer(buf[off_n:off_s], DISK_NEURON))
    row_base = np.zeros(nn + 1, np.uint64)
    np.cumsum(neurons["row_len"], out=row_base[1:])
    if int(row_base[-1]) != ns:
        raise SimError(f"row lengths do not add up to synapse count: {path}")
    end = off_s + ns * SYN_DTYPE.itemsize
    if end > size:
        raise SimError(f"truncated table file: {path}")
    if end != size:
        raise SimError(f"trailing bytes in table file: {path}")
    syn = np.frombuffer(buf[off_s:end], SYN_DTYPE) if ns else np.zeros(0, SYN_DTYPE)
    return WorkerTable(int(h["worker"]), int(h["worker_count"]), int(h["seed"]), neurons, syn,
                       row_base)


def save_tables(tables: NetworkTables, directory) -> None:
    """netgen.cpp:466-500 (manifest.json with per-file FNV-1a)."""
    d = Path(directory)
    d.mkdir(parents=True, exist_ok=True)
    files, neurons, synapses = [], 0, 0
    for t in tables.workers:
        name = f"worker_{t.worker:03d}.bin"
        save_worker_table(t, d / name)
        files.append({"file": name, "worker": t.worker, "neurons": int(t.neurons.shape[0]),
                      "synapses": int(t.synapses.shape[0]),
                      "fnv1a": f"{fnv1a((d / name).read_bytes()):016x}"})
        neurons += t.neurons.shape[0]
        synapses += t.synapses.shape[0]
    manifest = {"version": VERSION, "workers": len(tables.workers),
                "seed": tables.workers[0].seed if tables.workers else 0,
                "neurons": int(neurons), "synapses": int(synapses), "files": files,
                "unit_worker": [int(x) for x in tables.unit_worker],
                "unit_local_base": [int(x) for x in tables.unit_local_base]}
    (d / "manifest.json").write_text(json.dumps(manifest, indent=2) + "\n")


def _file_hash(path: str) -> int:
    size = os.path.getsize(path)
    if size == 0:
        return FNV_OFFSET
    with open(path, "rb") as f, mmap.mmap(f.fileno(), 0, access=mmap.ACCESS_READ) as mm:
        return fnv1a(mm)


def load_tables(directory, units: np.ndarray, n_voxels: int) -> NetworkTables:
    """netgen.cpp:502-539: verify every file's FNV-1a against the manifest,
    load, sort by worker, check the worker set.  `units` / `n_voxels` come from
    the layout rebuilt from the run's config (voxsim.cpp:151-156)."""
    d = Path(directory)
    try:
        manifest = json.loads((d / "manifest.json").read_text())
    except OSError:
        raise SimError(f"cannot open manifest in {directory}")
    workers = []
    for f in manifest["files"]:
        path = str(d / f["file"])
        want = int(f["fnv1a"], 16)
        got = _file_hash(path)
        if want != got:
            raise SimError(f"table hash mismatch for {path}: manifest {want:016x} vs file "
                           f"{got:016x}")
        workers.append(load_worker_table(path))
    workers.sort(key=lambda t: t.worker)
    for w, t in enumerate(workers):
        if t.worker != w or t.worker_count != len(workers):
            raise SimError("manifest worker set is inconsistent")
    return NetworkTables(workers, np.asarray(manifest["unit_worker"], np.uint16),
                         np.asarray(manifest["unit_local_base"], np.uint32), units, n_voxels)
