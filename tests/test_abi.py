"""CPU tests of the drop-in boundary: libvxb.so builds for sm_100a, loads, and
exports every entry point include/vxb.h declares; the numpy/ctypes mirrors
match the C struct layouts; without a GPU the engine fails loudly (there is
no CPU fallback)."""
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2308_01241_b200 import _abi
from paper_2308_01241_b200.engine import SimError, SimInstance, SimOptions

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "vxb.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*[\w\s\*]+?\b(vxb_\w+)\s*\(", text, re.M)))


def test_header_declarations_are_mirrored():
    assert set(declared_functions()) == set(_abi.EXPORTS)


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", str(_abi.LIB_PATH)], check=True,
                         capture_output=True, text=True).stdout
    syms = {l.split()[-1] for l in out.splitlines() if l.strip()}
    missing = [f for f in declared_functions() if f not in syms]
    assert not missing, missing
    lib = _abi.load_library()
    assert lib.vxb_abi_version() == 1


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_abi.LIB_PATH)], check=True,
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_header():
    # offsets/sizes fixed in vxb.h; see the comments there
    assert _abi.SYN_DTYPE.itemsize == 16
    assert _abi.NEURON_DTYPE.itemsize == 136
    assert _abi.UNIT_DTYPE.itemsize == 24
    assert _abi.RASTER_DTYPE.itemsize == 24
    assert _abi.TIMINGS_DTYPE.itemsize == 168


def test_struct_layouts_compiled():
    """Compile a probe against vxb.h and compare sizeof/offsetof with numpy."""
    src = r'''
#include <stddef.h>
#include <stdio.h>
#include "vxb.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(vxb_syn_entry), sizeof(vxb_neuron),
         sizeof(vxb_unit), sizeof(vxb_raster_event), sizeof(vxb_step_timings),
         sizeof(vxb_worker_table), sizeof(vxb_network), sizeof(vxb_options));
  printf("%zu %zu %zu %zu %zu\n", offsetof(vxb_neuron, capacitance), offsetof(vxb_neuron, g),
         offsetof(vxb_neuron, v_init), offsetof(vxb_step_timings, bytes_sent_intra),
         offsetof(vxb_options, device));
  return 0;
}
'''
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        p = Path(d) / "probe.c"
        p.write_text(src)
        exe = Path(d) / "probe"
        subprocess.run(["gcc", "-I", str(ROOT / "include"), str(p), "-o", str(exe)], check=True)
        out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    sizes, offs = [list(map(int, l.split())) for l in out.splitlines()]
    import ctypes as C
    assert sizes == [16, 136, 24, 24, 168, C.sizeof(_abi.WorkerTable), C.sizeof(_abi.Network),
                     C.sizeof(_abi.Options)]
    assert offs[0] == _abi.NEURON_DTYPE.fields["capacitance"][1]
    assert offs[1] == _abi.NEURON_DTYPE.fields["g"][1]
    assert offs[2] == _abi.NEURON_DTYPE.fields["v_init"][1]
    assert offs[3] == _abi.TIMINGS_DTYPE.fields["bytes_sent_intra"][1]
    assert offs[4] == _abi.Options.device.offset


def _gpu_present():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_gpu_present(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback_without_gpu():
    from refnet import RefNet, make_config
    net = RefNet(make_config(seed=1, voxels=1, npv=20, k_in=3))
    with pytest.raises(SimError, match="no CUDA device"):
        SimInstance(net.tables, SimOptions(steps=5))


def test_product_does_not_reference_oracle():
    """The product package never imports, links or loads anything under oracle/."""
    pkg = ROOT / "paper_2308_01241_b200"
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        text = f.read_text()
        for bad in ("refnet", "voxsim_ref", "vxo_", "oracle/_ref", "voxsim_oracle"):
            assert bad not in text, (f, bad)
