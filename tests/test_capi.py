"""CPU checks of the boundary: the product library loads, exports exactly the
entry points include/dynwalk_b200.h declares, and fails loudly (no CPU
fallback) when no GPU is present."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dynwalk_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(dw_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("dw_graph_create", "dw_run", "dw_calibrate", "dw_last_error", "dw_graph_destroy"):
        assert s in syms


def test_library_exports_every_declared_symbol(dw):
    lib = dw.load_library()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert sorted(dw.EXPORTED_SYMBOLS) == declared_symbols()
    out = subprocess.run(["nm", "-D", "--defined-only", dw.library_path()], capture_output=True,
                         text=True).stdout
    exported = sorted(set(re.findall(r" T (dw_\w+)", out)))
    assert exported == declared_symbols()


def test_library_is_sm100a(dw):
    out = subprocess.run(["cuobjdump", "--list-elf", dw.library_path()], capture_output=True,
                         text=True)
    assert "sm_100a" in out.stdout


def test_abi_version(dw):
    assert dw.load_library().dw_abi_version() == 2


def test_no_cpu_fallback_without_gpu(dw):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(dw.DynwalkError) as ei:
        dw.DeviceGraph.from_csr(np.array([0, 1, 1], np.uint64), np.array([1], np.uint32),
                                np.array([1.0], np.float32))
    assert ei.value.code == -2  # DW_ECUDA


def test_model_and_mode_validation(dw):
    with pytest.raises(dw.DynwalkError, match="unknown model"):
        dw.Model(kind="dsl").c()
    with pytest.raises(dw.DynwalkError, match="unknown sampler mode"):
        dw.RunOptions(mode="bogus").c()


def test_struct_layouts_match_header(dw):
    """ctypes mirrors of the ABI structs have the C sizes (gcc, x86-64)."""
    src = r'''
#include <stdio.h>
#include "dynwalk_b200.h"
int main(void){printf("%zu %zu %zu %zu %zu %zu\n", sizeof(dw_graph_desc), sizeof(dw_rmat_desc),
 sizeof(dw_model_desc), sizeof(dw_run_opts), sizeof(dw_run_stats), sizeof(void*));return 0;}
'''
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "s.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "s")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", exe, c], check=True)
        sizes = list(map(int, subprocess.run([exe], capture_output=True, text=True).stdout.split()))
    want = [C.sizeof(dw.GraphDesc), C.sizeof(dw.RmatDesc), C.sizeof(dw.ModelDesc),
            C.sizeof(dw.RunOptsC), C.sizeof(dw.RunStatsC), C.sizeof(C.c_void_p)]
    assert sizes == want


def test_dwg1_header_errors(dw, tmp_path):
    """dw_graph_load_dwg1 rejects bad files with load_binary's messages
    (graph.cpp:258-276) before touching a device."""
    with pytest.raises(dw.DynwalkError, match="cannot open graph file"):
        dw.DeviceGraph.load_dwg1(str(tmp_path / "missing.dwg1"))
    bad = tmp_path / "bad.dwg1"
    bad.write_bytes(b"XXXX" + b"\0" * 32)
    with pytest.raises(dw.DynwalkError, match="not a binary graph file"):
        dw.DeviceGraph.load_dwg1(str(bad))
    v2 = tmp_path / "v2.dwg1"
    v2.write_bytes(b"DWG1" + (2).to_bytes(4, "little") + b"\0" + b"\0" * 8)
    with pytest.raises(dw.DynwalkError, match="unsupported binary graph version 2"):
        dw.DeviceGraph.load_dwg1(str(v2))
    empty = tmp_path / "empty.dwg1"
    empty.write_bytes(b"DWG1" + (1).to_bytes(4, "little") + b"\0" + (0).to_bytes(8, "little"))
    with pytest.raises(dw.DynwalkError, match="corrupt binary graph file"):
        dw.DeviceGraph.load_dwg1(str(empty))
