"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/ckmpm_b200.h declares, and the ctypes mirrors match the C
struct layouts (compiled here with gcc against the header)."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

from paper_2412_10399_b200 import abi
from paper_2412_10399_b200._lib import EXPORTED, LIB_PATH, lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ckmpm_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(ckg_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB_PATH), "libckmpm_b200.so not built"
    l = lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(l, s), s
    assert set(syms) == set(EXPORTED)
    assert l.ckg_abi_version() == abi.ABI_VERSION


def test_struct_layouts_match_header():
    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "ckmpm_b200.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu\n", sizeof(ckg_config), sizeof(ckg_material), sizeof(ckg_boundary),
         sizeof(ckg_step_out), sizeof(ckg_diagnostics), sizeof(ckg_particle_f64), sizeof(ckg_particle_f32));
  printf("%zu %zu %zu\n", offsetof(ckg_config, materials), offsetof(ckg_config, boundaries),
         offsetof(ckg_step_out, status));
  printf("%zu %zu %zu\n", sizeof(ckg_frame_in), sizeof(ckg_frame_out), offsetof(ckg_frame_out, status));
  return 0;
}
'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "t")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    got = list(map(int, out))
    want = [C.sizeof(abi.Config), C.sizeof(abi.Material), C.sizeof(abi.Boundary), C.sizeof(abi.StepOut),
            C.sizeof(abi.Diagnostics), abi.particle_dtype(8).itemsize, abi.particle_dtype(4).itemsize,
            abi.Config.materials.offset, abi.Config.boundaries.offset, abi.StepOut.status.offset,
            C.sizeof(abi.FrameIn), C.sizeof(abi.FrameOut), abi.FrameOut.status.offset]
    assert got == want


def test_create_rejects_bad_config_without_gpu():
    c = abi.Config()
    c.abi_version = 999
    ctx = C.c_void_p()
    assert lib().ckg_create(C.byref(c), C.byref(ctx)) == abi.ERR_CONFIG
    assert not ctx.value


def test_no_cpu_fallback_in_product():
    """The product package never imports the oracle/checker code."""
    pkg = os.path.join(ROOT, "paper_2412_10399_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".hpp")):
                t = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", t).replace("oracle/", ""), f
