"""The C-ABI library builds for sm_100a, loads without a GPU, and exports
every entry point include/moep_b200.h declares (no compute calls here)."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "moep_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = set(re.findall(r"\b(?:int|int64_t|const char\*)\s+(moep_\w+)\s*\(", text))
    return sorted(names)


@pytest.fixture(scope="module")
def libpath():
    from paper_2511_10676_b200 import build
    return build.build()


def test_header_declares_entry_points():
    names = declared_symbols()
    for must in ("moep_predict_bf16", "moep_predict_fp64", "moep_eval_logits", "moep_counters_reduce",
                 "moep_input_norm", "moep_topk_logits", "moep_rank_order"):
        assert must in names


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    for name in declared_symbols():
        assert re.search(rf"\bT {name}\b", out), name


def test_version_string(libpath):
    lib = ctypes.CDLL(libpath)
    lib.moep_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.moep_version()


def test_cubin_is_sm100a_with_tcgen05(libpath):
    out = subprocess.run(["cuobjdump", "-sass", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", libpath], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out  # tcgen05.mma
    assert "UTMALDG" in out  # TMA tensor loads
    assert "LDTM" in out     # tcgen05.ld


def test_struct_layouts_match_header(libpath):
    # ctypes mirrors of the arg structs must have the C sizes (checked via a tiny C probe)
    from paper_2511_10676_b200 import _lib
    src = f'''#include "{HEADER}"
#include <stdio.h>
#include <stddef.h>
int main(){{printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(moep_predict_args), offsetof(moep_predict_args, partials),
 sizeof(moep_fp64_args), offsetof(moep_fp64_args, partials), offsetof(moep_predict_args, status),
 offsetof(moep_predict_args, kernel));return 0;}}'''
    tmp = "/tmp/moep_layout_probe"
    with open(tmp + ".c", "w") as f:
        f.write(src)
    subprocess.run(["gcc", "-o", tmp, tmp + ".c"], check=True)
    got = [int(v) for v in subprocess.run([tmp], capture_output=True, text=True).stdout.split()]
    assert got == [ctypes.sizeof(_lib.PredictArgs), _lib.PredictArgs.partials.offset,
                   ctypes.sizeof(_lib.Fp64Args), _lib.Fp64Args.partials.offset,
                   _lib.PredictArgs.status.offset, _lib.PredictArgs.kernel.offset]


def test_loss_and_optim_struct_layouts(libpath):
    from paper_2511_10676_b200 import _lib
    src = f'''#include "{HEADER}"
#include <stdio.h>
#include <stddef.h>
int main(){{printf("%zu %zu %zu %zu\\n", sizeof(moep_loss_args), offsetof(moep_loss_args, n_blocks),
 sizeof(moep_optim_args), offsetof(moep_optim_args, nonfinite));return 0;}}'''
    tmp = "/tmp/moep_layout_probe2"
    with open(tmp + ".c", "w") as f:
        f.write(src)
    subprocess.run(["gcc", "-o", tmp, tmp + ".c"], check=True)
    got = [int(v) for v in subprocess.run([tmp], capture_output=True, text=True).stdout.split()]
    assert got == [ctypes.sizeof(_lib.LossArgs), _lib.LossArgs.n_blocks.offset,
                   ctypes.sizeof(_lib.OptimArgs), _lib.OptimArgs.nonfinite.offset]


def test_python_binding_covers_header():
    from paper_2511_10676_b200 import _lib
    assert set(declared_symbols()) == set(_lib.EXPORTED)
