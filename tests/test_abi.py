"""The C-ABI library (CPU-side checks; no compute without a GPU).

* libzxs_b200.so loads and exports every function include/zxs_b200.h declares.
* The ctypes mirrors of zxs_model_desc / zxs_sampler_info have the header's
  layout (offsets measured by compiling a probe against the header).
* Without a GPU, create fails loudly (there is no CPU fallback).
* The product package never imports the oracle.
"""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT, golden_path, has_cuda
from paper_2604_01059_b200 import _native, zxs_format

HEADER = os.path.join(ROOT, "include", "zxs_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w ]+?\*?\s*\b(zxs_\w+)\s*\(", text, re.M)))


def test_header_declares_api():
    fns = declared_functions()
    for must in ("zxs_sampler_create", "zxs_sample", "zxs_sample_device", "zxs_count", "zxs_eval_batch",
                 "zxs_sample_error_batch", "zxs_probability_of_at", "zxs_last_error"):
        assert must in fns


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(_native.LIB_PATH)
    missing = [f for f in declared_functions() if not hasattr(L, f)]
    assert not missing, missing
    assert {name for name, _, _ in _native.SIGNATURES} == set(declared_functions())


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _probe_offsets(struct_name, fields):
    src = "#include <stddef.h>\n#include <stdio.h>\n#include \"zxs_b200.h\"\nint main(){\n"
    src += f'printf("%zu\\n", sizeof({struct_name}));\n'
    for f in fields:
        src += f'printf("%zu\\n", offsetof({struct_name}, {f}));\n'
    src += "return 0;}\n"
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "p.c")
        exe = os.path.join(d, "p")
        open(c, "w").write(src)
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        vals = [int(x) for x in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    return vals[0], vals[1:]


@pytest.mark.parametrize("cls,cname", [(zxs_format.ModelDesc, "zxs_model_desc"),
                                       (_native.SamplerInfo, "zxs_sampler_info"),
                                       (_native.SampleOptions, "zxs_sample_options")])
def test_ctypes_layout_matches_header(cls, cname):
    names = [n for n, _ in cls._fields_]
    size, offs = _probe_offsets(cname, names)
    assert ctypes.sizeof(cls) == size
    assert [getattr(cls, n).offset for n in names] == offs


@pytest.mark.skipif(has_cuda(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback():
    from paper_2604_01059_b200 import CompiledSampler
    with pytest.raises(RuntimeError, match="no CUDA device"):
        CompiledSampler.load(golden_path("c2_surface_d3_xmem_t"))


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2604_01059_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*|\"\"\"[\s\S]*?\"\"\"", "", text), f
