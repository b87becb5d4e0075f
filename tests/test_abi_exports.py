"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
entry point include/snn.h declares (no compute calls here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2107_04092_b200 import build_ext
    return build_ext.build()


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "snn.h")).read()
    return sorted(set(re.findall(r"^\s*(?:snn_status|void|const char \*|uint32_t)\s*\*?\s*(snn_\w+)\s*\(", hdr, re.M)))


def test_header_declares_the_five_entry_points():
    syms = declared_symbols()
    for s in ["snn_create", "snn_add_population", "snn_connect", "snn_step", "snn_read_state",
              "snn_destroy", "snn_last_error", "snn_abi_version"]:
        assert s in syms


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.check_output(["nm", "-D", "--defined-only", libpath], text=True)
    exported = set(l.split()[-1] for l in out.splitlines() if l.strip())
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing


def test_library_loads_and_reports_abi_without_gpu(libpath):
    lib = ctypes.CDLL(libpath)
    lib.snn_abi_version.restype = ctypes.c_uint32
    import paper_2107_04092_b200 as P
    assert lib.snn_abi_version() == P.SNN_ABI_VERSION == 4
    assert P.snn_abi_version() == 4
    for s in P.EXPORTS:
        assert hasattr(P, s)


def test_binding_struct_sizes_match_header(libpath):
    """ctypes mirrors of snn_config / snn_pop_params / snn_syn_params have the C
    sizes (checked by compiling a tiny probe against include/snn.h)."""
    import tempfile
    import paper_2107_04092_b200 as P
    src = ('#include "snn.h"\n#include <stdio.h>\nint main(){printf("%zu %zu %zu\\n", sizeof(snn_config),'
           ' sizeof(snn_pop_params), sizeof(snn_syn_params));return 0;}\n')
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "p.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "p")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
        sizes = [int(x) for x in subprocess.check_output([exe], text=True).split()]
    assert sizes == [ctypes.sizeof(P.snn_config), ctypes.sizeof(P.snn_pop_params), ctypes.sizeof(P.snn_syn_params)]


def test_kernels_compiled_for_sm100a(libpath):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath], text=True)
    assert "sm_100a" in out


def test_product_path_has_no_oracle_dependency():
    """The product package never imports / links the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2107_04092_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle|#include.*oracle|snn_oracle|liboracle",
                                     txt, re.M), f
