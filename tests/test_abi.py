"""CPU checks of the boundary: the C-ABI library loads, exports every symbol
include/mds.h declares, and the product path is independent of the oracle."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mds.h")
PKG = os.path.join(ROOT, "paper_2605_13736_b200")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mds_[a-z0-9_]+|ipm_[a-z0-9_]+)\s*\(", src)))


def lib_path():
    from paper_2605_13736_b200 import build
    return build.build()


def test_header_declares_the_four_calls():
    fns = declared_functions()
    for f in ("mds_condense", "mds_factor", "mds_solve", "ipm_step_vectors"):
        assert f in fns


def test_library_loads_and_exports_every_declared_symbol():
    lib = ctypes.CDLL(lib_path())
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing
    lib.mds_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.mds_version()


def test_binding_names_match_header():
    import paper_2605_13736_b200 as mds
    assert sorted(mds.EXPORTS) == declared_functions()


def test_sass_is_sm100a_with_dmma():
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump missing")
    out = subprocess.run(["cuobjdump", "-sass", lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "DMMA" in out          # FP64 tensor-core trailing update


def test_product_path_never_touches_the_oracle():
    # the product package may mention the oracle in comments, but never import, link or include it
    bad = ("import oracle", "from oracle", "liboracle", "oracle.c", '#include "../../oracle', "mdsgen")
    for dirpath, _, files in os.walk(PKG):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, fn)).read()
                for b in bad:
                    assert b not in src, (fn, b)


def test_plan_rejects_bad_pattern_without_gpu():
    # plan validation happens on the host before any device call
    import numpy as np
    lib = ctypes.CDLL(lib_path())
    rowptr = np.array([0, 2], dtype=np.int32)
    colidx = np.array([1, 0], dtype=np.int32)   # unsorted
    h = ctypes.c_void_p()
    lib.mds_plan_create.argtypes = [ctypes.c_int64] * 4 + [ctypes.c_void_p] * 2 + [ctypes.POINTER(ctypes.c_void_p)]
    code = lib.mds_plan_create(1, 0, 2, 0, rowptr.ctypes.data, colidx.ctypes.data, ctypes.byref(h))
    assert code == -2
