"""CPU-side checks of the C ABI boundary: the library loads and exports every
function include/lorpc.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "lorpc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lorpc_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1908_07071_b200 import build
    path = build.build()
    lib = ctypes.CDLL(path)
    names = declared_functions()
    assert len(names) >= 17
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_names_match_header():
    from paper_1908_07071_b200 import lorpc
    assert sorted(lorpc.SYMBOLS) == declared_functions()


def test_no_oracle_import_in_product():
    pkg = os.path.join(ROOT, "paper_1908_07071_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in txt.replace("no CPU fallback", ""), f
