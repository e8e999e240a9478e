"""CPU checks of the C-ABI library: it loads and exports every symbol include/rtk_b200.h declares."""
import os
import re

from paper_2602_21958_b200 import _native

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "rtk_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rtk_[A-Za-z0-9_]+)\s*\(", text)) - {"rtk_matvec_fn"})


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    names = declared_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_signatures_cover_header():
    assert sorted(n for n, _, _ in _native.SIGNATURES) == declared_functions()


def test_version_and_counter_without_gpu():
    lib = _native.lib()
    assert lib.rtk_version() == 1
    assert lib.rtk_kernel_launch_count() >= 0
