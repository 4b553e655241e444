"""The C-ABI library builds, loads without a GPU and exports every declared symbol."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2604_02715_b200 import _lib
from paper_2604_02715_b200.build import OUT, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "xpgb.h")


@pytest.fixture(scope="module")
def libpath():
    return build()


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|uint64_t|const char\*)\s+(xpgb_\w+)\s*\(", text, flags=re.M)))


def test_header_and_binding_agree():
    assert set(header_functions()) == set(_lib.DECLARED)


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (xpgb_\w+)", out))
    missing = set(header_functions()) - exported
    assert not missing, missing


def test_library_loads_without_gpu(libpath):
    handle = ctypes.CDLL(libpath)
    assert handle.xpgb_abi_version() == 1
    for name in header_functions():
        assert hasattr(handle, name)


def test_binding_loads(libpath):
    lib = _lib.lib()
    assert lib.xpgb_abi_version() == 1


def test_sass_has_tcgen05_and_tma(libpath):
    sass = subprocess.run(["cuobjdump", "-sass", libpath], capture_output=True, text=True, check=True).stdout
    assert "UTCHMMA" in sass  # tcgen05.mma
    assert "UTMALDG" in sass  # TMA tensor loads
    assert "LDTM" in sass  # tcgen05.ld (TMEM -> registers)
    assert re.search(r"\bHMMA\b", sass) is None  # no legacy mma.sync path
