"""The C-ABI library loads and exports every symbol include/hm.h declares
(CPU-only: no compute calls)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "hm.h")
LIB = os.path.join(ROOT, "paper_1703_09085_b200", "lib", "libhm.so")


def declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hm_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib_path():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_1703_09085_b200"), "-j8"], check=True,
                       capture_output=True)
    return LIB


def test_header_declares_boundary():
    names = declared()
    for n in ("hm_build", "hm_addmul", "hm_lr", "hm_chol", "hm_matvec_thin", "hm_import", "hm_export"):
        assert n in names


def test_library_exports_every_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], check=True, capture_output=True,
                         text=True).stdout
    syms = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [n for n in declared() if n not in syms]
    assert not missing, missing


def test_ctypes_load_and_version(lib_path):
    from paper_1703_09085_b200 import _lib
    lib = _lib.load(lib_path)
    assert b"sm_100a" in lib.hm_version()
    for n in _lib.EXPORTS:
        assert hasattr(lib, n)


def test_sass_is_sm100a(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
