"""C-ABI boundary checks that need no GPU: the library loads and exports
every entry point include/xstrace_b200.h declares, with no extras missing."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2102_04285_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "xstrace_b200.h")


def header_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(xs_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_expected_entry_points():
    syms = header_symbols()
    for s in ("xs_overlap", "xs_correct", "xs_analyze", "xs_transition_sites", "xs_validate", "xs_remap"):
        assert s in syms


def test_library_exports_every_header_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_lib.LIB_PATH, mode=os.RTLD_NOW)  # resolve every symbol now
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (xs_[a-z0-9_]+)$", out, flags=re.M))
    assert set(header_symbols()) <= exported
    # python binding covers the whole ABI
    assert set(_lib.SIGNATURES) == set(header_symbols())


def test_status_strings_without_gpu():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    lib = _lib.load()
    assert lib.xs_status_str(1) == b"invalid trace"
    assert lib.xs_status_str(2) == b"uncalibrated hook"
    assert lib.xs_version() == 1


def test_sm100a_cubin_present():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
