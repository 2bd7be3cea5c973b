"""The C-ABI library loads without a GPU and exports every symbol that
include/treedec_b200.h declares (no compute calls here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "treedec_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(td_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_api():
    names = declared()
    for must in ("td_tree_decode", "td_ring_decode", "td_decode_partial", "td_combine_partials",
                 "td_kv_place", "td_comm_init", "td_seeded_fill"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2408_04093_b200._capi import EXPORTS, LIB_PATH
    names = declared()
    assert sorted(EXPORTS) == names
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (td_[a-z0-9_]+)", out))
    assert set(names) <= exported


def test_library_is_sm100a(lib):
    from paper_2408_04093_b200._capi import LIB_PATH
    out = subprocess.run(["cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_error_string(lib):
    assert lib.td_version() >= 1
    assert isinstance(lib.td_last_error(), bytes)


def test_header_compiles_as_c(tmp_path):
    c = tmp_path / "t.c"
    c.write_text('#include "treedec_b200.h"\nint main(void){return td_version() > 0 ? 0 : 1;}\n')
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-c", str(c),
                        "-o", str(tmp_path / "t.o")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_no_cpu_fallback_in_product():
    """The product package never imports the oracle."""
    pkg = os.path.join(ROOT, "paper_2408_04093_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in src.replace("oracle/_ref", ""), f


def test_header_flags_match_python(tmp_path):
    """Every TD_* flag / status / dtype value of the header, compiled by a C
    compiler, equals the constant the Python mirror passes."""
    from paper_2408_04093_b200 import _capi
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    names = sorted(set(re.findall(r"\b(TD_[A-Z0-9_]+)\s*=", src)))
    assert "TD_NCCL_DEVICE" in names and "TD_P2P" in names
    c = tmp_path / "f.c"
    c.write_text('#include <stdio.h>\n#include "treedec_b200.h"\nint main(void){\n' +
                 "".join(f'printf("{n} %d\\n", (int){n});\n' for n in names) + "return 0;}\n")
    exe = tmp_path / "f"
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), str(c), "-o",
                        str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split("\n")
               if line)
    for n, v in got.items():
        if hasattr(_capi, n):
            assert getattr(_capi, n) == int(v), n
    for flag in ("TD_HOST_IO", "TD_P2P", "TD_PINNED_IO", "TD_DYNAMIC", "TD_GRAPH", "TD_NCCL_DEVICE"):
        assert hasattr(_capi, flag) and int(got[flag]) == getattr(_capi, flag), flag
