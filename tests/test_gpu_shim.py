"""The C++ drop-in (include/treedec_gpu.hpp) against the reference library
itself, with the reference's own types: tests/cpp/shim_parity.cpp replays the
reference's decode grid through treedec::gpu::tree_decode / ring_decode and
compares with treedec::tree_decode / ring_decode (Float64 on the same values)
within the reference tolerance table, plus the reporting counters."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "shim_parity")


def test_cpp_shim_matches_reference(lib):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/shim_parity not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "0 failures" in r.stdout
