"""The C-ABI from plain C (tests/cpp/capi_c_demo.c): one rank, and two ranks
bootstrapped with fork + pipes (NCCL path and one-shot NVLink exchange), each
checked against a one-rank decode. No Python or torch in the decoding process."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    exe = str(tmp_path / "capi_c_demo")
    lib = os.path.join(ROOT, "paper_2408_04093_b200")
    cmd = ["gcc", "-std=c11", "-O2", os.path.join(ROOT, "tests", "cpp", "capi_c_demo.c"),
           "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include", "-L" + lib, "-ltreedec_b200",
           "-L/usr/local/cuda/lib64", "-lcudart", "-lm", "-Wl,-rpath," + lib, "-Wl,-rpath,/usr/local/cuda/lib64",
           "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def _gpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("ranks", [1, 2])
def test_c_program(lib, tmp_path, ranks):
    if _gpus() < ranks:
        pytest.skip(f"needs {ranks} GPUs")
    exe = _build(tmp_path)
    r = subprocess.run([exe, str(ranks)], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr[-2000:])
    assert r.returncode == 0 and r.stdout.strip().endswith("ok")
