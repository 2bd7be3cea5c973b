import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libtreedec_b200.so)")
    config.addinivalue_line("markers", "slow: full-size parity cases")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle, build
    build(ref=False)
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    """The reference library built by path (oracle/_ref); skipped where absent."""
    from oracle.oracle import REF_SO, REF_SRC, Reference, build
    if not os.path.exists(REF_SO):
        if not os.path.isdir(REF_SRC):
            pytest.skip("oracle/_ref not built and /root/reference absent")
        build(ref=True)
    return Reference()


@pytest.fixture(scope="session")
def lib():
    """The product library; built in-tree if stale (nvcc works without a GPU)."""
    from paper_2408_04093_b200 import build as b
    b.build()
    from paper_2408_04093_b200 import _capi
    return _capi.lib()


def make_inputs(oracle, seed, b, n_q, n_kv, n, d, dtype):
    """The reference seeding convention (bench.cpp:73-79 / test_decode.cpp:18-23):
    q, k, v from seeds mix64(seed, 1..3), rounded to dtype."""
    q = oracle.seeded(oracle.mix64(seed, 1), b * n_q * d, dtype).reshape(b, n_q, d)
    k = oracle.seeded(oracle.mix64(seed, 2), b * n_kv * n * d, dtype).reshape(b, n_kv, n, d)
    v = oracle.seeded(oracle.mix64(seed, 3), b * n_kv * n * d, dtype).reshape(b, n_kv, n, d)
    return q, k, v


def rel_err(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300))
