"""Full-output parity at the benchmarked configurations (BASELINE.json configs).

Every output row of the decode the bench times is compared with the oracle:
the reference algorithm in Float64 on the same dtype-rounded inputs
(oracle/full.py runs it per (batch, kv-head) row so host memory stays
near 2 GB), max|gpu - ref| <= tol * max|ref| with tol = 1e-3 for bf16 inputs
and 1e-5 for fp32 (BASELINE.json north_star). The reference's own grids
check every head (test_decode.cpp:44-58, acceptance_main.cpp:154-187); so do
these, at the sizes bench.py measures:

* cfg3: Llama-3-8B attention, 32 q / 8 kv heads, d 128, 1,048,576 tokens --
  the default N=1 path (calibrated static partition), through the device and
  the host-buffer (e2e) calls, and the opt-in dynamic pool with cross-row
  stealing;
* cfg4: batch 16, 64 q / 8 kv heads, 131,072 tokens per sequence (1024 rows);
* cfg2: 32-head MHA, 262,144 tokens, one GPU and p = 8 in-process workers;
* one p = 8 shard of cfg3 (131,072 tokens), the per-GPU work of the north star.
"""
import math

import numpy as np
import pytest

from oracle.full import full_decode, rel_err_rows
from oracle.oracle import BF16, F32

pytestmark = pytest.mark.gpu

TOL = {BF16: 1e-3, F32: 1e-5}


@pytest.fixture(scope="module")
def td(lib):
    import paper_2408_04093_b200 as td
    return td


def _seeded_case(td, oracle, dt, b, n_q, n_kv, n, d):
    """The bench's inputs (bench.cpp:73-79 seeding): cache generated on the device
    by the bit-exact generator, q on the device, q's values on the host."""
    seed = oracle.mix64(0, n)
    w = td.Worker(0)
    w.generate_kv(td.DType(dt), b, n_kv, n, d, oracle.mix64(seed, 2), oracle.mix64(seed, 3))
    q = td.seeded_tensor([b, n_q, d], oracle.mix64(seed, 1), 1.0, td.DType(dt))
    qh = oracle.seeded(oracle.mix64(seed, 1), b * n_q * d, dt).reshape(b, n_q, d)
    assert np.array_equal(q.double().cpu().numpy(), qh)
    return w, q, qh, oracle.mix64(seed, 2), oracle.mix64(seed, 3)


def _host(t):
    return t.detach().double().cpu().numpy()


@pytest.mark.parametrize("scale", [1.0, 1 / math.sqrt(128)])
def test_cfg3_1m_every_row(td, oracle, scale):
    import torch
    b, n_q, n_kv, n, d = 1, 32, 8, 1 << 20, 128
    w, q, qh, sk, sv = _seeded_case(td, oracle, BF16, b, n_q, n_kv, n, d)
    outs = [w.tree_decode(q, scale) for _ in range(3)]  # the first call calibrates the partition
    qhost = q.cpu()
    outs.append(w.tree_decode(qhost, scale))                           # host buffers (the e2e call)
    outs.append(w.tree_decode(q, scale, flags=td._capi.TD_DYNAMIC))  # dynamic pool + cross-row stealing
    gain, state = w.calibration_info()
    w.close()
    torch.cuda.synchronize()
    want = full_decode(oracle, qh, n_kv, n, sk, sv, BF16, scale)
    assert len(want) == b * n_q
    errs = [rel_err_rows(_host(o), want) for o in outs]
    print({"scale": scale, "errs": errs, "calibration": (gain, state)})
    assert max(errs) <= TOL[BF16], errs


def test_cfg3_p8_shard_every_row(td, oracle):
    """One rank's share of the north star (131,072 tokens): stealing off, pool on."""
    b, n_q, n_kv, n, d = 1, 32, 8, 1 << 17, 128
    w, q, qh, sk, sv = _seeded_case(td, oracle, BF16, b, n_q, n_kv, n, d)
    outs = [w.tree_decode(q) for _ in range(3)]
    w.close()
    want = full_decode(oracle, qh, n_kv, n, sk, sv, BF16)
    errs = [rel_err_rows(_host(o), want) for o in outs]
    assert max(errs) <= TOL[BF16], errs


def test_cfg4_batch16_every_row(td, oracle):
    b, n_q, n_kv, n, d = 16, 64, 8, 131072, 128
    w, q, qh, sk, sv = _seeded_case(td, oracle, BF16, b, n_q, n_kv, n, d)
    outs = [w.tree_decode(q), w.tree_decode(q, flags=td._capi.TD_DYNAMIC)]
    w.close()
    want = full_decode(oracle, qh, n_kv, n, sk, sv, BF16)
    assert len(want) == b * n_q == 1024
    errs = [rel_err_rows(_host(o), want) for o in outs]
    assert max(errs) <= TOL[BF16], errs


def test_cfg2_mha_256k_every_row(td, oracle):
    """32-head MHA at 256K: one worker, then the in-process p = 8 workers of the
    reference API (tree and ring) over the same cache."""
    import torch
    b, n_q, n_kv, n, d = 1, 32, 32, 262144, 128
    w, q, qh, sk, sv = _seeded_case(td, oracle, BF16, b, n_q, n_kv, n, d)
    one = w.tree_decode(q)
    w.close()
    want = full_decode(oracle, qh, n_kv, n, sk, sv, BF16)
    assert rel_err_rows(_host(one), want) <= TOL[BF16]
    k = td.seeded_tensor([b, n_kv, n, d], sk, 1.0, td.DType.Bf16)
    v = td.seeded_tensor([b, n_kv, n, d], sv, 1.0, td.DType.Bf16)
    cache = td.shard_kv(k, v, 8)
    del k, v
    topo = td.topology_for_workers(8)
    tree = td.tree_decode(q, cache, topo).output
    ring = td.ring_decode(q, cache, topo).output
    torch.cuda.synchronize()
    assert rel_err_rows(_host(tree), want) <= TOL[BF16]
    assert rel_err_rows(_host(ring), want) <= TOL[BF16]


def test_cfg1_f32_64k(td, oracle):
    b, n_q, n_kv, n, d = 1, 1, 1, 65536, 128
    w, q, qh, sk, sv = _seeded_case(td, oracle, F32, b, n_q, n_kv, n, d)
    outs = [w.tree_decode(q), w.tree_decode(q.cpu())]
    w.close()
    want = full_decode(oracle, qh, n_kv, n, sk, sv, F32)
    errs = [rel_err_rows(_host(o), want) for o in outs]
    assert max(errs) <= TOL[F32], errs
