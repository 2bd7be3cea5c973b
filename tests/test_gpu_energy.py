"""GPU parity of the energy formulation (
energy_forward_parallel / energy_grad_parallel, energy.cpp:152-259) against
the CPU oracle (the reference algorithm in Float64 on the same dtype-rounded
inputs; the oracle equals the reference bitwise, tests/test_oracle.py).
Stats (value, row_max, shifted_lse) are compared as max|gpu - ref| <= tol *
max(1, max|ref|); the gradient as max|gpu - ref| <= tol * max|ref|; tol 1e-3
for bf16 inputs, 1e-5 for fp32 inputs."""
import numpy as np
import pytest

from conftest import rel_err
from oracle.oracle import BF16, F32, F64, HIER

pytestmark = pytest.mark.gpu

TOL = {BF16: 1e-3, F32: 1e-5}


@pytest.fixture(scope="module")
def td(lib):
    import paper_2408_04093_b200 as td
    return td


def dev(x, dtype):
    import torch
    tdt = {BF16: torch.bfloat16, F32: torch.float32}[dtype]
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda").to(tdt)


def host(t):
    return t.detach().double().cpu().numpy()


def inputs(oracle, seed, b, h, nq, n, d, dt):
    q = oracle.seeded(oracle.mix64(seed, 1), b * h * nq * d, dt).reshape(b, h, nq, d)
    k = oracle.seeded(oracle.mix64(seed, 2), b * h * n * d, dt).reshape(b, h, n, d)
    v = oracle.seeded(oracle.mix64(seed, 3), b * h * n * d, dt).reshape(b, h, n, d)
    src = oracle.seeded(oracle.mix64(seed, 4), b * h * nq * d, dt, scale=0.5).reshape(b, h, nq, d)
    return q, k, v, src


def stat_err(got, want):
    return float(np.max(np.abs(host(got) - want)) / max(1.0, np.max(np.abs(want))))


SHAPES = [(1, 2, 3, 300, 64), (2, 4, 1, 1000, 128), (1, 1, 5, 77, 16), (1, 8, 2, 4096, 128)]


@pytest.mark.parametrize("dt", [BF16, F32])
@pytest.mark.parametrize("shape", SHAPES)
def test_energy_forward_parallel(td, oracle, dt, shape):
    b, h, nq, n, d = shape
    q, k, v, src = inputs(oracle, 41, b, h, nq, n, d, dt)
    for chunks in (1, 3, 8):
        for s_ in (None, src):
            got = td.energy_forward_parallel(dev(q, dt), dev(k, dt), dev(v, dt),
                                             None if s_ is None else dev(s_, dt), chunks)
            want = oracle.energy_forward_parallel(q, k, v, s_, chunks, F64)
            for g, w in zip((got.value, got.row_max, got.shifted_lse), want):
                assert stat_err(g, w) <= TOL[dt], (chunks, s_ is None, stat_err(g, w))


@pytest.mark.parametrize("dt", [BF16, F32])
@pytest.mark.parametrize("shape", SHAPES)
def test_energy_grad_parallel(td, oracle, dt, shape):
    b, h, nq, n, d = shape
    q, k, v, _ = inputs(oracle, 42, b, h, nq, n, d, dt)
    qd, kd, vd = dev(q, dt), dev(k, dt), dev(v, dt)
    saved = td.energy_forward_parallel(qd, kd, vd, None, 4)
    _, rm, sh = oracle.energy_forward_parallel(q, k, v, None, 4, F64)
    for chunks in (1, 5):
        g = td.energy_grad_parallel(qd, kd, vd, saved, chunks)
        want = oracle.energy_grad_parallel(q, k, v, rm, sh, chunks, F64)
        assert rel_err(host(g), want) <= TOL[dt]
    # at zero source the gradient is the attention output (tree_decode, scale 1)
    if nq == 1:
        out = td.tree_decode(qd[:, :, 0], td.shard_kv(kd, vd, 1), td.topology_for_workers(1)).output
        assert rel_err(host(g[:, :, 0]), host(out)) <= 1e-5


def test_energy_properties_on_gpu(td, oracle):
    q, k, v, src = inputs(oracle, 43, 1, 2, 1, 500, 64, F32)
    qd, kd, vd, sd = dev(q, F32), dev(k, F32), dev(v, F32), dev(src, F32)
    e = td.energy(qd, kd, vd, sd)
    assert np.allclose(host(e.value), host(e.row_max) + host(e.shifted_lse), atol=1e-5)
    # a constant shift of every key's score (energy.cpp: log Z moves by the shift)
    import torch
    e2 = td.energy(qd, kd, vd, torch.zeros_like(sd))
    e0 = td.energy(qd, kd, vd, None)
    assert np.allclose(host(e2.value), host(e0.value), atol=1e-6)
    with pytest.raises(td.InvalidArgument):
        td.energy_forward_parallel(qd, kd, vd, None, 0)
    with pytest.raises(td.InvalidArgument):
        td.energy_forward_parallel(qd, kd, vd, None, 501)
    with pytest.raises(td.InvalidArgument):
        td.energy_partial(qd, kd[:, :1], vd, None)


@pytest.mark.parametrize("dt", [BF16, F32])
def test_worker_energy(td, oracle, dt):
    """Alg. 1 / Alg. 2 through a context over a placed shard (p = 1)."""
    b, h, nq, n, d = 1, 4, 2, 3000, 128
    q, k, v, src = inputs(oracle, 44, b, h, nq, n, d, dt)
    w = td.Worker(0)
    w.place_kv(dev(k, dt), dev(v, dt))
    e = w.energy_forward(dev(q, dt), dev(src, dt))
    want = oracle.energy_forward_parallel(q, k, v, src, 1, F64)
    for g, wv in zip((e.value, e.row_max, e.shifted_lse), want):
        assert stat_err(g, wv) <= TOL[dt]
    e0 = w.energy_forward(dev(q, dt))
    g = w.energy_grad(dev(q, dt), e0)
    _, rm, sh = oracle.energy_forward_parallel(q, k, v, None, 1, F64)
    assert rel_err(host(g), oracle.energy_grad_parallel(q, k, v, rm, sh, 1, F64)) <= TOL[dt]
    w.close()
