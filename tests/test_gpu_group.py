"""Single-process worker group (td_group_*): the reference's p in-process
workers (decode.hpp:70-72, decode.cpp:37-41) as p contexts, several of them
sharing one GPU when the box has fewer GPUs than workers. Every worker runs K1
and the one-shot exchange combine K2x (allreduce(max) + rescale +
allreduce(sum) + divide of decode.cpp:129-173 in one NVLink / HBM exchange),
so a one-GPU box exercises the multi-rank combine end to end. Every output
row is compared with the oracle (reference decode in Float64 on the same
inputs)."""
import math
import time

import numpy as np
import pytest

from oracle.full import full_decode, rel_err_rows
from oracle.oracle import BF16, F32

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def td(lib):
    import paper_2408_04093_b200 as td
    return td


def _group_case(td, oracle, p, dt, b, n_q, n_kv, n, d, devices=None):
    seed = oracle.mix64(0, n)
    g = td.WorkerGroup(p, devices or [0])
    for w in g.workers:
        w.generate_kv(td.DType(dt), b, n_kv, n, d, oracle.mix64(seed, 2), oracle.mix64(seed, 3))
    g.enable_p2p(b * n_q, d)
    q = td.seeded_tensor([b, n_q, d], oracle.mix64(seed, 1), 1.0, td.DType(dt), device=f"cuda:{g.devices[0]}")
    qh = oracle.seeded(oracle.mix64(seed, 1), b * n_q * d, dt).reshape(b, n_q, d)
    return g, q, qh, oracle.mix64(seed, 2), oracle.mix64(seed, 3)


@pytest.mark.parametrize("p", [2, 4, 8])
def test_virtual_ranks_one_gpu_every_row(td, oracle, p):
    """p workers on GPU 0: the K2x exchange between contexts sharing the HBM."""
    import torch
    b, n_q, n_kv, n, d = 1, 32, 8, 262144 + 5, 128
    g, q, qh, sk, sv = _group_case(td, oracle, p, BF16, b, n_q, n_kv, n, d)
    starts = [w.kv_info()[0] for w in g.workers]
    lens = [w.kv_info()[1] for w in g.workers]
    assert starts == [sum(td.chunk_extents(n, p)[:i]) for i in range(p)] and lens == td.chunk_extents(n, p)
    outs = [g.tree_decode(q).clone() for _ in range(3)]
    outs.append(g.tree_decode(q.cpu()))  # host buffers
    # a decode loop without host synchronisation: epochs advance on every worker
    loop = torch.empty(12, b, n_q, d, dtype=torch.float32, device="cuda:0")
    for s in range(12):
        g.tree_decode_async(q.data_ptr(), n_q, loop[s].data_ptr())
    for w in g.workers:
        w._sync_worker()
        assert w.p2p_status() == 0
    outs += [loop[0], loop[11]]
    g.close()
    want = full_decode(oracle, qh, n_kv, n, sk, sv, BF16)
    errs = [rel_err_rows(o.double().cpu().numpy(), want) for o in outs]
    assert max(errs) <= 1e-3, errs


def test_virtual_ranks_f32_and_scale(td, oracle):
    b, n_q, n_kv, n, d = 1, 2, 2, 65536 + 3, 128
    g, q, qh, sk, sv = _group_case(td, oracle, 3, F32, b, n_q, n_kv, n, d)
    scale = 1 / math.sqrt(d)
    out = g.tree_decode(q, scale)
    g.close()
    want = full_decode(oracle, qh, n_kv, n, sk, sv, F32, scale)
    assert rel_err_rows(out.double().cpu().numpy(), want) <= 1e-5


def test_exchange_timeout_is_an_error(td, oracle):
    """A worker whose peer never delivers fails the call (TD_ECUDA) instead of
    returning stale words; re-opening the exchange resumes exact decoding."""
    b, n_q, n_kv, n, d = 1, 8, 2, 4096, 128
    g, q, qh, sk, sv = _group_case(td, oracle, 2, BF16, b, n_q, n_kv, n, d)
    w0 = g.workers[0]
    t0 = time.time()
    with pytest.raises(td.TreeDecError) as e:  # worker 1 never launches: worker 0's K2x times out
        w0.tree_decode(q.cpu(), flags=td._capi.TD_P2P)
    assert "timed out" in str(e.value) and time.time() - t0 < 60
    with pytest.raises(td.TreeDecError):  # the exchange stays closed until re-opened
        w0.tree_decode(q, flags=td._capi.TD_P2P)
    g.enable_p2p(b * n_q, d)
    out = g.tree_decode(q)
    g.close()
    want = full_decode(oracle, qh, n_kv, n, sk, sv, BF16)
    assert rel_err_rows(out.double().cpu().numpy(), want) <= 1e-3


def test_group_validation(td, oracle):
    with pytest.raises(td.InvalidArgument):
        td.WorkerGroup(0, [0])
    with pytest.raises(td.InvalidArgument):
        td.WorkerGroup(2, [99])
    g = td.WorkerGroup(2, [0])
    q = td.seeded_tensor([1, 8, 128], 1, 1.0, td.DType.Bf16)
    with pytest.raises(td.TreeDecError):  # no shard placed
        g.tree_decode(q)
    seed = oracle.mix64(0, 1000)
    g.workers[0].generate_kv(td.DType.Bf16, 1, 2, 1000, 128, seed, seed + 1)
    g.workers[1].generate_kv(td.DType.Bf16, 1, 2, 1001, 128, seed, seed + 1)  # another cache
    g.enable_p2p(8, 128)
    with pytest.raises(td.InvalidArgument):
        g.tree_decode(q)
    g.close()


def test_group_over_every_gpu(td, oracle):
    """Workers spread over all visible GPUs (two workers per GPU when p = 2 x
    GPUs): peers across NVLink and in the same HBM in one exchange."""
    import torch
    ng = torch.cuda.device_count()
    if ng < 2:
        pytest.skip("needs 2 GPUs")
    b, n_q, n_kv, n, d = 2, 32, 8, 131072 + 7, 128
    for p in (ng, 2 * ng):
        g, q, qh, sk, sv = _group_case(td, oracle, p, BF16, b, n_q, n_kv, n, d, devices=list(range(ng)))
        assert sorted({w.device for w in g.workers}) == list(range(ng))
        a = g.tree_decode(q)
        h = g.tree_decode(q.cpu())
        g.close()
        want = full_decode(oracle, qh, n_kv, n, sk, sv, BF16)
        assert rel_err_rows(a.double().cpu().numpy(), want) <= 1e-3
        assert rel_err_rows(h.double().numpy(), want) <= 1e-3


def test_group_host_buffers_large_output(td, oracle):
    """A host-buffer call whose output exceeds what the exchange stores in place
    (b * n_q * d * 4 > 64 KB): the exchange writes a device buffer, the call copies
    it once (td_capi.cu xchg_in_place). Pinned and pageable outputs, every row."""
    import torch
    b, n_q, n_kv, n, d = 8, 32, 8, 4096 + 3, 128
    g, q, qh, sk, sv = _group_case(td, oracle, 2, BF16, b, n_q, n_kv, n, d)
    dev_out = g.tree_decode(q).double().cpu().numpy()
    pinned = g.tree_decode(q.cpu()).double().numpy()  # the default host output is pinned
    pageable = torch.empty(b, n_q, d, dtype=torch.float32)
    g.tree_decode(q.cpu(), out=pageable)
    g.close()
    want = full_decode(oracle, qh, n_kv, n, sk, sv, BF16)
    for got in (dev_out, pinned, pageable.double().numpy()):
        assert rel_err_rows(got, want) <= 1e-3
