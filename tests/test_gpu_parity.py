"""GPU parity of the B200 decode path against the CPU oracle.

Parity rule: inputs are generated with the
reference generator and rounded to the data dtype; the oracle is the
reference algorithm run in Float64 on those same values; the GPU result is
compared in fp32 with max|gpu - ref| <= tol * max|ref|, tol = 1e-3 for bf16
inputs and 1e-5 for fp32 inputs (BASELINE.json north_star).
"""
import math

import numpy as np
import pytest

from conftest import make_inputs, rel_err
from oracle.full import full_decode, rel_err_rows
from oracle.oracle import BF16, F32, F64, HIER

pytestmark = pytest.mark.gpu

TOL = {BF16: 1e-3, F32: 1e-5}


@pytest.fixture(scope="module")
def td(lib):
    import paper_2408_04093_b200 as td
    return td


def dev(x, dtype):
    import torch
    tdt = {BF16: torch.bfloat16, F32: torch.float32, F64: torch.float64}[dtype]
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda").to(tdt)


def host(t):
    return t.detach().double().cpu().numpy()


# ---------------------------------------------------------------- K6 generator
@pytest.mark.parametrize("dtype", [BF16, F32, F64])
@pytest.mark.parametrize("seed", [0, 1, 2 ** 64 - 1, 0x9E3779B97F4A7C15])
def test_generator_bit_exact(td, oracle, dtype, seed):
    import torch
    shape = [2, 3, 257, 16]
    t = td.seeded_tensor(shape, seed, 1.0, td.DType(dtype))
    want = oracle.seeded(seed, int(np.prod(shape)), dtype).reshape(shape)
    got = t.double().cpu().numpy()
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    # a shard (rows [start, start+len) of every (b, h)) is the slice of the whole
    sh = td.seeded_tensor(shape, seed, 0.5, td.DType(dtype), start=100, length=57)
    whole = oracle.seeded(seed, int(np.prod(shape)), dtype, scale=0.5).reshape(shape)
    assert np.array_equal(sh.double().cpu().numpy(), whole[:, :, 100:157])
    torch.cuda.synchronize()


def test_generator_rejects_bad_scale(td):
    with pytest.raises(td.InvalidArgument):
        td.seeded_tensor([4, 4], 1, 0.0)


# ---------------------------------------------------------------- K1 + K2 partial
PARTIAL_CASES = [
    # dtype, b, n_q, n_kv, t, d, scale
    (BF16, 1, 1, 1, 1, 128, 1.0),
    (BF16, 1, 4, 1, 17, 128, 1.0),
    (BF16, 1, 32, 8, 4096, 128, 1.0),
    (BF16, 2, 8, 8, 1000, 128, 1 / math.sqrt(128)),
    (BF16, 1, 64, 8, 3000, 128, 1.0),
    (BF16, 3, 16, 2, 555, 64, 1.0),
    (BF16, 1, 4, 2, 300, 256, 1.0),
    (BF16, 1, 2, 1, 65536, 128, 1.0),
    (F32, 1, 1, 1, 65536, 128, 1.0),
    (F32, 2, 4, 2, 999, 128, 1.0),
    (F32, 1, 2, 2, 33, 128, 1 / math.sqrt(128)),
    (F32, 1, 2, 2, 40, 8, 1.0),       # generic kernel (reference test shapes)
    (BF16, 1, 2, 2, 96, 8, 1.0),
    (BF16, 1, 3, 1, 50, 4, 0.5),
    (F32, 2, 16, 16, 64, 100, 1.0),   # ragged head dim
    (BF16, 1, 16, 1, 200, 128, 1.0),  # group 16 -> generic
]


@pytest.mark.parametrize("case", PARTIAL_CASES, ids=lambda c: "-".join(map(str, c)))
def test_chunk_partial_matches_oracle(td, oracle, case):
    dtype, b, n_q, n_kv, t, d, scale = case
    q, k, v = make_inputs(oracle, 7 + t, b, n_q, n_kv, t, d, dtype)
    part = td.attention_chunk_partial(dev(q, dtype), dev(k, dtype), dev(v, dtype), scale)
    m, lse, out = oracle.chunk_partial(q, k, v, 0, t, scale, F64, nthreads=8)
    assert rel_err(host(part.out), out) <= TOL[dtype]
    # lse / row_max are fp32 statistics: compare in absolute terms
    assert np.max(np.abs(host(part.lse) - lse)) <= 1e-5 * max(1.0, np.max(np.abs(lse)))
    assert np.max(np.abs(host(part.row_max) - m)) <= 1e-5 * max(1.0, np.max(np.abs(m)))


def test_empty_chunk_is_identity(td, oracle):
    import torch
    q, k, v = make_inputs(oracle, 9, 1, 4, 1, 5, 128, BF16)
    part = td.attention_chunk_partial(dev(q, BF16), dev(k, BF16)[:, :, :0], dev(v, BF16)[:, :, :0])
    assert torch.isneginf(part.lse).all() and torch.isneginf(part.row_max).all()
    assert (part.out == 0).all()


def test_single_key_returns_value_row(td, oracle):
    q, k, v = make_inputs(oracle, 1, 1, 8, 8, 1, 128, BF16)
    part = td.attention_chunk_partial(dev(q, BF16), dev(k, BF16), dev(v, BF16))
    assert np.array_equal(host(part.out), v[:, :, 0, :])


def test_zero_query_averages_values(td, oracle):
    q, k, v = make_inputs(oracle, 2, 1, 4, 4, 1000, 128, F32)
    part = td.attention_chunk_partial(dev(np.zeros_like(q), F32), dev(k, F32), dev(v, F32))
    assert rel_err(host(part.out), v.mean(axis=2)) <= 1e-5


@pytest.mark.parametrize("dtype", [BF16, F32])
def test_large_score_is_stable(td, oracle, dtype):
    """attention.cpp test: a +300 score must not overflow the accumulation."""
    q, k, v = make_inputs(oracle, 55, 1, 1, 1, 600, 128, dtype)
    q[:] = 0.0
    q[0, 0, 0] = 1.0
    k[0, 0, 5, 0] = 300.0
    part = td.attention_chunk_partial(dev(q, dtype), dev(k, dtype), dev(v, dtype))
    _, lse, out = oracle.chunk_partial(q, k, v, 0, 600, 1.0, F64)
    got = host(part.out)
    assert np.isfinite(got).all()
    assert rel_err(got, out) <= TOL[dtype]


def test_partial_rejects_bad_shapes(td, oracle):
    import torch
    q, k, v = make_inputs(oracle, 13, 1, 2, 2, 6, 128, BF16)
    with pytest.raises(td.InvalidArgument):
        td.attention_chunk_partial(dev(q, BF16), dev(k, BF16)[..., :64], dev(v, BF16))
    with pytest.raises(td.InvalidArgument):
        td.attention_chunk_partial(dev(q, BF16), dev(k, BF16), dev(v, F32))
    with pytest.raises(td.InvalidArgument):  # 3 q heads over 2 kv heads
        td.attention_chunk_partial(dev(q, BF16)[:, :1].expand(1, 3, 128).contiguous(), dev(k, BF16), dev(v, BF16))
    torch.cuda.synchronize()


# ---------------------------------------------------------------- combine primitives
def test_combine_partials_partition_invariant(td, oracle):
    """attention.cpp test: {4,4}, {1,7}, {2,2,2,2} partitions combine to the kernel."""
    import torch
    q, k, v = make_inputs(oracle, 10, 1, 2, 2, 8 * 512, 128, BF16)
    ref = oracle.attention_naive(q, k, v)
    qd, kd, vd = dev(q, BF16), dev(k, BF16), dev(v, BF16)
    for sizes in ([4, 4], [1, 7], [2, 2, 2, 2]):
        parts, begin = [], 0
        for s in sizes:
            ext = s * 512
            parts.append(td.attention_chunk_partial(qd, kd[:, :, begin:begin + ext].contiguous(),
                                                    vd[:, :, begin:begin + ext].contiguous()))
            begin += ext
        assert rel_err(host(td.combine_partials(parts)), ref) <= 1e-3
    # pairwise fold, left to right
    fold = parts[0]
    for p_ in parts[1:]:
        fold = td.combine_pair(fold, p_)
    assert rel_err(host(fold.out), ref) <= 1e-3
    # all-empty rows are rejected like the reference (invalid_argument)
    empty = td.SoftmaxPartial(torch.full_like(parts[0].lse, -math.inf), torch.full_like(parts[0].lse, -math.inf),
                              torch.zeros_like(parts[0].out))
    with pytest.raises(td.InvalidArgument):
        td.combine_partials([empty])
    # identity absorbs exactly
    right = td.combine_pair(parts[0], empty)
    assert torch.equal(right.out, parts[0].out) and torch.equal(right.lse, parts[0].lse)


def test_numerator_and_finalize(td, oracle):
    import torch
    q, k, v = make_inputs(oracle, 11, 1, 4, 4, 2000, 128, F32)
    qd, kd, vd = dev(q, F32), dev(k, F32), dev(v, F32)
    parts = [td.attention_chunk_partial(qd, kd[:, :, a:a + 500].contiguous(), vd[:, :, a:a + 500].contiguous())
             for a in range(0, 2000, 500)]
    shift = torch.stack([p_.lse for p_ in parts]).amax(0)
    nds = [td.partial_to_numerator(p_, shift) for p_ in parts]
    num = sum(n for n, _ in nds)
    den = sum(d_ for _, d_ in nds)
    out = td.finalize(num, den)
    assert rel_err(host(out), oracle.attention_naive(q, k, v)) <= 1e-5


# ---------------------------------------------------------------- single-process tree / ring
@pytest.mark.parametrize("dtype", [BF16, F32])
def test_tree_decode_grid(td, oracle, dtype):
    """test_decode.cpp:44-58 / acceptance criterion 3 grid at GPU shapes."""
    for n in (17, 64, 1024, 5000):
        q, k, v = make_inputs(oracle, 2 + n, 1, 8, 2, n, 128, dtype)
        qd, kd, vd = dev(q, dtype), dev(k, dtype), dev(v, dtype)
        for p in (1, 2, 3, 4, 7, 8, 16):
            if p > n:
                continue
            want = oracle.tree_decode(q, k, v, p, HIER, 1.0, F64)
            cache = td.shard_kv(kd, vd, p)
            topo = td.topology_for_workers(p)
            tree = td.tree_decode(qd, cache, topo).output
            ring = td.ring_decode(qd, cache, topo).output
            assert rel_err(host(tree), want) <= TOL[dtype], (n, p)
            assert rel_err(host(ring), want) <= TOL[dtype], (n, p)


def test_tree_decode_validation(td, oracle):
    q, k, v = make_inputs(oracle, 12, 1, 2, 2, 16, 128, BF16)
    qd, kd, vd = dev(q, BF16), dev(k, BF16), dev(v, BF16)
    cache = td.shard_kv(kd, vd, 4)
    with pytest.raises(td.InvalidArgument):
        td.tree_decode(qd, cache, td.topology_for_workers(8))
    with pytest.raises(td.InvalidArgument):
        td.ring_decode(qd, cache, td.topology_for_workers(2))
    with pytest.raises(td.InvalidArgument):
        td.shard_kv(kd, vd, 17)
    with pytest.raises(td.InvalidArgument):
        td.shard_kv(kd, vd, 0)
    with pytest.raises(td.InvalidArgument):
        td.tree_decode(qd, td.ShardedKVCache([], [], 0), td.topology_for_workers(1))


def test_decode_is_deterministic(td, oracle):
    """test_decode.cpp:185-202: bitwise-identical results by default (the static
    calibrated split); the opt-in dynamic pool (TD_DYNAMIC / set_deterministic(False))
    agrees to ~1e-7."""
    import torch
    q, k, v = make_inputs(oracle, 9, 1, 32, 8, 400000, 128, BF16)
    qd, kd, vd = dev(q, BF16), dev(k, BF16), dev(v, BF16)
    cache = td.shard_kv(kd, vd, 8)
    a = td.tree_decode(qd, cache, td.topology_for_workers(8)).output
    b = td.tree_decode(qd, cache, td.topology_for_workers(8)).output
    assert torch.equal(a, b)
    w = td.Worker(0)
    w.place_kv(kd, vd)
    x = w.tree_decode(qd)
    y = w.tree_decode(qd)
    h = w.tree_decode(qd.cpu())  # the host-buffer path computes the same split
    assert torch.equal(x, y) and torch.equal(x.cpu(), h)
    dyn = [w.tree_decode(qd, flags=td._capi.TD_DYNAMIC) for _ in range(3)]
    try:
        td.set_deterministic(False)
        c = td.tree_decode(qd, cache, td.topology_for_workers(8)).output
        z = w.tree_decode(qd)
    finally:
        td.set_deterministic(True)
    w.close()
    assert rel_err(host(c), host(a)) <= 5e-6 and rel_err(host(z), host(x)) <= 5e-6
    assert max(rel_err(host(o), host(x)) for o in dyn) <= 5e-6
    want = oracle.tree_decode(q, k, v, 1, HIER, 1.0, F64, nthreads=8)
    assert rel_err(host(x), want) <= 1e-3 and rel_err(host(dyn[0]), want) <= 1e-3


# ---------------------------------------------------------------- the Worker (C-ABI context) path
@pytest.mark.parametrize("dtype,n_q,n_kv,n", [(F32, 1, 1, 65536), (BF16, 32, 8, 262144), (BF16, 8, 8, 70001)])
def test_worker_generate_and_decode(td, oracle, dtype, n_q, n_kv, n):
    """cfg1 at full size; GQA / MHA at reduced length. Inputs generated on the
    device with the bit-exact generator, oracle on the same seeds."""
    import torch
    seed = oracle.mix64(0, n)  # data_seed = mix64(seed, N), bench.cpp:73
    w = td.Worker(0)
    w.generate_kv(td.DType(dtype), 1, n_kv, n, 128, oracle.mix64(seed, 2), oracle.mix64(seed, 3))
    q = oracle.seeded(oracle.mix64(seed, 1), n_q * 128, dtype).reshape(1, n_q, 128)
    out = w.tree_decode(dev(q, dtype))
    want = full_decode(oracle, q, n_kv, n, oracle.mix64(seed, 2), oracle.mix64(seed, 3), dtype)  # every row
    assert rel_err_rows(host(out), want) <= TOL[dtype]
    # host buffers through the same call (the e2e path)
    out_h = w.tree_decode(torch.from_numpy(np.ascontiguousarray(q)).to(dev(q, dtype).dtype))
    assert rel_err(out_h.double().numpy(), host(out)) <= 5e-6  # default mode: ~1e-7..1e-6 between calls
    kernels, kv_bytes, split = w.last_launch_stats()
    assert kernels >= 2 and kv_bytes == 2 * n_kv * n * 128 * (2 if dtype == BF16 else 4)
    w.close()


@pytest.mark.parametrize("dtype", [BF16, F32])
def test_worker_append_loop(td, oracle, dtype):
    """Multi-step decode: append one token per step (through capacity growth,
    from host and device), decode the grown cache; equals the reference's
    decode over the concatenated cache."""
    import torch
    b, n_q, n_kv, n, d, steps = 2, 8, 2, 1500, 128, 1100
    q, k, v = make_inputs(oracle, 33, b, n_q, n_kv, n + steps, d, dtype)
    w = td.Worker(0)
    w.place_kv(dev(np.ascontiguousarray(k[:, :, :n]), dtype), dev(np.ascontiguousarray(v[:, :, :n]), dtype))
    tdt = dev(q, dtype).dtype
    for s in range(steps):
        kt = torch.from_numpy(np.ascontiguousarray(k[:, :, n + s:n + s + 1])).to(tdt)
        vt = torch.from_numpy(np.ascontiguousarray(v[:, :, n + s:n + s + 1])).to(tdt)
        if s % 2:
            kt, vt = kt.cuda(), vt.cuda()
        w.append_kv(kt, vt)
        if s in (0, 1, 1023, 1024, steps - 1):  # around the first capacity growth (+1024)
            m = n + s + 1
            out = w.tree_decode(dev(q, dtype))
            want = oracle.tree_decode(q, np.ascontiguousarray(k[:, :, :m]), np.ascontiguousarray(v[:, :, :m]),
                                      1, HIER, 1.0, F64)
            assert rel_err(host(out), want) <= TOL[dtype], (s, rel_err(host(out), want))
            r = w.ring_decode(dev(q, dtype))
            assert rel_err(host(r), want) <= TOL[dtype]
    assert w.kv_info()[1] == n + steps and w.seq_len == n + steps
    w.reserve_kv(5000)
    out = w.tree_decode(dev(q, dtype))
    assert rel_err(host(out), oracle.tree_decode(q, k, v, 1, HIER, 1.0, F64)) <= TOL[dtype]
    w.close()


def test_append_decode_loop_without_host_sync(td, oracle):
    """A generation loop with no host synchronisation: device-source append
    (kernel), then an async decode into its own output slot, 150 times. Each
    appended key points along the group's first query (score ~15-30 against
    ~0.3), so a tile read before its token landed -- K1 streams tiles below
    the last decode's length before its PDL wait -- would move the output far
    past the tolerance. Covers the capacity growth on the first append."""
    import torch
    b, n_q, n_kv, n, d, steps = 1, 32, 8, 700, 128, 150
    scale = 1.0 / math.sqrt(d)
    q, k, v = make_inputs(oracle, 41, b, n_q, n_kv, n + steps, d, BF16)
    g = n_q // n_kv
    qb = q.reshape(b, n_kv, g, d)[:, :, 0]  # [b, n_kv, d]
    k = k.copy()
    for s in range(steps):  # bf16-exact needles: q times a power of two (scores ~15 / ~30)
        k[:, :, n + s] = qb * float(2 << (s % 2))
    w = td.Worker(0)
    w.place_kv(dev(np.ascontiguousarray(k[:, :, :n]), BF16), dev(np.ascontiguousarray(v[:, :, :n]), BF16))
    qd = dev(q, BF16)
    kn = dev(np.ascontiguousarray(np.moveaxis(k[:, :, n:], 2, 0)[:, :, :, None]), BF16)  # [steps, b, n_kv, 1, d]
    vn = dev(np.ascontiguousarray(np.moveaxis(v[:, :, n:], 2, 0)[:, :, :, None]), BF16)
    out = torch.empty(steps, b, n_q, d, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    for s in range(steps):
        w.append_kv(kn[s], vn[s])
        w.tree_decode_async(qd.data_ptr(), n_q, out[s].data_ptr(), scale)
    w._sync_worker()
    got = out.cpu().double().numpy()
    for s in range(steps):
        m = n + s + 1
        want = oracle.tree_decode(q, np.ascontiguousarray(k[:, :, :m]), np.ascontiguousarray(v[:, :, :m]), 1, HIER,
                                  scale, F64)
        assert rel_err(got[s], want) <= TOL[BF16], (s, rel_err(got[s], want))
    w.close()


def test_group_fused_append_loop(td, oracle):
    """Device-token appends into a 3-worker group on one GPU, decoded through the
    exchange combine with no host synchronisation. The last worker's split kernel
    writes each token as it streams (fused append); on every third step two tokens
    are appended before one decode, so the first is written by the append kernel
    the second append enqueues. A token read before it landed, or written twice at
    the wrong position, moves the output past the tolerance (needle keys as above)."""
    import torch
    b, n_q, n_kv, n, d, steps, p = 1, 32, 8, 5000, 128, 40, 3
    q, k, v = make_inputs(oracle, 47, b, n_q, n_kv, n + steps, d, BF16)
    qb = q.reshape(b, n_kv, n_q // n_kv, d)[:, :, 0]
    k = k.copy()
    for s in range(steps):
        k[:, :, n + s] = qb * float(2 << (s % 2))
    g = td.WorkerGroup(p, [0])
    start = 0
    for w, e in zip(g.workers, td.chunk_extents(n, p)):
        w.place_kv(dev(np.ascontiguousarray(k[:, :, start:start + e]), BF16),
                   dev(np.ascontiguousarray(v[:, :, start:start + e]), BF16), seq_len=n, start=start)
        start += e
    g.enable_p2p(b * n_q, d)
    qd = dev(q, BF16)
    kn = dev(np.ascontiguousarray(np.moveaxis(k[:, :, n:], 2, 0)[:, :, :, None]), BF16)
    vn = dev(np.ascontiguousarray(np.moveaxis(v[:, :, n:], 2, 0)[:, :, :, None]), BF16)
    out = torch.empty(steps, b, n_q, d, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    decoded = []
    for s in range(steps):
        for w in g.workers:
            w.append_kv(kn[s], vn[s])
        if s % 3 != 1:
            g.tree_decode_async(qd.data_ptr(), n_q, out[s].data_ptr())
            decoded.append(s)
    for w in g.workers:
        w._sync_worker()
        assert w.p2p_status() == 0
    assert g.workers[-1].kv_info()[1] == td.chunk_extents(n, p)[-1] + steps
    got = out.cpu().double().numpy()
    g.close()
    for s in decoded:
        m = n + s + 1
        want = oracle.tree_decode(q, np.ascontiguousarray(k[:, :, :m]), np.ascontiguousarray(v[:, :, :m]), 1, HIER,
                                  1.0, F64)
        assert rel_err(got[s], want) <= TOL[BF16], (s, rel_err(got[s], want))


def test_worker_append_validation_and_output_buffers(td, oracle):
    """Append errors leave the cache unchanged; host outputs work pinned
    (zero-copy store) and pageable (D2H copy) alike."""
    import torch
    q, k, v = make_inputs(oracle, 35, 1, 8, 2, 700, 128, BF16)
    w = td.Worker(0)
    w.place_kv(dev(k, BF16), dev(v, BF16))
    with pytest.raises(td.InvalidArgument):
        w.append_kv(torch.zeros(1, 2, 1, 128, dtype=torch.float32), torch.zeros(1, 2, 1, 128, dtype=torch.float32))
    with pytest.raises(td.InvalidArgument):
        w.append_kv(torch.zeros(1, 2, 2, 128, dtype=torch.bfloat16), torch.zeros(1, 2, 2, 128, dtype=torch.bfloat16))
    assert w.kv_info()[1] == 700
    qh = torch.from_numpy(np.ascontiguousarray(q)).to(torch.bfloat16)
    pinned = torch.empty(1, 8, 128, dtype=torch.float32).pin_memory()
    pageable = torch.empty(1, 8, 128, dtype=torch.float32)
    a = w.tree_decode(qh, out=pinned)
    b = w.tree_decode(qh, out=pageable)
    want = oracle.tree_decode(q, k, v, 1, HIER, 1.0, F64)
    assert rel_err(a.double().numpy(), want) <= 1e-3 and rel_err(b.double().numpy(), want) <= 1e-3
    assert a.data_ptr() == pinned.data_ptr() and b.data_ptr() == pageable.data_ptr()
    w.close()


def test_long_shard_default_path(td, oracle):
    """A shard long enough (>= 1024 tiles per CTA) for the dynamic mode to turn
    cross-row stealing on, with the calibrated partition; and the default static
    split (the bench's N=1 path)."""
    n, n_q, n_kv = 655360, 32, 8
    seed = oracle.mix64(0, n)
    w = td.Worker(0)
    w.generate_kv(td.DType(BF16), 1, n_kv, n, 128, oracle.mix64(seed, 2), oracle.mix64(seed, 3))
    q = oracle.seeded(oracle.mix64(seed, 1), n_q * 128, BF16).reshape(1, n_q, 128)
    outs = [w.tree_decode(dev(q, BF16)) for _ in range(2)]
    outs += [w.tree_decode(dev(q, BF16), flags=td._capi.TD_DYNAMIC) for _ in range(2)]  # pool + stealing
    w.close()
    want = full_decode(oracle, q, n_kv, n, oracle.mix64(seed, 2), oracle.mix64(seed, 3), BF16)  # every row
    for o in outs:
        assert rel_err_rows(host(o), want) <= TOL[BF16]


def test_cross_row_stealing_parity(lib):
    """Stealing (foreign states merged by K2) forced on small shards, in a
    subprocess because the switch is read once per process."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TD_STEAL_SLOTS="16", TD_STEAL_MIN="1", TD_STEAL_SCANS="8")
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "steal_check.py")], capture_output=True,
                       text=True, timeout=600, env=env, cwd=root)
    print(r.stdout[-2000:])
    assert r.returncode == 0, r.stderr[-3000:]


def test_streamed_combine_matches_cta_merge(lib, tmp_path):
    """The streamed combine (default: K2 folds K1's warp and chunk states as they
    are published) against the CTA-merge combine (TD_K2_STREAM=0): each is bitwise
    reproducible across calls, entry points and buffers, matches the oracle, and
    the two agree to fp32 regrouping."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    dirs = {}
    for mode in ("1", "0"):
        d = tmp_path / f"mode{mode}"
        d.mkdir()
        env = dict(os.environ, TD_STREAM_CHECK_MODE=mode)
        r = subprocess.run([sys.executable, os.path.join(root, "tests", "stream_check.py"), str(d)],
                           capture_output=True, text=True, timeout=600, env=env, cwd=root)
        print(r.stdout[-2000:])
        assert r.returncode == 0, r.stderr[-3000:]
        dirs[mode] = d
    for f in sorted(os.listdir(dirs["1"])):
        a, b = np.load(dirs["1"] / f), np.load(dirs["0"] / f)
        assert rel_err(a, b) <= 5e-6, f


def test_streamed_combine_timeout_is_an_error(lib):
    """A split-kernel state that is never published (debug hook) makes the streamed
    combine give up after ~1 s and the call fail with TD_ECUDA."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TD_DEBUG_REVERSE="4")
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "stream_timeout_check.py")], capture_output=True,
                       text=True, timeout=300, env=env, cwd=root)
    print(r.stdout[-2000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]


def test_worker_place_matches_generate(td, oracle):
    import torch
    q, k, v = make_inputs(oracle, 21, 2, 8, 4, 3000, 128, BF16)
    w = td.Worker(0)
    w.place_kv(dev(k, BF16), dev(v, BF16))
    a = w.tree_decode(dev(q, BF16))
    w.place_kv(torch.from_numpy(k).to(torch.bfloat16), torch.from_numpy(v).to(torch.bfloat16))  # from host
    b = w.tree_decode(dev(q, BF16))
    assert rel_err(host(a), host(b)) <= 5e-6
    assert rel_err(host(a), oracle.tree_decode(q, k, v, 1, HIER, 1.0, F64)) <= 1e-3
    r = w.ring_decode(dev(q, BF16))  # p = 1: ring is the local partial
    assert rel_err(host(r), host(a)) <= 5e-6
    # deterministic mode: bitwise-identical repeated calls through every entry point
    x = w.tree_decode(dev(q, BF16), flags=td._capi.TD_DETERMINISTIC)
    y = w.tree_decode(dev(q, BF16), flags=td._capi.TD_DETERMINISTIC)
    z = w.ring_decode(dev(q, BF16), flags=td._capi.TD_DETERMINISTIC)
    assert torch.equal(x, y) and torch.equal(x, z)
    w.close()
