"""The multi-rank decomposition on CPU (world_size 2 and 4, gloo): each rank
holds the shard shard_range(N, p, rank) gives it, computes its partial, and
the ranks run the tree exchange (allreduce max -> rescale -> allreduce sum ->
divide) and the ring pass-KV exchange (send to rank+1, receive from rank-1,
fold in ring_fold_order) with real torch.distributed collectives. The result
must equal the reference algorithm (oracle) on the unsharded cache. This is
the host-side logic the GPU ranks run, with the GPU kernels replaced by the
oracle's chunk partial."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, k, v, ret):
    import sys
    sys.path.insert(0, ROOT)
    import paper_2408_04093_b200 as td
    from oracle.oracle import F64, Oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    n = k.shape[2]
    start, ln = td.shard_range(n, world, rank)
    b, n_q, d = q.shape
    rows = b * n_q
    # --- tree: local partial, allreduce(max), rescale, allreduce(sum), divide
    _, lse, out = orc.chunk_partial(q, k, v, start, ln, 1.0, F64)
    shift = torch.from_numpy(lse.copy())
    dist.all_reduce(shift, op=dist.ReduceOp.MAX)
    w = np.exp(lse - shift.numpy())
    nd = torch.from_numpy(np.concatenate([(out * w[..., None]).reshape(-1), w.reshape(-1)]))
    dist.all_reduce(nd, op=dist.ReduceOp.SUM)
    nd = nd.numpy()
    tree = nd[: rows * d].reshape(b, n_q, d) / nd[rows * d:].reshape(b, n_q)[..., None]
    # --- ring pass-KV: chunks really move between ranks
    ext = td.chunk_extents(n, world)
    kv_in = np.ascontiguousarray(np.concatenate([k[:, :, start:start + ln], v[:, :, start:start + ln]], axis=2))
    m0, l0, o0 = orc.chunk_partial(q, k, v, start, ln, 1.0, F64)
    root = (m0, l0, o0)
    held = kv_in
    for r, chunk in enumerate(td.ring_fold_order(world, rank)[1:]):
        incoming = np.empty((b, k.shape[1], 2 * ext[chunk], d))
        sreq = dist.isend(torch.from_numpy(held), (rank + 1) % world)
        rbuf = torch.from_numpy(incoming)
        dist.recv(rbuf, (rank - 1) % world)
        sreq.wait()
        held = rbuf.numpy().copy()
        kc, vc = held[:, :, : ext[chunk]].copy(), held[:, :, ext[chunk]:].copy()
        mp_, lp, op = orc.chunk_partial(q, kc, vc, 0, ext[chunk], 1.0, F64)
        lm, ll, lo = root
        nm, nl, no = np.empty_like(lm), np.empty_like(ll), np.empty_like(lo)
        orc.lib.orc_combine_pair(*[orc_ptr(x) for x in (lm, ll, lo, mp_, lp, op)], rows, d, F64,
                                 *[orc_ptr(x) for x in (nm, nl, no)])
        root = (nm, nl, no)
    ret[rank] = (tree, root[2])
    dist.destroy_process_group()


def orc_ptr(a):
    import ctypes
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


@pytest.mark.parametrize("world", [2, 4])
def test_tree_and_ring_exchange_gloo(oracle, world):
    from conftest import make_inputs
    from oracle.oracle import F64, HIER
    q, k, v = make_inputs(oracle, 31 + world, 2, 4, 2, 1001, 16, F64)
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    ret = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, k, v, ret)) for r in range(world)]
    for p_ in procs:
        p_.start()
    for p_ in procs:
        p_.join(120)
        assert p_.exitcode == 0
    want = oracle.tree_decode(q, k, v, world, HIER, 1.0, F64)
    want_ring = oracle.ring_decode(q, k, v, world, 1.0, F64)
    for r in range(world):
        tree, ring = ret[r]
        assert np.max(np.abs(tree - want)) <= 1e-12
        assert np.max(np.abs(ring - want_ring)) <= 1e-12
    # rank 0's ring fold is the reference's root: bitwise
    assert np.array_equal(ret[0][1], want_ring)
