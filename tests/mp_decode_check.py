#!/usr/bin/env python3
"""Multi-GPU parity check, one process per GPU (launched by torchrun; used by
tests/test_gpu_multi.py). Every rank generates its own shard of the seeded
cache on its GPU, runs the NCCL tree decode and the ring pass-KV decode, and
rank 0 compares every output row of both against the CPU oracle (reference
algorithm in Float64 on the same bf16 / f32 values).

Prints one JSON line per rank-0 case; exits non-zero on any parity failure.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2408_04093_b200 as td
    from oracle.full import full_decode, rel_err_rows
    from oracle.oracle import BF16, F32, F64, HIER, Oracle

    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    orc = Oracle()
    w = td.Worker.from_torch_distributed(local)
    w.enable_p2p(2 * 32, 128)
    cases = [  # dtype, b, n_q, n_kv, n, d, scale
        (BF16, 1, 32, 8, 262144 + 3, 128, 1.0),
        (BF16, 2, 8, 8, 20001, 128, 0.0883883476),
        (F32, 1, 2, 2, 65536, 128, 1.0),
        (BF16, 1, 4, 2, 3 * world + 1, 64, 1.0),   # tiny shards, ragged extents
    ]
    ok = True
    for dt, b, n_q, n_kv, n, d, scale in cases:
        seed = orc.mix64(0, n)
        w.generate_kv(td.DType(dt), b, n_kv, n, d, orc.mix64(seed, 2), orc.mix64(seed, 3))
        q = td.seeded_tensor([b, n_q, d], orc.mix64(seed, 1), 1.0, td.DType(dt))
        tree = w.tree_decode(q, scale)
        ring = w.ring_decode(q, scale)
        # the same NCCL step replayed as a CUDA graph (captured on the first call)
        gbuf = torch.empty_like(tree)  # one output buffer: captured once per pool parity, then replayed
        graphed = [w.tree_decode(q, scale, out=gbuf, flags=td._capi.TD_GRAPH).clone() for _ in range(5)]
        fits = b * n_q <= 64 and d == 128
        p2p = w.tree_decode(q, scale, flags=td._capi.TD_P2P) if fits else tree
        # the two allreduces inside one kernel through NCCL's device API (several
        # calls: the window's parities alternate), device and host buffers
        ndev = [w.tree_decode(q, scale, flags=td._capi.TD_NCCL_DEVICE).clone() for _ in range(3)]
        ndev.append(w.tree_decode(q.cpu(), scale, flags=td._capi.TD_NCCL_DEVICE))
        # every rank must hold the same output
        t_all = [torch.empty_like(tree) for _ in range(world)]
        dist.all_gather(t_all, tree)
        if rank == 0:
            qh = orc.seeded(orc.mix64(seed, 1), b * n_q * d, dt).reshape(b, n_q, d)
            want = full_decode(orc, qh, n_kv, n, orc.mix64(seed, 2), orc.mix64(seed, 3), dt, scale)  # every row
            tol = 1e-3 if dt == BF16 else 1e-5
            e_tree = rel_err_rows(tree.double().cpu().numpy(), want)
            e_ring = rel_err_rows(ring.double().cpu().numpy(), want)
            e_p2p = rel_err_rows(p2p.double().cpu().numpy(), want)
            e_ndev = max(rel_err_rows(x.double().cpu().numpy(), want) for x in ndev)
            same = all(torch.equal(t_all[0], x) for x in t_all)
            same_graph = all(torch.equal(tree, x) for x in graphed)  # static split: bitwise
            good = (e_tree <= tol and e_ring <= tol and e_p2p <= tol and e_ndev <= tol and same and same_graph
                    and w.p2p_status() == 0)
            ok &= good
            print(json.dumps({"world": world, "dtype": "bf16" if dt == BF16 else "f32", "n": n, "b": b, "n_q": n_q,
                              "n_kv": n_kv, "tree_rel_err": e_tree, "ring_rel_err": e_ring, "p2p_rel_err": e_p2p,
                              "nccl_device_rel_err": e_ndev,
                              "ranks_agree": same, "graph_equals_stream": same_graph, "ok": good}), flush=True)
    # generation loop: append tokens to rank p-1's shard, decode the grown cache
    b, n_q, n_kv, d, n0, steps = 1, 8, 2, 128, 4096 * world + 5, 40
    seed = orc.mix64(7, n0)
    qh = orc.seeded(orc.mix64(seed, 1), b * n_q * d, BF16).reshape(b, n_q, d)
    kh = orc.seeded(orc.mix64(seed, 2), b * n_kv * (n0 + steps) * d, BF16).reshape(b, n_kv, n0 + steps, d)
    vh = orc.seeded(orc.mix64(seed, 3), b * n_kv * (n0 + steps) * d, BF16).reshape(b, n_kv, n0 + steps, d)
    s0, ln = td.shard_range(n0, world, rank)
    bf = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16)  # noqa: E731
    w.place_kv(bf(kh[:, :, s0:s0 + ln]).cuda(), bf(vh[:, :, s0:s0 + ln]).cuda(), seq_len=n0)
    q = bf(qh).cuda()
    for s in range(steps):
        w.append_kv(bf(kh[:, :, n0 + s:n0 + s + 1]).cuda(), bf(vh[:, :, n0 + s:n0 + s + 1]).cuda())
        if s not in (0, steps - 1):
            continue
        # the first decode after a device append writes the token (fused): a different
        # combine takes it at the first and at the last step
        fl = {"tree": 0, "p2p": td._capi.TD_P2P, "nccl_device": td._capi.TD_NCCL_DEVICE}
        order = ["tree", "ring", "p2p", "nccl_device"] if s == 0 else ["nccl_device", "p2p", "ring", "tree"]
        res = {k: (w.ring_decode(q) if k == "ring" else w.tree_decode(q, flags=fl[k])) for k in order}
        if rank == 0:
            m = n0 + s + 1
            want = orc.tree_decode(qh, np.ascontiguousarray(kh[:, :, :m]), np.ascontiguousarray(vh[:, :, :m]),
                                   world, HIER, 1.0, F64, nthreads=8)
            mx = np.max(np.abs(want))
            errs = {k + "_rel_err": float(np.max(np.abs(x.double().cpu().numpy() - want)) / mx) for k, x in res.items()}
            good = max(errs.values()) <= 1e-3
            ok &= good
            print(json.dumps({"world": world, "append_step": s, "n": m, **errs, "ok": good}), flush=True)
    # energy formulation across the ranks (Alg. 1 / Alg. 2, energy.cpp:152-259)
    b, h, nq, n, d = 1, 4, 2, 2048 * world + 3, 128
    seed = orc.mix64(9, n)
    qe = orc.seeded(orc.mix64(seed, 1), b * h * nq * d, BF16).reshape(b, h, nq, d)
    ke = orc.seeded(orc.mix64(seed, 2), b * h * n * d, BF16).reshape(b, h, n, d)
    ve = orc.seeded(orc.mix64(seed, 3), b * h * n * d, BF16).reshape(b, h, n, d)
    se = orc.seeded(orc.mix64(seed, 4), b * h * nq * d, BF16, scale=0.5).reshape(b, h, nq, d)
    s0, ln = td.shard_range(n, world, rank)
    w.place_kv(bf(ke[:, :, s0:s0 + ln]).cuda(), bf(ve[:, :, s0:s0 + ln]).cuda(), seq_len=n)
    ev = w.energy_forward(bf(qe).cuda(), bf(se).cuda())
    e0 = w.energy_forward(bf(qe).cuda())
    gr = w.energy_grad(bf(qe).cuda(), e0)
    if rank == 0:
        want = orc.energy_forward_parallel(qe, ke, ve, se, world, F64)
        errs = [float(np.max(np.abs(x.double().cpu().numpy() - y)) / max(1.0, np.max(np.abs(y))))
                for x, y in zip((ev.value, ev.row_max, ev.shifted_lse), want)]
        _, rm, sh = orc.energy_forward_parallel(qe, ke, ve, None, world, F64)
        gw = orc.energy_grad_parallel(qe, ke, ve, rm, sh, world, F64)
        eg = float(np.max(np.abs(gr.double().cpu().numpy() - gw)) / np.max(np.abs(gw)))
        good = max(errs) <= 1e-3 and eg <= 1e-3
        ok &= good
        print(json.dumps({"world": world, "energy_forward_errs": errs, "energy_grad_err": eg, "ok": good}), flush=True)
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.broadcast(flag, 0)
    w.close()
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
