#!/usr/bin/env python3
"""Decode through the default deterministic path with the streamed combine on or
off (TD_STREAM_CHECK_MODE sets TD_K2_STREAM, read once per process, hence a
subprocess of tests/test_gpu_parity.py). Per shape: three device-buffer calls, a
host-buffer call and the ring at p = 1 must be bitwise equal; the result must
match the CPU oracle on every row; a short append + decode loop must match the
oracle on its last step. Outputs are saved to argv[1] so the caller can compare
the two modes. Exits non-zero on a failure."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

SHAPES = [(1, 32, 8, 150001), (2, 8, 4, 70001), (1, 32, 8, 131072)]


def main():
    os.environ["TD_K2_STREAM"] = os.environ.get("TD_STREAM_CHECK_MODE", "1")
    import numpy as np
    import torch

    import paper_2408_04093_b200 as td
    from conftest import make_inputs, rel_err
    from oracle.oracle import BF16, F64, HIER, Oracle
    out_dir = sys.argv[1]
    orc = Oracle()
    ok = True
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to("cuda").to(torch.bfloat16)  # noqa: E731
    for b, n_q, n_kv, n in SHAPES:
        q, k, v = make_inputs(orc, 17 + n, b, n_q, n_kv, n, 128, BF16)
        w = td.Worker(0)
        w.place_kv(dev(k), dev(v))
        qd = dev(q)
        q2 = make_inputs(orc, 29 + n, b, n_q, n_kv, 1, 128, BF16)[0]  # another query, same cache
        outs, other = [], []
        for _ in range(3):  # alternating queries: a step must never see the previous step's states
            outs.append(w.tree_decode(qd))
            other.append(w.tree_decode(dev(q2)))
        hout = w.tree_decode(qd.cpu())
        ring = w.ring_decode(qd)
        same = all(torch.equal(outs[0], o) for o in outs[1:]) and torch.equal(outs[0].cpu(), hout) \
            and torch.equal(outs[0], ring) and all(torch.equal(other[0], o) for o in other[1:])
        want = orc.tree_decode(q, k, v, 1, HIER, 1.0, F64, nthreads=os.cpu_count() or 8)
        want2 = orc.tree_decode(q2, k, v, 1, HIER, 1.0, F64, nthreads=os.cpu_count() or 8)
        err = max(rel_err(outs[0].double().cpu().numpy(), want), rel_err(other[0].double().cpu().numpy(), want2))
        np.save(os.path.join(out_dir, f"out_{b}_{n_q}_{n_kv}_{n}.npy"), outs[0].float().cpu().numpy())
        good = same and err <= 1e-3
        ok &= good
        print(json.dumps({"b": b, "n_q": n_q, "n_kv": n_kv, "n": n, "bitwise_repeat": same, "err": err,
                          "ok": good}), flush=True)
        w.close()
    # append + decode loop (the fused append rides on the streamed K1)
    b, n_q, n_kv, n0, steps = 1, 32, 8, 65536 + 7, 6
    q, k, v = make_inputs(orc, 5, b, n_q, n_kv, n0 + steps, 128, BF16)
    w = td.Worker(0)
    w.place_kv(dev(k[:, :, :n0]), dev(v[:, :, :n0]))
    qd = dev(q)
    for s in range(steps):
        w.append_kv(dev(k[:, :, n0 + s:n0 + s + 1]), dev(v[:, :, n0 + s:n0 + s + 1]))
        out = w.tree_decode(qd)
    want = orc.tree_decode(q, k, v, 1, HIER, 1.0, F64, nthreads=os.cpu_count() or 8)
    err = rel_err(out.double().cpu().numpy(), want)
    good = err <= 1e-3
    ok &= good
    print(json.dumps({"append_loop": steps, "n": n0 + steps, "err": err, "ok": good}), flush=True)
    w.close()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
