#!/usr/bin/env python3
"""A generation loop on the GPU path: every step
appends the new token's K/V (to rank p-1's shard) and runs the exact tree
decode over the grown cache. Prints one JSON line with the device time per
step (CUDA events around K back-to-back steps, max over ranks), the append's
share, and a final parity check of the last step against the CPU oracle on
the first kv group.

  python scripts/decode_loop.py [--seq-len N] [--steps K]
  torchrun --nproc-per-node P scripts/decode_loop.py --seq-len N
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq-len", type=int, default=1 << 20)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--no-check", action="store_true")
    args = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2408_04093_b200 as td
    from paper_2408_04093_b200 import _capi
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    flags = 0
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        w = td.Worker.from_torch_distributed(local)
        w.enable_p2p(32, 128)
        flags = _capi.TD_P2P
    else:
        w = td.Worker(local)
    b, n_q, n_kv, d, n, K = 1, 32, 8, 128, args.seq_len, args.steps
    w.generate_kv(td.DType.Bf16, b, n_kv, n, d, 2, 3)
    w.reserve_kv(K + 8)  # capacity for the loop: no growth inside the timed region
    q = td.seeded_tensor([b, n_q, d], 1, 1.0, td.DType.Bf16)
    # the new tokens' K/V (on the device, like a projection's output)
    ks = td.seeded_tensor([K, b, n_kv, d], 4, 1.0, td.DType.Bf16)
    vs = td.seeded_tensor([K, b, n_kv, d], 5, 1.0, td.DType.Bf16)
    out = torch.empty(b, n_q, d, device="cuda")
    stream = torch.cuda.ExternalStream(w.stream)
    for _ in range(3):  # warm-up (and calibration) on the placed cache
        w.tree_decode_async(q.data_ptr(), n_q, out.data_ptr(), 1.0, flags)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    import time
    host_us = {}

    def timed(do_append, do_decode):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t0 = time.perf_counter()
        t_app = 0.0
        for s in range(K):
            if do_append:
                ta = time.perf_counter()
                w.append_kv(ks[s], vs[s])
                t_app += time.perf_counter() - ta
            if do_decode:
                w.tree_decode_async(q.data_ptr(), n_q, out.data_ptr(), 1.0, flags)
        host_us[(do_append, do_decode)] = (time.perf_counter() - t0) / K * 1e6
        if do_append:
            host_us[("append only", True)] = t_app / K * 1e6
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / K

    decode_only = timed(False, True)
    ms = timed(True, True)
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    err = None
    if rank == 0 and not args.no_check:
        from conftest import rel_err
        from oracle.oracle import BF16, F64, HIER, Oracle
        orc = Oracle()
        g = n_q // n_kv
        qh = orc.seeded(1, b * n_q * d, BF16).reshape(b, n_q, d)[:, :g]
        k0 = orc.seeded(2, n * d, BF16).reshape(1, 1, n, d)
        v0 = orc.seeded(3, n * d, BF16).reshape(1, 1, n, d)
        kn = ks[:, 0, 0].float().cpu().double().numpy().reshape(1, 1, K, d)
        vn = vs[:, 0, 0].float().cpu().double().numpy().reshape(1, 1, K, d)
        kk, vv = np.concatenate([k0, kn], axis=2), np.concatenate([v0, vn], axis=2)
        want = orc.tree_decode(np.ascontiguousarray(qh), kk, vv, 1, HIER, 1.0, F64, nthreads=16)
        err = rel_err(out[:, :g].double().cpu().numpy(), want)
    if rank == 0:
        print(json.dumps({"metric": "generation loop: append + exact tree decode, us per token", "n_gpus": world,
                          "start_len": n, "steps": K, "us_per_token": ms * 1000.0,
                          "decode_only_us_per_token": decode_only * 1000.0,
                          "host_enqueue_us_per_step": {(a if isinstance(a, str) else ("append+decode" if a else "decode")):
                                                       round(v, 1) for (a, _), v in host_us.items()},
                          "final_len": n + K, "rel_err_vs_oracle": err}), flush=True)
    w.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
