#!/usr/bin/env python3
"""Device timeline of back-to-back decode steps (TD_DEBUG_TIMELINE=1): per step
the first K1 CTA start, the first CTA past K1's PDL wait, the last K1 CTA end
and the last K2 warp done (globaltimer, no extra stream operations).
  TD_DEBUG_TIMELINE=1 python scripts/timeline_probe.py [--seq-len N] [--steps K]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq-len", type=int, default=131072)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--b", type=int, default=1)
    ap.add_argument("--nq", type=int, default=32)
    ap.add_argument("--nkv", type=int, default=8)
    ap.add_argument("--append", action="store_true", help="append one token before every step")
    ap.add_argument("--isolated", action="store_true", help="synchronise after every step (a cold call each time)")
    ap.add_argument("--dynamic", action="store_true", help="TD_DYNAMIC: the dynamic tile pool")
    ap.add_argument("--f32", action="store_true", help="fp32 cache and query (the cfg1 kernel)")
    ap.add_argument("--reserve", type=int, default=0, help="reserve this many extra tokens per row first")
    ap.add_argument("--distinct", action="store_true", help="with --append: a different token every step")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_2408_04093_b200 as td
    from paper_2408_04093_b200 import _capi
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    flags = 0
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        w = td.Worker.from_torch_distributed(local)
        w.enable_p2p(args.b * args.nq, 128)
        flags = _capi.TD_P2P
    else:
        w = td.Worker(local)
    if args.dynamic:
        flags |= _capi.TD_DYNAMIC
    dt = td.DType.Float32 if args.f32 else td.DType.Bf16
    w.generate_kv(dt, args.b, args.nkv, args.seq_len, 128, 2, 3)
    q = td.seeded_tensor([args.b, args.nq, 128], 1, 1.0, dt)
    out = torch.empty(args.b, args.nq, 128, device="cuda")
    for _ in range(3):
        w.tree_decode_async(q.data_ptr(), args.nq, out.data_ptr(), 1.0, flags)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    if args.reserve:
        w.reserve_kv(args.reserve)
        torch.cuda.synchronize()
        for _ in range(3):
            w.tree_decode_async(q.data_ptr(), args.nq, out.data_ptr(), 1.0, flags)
        torch.cuda.synchronize()
    if args.append:
        w.reserve_kv(args.steps + 8)
        tok = td.seeded_tensor([args.b, args.nkv, 128], 9, 1.0, td.DType.Bf16)
        toks = td.seeded_tensor([args.steps, args.b, args.nkv, 128], 4, 1.0, td.DType.Bf16)
        torch.cuda.synchronize()
    import time
    t_host = time.perf_counter()
    for i in range(args.steps):
        if args.append:
            if args.distinct:
                w.append_kv(toks[i], toks[i])
            else:
                w.append_kv(tok, tok)
        w.tree_decode_async(q.data_ptr(), args.nq, out.data_ptr(), 1.0, flags)
        if args.isolated:
            w._sync_worker()
    host_us = (time.perf_counter() - t_host) / args.steps * 1e6
    torch.cuda.synchronize()
    st = w.debug_stamps(6144)
    rows = [st[5000 + 4 * i: 5004 + 4 * i] for i in range(3, 3 + args.steps)]
    t0 = rows[0][0]
    us = lambda x: round((x - t0) / 1000.0, 2)  # noqa: E731
    tl = [[us(x) for x in r] for r in rows]
    gaps = [round(tl[i + 1][0] - tl[i][3], 2) for i in range(len(tl) - 1)]
    waits = [round(tl[i + 1][1] - tl[i][3], 2) for i in range(len(tl) - 1)]
    steps = [round(tl[i + 1][1] - tl[i][1], 2) for i in range(len(tl) - 1)]
    print(json.dumps({"rank": local, "world": world, "seq_len": args.seq_len, "pdl": os.environ.get("TD_K1_PDL", "1"),
                      "isolated": args.isolated, "host_us_per_step": round(host_us, 2),
                      "k1_first_start_to_first_past_wait": [round(r[1] - r[0], 2) for r in tl],
                      "abs_k1_start_us": [round(r[0] / 1000.0, 2) for r in rows],
                      "abs_k1_end_us": [round(r[2] / 1000.0, 2) for r in rows],
                      "abs_k2_done_us": [round(r[3] / 1000.0, 2) for r in rows],
                      "k1_start_minus_prev_k2_done": gaps, "k1_past_wait_minus_prev_k2_done": waits,
                      "step_period": steps, "k1_span": [round(r[2] - r[1], 2) for r in tl],
                      "tail": [round(r[3] - r[2], 2) for r in tl]}))
    if os.environ.get("TL_DUMP_CTAS"):  # the last step, per CTA index: (c, smid, past-wait, end)
        nc = 452  # CTA slots [4096 + 2c] below the per-step rows at [5000 + 4i]
        g0 = min(st[4096 + 2 * c] for c in range(nc) if st[4096 + 2 * c])
        print(json.dumps({"rank": local, "ctas": [(c, st[2048 + c], round((st[4096 + 2 * c] - g0) / 1000.0, 2),
                                                   round((st[4097 + 2 * c] - g0) / 1000.0, 2))
                                                  for c in range(nc) if st[4097 + 2 * c]]}))
    w.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
