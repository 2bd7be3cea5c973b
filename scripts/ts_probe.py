#!/usr/bin/env python3
"""Per-stage device timestamps of one decode step (TD_DEBUG_TS), per rank.
torchrun --nproc-per-node N scripts/ts_probe.py [--combine p2p|nccl] [--seq-len N]
Prints, per rank, microseconds relative to the first K1 CTA start:
K1 end, and for the K2 blocks the max over blocks of each stage."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--combine", default="p2p")
    ap.add_argument("--seq-len", type=int, default=1 << 20)
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_2408_04093_b200 as td
    from paper_2408_04093_b200 import _capi
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = td.Worker.from_torch_distributed(local) if world > 1 else td.Worker(local)
    b, n_q, n_kv, d = 1, 32, 8, 128
    w.generate_kv(td.DType.Bf16, b, n_kv, args.seq_len, d, 11, 12)
    q = td.seeded_tensor([b, n_q, d], 13, 1.0, td.DType.Bf16)
    out = torch.empty(b, n_q, d, device="cuda")
    flags = 0
    if args.combine == "p2p" and world > 1:
        w.enable_p2p(b * n_q, d)
        flags = _capi.TD_P2P
    torch.cuda.synchronize()
    for _ in range(args.steps):
        w.tree_decode_async(q.data_ptr(), n_q, out.data_ptr(), 1.0, flags)
    res = []
    for _ in range(5):
        w.tree_decode_async(q.data_ptr(), n_q, out.data_ptr(), 1.0, flags | _capi.TD_DEBUG_TS)
        st = w.debug_stamps(6144)
        t0 = st[0]
        ends = sorted((st[4097 + 2 * c] - t0) / 1000.0 for c in range(1024) if st[4097 + 2 * c])
        starts = sorted((st[4096 + 2 * c] - t0) / 1000.0 for c in range(1024) if st[4096 + 2 * c])
        blocks = [st[8 + 8 * i: 8 + 8 * i + 8] for i in range(64) if st[8 + 8 * i] != 0]
        rel = lambda x: round((x - t0) / 1000.0, 2) if x else None
        summary = {"k1_end": rel(st[1]), "pre_k1_stamp": rel(st[2]), "post_k2_stamp": rel(st[3]),
                   "abs_k1_start_ns": int(t0), "abs_k1_end_ns": int(st[1])}
        if ends:
            qt = lambda xs, f: round(xs[min(len(xs) - 1, int(f * len(xs)))], 2)
            summary["cta_start_q"] = [qt(starts, f) for f in (0.0, 0.5, 1.0)]
            summary["cta_end_q"] = [qt(ends, f) for f in (0.0, 0.1, 0.5, 0.9, 1.0)]
        names = ["k2_entry", "pushed", "merged", "seen", "done"]
        if world == 1:
            names[1] = "probe_load"
            names[3] = "k2_prewait"
        for k, name in enumerate(names):
            vals = [bl[k] for bl in blocks if bl[k]]
            if vals:
                summary[name + "_min"] = rel(min(vals))
                summary[name + "_max"] = rel(max(vals))
                summary["abs_" + name + "_max_ns"] = int(max(vals))
        if os.environ.get("TS_DUMP_CTAS"):
            summary["ctas"] = [(c, st[2048 + c], round((st[4097 + 2 * c] - t0) / 1000.0, 2))
                               for c in range(1024) if st[4097 + 2 * c]]
        res.append(summary)
    print(json.dumps({"rank": local, "world": world, "combine": args.combine, "steps": res[1:]}), flush=True)
    w.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
