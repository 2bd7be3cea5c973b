#!/usr/bin/env python3
"""Sequence-length sweep (BASELINE.json configs[4]): Llama-3-8B attention shape
(32 q / 8 kv heads, d 128, bf16), N = 16K ... 4M tokens, on the GPUs of one box.

  torchrun --nproc-per-node P scripts/sweep.py [--seq 16384,...] [--out sweep_pP.csv]

Writes the reference's bench CSV schema (bench.cpp:18-19, parsed by
`treedec report`, bench.cpp:193-302) with sim_time_s replaced by the MEASURED
device time of one decode step (max over ranks; meta key time=measured), and
prints one JSON line per point with us/token, HBM GB/s and the roofline
fraction. Rows: tree (NCCL max + sum allreduce), tree-p2p (one-shot NVLink
exchange, algo column 'tree' with meta combine), ring (pass-KV).
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

L2_BYTES = 126 * 1024 * 1024


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", default="16384,32768,65536,131072,262144,524288,1048576,2097152,4194304")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--ring-steps", type=int, default=3)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    import paper_2408_04093_b200 as td
    from paper_2408_04093_b200 import _capi, report  # noqa: F401

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def mx(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    b, n_q, n_kv, d = 1, 32, 8, 128
    w = td.Worker.from_torch_distributed(local) if world > 1 else td.Worker(local)
    if world > 1:
        w.enable_p2p(b * n_q, d)
    q = td.seeded_tensor([b, n_q, d], 1, 1.0, td.DType.Bf16)
    out = torch.empty(b, n_q, d, device="cuda")
    stream = torch.cuda.ExternalStream(w.stream)
    # L2 flush between steps of small shards: a read-only 256 MB sweep (a write flush
    # would leave dirty lines whose write-back lands in the timed step)
    scratch = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
    sink = torch.empty((), dtype=torch.float32, device="cuda")
    rows, lines = [], []
    first = True
    for n in [int(x) for x in args.seq.split(",")]:
        if n < world:
            continue
        w.generate_kv(td.DType.Bf16, b, n_kv, n, d, 2 + n, 3 + n)
        _, shard, shard_bytes = w.kv_info()
        flush = shard_bytes < 4 * L2_BYTES
        kv_rank = 2 * b * n_kv * math.ceil(n / world) * d * 2
        variants = [("tree", "nccl", 0, args.steps)]
        if world > 1:
            variants += [("tree", "p2p", _capi.TD_P2P, args.steps), ("ring", "nccl", 0, args.ring_steps)]
        for algo, comb, flags, steps in variants:
            fn = w.tree_decode_async if algo == "tree" else w.ring_decode_async
            # the first point also pays one-time costs (NCCL's lazily loaded kernels,
            # connection setup): it gets a longer warm-up
            for _ in range(args.warmup if not first else max(args.warmup, 30)):
                if flush:  # (the flush's own first-use costs stay out of the timed steps too)
                    with torch.cuda.stream(stream):
                        torch.sum(scratch, dim=0, out=sink)
                fn(q.data_ptr(), n_q, out.data_ptr(), 1.0, flags)
            barrier()
            if world > 1:  # release every rank's first step together (see bench.align_streams)
                t1 = torch.ones(1, device="cuda")
                dist.all_reduce(t1)
                ev = torch.cuda.Event()
                ev.record(torch.cuda.current_stream())
                stream.wait_event(ev)
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
            for i in range(steps):
                if flush:
                    with torch.cuda.stream(stream):
                        torch.sum(scratch, dim=0, out=sink)
                evs[i][0].record(stream)
                fn(q.data_ptr(), n_q, out.data_ptr(), 1.0, flags)
                evs[i][1].record(stream)
            barrier()
            ms = mx(sum(a.elapsed_time(e) for a, e in evs) / steps)
            if rank == 0:
                tc = td.tree_cost(b, n_q, n_kv, n, d, world) if algo == "tree" else td.ring_cost(b, n_q, n_kv, n, d, world)
                rounds = (2 if comb == "nccl" else 1) if algo == "tree" else world - 1
                rec = td.report.BenchRecord(algo, n, world, 1, ms * 1e-3, float(tc.elems_sent_total()), 0.0,
                                            int(tc.peak_elems_per_worker), rounds, math.nan)
                lines.append((comb, rec))
                rec = {"algo": algo, "combine": comb if world > 1 else "none", "N": n, "p": world,
                       "us_per_token": ms * 1000.0, "hbm_gbs": kv_rank / (ms * 1e-3) / 1e9,
                       "roofline_frac_of_measured": kv_rank / (ms * 1e-3) / 1e9 / peak,
                       "l2": "flushed" if flush else "inputs > L2"}
                rows.append(rec)
                print(json.dumps(rec), flush=True)
        first = False
    if rank == 0:
        for comb in ("nccl", "p2p"):
            sel = [r for c, r in lines if c == comb or (comb == "p2p" and r.algo == "ring")]
            if not sel or (comb == "p2p" and world == 1):
                continue
            path = args.out or os.path.join(ROOT, "gpurun_out", f"sweep_p{world}_{comb}.csv")
            if args.out:
                path = path.replace(".csv", f"_{comb}.csv")
            os.makedirs(os.path.dirname(path), exist_ok=True)
            seqs = sorted({r.seq_len for r in sel})
            meta = {"time": "measured (CUDA events, max over ranks)", "device": "B200", "dtype": "bf16",
                    "batch": str(b), "heads": f"{n_q}q/{n_kv}kv", "head_dim": str(d), "combine": comb,
                    "algos": "tree ring" if world > 1 else "tree", "clusters": f"1x{world}",
                    "seq_lens": " ".join(str(x) for x in seqs), "element_bytes": "2", "seed": "synthetic",
                    "max_abs_err": "nan (parity is checked by tests/, not re-measured at sweep sizes)"}
            out_ = td.report.SweepOutcome(records=sel, meta=meta)
            with open(path, "w") as f:
                td.report.write_csv(out_, f)
            with open(path.replace(".csv", ".json"), "w") as f:
                td.report.write_json(out_, f)
    w.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
