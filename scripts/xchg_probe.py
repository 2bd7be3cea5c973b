#!/usr/bin/env python3
"""Exchange-latency probe: a tiny KV shard (K1 ~ microseconds) so the step is
the exchange itself; per-stage in-kernel stamps and per-step CUDA-event
times, for the P2P exchange (TD_XCHG_VARIANT selects the flag protocol) and
the NCCL path, with the steps captured in a CUDA graph so the host launch
rate does not bound the measurement.
torchrun --nproc-per-node N scripts/xchg_probe.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    import paper_2408_04093_b200 as td
    from paper_2408_04093_b200 import _capi
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world, rank = dist.get_world_size(), dist.get_rank()
    w = td.Worker.from_torch_distributed(local)
    b, n_q, n_kv, d = 1, 32, 8, 128
    n = int(os.environ.get("PROBE_N", str(4096 * world)))
    w.generate_kv(td.DType.Bf16, b, n_kv, n, d, 5, 6)
    w.enable_p2p(b * n_q, d)
    q = td.seeded_tensor([b, n_q, d], 7, 1.0, td.DType.Bf16)
    out = torch.empty(b, n_q, d, device="cuda")
    stream = torch.cuda.ExternalStream(w.stream)
    res = {"rank": rank, "world": world, "n": n, "variant": os.environ.get("TD_XCHG_VARIANT", "0")}
    for name, flags in (("p2p", _capi.TD_P2P), ("nccl", 0)):
        for _ in range(10):
            w.tree_decode_async(q.data_ptr(), n_q, out.data_ptr(), 1.0, flags)
        torch.cuda.synchronize()
        dist.barrier()
        # back-to-back steps, events only at the ends (host far ahead after the first few)
        steps = 200
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = torch.ones(1, device="cuda")
        dist.all_reduce(t)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        stream.wait_event(ev)
        e0.record(stream)
        for _ in range(steps):
            w.tree_decode_async(q.data_ptr(), n_q, out.data_ptr(), 1.0, flags)
        e1.record(stream)
        torch.cuda.synchronize()
        res[name + "_us_per_step"] = round(e0.elapsed_time(e1) * 1000.0 / steps, 2)
        if name == "p2p":
            stamps = []
            for _ in range(4):
                w.tree_decode_async(q.data_ptr(), n_q, out.data_ptr(), 1.0, flags | _capi.TD_DEBUG_TS)
                st = w.debug_stamps(8 + 8 * 64)
                blocks = [st[8 + 8 * i: 8 + 8 * i + 5] for i in range(64) if st[8 + 8 * i]]
                t0 = min(bl[0] for bl in blocks)
                stamps.append([round((max(bl[k] for bl in blocks) - t0) / 1000.0, 2) for k in range(5)])
            res["p2p_stage_max_us(entry,pushed,merged_row0,seen,done)"] = stamps[1:]
    print(json.dumps(res), flush=True)
    w.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
