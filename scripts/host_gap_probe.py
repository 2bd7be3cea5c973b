#!/usr/bin/env python3
"""Is the decode step host-bound? Times K steps three ways on one GPU:
A per-step CUDA events as bench.py does; B the same after a long device
sleep (the host runs ahead, so no host gap can land inside an event window);
C host-side cost of one async call (perf_counter, no sync)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2408_04093_b200 as td
    n = int(os.environ.get("N", 131072))
    K = 30
    w = td.Worker(0)
    w.generate_kv(td.DType.Bf16, 1, 8, n, 128, 2, 3)
    q = td.seeded_tensor([1, 32, 128], 1, 1.0, td.DType.Bf16)
    out = torch.empty(1, 32, 128, device="cuda")
    stream = torch.cuda.ExternalStream(w.stream)

    def step():
        w.tree_decode_async(q.data_ptr(), 32, out.data_ptr(), 1.0, 0)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    res = {}
    for mode in ("A", "B"):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        tot0, tot1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        if mode == "B":
            with torch.cuda.stream(stream):
                torch.cuda._sleep(50_000_000)
        tot0.record(stream)
        for i in range(K):
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        tot1.record(stream)
        torch.cuda.synchronize()
        per = [a.elapsed_time(b) * 1000 for a, b in evs]
        res[mode] = {"per_step_us": round(sum(per) / K, 2), "min_us": round(min(per), 2),
                     "total_over_K_us": round(tot0.elapsed_time(tot1) * 1000 / K, 2)}
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        torch.cuda._sleep(200_000_000)
    t0 = time.perf_counter()
    for _ in range(K):
        step()
    res["C_host_us_per_call"] = round((time.perf_counter() - t0) / K * 1e6, 2)
    torch.cuda.synchronize()
    print(json.dumps(res))
    w.close()


if __name__ == "__main__":
    main()
