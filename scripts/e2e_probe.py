#!/usr/bin/env python3
"""Where does the end-to-end (host q in, host out) decode call spend its time?

One GPU, one shard (N tokens, Llama-3-8B heads). Per mode, 40 calls, each
bracketed by host perf_counter and by CUDA events on the library stream
recorded right before and after the call (the GPU span: from the moment the
idle stream reaches the call to the end of its last kernel):

  device  device q / out, async call + stream synchronize
  host    TD_HOST_IO (q copied H2D, output stored into pinned host memory, stream sync)
  pinned  TD_HOST_IO | TD_PINNED_IO (K1 stages q from host, K2 signals through host memory)

Prints one JSON line per mode: host wall per call, GPU span, K1 event time."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2408_04093_b200 as td
    from paper_2408_04093_b200 import _capi
    n = int(os.environ.get("N", 131072))
    K = 40
    w = td.Worker(0)
    w.generate_kv(td.DType.Bf16, 1, 8, n, 128, 2, 3)
    q = td.seeded_tensor([1, 32, 128], 1, 1.0, td.DType.Bf16)
    out = torch.empty(1, 32, 128, device="cuda")
    qh = q.cpu().pin_memory()
    oh = torch.empty(1, 32, 128).pin_memory()
    stream = torch.cuda.ExternalStream(w.stream)
    modes = {
        "device": (q.data_ptr(), out.data_ptr(), 0, True),
        "host": (qh.data_ptr(), oh.data_ptr(), _capi.TD_HOST_IO, False),
        "pinned": (qh.data_ptr(), oh.data_ptr(), _capi.TD_HOST_IO | _capi.TD_PINNED_IO, False),
    }
    for _ in range(5):
        w.tree_decode_async(q.data_ptr(), 32, out.data_ptr())
    torch.cuda.synchronize()
    for name, (qp, op, flags, sync) in modes.items():
        for timed in (False, True):
            walls, spans = [], []
            w.reset_kernel_timer()
            for i in range(K):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                t0 = time.perf_counter()
                w.tree_decode_async(qp, 32, op, 1.0, flags | (_capi.TD_TIME_KERNELS if timed else 0))
                if sync:
                    stream.synchronize()
                t1 = time.perf_counter()
                e1.record(stream)
                stream.synchronize()
                walls.append((t1 - t0) * 1e6)
                spans.append(e0.elapsed_time(e1) * 1000)
            walls.sort()
            spans.sort()
            rec = {"mode": name, "k1_event_timed": timed, "n": n, "wall_us_median": round(walls[K // 2], 2),
                   "wall_us_min": round(walls[0], 2), "gpu_span_us_median": round(spans[K // 2], 2)}
            if timed:
                rec["k1_us"] = round(w.kernel_time()[0] * 1000, 2)
            print(json.dumps(rec), flush=True)
    # back-to-back async (the bench's device value)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(K):
        w.tree_decode_async(q.data_ptr(), 32, out.data_ptr())
    b.record(stream)
    torch.cuda.synchronize()
    print(json.dumps({"mode": "back_to_back", "us_per_step": round(a.elapsed_time(b) * 1000 / K, 2)}))
    assert torch.allclose(oh, out.cpu(), rtol=0, atol=1e-5 * float(out.abs().max()))
    w.close()


if __name__ == "__main__":
    main()
