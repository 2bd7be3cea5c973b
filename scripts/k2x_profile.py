#!/usr/bin/env python3
"""Target program for an ncu capture of the one-shot exchange combine (K2x).

A single-process worker group (td_group) of P workers over the visible GPUs
(P = 2 by default: one worker per GPU on a 2-GPU box, or two workers sharing
GPU 0), a north-star shard per worker (131,072 tokens, 32 q / 8 kv heads,
bf16), a few decode steps. ncu serialises kernels, so a worker's K2x that runs
before its peer's has pushed spins into its ~2 s timeout; the LAST K2x of a
step finds every peer's words already delivered and is the one to capture:

  ncu --set full -k regex:k2_exchange --launch-skip 1 --launch-count 1 \\
      python scripts/k2x_profile.py

(with P = 2, launch index 1 is worker 1's K2x of the first step). Exit code 0
even when an earlier K2x reported the timeout (expected under ncu)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2408_04093_b200 as td
    p = int(os.environ.get("P", 2))
    n = int(os.environ.get("N", 131072)) * p
    steps = int(os.environ.get("STEPS", 1))
    ng = torch.cuda.device_count()
    g = td.WorkerGroup(p, list(range(min(ng, p))))
    for w in g.workers:
        w.generate_kv(td.DType.Bf16, 1, 8, n, 128, 2, 3)
    g.enable_p2p(32, 128)
    q = td.seeded_tensor([1, 32, 128], 1, 1.0, td.DType.Bf16)
    out = torch.empty(1, 32, 128, device="cuda")
    torch.cuda.synchronize()
    for _ in range(steps):
        g.tree_decode_async(q.data_ptr(), 32, out.data_ptr())
    for w in g.workers:
        w._sync_worker()
    print("k2x_profile: workers", p, "gpus", min(ng, p), "timeouts", [w.p2p_status() for w in g.workers])
    g.close()


if __name__ == "__main__":
    main()
