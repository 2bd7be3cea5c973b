#!/usr/bin/env python3
"""The streamed combine's failure path: with TD_DEBUG_REVERSE=4 (read once per
process, hence a subprocess of tests/test_gpu_parity.py) the split kernel never
publishes one warp's state, so the combine kernel gives up after ~1 s; the call
must fail with TD_ECUDA instead of returning a wrong result. Exits non-zero
otherwise."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2408_04093_b200 as td
    from paper_2408_04093_b200 import _capi
    w = td.Worker(0)
    w.generate_kv(td.DType.Bf16, 1, 8, 131072, 128, 2, 3)
    q = td.seeded_tensor([1, 32, 128], 1, 1.0, td.DType.Bf16)
    try:
        w.tree_decode(q.cpu())  # host buffers: the call synchronises and reports this step
    except _capi.TreeDecError as e:
        ok = e.status == _capi.TD_ECUDA and "timed out waiting" in str(e)
        print("raised:", e, flush=True)
        w.close()
        sys.exit(0 if ok else 1)
    print("no error raised", flush=True)
    torch.cuda.synchronize()
    sys.exit(1)


if __name__ == "__main__":
    main()
