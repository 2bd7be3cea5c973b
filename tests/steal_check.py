#!/usr/bin/env python3
"""Decode with cross-row stealing forced on (TD_STEAL_SLOTS, read once per
process, hence a subprocess of tests/test_gpu_parity.py) and compare every
output row with the CPU oracle (foreign states can belong to any (batch,
kv-head) row); exits non-zero on a parity failure."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import numpy as np
    import torch

    import paper_2408_04093_b200 as td
    from conftest import make_inputs, rel_err
    from oracle.oracle import BF16, F64, HIER, Oracle
    orc = Oracle()
    ok = True
    for b, n_q, n_kv, n in [(1, 32, 8, 150001), (2, 8, 4, 70001)]:
        q, k, v = make_inputs(orc, 61 + n, b, n_q, n_kv, n, 128, BF16)
        dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to("cuda").to(torch.bfloat16)  # noqa: E731
        w = td.Worker(0)
        w.place_kv(dev(k), dev(v))
        outs = [w.tree_decode(dev(q), flags=td._capi.TD_DYNAMIC) for _ in range(3)]  # the pool feeds the stealing
        want = orc.tree_decode(q, k, v, 1, HIER, 1.0, F64, nthreads=os.cpu_count() or 8)
        errs = [rel_err(o.double().cpu().numpy(), want) for o in outs]
        good = max(errs) <= 1e-3
        ok &= good
        print(json.dumps({"b": b, "n_q": n_q, "n_kv": n_kv, "n": n, "errs": errs, "ok": good}), flush=True)
        w.close()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
