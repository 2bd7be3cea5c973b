"""The append-loop GPU test body with progress prints (debug aid)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2408_04093_b200 as td  # noqa: E402
from oracle.oracle import BF16, F64, HIER, Oracle  # noqa: E402
from conftest import make_inputs, rel_err  # noqa: E402

oracle = Oracle()
dtype = BF16
b, n_q, n_kv, n, d, steps = 2, 8, 2, 1500, 128, int(os.environ.get("STEPS", 1100))
q, k, v = make_inputs(oracle, 33, b, n_q, n_kv, n + steps, d, dtype)
print("inputs", flush=True)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to("cuda").to(torch.bfloat16)  # noqa: E731
w = td.Worker(0)
w.place_kv(dev(k[:, :, :n]), dev(v[:, :, :n]))
print("placed", flush=True)
for s in range(steps):
    kt = torch.from_numpy(np.ascontiguousarray(k[:, :, n + s:n + s + 1])).to(torch.bfloat16)
    vt = torch.from_numpy(np.ascontiguousarray(v[:, :, n + s:n + s + 1])).to(torch.bfloat16)
    if s % 2:
        kt, vt = kt.cuda(), vt.cuda()
    w.append_kv(kt, vt)
    if s < 4 or s % 100 == 0:
        print("appended", s, w.kv_info(), flush=True)
    if s in (0, 1, 1023, 1024, steps - 1):
        m = n + s + 1
        out = w.tree_decode(dev(q))
        torch.cuda.synchronize()
        print("tree", s, flush=True)
        want = oracle.tree_decode(q, np.ascontiguousarray(k[:, :, :m]), np.ascontiguousarray(v[:, :, :m]),
                                  1, HIER, 1.0, F64)
        print("oracle", s, rel_err(out.double().cpu().numpy(), want), flush=True)
        r = w.ring_decode(dev(q))
        torch.cuda.synchronize()
        print("ring", s, rel_err(r.double().cpu().numpy(), want), flush=True)
w.reserve_kv(5000)
print("reserved", flush=True)
out = w.tree_decode(dev(q))
print("final", rel_err(out.double().cpu().numpy(), oracle.tree_decode(q, k, v, 1, HIER, 1.0, F64)), flush=True)
w.close()
print("ok")
