"""Small append loop on one GPU (debug aid for td_kv_append)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04093_b200 as td  # noqa: E402

b, n_kv, n_q, d, n, steps = 2, 2, 8, 128, int(os.environ.get("N0", 1500)), int(os.environ.get("STEPS", 40))
w = td.Worker(0)
k = torch.randn(b, n_kv, n + steps, d).to(torch.bfloat16)
v = torch.randn(b, n_kv, n + steps, d).to(torch.bfloat16)
q = torch.randn(b, n_q, d).to(torch.bfloat16).cuda()
w.place_kv(k[:, :, :n].contiguous().cuda(), v[:, :, :n].contiguous().cuda())
print("placed", flush=True)
for s in range(steps):
    w.append_kv(k[:, :, n + s:n + s + 1].contiguous(), v[:, :, n + s:n + s + 1].contiguous())
    print("appended", s, w.kv_info(), flush=True)
    out = w.tree_decode(q)
    torch.cuda.synchronize()
    print("decoded", s, float(out.abs().max()), flush=True)
w.close()
print("ok")
