"""Full-size oracle runs for the parity checks. TEST INFRASTRUCTURE ONLY
(tests/ and bench.py's parity leg -- the checker, never the product).

The oracle (oracle/treedec_oracle.c) restates the reference's decode in
IEEE double. At the benchmarked sizes (1M tokens x 32 heads, or 16 x 128K x
64 heads) a single call would need the whole cache as doubles (17 GB at
cfg3) and hours of one core, so the helpers here run it per (batch, kv-head)
row -- only that row's K/V as doubles, about 2 GB at 1M tokens -- and spread
both the generator and the partials over host threads (ctypes releases the
GIL):

* the row's K and V come from ``Oracle.seeded`` with the element offset of
  that row (``seeded_random_tensor`` is counter-based, numerics.cpp:41-50), in
  slices, one per thread;
* the group's query rows are reduced over T contiguous token ranges with
  ``orc_chunk_partial`` (attention.cpp:146-168) and combined with
  ``orc_combine_partials`` (attention.cpp:207-241) -- the reference's
  tree_decode with T workers, in Float64 (decode.cpp:100-184; exact under any
  partition, test_decode.cpp:69-80 / attention tests :143-186).
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from oracle.oracle import F64


def host_threads() -> int:
    return max(1, min(32, os.cpu_count() or 1))


def seeded_threaded(oracle, pool, seed: int, n: int, dtype: int, offset: int, parts: int) -> np.ndarray:
    """oracle.seeded(seed, n, dtype, offset=offset) computed in `parts` slices."""
    out = np.empty(n, dtype=np.float64)
    bounds = [n * i // parts for i in range(parts + 1)]

    def fill(i):
        a, e = bounds[i], bounds[i + 1]
        if e > a:
            out[a:e] = oracle.seeded(seed, e - a, dtype, offset=offset + a)

    list(pool.map(fill, range(parts)))
    return out


def rows_partials(oracle, pool, q_rows: np.ndarray, k_row: np.ndarray, v_row: np.ndarray, scale: float,
                  parts: int) -> np.ndarray:
    """Exact attention of q_rows [g, d] against one kv row k_row / v_row [n, d]:
    T token-range partials in Float64, then combine_partials."""
    g, d = q_rows.shape
    n = k_row.shape[0]
    q = np.ascontiguousarray(q_rows.reshape(1, g, d))
    k = k_row.reshape(1, 1, n, d)
    v = v_row.reshape(1, 1, n, d)
    parts = max(1, min(parts, n))
    bounds = [n * i // parts for i in range(parts + 1)]

    def one(i):
        _, lse, out = oracle.chunk_partial(q, k, v, bounds[i], bounds[i + 1] - bounds[i], scale, F64)
        return lse, out

    res = list(pool.map(one, range(parts)))
    lse = np.stack([r[0].reshape(g) for r in res])
    out = np.stack([r[1].reshape(g, d) for r in res])
    return oracle.combine_partials(lse, out, F64).reshape(g, d)


def full_decode(oracle, q: np.ndarray, n_kv: int, n: int, seed_k: int, seed_v: int, dtype: int,
                scale: float = 1.0, rows=None, kv_source=None) -> dict:
    """Oracle output of the single-query decode q [b, n_q, d] against the
    seeded cache k, v = seeded_random_tensor([b, n_kv, n, d], seed_k / seed_v,
    1.0, dtype), for every (b, q-head) row (or only the (b, q-head) pairs in
    `rows`). kv_source(bh) -> (k_row, v_row) as float64 [n, d] replaces the
    generator (e.g. a host copy of the device cache). Returns {(b, h): [d]}."""
    b, n_q, d = q.shape
    g = n_q // n_kv
    want = {}
    if rows is None:
        rows = [(ib, h) for ib in range(b) for h in range(n_q)]
    by_bh = {}
    for ib, h in rows:
        by_bh.setdefault(ib * n_kv + h // g, []).append((ib, h))
    nt = host_threads()
    with ThreadPoolExecutor(nt) as pool:
        for bh, members in sorted(by_bh.items()):
            if kv_source is not None:
                k_row, v_row = kv_source(bh)
            else:
                k_row = seeded_threaded(oracle, pool, seed_k, n * d, dtype, bh * n * d, nt).reshape(n, d)
                v_row = seeded_threaded(oracle, pool, seed_v, n * d, dtype, bh * n * d, nt).reshape(n, d)
            heads = [h for _, h in members]
            ib = members[0][0]
            res = rows_partials(oracle, pool, q[ib, heads], k_row, v_row, scale, nt)
            for i, key in enumerate(members):
                want[key] = res[i]
            del k_row, v_row
    return want


def rel_err_rows(got: np.ndarray, want: dict) -> float:
    """max |got - want| / max |want| over the rows in want (the decode.cpp:253-260 convention)."""
    num = max(float(np.max(np.abs(got[ib, h] - w))) for (ib, h), w in want.items())
    den = max(float(np.max(np.abs(w))) for w in want.values())
    return num / max(den, 1e-300)
