#!/usr/bin/env python3
"""Regenerates the golden fixtures in tests/golden/ from the REFERENCE itself
(oracle/_ref/libtreedec_ref.so, built by `make -C oracle ref` from
/root/reference/proj/core). Run in a container that has /root/reference:

    python tests/golden/make_golden.py

Fixtures:
  rng_vectors.json   the (seed, index, scale) triples of the reference's
                     proj/tests/data/rng_vectors.csv with the bits of
                     seeded_random_tensor produced by the reference library
                     (plus bf16 / f32 rounded values).
  decode_cases.json  small tree/ring decode problems (seeded inputs, the
                     reference seeding convention of test_decode.cpp:18-23)
                     with the reference's outputs at every dtype, strategy and
                     worker count; doubles stored as 16-hex-digit bit patterns.
"""
from __future__ import annotations

import json
import os
import struct
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import BF16, F32, F64, HIER, RING, TREE_BINARY, Oracle, Reference, build  # noqa: E402

RNG_CSV = "/root/reference/proj/tests/data/rng_vectors.csv"


def hexd(x: float) -> str:
    return struct.pack("<d", float(x)).hex()


def hexarr(a) -> list[str]:
    return [hexd(x) for x in np.asarray(a, dtype=np.float64).reshape(-1)]


def rng_vectors(ref: Reference):
    triples = []
    with open(RNG_CSV) as f:
        for line in f:
            if not line.strip() or line.startswith("#"):
                continue
            seed, idx, scale = line.split(",")[:3]
            triples.append((int(seed), int(idx), float(scale)))
    out = []
    for seed, idx, scale in triples:
        vals = {name: hexd(ref.seeded(seed, idx + 1, code, scale)[idx]) for name, code in
                (("f64", F64), ("f32", F32), ("bf16", BF16))}
        out.append({"seed": seed, "index": idx, "scale": scale, **vals})
    return out


def decode_cases(ref: Reference, orc: Oracle):
    cases = []
    spec = [  # seed, b, n_h, n, d_h, ps
        (2 + 17, 1, 2, 17, 4, [1, 2, 3, 4, 8, 16]),
        (2 + 64, 1, 2, 64, 4, [1, 2, 3, 4, 8, 16]),
        (5, 1, 2, 96, 8, [8]),
        (9, 1, 2, 40, 4, [8]),
        (77, 2, 3, 33, 8, [1, 2, 5, 7]),
    ]
    for seed, b, n_h, n, d, ps in spec:
        for dt_name, dt in (("f64", F64), ("f32", F32), ("bf16", BF16)):
            q = orc.seeded(orc.mix64(seed, 1), b * n_h * d, dt).reshape(b, n_h, d)
            k = orc.seeded(orc.mix64(seed, 2), b * n_h * n * d, dt).reshape(b, n_h, n, d)
            v = orc.seeded(orc.mix64(seed, 3), b * n_h * n * d, dt).reshape(b, n_h, n, d)
            for p in ps:
                entry = {"seed": seed, "b": b, "n_h": n_h, "n": n, "d_h": d, "p": p, "dtype": dt_name,
                         "scale": 1.0, "tree": {}}
                for st_name, st in (("tree", TREE_BINARY), ("ring", RING), ("hier", HIER)):
                    entry["tree"][st_name] = hexarr(ref.tree_decode(q, k, v, p, st, 1.0, dt))
                entry["ring"] = hexarr(ref.ring_decode(q, k, v, p, 1.0, dt))
                cases.append(entry)
    return cases


def main():
    build(ref=True)
    ref, orc = Reference(), Oracle()
    with open(os.path.join(HERE, "rng_vectors.json"), "w") as f:
        json.dump({"source": "reference seeded_random_tensor via oracle/_ref; triples from "
                             "proj/tests/data/rng_vectors.csv", "vectors": rng_vectors(ref)}, f, indent=0)
    with open(os.path.join(HERE, "decode_cases.json"), "w") as f:
        json.dump({"source": "reference tree_decode / ring_decode via oracle/_ref; inputs "
                             "q,k,v = seeded_random_tensor(shape, mix64(seed, 1|2|3), 1.0, dtype)",
                   "cases": decode_cases(ref, orc)}, f, separators=(",", ":"))
    print("wrote", HERE)


if __name__ == "__main__":
    main()
