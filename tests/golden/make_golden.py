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
  bench_io.json      `treedec report` file compatibility: inputs (reference
                     sweeps, measured GPU sweeps, hand-made edge and malformed
                     files) with the reference bench.cpp's re-emitted CSV/JSON,
                     report text and exit status (oracle/_ref/ref_bench_tool).
  energy_cases.json  energy_forward_parallel / energy_grad_parallel
                     (energy.cpp:152-259) outputs of the reference, with and
                     without a source, every dtype and several chunk counts.
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


def energy_cases(ref: Reference, orc: Oracle):
    """Inputs q, k, v from seeds mix64(seed, 1..3); source from mix64(seed, 4)
    at scale 0.5; shapes [b, h, nq, d] / [b, h, n, d]."""
    cases = []
    for seed, b, h, nq, n, d, chunks in [(31, 1, 2, 3, 17, 4, [1, 2, 5, 17]),
                                          (32, 2, 1, 1, 64, 8, [1, 3, 8]),
                                          (33, 1, 3, 2, 40, 16, [1, 4, 7])]:
        for dt_name, dt in (("f64", F64), ("f32", F32), ("bf16", BF16)):
            q = orc.seeded(orc.mix64(seed, 1), b * h * nq * d, dt).reshape(b, h, nq, d)
            k = orc.seeded(orc.mix64(seed, 2), b * h * n * d, dt).reshape(b, h, n, d)
            v = orc.seeded(orc.mix64(seed, 3), b * h * n * d, dt).reshape(b, h, n, d)
            src = orc.seeded(orc.mix64(seed, 4), b * h * nq * d, dt, scale=0.5).reshape(b, h, nq, d)
            for c in chunks:
                entry = {"seed": seed, "b": b, "h": h, "nq": nq, "n": n, "d": d, "chunks": c, "dtype": dt_name}
                for tag, s_ in (("zero", None), ("source", src)):
                    val, rm, sh = ref.energy_forward_parallel(q, k, v, s_, c, dt)
                    entry[tag] = {"value": hexarr(val), "row_max": hexarr(rm), "shifted": hexarr(sh)}
                val, rm, sh = ref.energy_forward_parallel(q, k, v, None, c, dt)
                entry["grad"] = hexarr(ref.energy_grad_parallel(q, k, v, val, rm, sh, c, dt))
                cases.append(entry)
    return cases


BENCH_TOOL = os.path.join(os.path.dirname(os.path.dirname(HERE)), "oracle", "_ref", "ref_bench_tool")
_HDR = "algo,N,p,nodes,sim_time_s,elems_intra,elems_inter,peak_elems,rounds,max_abs_err"


def _tool(*args) -> tuple[int, str]:
    import subprocess
    r = subprocess.run([BENCH_TOOL, *args], capture_output=True, text=True)
    return r.returncode, r.stdout


def bench_io_cases() -> list[dict]:
    import tempfile
    inputs = []
    for fmt in ("csv", "json"):
        for name, spec in (("f64_small", ("11", "f64", "2", "4", "64,128", "1x1,1x8,2x4")),
                           ("bf16_mixed", ("5", "bf16", "4", "8", "96,200", "1x2,2x2,1x16"))):
            rc, text = _tool("sweep", fmt, *spec)
            assert rc == 0
            inputs.append((f"ref_sweep_{name}.{fmt}", text))
    root = os.path.dirname(os.path.dirname(HERE))
    for fn in ("r1_sweep_p4_nccl.csv", "r1_sweep_p4_p2p.csv"):
        path = os.path.join(root, "profiles", fn)
        if os.path.exists(path):
            inputs.append((f"measured_{fn}", open(path).read()))
    edge_rows = "\n".join([
        "tree,64,2,1,0.5,10,0,100,3,0", "ring,64,2,1,0.25,40,0,160,1,0",        # tree slower
        "tree,128,4,1,0,0,0,0,0,0", "ring,128,4,1,0,0,0,0,0,0",                 # 0/0 cells
        "tree,256,8,2,1e-300,1e20,1e-7,9223372036854775807,7,nan",             # unpaired, extremes
        "ring,512,8,1, 2.5e-6,+3,-0,42,1,inf", "tree,512,8,1,0x1p-3,.5,5.,1,1,-inf",
        "tree,1024,8,1,1.7976931348623157e308,123456789012345678,1e15,5,2,4.9e-300",
        "ring,1024,8,1,1e16,0.1,1234567890123456,-1,2,2.2250738585072014e-308",
        "tree,2048,3,1,3,3,3,3,3,3", "tree,2048,3,1,1,1,1,1,1,1", "ring,2048,3,1,2,2,2,2,2,2",  # duplicate: last wins
    ])
    inputs += [
        ("edge_rows.csv", "# note=edge cases\n#novalue\n#  spaced = x=y\n" + _HDR + "\n" + edge_rows + "\n"),
        ("crlf.csv", "# a=1\r\n" + _HDR + "\r\n\r\ntree,8,2,1,1,2,0,3,1,0\r\nring,8,2,1,2,4,0,5,1,0\r\n"),
        ("no_trailing_newline.csv", _HDR + "\ntree,8,2,1,1,2,0,3,1,0"),
        ("header_only.csv", _HDR + "\n"),
        ("empty.csv", ""),
        ("underflow.csv", _HDR + "\ntree,64,2,1,0,0,0,0,0,5e-324\n"),
        ("underflow_zero.csv", _HDR + "\ntree,64,2,1,0,1e-400,0,0,0,0\n"),
        ("u64_peak.csv", _HDR + "\ntree,64,2,1,0,0,0,18446744073709551615,0,0\n"),
        ("comments_only.csv", "# a=1\n# b=2\n"),
        ("missing_header.csv", "tree,64,2,1,0,0,0,0,0,0\n"),
        ("short_row.csv", _HDR + "\ntree,64,2\n"),
        ("bad_int.csv", _HDR + "\ntree,64,2,1,0,0,0,0,0,0\nring,sixty,2,1,0,0,0,0,0,0\n"),
        ("trailing_chars.csv", _HDR + "\ntree,64,2,1,0.5x,0,0,0,0,0\n"),
        ("bad_algo.csv", _HDR + "\nstar,64,2,1,0,0,0,0,0,0\n"),
        ("int_overflow.csv", _HDR + "\ntree,99999999999999999999,2,1,0,0,0,0,0,0\n"),
        ("double_overflow.csv", _HDR + "\ntree,64,2,1,1e999,0,0,0,0,0\n"),
        ("space_int.csv", _HDR + "\ntree, 64,2,1,0,0,0,0,0,0\n"),
        ("wrong_header.csv", "algo,N,p\n"),
        ("bare_array.json", '[{"algo":"tree","N":64,"p":2,"nodes":1,"sim_time_s":0.5,\n"elems_intra":1.0,'
                            '"elems_inter":2.0,"peak_elems":10,"rounds":3,"max_abs_err":0.0}]'),
        ("json_int_fields_as_float.json", '{"meta":{"x":"y"},"records":[{"algo":"ring","N":64.0,"p":2,"nodes":1,'
                                          '"sim_time_s":1,"elems_intra":3,"elems_inter":0,"peak_elems":7,'
                                          '"rounds":1,"max_abs_err":0}]}'),
        ("json_truncated.json", '{"records": [{"algo": "tree"'),
        ("json_missing_key.json", '{"records": [{"algo": "tree", "N": 1}]}'),
        ("json_no_records.json", '{"meta": {}}'),
        ("json_multiline_error.json", '{\n  "records": [\n    {"algo": "tree",\n     "N": 12,,\n  ]\n}'),
        ("leading_blank.json", '\n\n  [ ]'),
    ]
    cases = []
    with tempfile.TemporaryDirectory() as tmp:
        for name, text in inputs:
            path = os.path.join(tmp, name)
            with open(path, "w", newline="") as f:
                f.write(text)
            c = {"name": name, "input": text}
            for key, args in (("report", ("report", path)), ("csv", ("reemit", "csv", path)),
                              ("json", ("reemit", "json", path))):
                rc, out = _tool(*args)
                c[key] = {"rc": rc, "stdout": out.replace(path, "FILE")}
            cases.append(c)
    return cases


def main():
    build(ref=True)
    if os.path.exists(BENCH_TOOL):
        with open(os.path.join(HERE, "bench_io.json"), "w") as f:
            json.dump({"source": "reference bench.cpp (write_csv / write_json / parse_bench_file / "
                                 "write_report) via oracle/_ref/ref_bench_tool", "cases": bench_io_cases()},
                      f, indent=1)
    ref, orc = Reference(), Oracle()
    with open(os.path.join(HERE, "rng_vectors.json"), "w") as f:
        json.dump({"source": "reference seeded_random_tensor via oracle/_ref; triples from "
                             "proj/tests/data/rng_vectors.csv", "vectors": rng_vectors(ref)}, f, indent=0)
    with open(os.path.join(HERE, "energy_cases.json"), "w") as f:
        json.dump({"source": "reference energy_forward_parallel / energy_grad_parallel via oracle/_ref",
                   "cases": energy_cases(ref, orc)}, f, separators=(",", ":"))
    with open(os.path.join(HERE, "decode_cases.json"), "w") as f:
        json.dump({"source": "reference tree_decode / ring_decode via oracle/_ref; inputs "
                             "q,k,v = seeded_random_tensor(shape, mix64(seed, 1|2|3), 1.0, dtype)",
                   "cases": decode_cases(ref, orc)}, f, separators=(",", ":"))
    print("wrote", HERE)


if __name__ == "__main__":
    main()
