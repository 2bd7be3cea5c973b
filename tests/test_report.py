"""`treedec report` compatibility: the host-side
mirror of the reference's bench record I/O (paper_2408_04093_b200/report.py)
against golden outputs of the reference's own bench.cpp
(tests/golden/bench_io.json, tests/golden/make_golden.py), plus the
reference's test_bench.cpp properties."""
import io
import json
import os
import subprocess

import pytest

from paper_2408_04093_b200 import report as rp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CASES = json.load(open(os.path.join(HERE, "golden", "bench_io.json")))["cases"]
TOOL = os.path.join(ROOT, "oracle", "_ref", "ref_bench_tool")


def _run(case, what):
    text = case["input"]
    stripped = text.lstrip(" \n\t\r")
    as_json = stripped[:1] in ("{", "[")
    try:
        out = rp.parse_bench_stream(stripped if as_json else text, as_json)
    except rp.ParseError as e:
        return 2, f"FILE:{e.line}: {e.message}\n"
    buf = io.StringIO()
    {"report": rp.write_report, "csv": rp.write_csv, "json": rp.write_json}[what](out, buf)
    return 0, buf.getvalue()


@pytest.mark.parametrize("what", ["report", "csv", "json"])
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_matches_reference_bench_io(case, what):
    rc, got = _run(case, what)
    want = case[what]
    assert rc == want["rc"], (got, want["stdout"])
    if rc == 0:
        assert got == want["stdout"]
    elif "json.exception" in want["stdout"]:
        # nlohmann's exception text is its own; the line number must agree
        assert got.split(":")[1] == want["stdout"].split(":")[1]
        if "bad record" in want["stdout"]:
            assert "bad record" in got
    else:
        assert got == want["stdout"]


def _sample():
    case = next(c for c in CASES if c["name"] == "ref_sweep_f64_small.csv")
    return rp.parse_bench_stream(case["input"], False)


def test_csv_parse_emit_parse_fixpoint():  # test_bench.cpp:57-71
    out = _sample()
    first = rp.to_text(rp.write_csv, out)
    parsed = rp.parse_bench_stream(first, False)
    assert parsed.records == out.records and parsed.meta == out.meta
    assert rp.to_text(rp.write_csv, parsed) == first


def test_json_round_trip():  # test_bench.cpp:73-90
    out = _sample()
    js = rp.to_text(rp.write_json, out)
    parsed = rp.parse_bench_stream(js, True)
    assert parsed.records == out.records and parsed.meta == out.meta


def test_malformed_line_numbers():  # test_bench.cpp:92-118
    with pytest.raises(rp.ParseError):
        rp.parse_bench_stream("tree,64,2,1,0,0,0,0,0,0\n", False)
    with pytest.raises(rp.ParseError) as e:
        rp.parse_bench_stream(rp.CSV_HEADER + "\ntree,64,2\n", False)
    assert e.value.line == 2
    with pytest.raises(rp.ParseError) as e:
        rp.parse_bench_stream(rp.CSV_HEADER + "\ntree,64,2,1,0,0,0,0,0,0\nring,sixty,2,1,0,0,0,0,0,0\n", False)
    assert e.value.line == 3


def test_report_flags_and_counts():
    out = rp.SweepOutcome(records=[
        rp.BenchRecord("tree", 64, 8, 1, 2.0, 10, 0, 100, 3, 0.0),
        rp.BenchRecord("ring", 64, 8, 1, 1.0, 70, 0, 170, 7, 0.0)])
    buf = io.StringIO()
    assert rp.write_report(out, buf) == 1
    assert "tree slower" in buf.getvalue()


def test_measured_sweep_files_are_reference_readable():
    """The measured GPU sweeps committed under profiles/ parse with this
    module (and, where built, with the reference's own parser)."""
    paths = [os.path.join(ROOT, "profiles", f) for f in sorted(os.listdir(os.path.join(ROOT, "profiles")))
             if f.startswith("r1_sweep") and f.endswith(".csv")]
    assert paths
    for p in paths:
        out = rp.parse_bench_file(p)
        assert out.records and {r.algo for r in out.records} <= {"tree", "ring"}
        if os.path.exists(TOOL):
            r = subprocess.run([TOOL, "report", p], capture_output=True, text=True)
            assert r.returncode == 0
            assert r.stdout == rp.to_text(rp.write_report, out)
