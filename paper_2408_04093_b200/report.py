"""`treedec report` compatibility: the reference's bench
record files, read and written byte-for-byte like `proj/core/src/bench.cpp`, so
measured B200 records (scripts/sweep.py, sim_time_s = measured device time)
can be compared with the reference's modeled sweeps by the same report.

  write_csv / write_json      bench.cpp:118-147 (format), bench.cpp:18-19 (header)
  parse_bench_stream / _file  bench.cpp:149-285 (CSV rules, JSON object / bare array)
  write_report                bench.cpp:287-355 (tree-vs-ring table, flagged cells)

Host-side file I/O only; nothing here touches the GPU. Checked against
golden files produced by the reference's own bench.cpp
(tests/golden/bench_io/, made by tests/golden/make_golden.py).
"""
from __future__ import annotations

import io
import json
import math
import re
from dataclasses import dataclass, field

CSV_HEADER = "algo,N,p,nodes,sim_time_s,elems_intra,elems_inter,peak_elems,rounds,max_abs_err"  # bench.cpp:18-19
_U64 = (1 << 64) - 1


@dataclass
class BenchRecord:  # bench.hpp:30-43
    algo: str = ""
    seq_len: int = 0
    p: int = 0
    nodes: int = 0
    sim_time_s: float = 0.0
    elems_intra: float = 0.0
    elems_inter: float = 0.0
    peak_elems: int = 0
    rounds: int = 0
    max_abs_err: float = 0.0

    def __eq__(self, other):  # `= default` comparison: NaN != NaN, like the C++ double members
        return isinstance(other, BenchRecord) and all(
            getattr(self, f) == getattr(other, f) for f in self.__dataclass_fields__)


@dataclass
class SweepOutcome:  # bench.hpp:45-49
    records: list = field(default_factory=list)
    meta: dict = field(default_factory=dict)  # std::map: iterated in key order
    all_within_tolerance: bool = True


class ParseError(Exception):  # bench.hpp:58-61: 1-based line number + message
    def __init__(self, line: int, message: str):
        super().__init__(f"{line}: {message}")
        self.line = line
        self.message = message


def fmt_double(x: float) -> str:
    """`%.17g` (bench.cpp:21-25)."""
    return _cfmt(".17g", x)


def _sorted_items(d: dict):
    # std::map<std::string, ...> orders keys by bytes
    return sorted(d.items(), key=lambda kv: kv[0].encode())


def write_csv(out: SweepOutcome, os_: io.TextIOBase) -> None:
    """bench.cpp:118-126: '# key=value' meta lines, the header, one row per record."""
    for k, v in _sorted_items(out.meta):
        os_.write(f"# {k}={v}\n")
    os_.write(CSV_HEADER + "\n")
    for r in out.records:
        os_.write(f"{r.algo},{r.seq_len},{r.p},{r.nodes},{fmt_double(r.sim_time_s)},"
                  f"{fmt_double(r.elems_intra)},{fmt_double(r.elems_inter)},{r.peak_elems},{r.rounds},"
                  f"{fmt_double(r.max_abs_err)}\n")


def _json_double(x: float) -> str:
    """A double the way nlohmann::json dump() prints it (shortest round-trip
    digits; fixed notation for decimal exponents -3..15, else d.ddde+XX;
    integral values keep '.0'; NaN / inf become null)."""
    if not math.isfinite(x):
        return "null"
    if x == 0.0:
        return "-0.0" if math.copysign(1.0, x) < 0 else "0.0"
    sign = "-" if x < 0 else ""
    digits, exp = _shortest_digits(abs(x))
    n = len(digits) + exp  # position of the decimal point
    k = len(digits)
    if k <= n <= 15:
        return sign + digits + "0" * (n - k) + ".0"
    if 0 < n <= 15:
        return sign + digits[:n] + "." + digits[n:]
    if -4 < n <= 0:
        return sign + "0." + "0" * (-n) + digits
    e = n - 1
    mant = digits[0] + ("." + digits[1:] if k > 1 else "")
    es = "-" if e < 0 else "+"
    return f"{sign}{mant}e{es}{abs(e):02d}"


def _shortest_digits(x: float):
    """(digits, exponent) with x == int(digits) * 10**exponent, shortest round trip."""
    s = repr(x)
    mant, _, e = s.partition("e")
    exp = int(e) if e else 0
    if "." in mant:
        ip, fp = mant.split(".")
    else:
        ip, fp = mant, ""
    if fp == "0":
        fp = ""
    digits = (ip + fp).lstrip("0")
    exp -= len(fp)
    stripped = digits.rstrip("0")
    exp += len(digits) - len(stripped)
    return stripped or "0", exp


def _json_str(s: str) -> str:
    return json.dumps(s, ensure_ascii=False)


def write_json(out: SweepOutcome, os_: io.TextIOBase) -> None:
    """bench.cpp:128-147: {"meta": {...}, "records": [...]}, dump(2); nlohmann
    objects are key-ordered, so the record fields come out sorted."""
    lines = ["{"]
    if out.meta:
        lines.append('  "meta": {')
        items = _sorted_items(out.meta)
        for i, (k, v) in enumerate(items):
            lines.append(f"    {_json_str(k)}: {_json_str(v)}" + ("," if i + 1 < len(items) else ""))
        lines.append("  },")
    else:
        lines.append('  "meta": {},')
    if out.records:
        lines.append('  "records": [')
        for i, r in enumerate(out.records):
            fields = {"N": str(r.seq_len), "algo": _json_str(r.algo), "elems_inter": _json_double(r.elems_inter),
                      "elems_intra": _json_double(r.elems_intra), "max_abs_err": _json_double(r.max_abs_err),
                      "nodes": str(r.nodes), "p": str(r.p), "peak_elems": str(r.peak_elems),
                      "rounds": str(r.rounds), "sim_time_s": _json_double(r.sim_time_s)}
            lines.append("    {")
            keys = sorted(fields)
            for j, k in enumerate(keys):
                lines.append(f'      "{k}": {fields[k]}' + ("," if j + 1 < len(keys) else ""))
            lines.append("    }" + ("," if i + 1 < len(out.records) else ""))
        lines.append("  ]")
    else:
        lines.append('  "records": []')
    lines.append("}")
    os_.write("\n".join(lines) + "\n")


# -------------------------------------------------------------- parsing
# std::stod / std::stoll accept leading whitespace and a sign; the whole field
# must be consumed (bench.cpp:165-191)
_DEC = r"[ \t\n\v\f\r]*[+-]?(?:0[xX](?:[0-9a-fA-F]+\.?[0-9a-fA-F]*|\.[0-9a-fA-F]+)(?:[pP][+-]?\d+)?|(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|inf(?:inity)?|nan(?:\([0-9A-Za-z_]*\))?)"
_FLOAT_RE = re.compile(_DEC, re.IGNORECASE)
_INT_RE = re.compile(r"[ \t\n\v\f\r]*[+-]?\d+")


def _to_double(s: str, line: int, what: str) -> float:
    m = _FLOAT_RE.match(s)
    if not m:
        raise ParseError(line, f"bad number for {what}")
    tok = m.group(0).strip()
    if m.end() != len(s):
        raise ParseError(line, f"trailing characters in {what}")
    low = tok.lower().lstrip("+-")
    neg = tok.startswith("-")
    if low.startswith("0x"):
        v = float.fromhex(tok)
    elif low.startswith("nan"):
        v = float("nan")
    elif low.startswith("inf"):
        v = -math.inf if neg else math.inf
    else:
        v = float(tok)
        # std::stod throws out_of_range when strtod reports ERANGE: overflow,
        # or a nonzero literal that underflows to a subnormal / zero
        tiny = abs(v) < 2.2250738585072014e-308 and any(ch in "123456789" for ch in tok.split("e")[0].split("E")[0])
        if math.isinf(v) or tiny:
            raise ParseError(line, f"bad number for {what}")
    return v


def _to_i64(s: str, line: int, what: str) -> int:
    m = _INT_RE.match(s)
    if not m:
        raise ParseError(line, f"bad integer for {what}")
    if m.end() != len(s):
        raise ParseError(line, f"trailing characters in {what}")
    v = int(m.group(0).strip())
    if not -(1 << 63) <= v < (1 << 63):
        raise ParseError(line, f"bad integer for {what}")
    return v


def _to_int32(v: int) -> int:  # static_cast<int>
    v &= 0xFFFFFFFF
    return v - (1 << 32) if v >= (1 << 31) else v


def _parse_csv(text: str) -> SweepOutcome:
    out = SweepOutcome()
    header_seen = False
    lineno = 0
    for line in text.split("\n") if text else []:
        lineno += 1
        if line.endswith("\r"):
            line = line[:-1]
        if not line:
            continue
        if line[0] == "#":
            body = line[1:]
            if body.startswith(" "):
                body = body[1:]
            eq = body.find("=")
            if eq >= 0:
                out.meta[body[:eq]] = body[eq + 1:]
            continue
        if not header_seen:
            if line != CSV_HEADER:
                raise ParseError(lineno, "unexpected CSV header")
            header_seen = True
            continue
        f = line.split(",")
        if len(f) != 10:
            raise ParseError(lineno, "expected 10 fields")
        if f[0] not in ("tree", "ring"):
            raise ParseError(lineno, f"unknown algo '{f[0]}'")
        out.records.append(BenchRecord(
            algo=f[0], seq_len=_to_i64(f[1], lineno, "N"), p=_to_int32(_to_i64(f[2], lineno, "p")),
            nodes=_to_int32(_to_i64(f[3], lineno, "nodes")), sim_time_s=_to_double(f[4], lineno, "sim_time_s"),
            elems_intra=_to_double(f[5], lineno, "elems_intra"), elems_inter=_to_double(f[6], lineno, "elems_inter"),
            peak_elems=_to_i64(f[7], lineno, "peak_elems") & _U64, rounds=_to_i64(f[8], lineno, "rounds") & _U64,
            max_abs_err=_to_double(f[9], lineno, "max_abs_err")))
    if text.endswith("\n"):
        lineno -= 1  # std::getline does not see a line after the final newline
    if not header_seen:
        raise ParseError(1 if lineno == 0 else lineno, "missing CSV header")
    return out


def _num(v, kind):
    if isinstance(v, bool) or not isinstance(v, (int, float)):
        if isinstance(v, bool):
            return int(v) if kind is int else float(v)
        raise TypeError(f"type must be number, but is {type(v).__name__}")
    if kind is int:
        return int(v)
    return float(v)


def _reject_constant(name):  # nlohmann rejects NaN / Infinity literals
    raise json.JSONDecodeError(f"invalid literal {name}", "", 0)


def _parse_json(text: str) -> SweepOutcome:
    try:
        doc = json.loads(text, parse_constant=_reject_constant)
    except json.JSONDecodeError as e:
        raise ParseError(e.lineno, e.msg) from None
    out = SweepOutcome()
    if isinstance(doc, list):
        records = doc
    elif isinstance(doc, dict) and "records" in doc:
        for k, v in (doc.get("meta") or {}).items():
            if not isinstance(v, str):
                raise TypeError(f"type must be string, but is {type(v).__name__}")
            out.meta[k] = v
        records = doc["records"]
    else:
        raise ParseError(1, "expected an array of records or an object with a 'records' field")
    try:
        for jr in records:
            algo = jr["algo"]
            if not isinstance(algo, str):
                raise TypeError("type must be string")
            out.records.append(BenchRecord(
                algo=algo, seq_len=_num(jr["N"], int), p=_to_int32(_num(jr["p"], int)),
                nodes=_to_int32(_num(jr["nodes"], int)), sim_time_s=_num(jr["sim_time_s"], float),
                elems_intra=_num(jr["elems_intra"], float), elems_inter=_num(jr["elems_inter"], float),
                peak_elems=_num(jr["peak_elems"], int) & _U64, rounds=_num(jr["rounds"], int) & _U64,
                max_abs_err=_num(jr["max_abs_err"], float)))
    except (KeyError, TypeError) as e:
        raise ParseError(1, f"bad record: {e}") from None
    return out


def parse_bench_stream(is_: io.TextIOBase | str, as_json: bool) -> SweepOutcome:
    """bench.cpp:269-271."""
    text = is_ if isinstance(is_, str) else is_.read()
    return _parse_json(text) if as_json else _parse_csv(text)


def parse_bench_file(path: str) -> SweepOutcome:
    """bench.cpp:273-285: JSON when the first non-blank byte is '{' or '['."""
    with open(path, newline="") as f:
        text = f.read()
    stripped = text.lstrip(" \n\t\r")
    as_json = stripped[:1] in ("{", "[")
    return parse_bench_stream(stripped if as_json else text, as_json)


def _div(a: float, b: float) -> float:
    """IEEE division on x86-64: 0/0 gives the default NaN, whose sign bit is
    set (glibc prints it as -nan)."""
    if math.isnan(a) or math.isnan(b):
        return a if math.isnan(a) else b
    if b == 0.0:
        if a == 0.0:
            return -math.nan
        return math.copysign(math.inf, a) * math.copysign(1.0, b)
    return a / b


def _cfmt(spec: str, x: float) -> str:
    """printf float conversion with glibc's NaN spelling (sign kept)."""
    if math.isnan(x):
        w = int(spec.split(".")[0] or 0)
        return (("-" if math.copysign(1.0, x) < 0 else "") + "nan").rjust(w)
    return ("%" + spec) % x


def write_report(out: SweepOutcome, os_: io.TextIOBase) -> int:
    """bench.cpp:287-355: pair tree / ring records per (N, p, nodes) cell in
    first-seen order; speedup = ring / tree time, volume and peak-memory
    ratios; returns the number of cells where tree is slower."""
    order, cells = [], {}
    for r in out.records:
        key = (r.seq_len, r.p, r.nodes)
        if key not in cells:
            order.append(key)
            cells[key] = [None, None]
        cells[key][0 if r.algo == "tree" else 1] = r
    os_.write("modeled tree-vs-ring comparison (sim_time is modeled, not measured)\n")
    os_.write("%10s %6s %6s %12s %14s %12s  %s\n" % ("N", "p", "nodes", "speedup", "volume_ratio", "mem_ratio",
                                                     "note"))
    flagged = 0
    for key in order:
        t, g = cells[key]
        if t is None or g is None:
            os_.write("%10d %6d %6d %12s %14s %12s  %s\n" % (key[0], key[1], key[2], "-", "-", "-", "unpaired cell"))
            continue
        speedup = 1.0 if (t.sim_time_s == 0.0 and g.sim_time_s == 0.0) else _div(g.sim_time_s, t.sim_time_s)
        tv, gv = t.elems_intra + t.elems_inter, g.elems_intra + g.elems_inter
        vol = 1.0 if (tv == 0.0 and gv == 0.0) else _div(gv, tv)
        mem = _div(float(g.peak_elems), float(t.peak_elems))
        loses = speedup < 1.0
        flagged += loses
        os_.write("%10d %6d %6d %s %s %s  %s\n" % (t.seq_len, t.p, t.nodes, _cfmt("12.2f", speedup),
                                                    _cfmt("14.4g", vol), _cfmt("12.4f", mem),
                                                    "tree slower" if loses else ""))
    os_.write("%d cells, %d flagged\n" % (len(order), flagged))
    return flagged


def to_text(fn, out: SweepOutcome) -> str:
    buf = io.StringIO()
    fn(out, buf)
    return buf.getvalue()


def main(argv=None) -> int:
    """`python -m paper_2408_04093_b200.report FILE`: the `treedec report`
    subcommand (tools/treedec_main.cpp:106-119, exit 2 on IO / parse errors)."""
    import sys
    args = sys.argv[1:] if argv is None else argv
    if len(args) != 1:
        print("usage: python -m paper_2408_04093_b200.report FILE", file=sys.stderr)
        return 2
    try:
        out = parse_bench_file(args[0])
    except ParseError as e:
        print(f"report: {args[0]}:{e.line}: {e.message}", file=sys.stderr)
        return 2
    except (OSError, TypeError, ValueError) as e:
        print(f"report: {e}", file=sys.stderr)
        return 2
    write_report(out, sys.stdout)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
