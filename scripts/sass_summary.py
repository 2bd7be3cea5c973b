#!/usr/bin/env python3
"""Static SASS summary of libtreedec_b200.so (cuobjdump -sass): per kernel, the
instruction counts that show how it is built -- TMA tensor loads (UTMALDG),
bulk copies (UBLKCP), mbarrier ops (SYNCS), mma.sync (HMMA), ldmatrix (LDSM),
global / shared loads and stores, shuffles, SFU (MUFU), tcgen05 (UTC*MMA,
LDTM: none expected).

  python scripts/sass_summary.py [--so PATH] > profiles/r2_sass_summary.md
"""
import argparse
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["UTMALDG", "UBLKCP", "SYNCS", "HMMA", "LDSM", "UTCHMMA", "UTCQMMA", "LDTM", "LDG", "STG", "LDS", "STS",
        "FFMA", "MUFU", "SHFL", "BAR", "ATOMG", "RED", "ELECT"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--so", default=os.path.join(ROOT, "paper_2408_04093_b200", "libtreedec_b200.so"))
    args = ap.parse_args()
    txt = subprocess.run(["cuobjdump", "-sass", args.so], capture_output=True, text=True, check=True).stdout
    arch = sorted(set(re.findall(r"arch = (sm_\w+)", txt)))
    rows = []
    for part in re.split(r"\n\t\tFunction : ", txt)[1:]:
        name = part.split("\n", 1)[0].strip()
        ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", part)
        c = collections.Counter(ops)
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        rows.append((dem, c, sum(c.values())))
    print(f"# SASS summary of `{os.path.relpath(args.so, ROOT)}` ({', '.join(arch)})\n")
    print("Static instruction counts per kernel (`cuobjdump -sass`, `scripts/sass_summary.py`).\n")
    print("| kernel | " + " | ".join(KEYS) + " | total |")
    print("|---|" + "---|" * (len(KEYS) + 1))
    for dem, c, tot in sorted(rows):
        print(f"| `{dem}` | " + " | ".join(str(c.get(k, 0)) for k in KEYS) + f" | {tot} |")


if __name__ == "__main__":
    main()
