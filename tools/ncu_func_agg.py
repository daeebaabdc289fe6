"""Aggregate an `ncu --page source --csv --print-source cuda` dump by enclosing
function (line ranges of __device__/__global__ definitions in the source
files), for a per-function instruction / stall-sample breakdown.

usage: ncu_func_agg.py <source.csv[.gz]> <csrc dir> [N] [stall column, e.g. stall_long_sb]
"""
import collections
import csv
import gzip
import io
import re
import sys
from pathlib import Path

path, csrc = sys.argv[1], Path(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
col = sys.argv[4] if len(sys.argv) > 4 else "Warp Stall Sampling (All Samples)"
opener = gzip.open if path.endswith(".gz") else open
rows = list(csv.reader(io.TextIOWrapper(opener(path, "rb"), encoding="utf-8", errors="replace")))

FUNC = re.compile(r"^(?:template\s*<[^>]*>\s*)?(?:SKG_HD\s+|__device__\s+|__global__\s+|__host__\s+|static\s+|inline\s+|"
                  r"__forceinline__\s+|__noinline__\s+|SKG_NOINLINE\s+|const\s+)+[\w:<>,\s\*&]+?\b(\w+)\s*\(")
ranges = {}
for f in csrc.glob("*.cu*"):
    starts = []
    for i, line in enumerate(f.read_text().splitlines(), 1):
        m = FUNC.match(line)
        if m:
            starts.append((i, m.group(1)))
    ranges[f.name] = starts


def func_of(fname, ln):
    best = "?"
    for s, name in ranges.get(fname, []):
        if s <= ln:
            best = name
        else:
            break
    return f"{fname}:{best}"


agg = collections.defaultdict(lambda: [0, 0])
cur, hdr = None, None
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit():
        d = dict(zip(hdr, r))
        s = d.get(col, "0")
        i = d.get("Instructions Executed", "0")
        a = agg[func_of(cur, int(r[0]))]
        a[0] += int(s) if s.isdigit() else 0
        a[1] += int(i) if i.isdigit() else 0
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"{col}: samples {ts}  instructions {ti}")
for k, (s, i) in sorted(agg.items(), key=lambda x: -x[1][1])[:n]:
    print(f"{100 * i / ti:5.1f}% ins {100 * s / ts:5.1f}% smp  {k}")
