"""Attribute ncu per-SASS-instruction metrics (--page source --print-source sass
--csv) to CUDA source lines using nvdisasm --print-line-info of the same cubin.

usage: ncu_sass_lines.py <sass.csv> <nvdisasm_lines.txt> <kernel mangled name> [N]
"""
import collections
import csv
import re
import sys

sass_csv, lines_txt, kname = sys.argv[1:4]
topn = int(sys.argv[4]) if len(sys.argv) > 4 else 40
locs, inside, loc = [], False, None
for line in open(lines_txt):
    s = line.strip()
    if s.startswith(".text.") and s.endswith(":"):
        inside = s[6:-1] == kname
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        if "inlined at" not in line:
            loc = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.match(r"\s+/\*[0-9a-f]+\*/", line):
        locs.append(loc)
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
data.sort(key=lambda d: int(d["Address"], 16))
print(f"sass rows {len(data)} nvdisasm instructions {len(locs)}")


def num(d, k):
    try:
        return float(d.get(k, 0) or 0)
    except ValueError:
        return 0.0


agg_i, agg_s = collections.Counter(), collections.Counter()
for k, d in enumerate(data):
    key = locs[k] if k < len(locs) else None
    agg_i[key] += num(d, "Instructions Executed")
    agg_s[key] += num(d, "Warp Stall Sampling (All Samples)")
ti, ts = sum(agg_i.values()) or 1, sum(agg_s.values()) or 1
src = {}
for key in sorted(agg_s, key=lambda k: -agg_s[k])[:topn]:
    f, ln = key if key else ("?", 0)
    if f not in src:
        try:
            src[f] = open(f"/root/repo/paper_2305_09493_b200/csrc/{f}").read().split("\n")
        except OSError:
            src[f] = []
    text = src[f][ln - 1].strip()[:80] if 0 < ln <= len(src[f]) else ""
    print(f"{100 * agg_s[key] / ts:5.1f}% stall {100 * agg_i[key] / ti:5.1f}% inst  {f}:{ln}  {text}")
