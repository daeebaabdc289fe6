"""Stall-reason breakdown of the instructions of one function (or phase) in an
ncu SASS dump, attributed like tools/ncu_sass_funcs.py.

usage: ncu_func_stalls.py <sass.csv> <nvdisasm_inline.txt> <kernel mangled name> <function substring>
"""
import collections
import csv
import subprocess
import sys
from pathlib import Path

sys.argv, argv = sys.argv[:4] + ["100000"], sys.argv
# reuse the attribution of ncu_sass_funcs.py (locs list) by importing its module body
src = (Path(__file__).parent / "ncu_sass_funcs.py").read_text()
cut = src.index("agg_i, agg_s")
ns = {"__name__": "x", "__file__": str(Path(__file__).parent / "ncu_sass_funcs.py")}
exec(compile(src[:cut], "ncu_sass_funcs", "exec"), ns)
data, locs = ns["data"], ns["locs"]
want = argv[4]
agg = collections.Counter()
for k, d in enumerate(data):
    key = locs[k] if k < len(locs) else None
    if not key or want not in key:
        continue
    for c, v in d.items():
        if c.startswith("stall_") and "Not Issued" not in c:
            try:
                agg[c] += float(v or 0)
            except ValueError:
                pass
tot = sum(agg.values()) or 1
for c, v in agg.most_common(12):
    print(f"{100 * v / tot:5.1f}%  {c}")
