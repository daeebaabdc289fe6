"""Summarise an `ncu --page source --csv --print-source cuda,sass` dump: top source lines."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur, hdr, out = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit():
        d = dict(zip(hdr, r))
        def num(k):
            v = d.get(k, "0")
            return int(v) if v.isdigit() else 0
        out.append((num("Warp Stall Sampling (All Samples)"), num("Instructions Executed"),
                    cur.split("/")[-1], int(r[0]), r[1][:90]))
tot_s = sum(o[0] for o in out) or 1
tot_i = sum(o[1] for o in out) or 1
print(f"total samples {tot_s}, instructions {tot_i}")
for s, i, f, ln, src in sorted(out, reverse=True)[:n]:
    print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% ins  {f}:{ln}  {src.strip()}")
