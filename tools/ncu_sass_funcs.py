"""Per-function / per-phase breakdown of an ncu SASS dump (--page source
--print-source sass --csv) using `nvdisasm --print-line-info-inline` of the same
cubin: every instruction is charged to the OUTERMOST frame of its inline chain
(the line in the enclosing non-inlined function), and that line to the
enclosing function by line ranges; lines of the phase driver (assemble_module /
disasm_one / validate_one) are further split by their `// -- X:` phase markers.

usage: ncu_sass_funcs.py <sass.csv> <nvdisasm_inline.txt> <kernel mangled name> [N] [opcode prefix, e.g. LDL]
"""
import collections
import csv
import re
import sys
from pathlib import Path

sass_csv, lines_txt, kname = sys.argv[1:4]
topn = int(sys.argv[4]) if len(sys.argv) > 4 else 40
op_prefix = sys.argv[5] if len(sys.argv) > 5 else ""
CSRC = Path(__file__).resolve().parents[1] / "paper_2305_09493_b200" / "csrc"
DRIVERS = {"assemble_module", "disasm_one", "validate_one"}

FUNC = re.compile(r"^(?:template\s*<[^>]*>\s*)?(?:SKG_HD\s+|__device__\s+|__global__\s+|__host__\s+|static\s+|inline\s+|"
                  r"__forceinline__\s+|__noinline__\s+|const\s+)+[\w:<>,\s\*&]+?\b(\w+)\s*\(")
PHASE = re.compile(r"^\s*// -- ([A-Z0-9]+):")
ranges, phases = {}, {}
for f in CSRC.glob("*.cu*"):
    starts, ph = [], []
    for i, line in enumerate(f.read_text().splitlines(), 1):
        m = FUNC.match(line)
        if m:
            starts.append((i, m.group(1)))
        p = PHASE.match(line)
        if p:
            ph.append((i, p.group(1)))
    ranges[f.name], phases[f.name] = starts, ph


def where(fname, ln):
    fn = "?"
    for s, name in ranges.get(fname, []):
        if s <= ln:
            fn = name
        else:
            break
    if fn in DRIVERS:
        tag = "pre"
        for s, name in phases.get(fname, []):
            if s <= ln:
                tag = name
            else:
                break
        fn = f"{fn}[{tag}]"
    return f"{fname}:{fn}"


locs, inside, loc = [], False, None
LOC = re.compile(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?')
for line in open(lines_txt):
    s = line.strip()
    if s.startswith(".text.") and s.endswith(":"):
        inside = s[6:-1] == kname
        continue
    if not inside:
        continue
    m = LOC.search(line)
    if m:
        # the last "inlined at" of the chain is the outermost frame
        chain = re.findall(r'inlined at "([^"]+)", line (\d+)', line)
        f, ln = (chain[-1] if chain else (m.group(1), m.group(2)))
        loc = where(f.split("/")[-1], int(ln))
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


agg_i, agg_s, agg_t = collections.Counter(), collections.Counter(), collections.Counter()
for k, d in enumerate(data):
    key = locs[k] if k < len(locs) else None
    if op_prefix:
        words = [w for w in d["Source"].split() if not w.startswith("@")]
        if not words or not words[0].startswith(op_prefix):
            continue
    agg_i[key] += num(d, "Instructions Executed")
    agg_s[key] += num(d, "Warp Stall Sampling (All Samples)")
    agg_t[key] += num(d, "Thread Instructions Executed")
ti, ts = sum(agg_i.values()) or 1, sum(agg_s.values()) or 1
for key in sorted(agg_s, key=lambda k: -agg_s[k])[:topn]:
    print(f"{100 * agg_s[key] / ts:5.1f}% stall {100 * agg_i[key] / ti:5.1f}% inst {agg_i[key] / 1e6:8.1f}M "
          f"{agg_t[key] / max(agg_i[key], 1):5.1f} lanes  {key}")
