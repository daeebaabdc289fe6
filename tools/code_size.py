"""Code bytes of one kernel attributed to source functions (nvdisasm --print-line-info).

usage: code_size.py <nvdisasm_lines.txt> <kernel mangled name> [N]"""
import bisect
import collections
import re
import sys

lines_txt, kname = sys.argv[1:3]
topn = int(sys.argv[3]) if len(sys.argv) > 3 else 40
inside, loc, chain = False, None, None
by = collections.Counter()
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
        by[loc] += 1


def heads(path):
    out = []
    for i, l in enumerate(open(path), 1):
        m = re.match(r"^(?:template <[^>]*>\s*)?(?:SKG_HD |__device__ |__global__ |__host__ )[^(]*?(\w+)\(", l)
        if m:
            out.append((i, m.group(1)))
    return out


cache, agg = {}, collections.Counter()
for key, v in by.items():
    if key is None:
        agg["?"] += v
        continue
    f, ln = key
    if f not in cache:
        try:
            cache[f] = heads("/root/repo/paper_2305_09493_b200/csrc/" + f)
        except OSError:
            cache[f] = []
    h = cache[f]
    i = bisect.bisect_right([x[0] for x in h], ln) - 1
    agg[f + ":" + (h[i][1] if i >= 0 else "?")] += v
tot = sum(agg.values())
print(f"{kname}: {tot} instructions, {tot * 16 // 1024} KB")
for k, v in agg.most_common(topn):
    print(f"{v * 16 / 1024:7.1f} KB {100 * v / tot:5.1f}%  {k}")
