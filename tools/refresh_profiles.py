"""Local side of the profile refresh: gpurun_out/rp_* -> profiles/ (bench line,
launch list, ncu summaries, per-kernel DRAM traffic for bench.py's roofline)."""
import csv
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT, PROF = ROOT / "gpurun_out", ROOT / "profiles"
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
line = [ln for ln in (OUT / "rp_bench.json").read_text().splitlines() if ln.startswith("{")][-1]
(PROF / f"{tag}_bench_roundtrip_1M.json").write_text(json.dumps(json.loads(line), indent=1) + "\n")
shutil.copy(OUT / "rp_launches.csv", PROF / f"{tag}_launches_roundtrip_1M.csv")
shutil.copy(OUT / "rp_kernels_200k.txt", PROF / f"{tag}_kernels_200k.txt")
traffic = {}
for k, name in (("disasm", "skg_disasm"), ("asm", "skg_asm")):
    rep = OUT / f"rp_{k}_1M.ncu-rep"
    summ = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), str(rep)],
                          capture_output=True, text=True).stdout
    (PROF / f"{tag}_{k}_ncu_summary.txt").write_text(
        f"ncu --set full --clock-control none -k regex:^{k}_kernel -c 1 python bench.py --steps 1 --warmup 3\n"
        f"(1M-module batch of the bench; report gpurun_out/rp_{k}_1M.ncu-rep)\n\n" + summ)
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    d = dict(zip(rows[0], rows[2]))
    unit = dict(zip(rows[0], rows[1]))

    def nbytes(key):
        v = float(d[key])
        return int(v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[unit[key]])
    rd, wr = nbytes("dram__bytes_read.sum"), nbytes("dram__bytes_write.sum")
    traffic[name] = {"kernel": f"{k}_kernel", "bytes_per_launch": rd + wr, "dram_read_bytes": rd,
                     "dram_write_bytes": wr,
                     "warp_inst_per_launch": int(float(d["smsp__inst_executed.sum"])),
                     "ncu_ms": float(d["gpu__time_duration.sum"]) * {"ms": 1.0, "us": 1e-3, "ns": 1e-6,
                                                                     "s": 1e3}[unit["gpu__time_duration.sum"]],
                     "source": f"profiles/{tag}_{k}_ncu_summary.txt (ncu --set full, 1M-module batch)"}
(PROF / "traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
# the bench line was taken before this traffic.json existed: same figure bench.py reads from it
bench = json.loads((PROF / f"{tag}_bench_roundtrip_1M.json").read_text())
bench["roofline"]["traffic"] = traffic[bench["roofline"]["kernel"]]["bytes_per_launch"]
t = traffic[bench["roofline"]["kernel"]]
ms = bench["roofline"]["per_kernel"][bench["roofline"]["kernel"]]["ms"]
peak_issue = 148 * 4 * 1.965e9
bench["roofline"]["issue"] = {"warp_inst_per_launch": t["warp_inst_per_launch"],
                              "achieved_warp_inst_per_s": t["warp_inst_per_launch"] / (ms / 1e3),
                              "peak_warp_inst_per_s": peak_issue,
                              "frac": t["warp_inst_per_launch"] / (ms / 1e3) / peak_issue}
(PROF / f"{tag}_bench_roundtrip_1M.json").write_text(json.dumps(bench, indent=1) + "\n")
print(json.dumps(traffic, indent=1))
