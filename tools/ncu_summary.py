"""One-screen summary of an ncu report: SOL, stalls, instruction mix (for profiles/)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2] if len(rows) > 2 else rows[1]
d = dict(zip(hdr, vals))
u = dict(zip(hdr, units))


def g(k):
    v = d.get(k)
    try:
        return float(v)
    except (TypeError, ValueError):
        return None


keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
        "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_shared_ld.sum",
        "smsp__sass_inst_executed_op_global_ld.sum", "smsp__sass_inst_executed_op_global_st.sum"]
for k in keys:
    print(f"{k}: {d.get(k)} {u.get(k, '')}")
st = {k: g(k) for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")}
tot = sum(v for v in st.values() if v) or 1
print("stall reasons (share of samples):")
for k, v in sorted(st.items(), key=lambda x: -(x[1] or 0))[:10]:
    print(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}: {100 * (v or 0) / tot:.1f}%")
