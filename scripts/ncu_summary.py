"""Write a committed text summary of an ncu report (key raw metrics, stall
reasons, top SASS lines):  python scripts/ncu_summary.py rep.ncu-rep out.txt"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg.per_second"]
lines = [f"ncu report: {rep}"]
for h, u, v in zip(hdr, units, vals):
    if h in want:
        lines.append(f"  {h:70s} {v} {u}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
if len(srows) > 2:
    sh = srows[1]
    col = {h: i for i, h in enumerate(sh)}
    reasons = [h for h in sh if h.startswith("stall_") and "Not Issued" not in h]
    tot = Counter()
    for r in srows[2:]:
        for h in reasons:
            if r[col[h]].isdigit():
                tot[h] += int(r[col[h]])
    S = sum(tot.values()) or 1
    lines.append("warp stall sampling (all samples):")
    for h, v in tot.most_common(10):
        lines.append(f"  {h:26s} {100 * v / S:5.1f}%")
    key = col["Warp Stall Sampling (All Samples)"]
    top = sorted(srows[2:], key=lambda r: -int(r[key]) if r[key].isdigit() else 0)[:15]
    lines.append("top SASS lines by stall samples:")
    for r in top:
        lines.append(f"  {r[key]:>7} ex={r[col['Instructions Executed']]:>10}  {r[col['Source']].strip()[:70]}")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
