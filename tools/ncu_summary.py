"""Summarise an ncu report: key throughput metrics, stall reasons, SASS opcode mix."""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2] if len(rows) > 2 else rows[1]
want = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_issued.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]
for k, x in zip(h, v):
    if k in want:
        print(f"{k} = {x}")
st = []
for k, x in zip(h, v):
    if "smsp__average_warps_issue_stalled" in k and k.endswith("ratio"):
        try:
            st.append((float(x), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        except ValueError:
            pass
print("stalls:", ", ".join(f"{k}={x:.2f}" for x, k in sorted(st, reverse=True)[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
c, cw = Counter(), Counter()
for r in rows[2:]:
    try:
        e, w = int(r[iE] or 0), int(r[iW] or 0)
    except (ValueError, IndexError):
        continue
    t = r[iS].strip().split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
    c[op.split(".")[0]] += e
    cw[op.split(".")[0]] += w
tot, totw = sum(c.values()), max(sum(cw.values()), 1)
print("opcode mix (dyn %, stall-sample %):",
      ", ".join(f"{o}={e / tot * 100:.1f}/{cw[o] / totw * 100:.1f}" for o, e in c.most_common(16)))
