"""Top stall-sampled SASS instructions of an ncu report (source page), with warp roles."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hi = next(i for i, r in enumerate(rows) if "Source" in r)
hdr = rows[hi]
iS, iW, iE = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = []
for r in rows[hi + 1:]:
    try:
        data.append((int(r[iW] or 0), int(r[iE] or 0), r[iS][:100]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
for i, (w, e, s) in enumerate(sorted(data, reverse=True)[:n]):
    print(f"{w / tot * 100:5.1f}% exec={e:9d} {s}")
