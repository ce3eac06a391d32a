"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv): per-kernel totals and
the per-launch sequence of the first window."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ik, iv, ig = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
tot, cnt, seq = collections.Counter(), collections.Counter(), []
for r in rows[hi + 1:]:
    try:
        v = float(r[iv].replace(",", ""))
    except (ValueError, IndexError):
        continue
    k = r[ik].split("(")[0].replace("void ", "").replace("goom::<unnamed>::", "")[:48] + " " + r[ig]
    tot[k] += v
    cnt[k] += 1
    seq.append((k, v))
s = sum(tot.values())
for k, v in tot.most_common(25):
    print(f"{k:70s} n={cnt[k]:5d} tot={v / 1e6:9.3f} ms avg={v / cnt[k] / 1e3:8.1f} us share={v / s * 100:5.1f}%")
