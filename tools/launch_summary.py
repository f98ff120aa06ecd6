"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel name,
launches, median and total time."""
import collections
import csv
import statistics
import sys

txt = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith('"')]
rows = list(csv.reader(txt))
h = rows[0]
iK, iV, iU = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
iM = h.index("Metric Name")
c = collections.defaultdict(list)
for r in rows[1:]:
    if r[iM] != "gpu__time_duration.sum":
        continue
    v = float(r[iV].replace(",", ""))
    v = v / 1e3 if r[iU] == "ns" else (v * 1e3 if r[iU] == "ms" else v)
    c[r[iK][:80]].append(v)
tot = sum(sum(v) for v in c.values())
for k, v in sorted(c.items(), key=lambda kv: -sum(kv[1]))[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{len(v):5d} {statistics.median(v):9.2f} us med {sum(v):10.1f} us tot  {k}")
print(f"total {tot:.1f} us")
