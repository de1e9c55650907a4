"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[hi + 1:]:
    name = re.sub(r"<.*", "", r[ki])[:56]
    v = float(r[vi].replace(",", "")) * {"usecond": 1e3, "msecond": 1e6, "nsecond": 1, "second": 1e9}.get(r[ui], 1)
    tot[name] += v
    cnt[name] += 1
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
allt = sum(tot.values())
for k, v in tot.most_common(20):
    print(f"{k:56s} {cnt[k] / div:8.1f} {v / div / 1e6:9.3f} ms {v / cnt[k] / 1e3:9.1f} us/launch {100 * v / allt:5.1f}%")
print(f"total {allt / div / 1e6:.3f} ms, {sum(cnt.values()) / div:.0f} launches")
