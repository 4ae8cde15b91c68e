"""Per-kernel totals from an ncu --metrics gpu__time_duration.sum launch list."""
import csv
import sys
from collections import defaultdict

lines = [l for l in open(sys.argv[1]) if not l.startswith("==")]
rd = csv.reader(lines)
h = next(rd)
kn, mv, mn = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
tot, cnt = defaultdict(float), defaultdict(int)
for r in rd:
    if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
        continue
    n = r[kn].split("(")[0]
    if "ls::" not in n and "CUB" not in n and (len(sys.argv) < 3):
        continue
    tot[n] += float(r[mv].replace(",", "")) / 1e3
    cnt[n] += 1
for n, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print("%-44s %5d %10.1f us  avg %8.1f" % (n[:44], cnt[n], v, v / cnt[n]))
