"""Summarize an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel."""
import collections
import csv
import re
import sys

path = sys.argv[1]
rows = list(csv.DictReader(l for l in open(path) if not l.startswith("==")))
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r["Kernel Name"])
    name = re.sub(r"\(anonymous namespace\)::|hy::|unnamed>::|void ", "", name)[:60]
    v = float(r["Metric Value"])
    unit = r["Metric Unit"]
    v = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)  # -> us
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':60s} {'launches':>8s} {'total ms':>9s} {'share':>6s} {'avg us':>9s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:60s} {v[0]:8d} {v[1]/1e3:9.2f} {100*v[1]/tot:5.1f}% {v[1]/v[0]:9.1f}")
print(f"{'TOTAL':60s} {sum(v[0] for v in agg.values()):8d} {tot/1e3:9.2f}")
