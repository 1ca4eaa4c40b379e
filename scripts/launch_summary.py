"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per
kernel count, total and mean time, and share of the sum."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr, data = rows[hi], rows[hi + 1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = {}
for r in data:
    if len(r) <= vi:
        continue
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "ms": 1.0, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(r[ui], 1.0)
    name = r[ki].split("(")[0].replace("void ", "").replace("me::<unnamed>::", "")[:60]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v * scale
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':60s} {'n':>5s} {'total ms':>10s} {'mean ms':>9s} {'share':>6s}")
for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:60s} {n:5d} {ms:10.3f} {ms / n:9.4f} {100 * ms / tot:5.1f}%")
