"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel.
usage: python tools/launch_table.py launches.csv [skip_first_n_launches]"""
import csv, collections, re, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
agg = collections.OrderedDict()
for r in rows[1 + skip:]:
    name = re.sub(r"\(.*", "", r[ik]).replace("void ", "").replace("hogb200::", "")
    v = float(r[iv].replace(",", ""))
    v = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r[iu]] * v
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':70s} {'n':>6s} {'total us':>12s} {'mean us':>10s} {'share':>7s}")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:70]:70s} {n:6d} {t:12.1f} {t / n:10.2f} {100 * t / tot:6.1f}%")
print(f"total {tot:.1f} us")
