"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel name."""
import csv, sys, collections, re
rows = []
with open(sys.argv[1]) as fh:
    lines = [l for l in fh if not l.startswith("==")]
rd = [r for r in csv.DictReader(lines) if r.get("Metric Name") == "gpu__time_duration.sum"]
if len(sys.argv) > 2 and sys.argv[2] == "second-half":
    rd = rd[len(rd) // 2:]
agg = collections.OrderedDict()
for r in rd:
    name = re.sub(r"\(.*", "", r["Kernel Name"])
    val = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    us = val / 1000.0 if unit in ("nsecond", "ns") else val if unit in ("usecond", "us") else val * 1000.0
    a = agg.setdefault(name, [0, 0.0, 0.0])
    a[0] += 1; a[1] += us; a[2] = max(a[2], us)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':48s} {'launches':>8s} {'total_us':>10s} {'mean_us':>9s} {'max_us':>9s} {'share':>7s}")
for k, (n, t, mx) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:48]:48s} {n:8d} {t:10.1f} {t/n:9.2f} {mx:9.2f} {100*t/tot:6.1f}%")
print(f"{'TOTAL':48s} {sum(a[0] for a in agg.values()):8d} {tot:10.1f}")
