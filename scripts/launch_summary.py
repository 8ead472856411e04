"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel name.
usage: python scripts/launch_summary.py launches.csv [steps]   (steps = timed steps in the run)"""
import collections, csv, re, sys

rows = list(csv.reader(open(sys.argv[1])))
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"^void |dtwlb::|<?unnamed>::|\(anonymous namespace\)::", "", d["Kernel Name"]).split("(")[0]
    agg[name][0] += 1
    agg[name][1] += float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1e-6)
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':58s} {'launches':>8s} {'ms total':>10s} {'ms/step':>9s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:58]:58s} {v[0]:8d} {v[1]:10.2f} {v[1] / steps:9.2f} {100 * v[1] / tot:5.1f}%")
print(f"{'total':58s} {sum(v[0] for v in agg.values()):8d} {tot:10.2f} {tot / steps:9.2f}")
