"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv): per kernel count, time, share.
usage: python tools/launch_summary.py LAUNCHES.csv"""
import csv, collections, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0]
    v = float(r[vi].replace(",", ""))
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
unit = rows[1][hdr.index("Metric Unit")] if "Metric Unit" in hdr else ""
print(f"launches {sum(v[0] for v in agg.values())}, total {tot:.1f} {unit}\n")
print("| kernel | launches | total | avg | share |\n|---|---|---|---|---|")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| {k} | {n} | {t:.1f} | {t/n:.2f} | {100*t/tot:.1f}% |")
