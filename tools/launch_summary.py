"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by
kernel name: launches, summed serialised kernel time and share.
  python tools/launch_summary.py gpurun_out/bench_launches.csv "<command line>" > profiles/...txt"""
import collections
import csv
import sys

path = sys.argv[1]
rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0] != "ID" and r[12] == "gpu__time_duration.sum"]
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    name = r[4].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    name = name.split("<")[0]
    agg[name][0] += 1
    agg[name][1] += float(r[14].replace(",", "")) / 1e6
tot = sum(v[1] for v in agg.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
print(f"launches {len(rows)} sum of kernel time {tot:.1f} ms")
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n[:40]:40s} {c:6d} launches {t:10.1f} ms {100 * t / tot:6.1f}%")
