"""Per-kernel totals of the last of R repetitions in an ncu launch list
(--metrics gpu__time_duration.sum --csv).  usage: launch_table.py FILE [R]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
last = data[len(data) * (reps - 1) // reps:]
tot, cnt = collections.OrderedDict(), collections.Counter()
for d in last:
    k = d["Kernel Name"].split("(")[0][-48:]
    v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1e-3)
    tot[k] = tot.get(k, 0) + v
    cnt[k] += 1
print(f"launches {len(last)}  sum {sum(tot.values()):.1f} us")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"  {v:9.1f} us  x{cnt[k]:4d}  {k}")
