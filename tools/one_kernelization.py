"""Per-launch device times of one kernelization in an ncu launch list
(--metrics gpu__time_duration.sum --csv), split at the first kernel of a
kernelization (its round-1 compactions before demand_range and the fused
validation's member scan, else validate_csr).
usage: one_kernelization.py FILE [K]   (K: the K-th such start, default the
last complete one; a streamed host-API call has one scan per chunk, so pick
a device-API kernelization, e.g. bench.py's last timed step: K = warmup +
steps - 1)"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
names = [d["Kernel Name"].split("(")[0][-44:] for d in data]
# a kernelization starts with round 1's compactions (two compact_1pass, then
# demand_range before the fused validation's scan, or validate_csr)
starts = []
for i, n in enumerate(names):
    if "validate_csr" in n or ("demand_range" in n and i + 1 < len(names) and "scan_members" in names[i + 1]):
        j = i
        while j > 0 and "compact_1pass" in names[j - 1] and (not starts or j - 1 > starts[-1]):
            j -= 1
        starts.append(j)
unit = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
if len(sys.argv) > 2:
    k = int(sys.argv[2])
    lo, hi = starts[k], starts[k + 1] if k + 1 < len(starts) else len(data)
else:
    lo, hi = (starts[-2], starts[-1]) if len(starts) > 1 else (starts[-1], len(data))
tot = 0.0
for i in range(lo, hi):
    v = float(data[i]["Metric Value"].replace(",", "")) * unit.get(data[i]["Metric Unit"], 1e-3)
    if "gen::" in names[i] or "Functor" in names[i]:
        continue
    tot += v
    print(f"{v:9.1f} us  {names[i]}")
print(f"{tot:9.1f} us  total (ours)")
