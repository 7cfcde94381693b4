"""Summarise ncu outputs into the text files committed under profiles/.

    python tools/ncu_summary.py full  gpurun_out/gram_full.ncu-rep  > profiles/rNN_gram_ncu.txt
    python tools/ncu_summary.py launches gpurun_out/launches.csv    > profiles/rNN_launches.txt
"""

from __future__ import annotations

import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "lts__t_sectors_srcunit_tex_op_read.sum",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "launch__cluster_dim_x",
    "smsp__inst_executed.sum",
]


def full(path: str) -> None:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {h: k for k, h in enumerate(hdr)}
    name_col = idx.get("Kernel Name")
    for r in rows[2:]:
        print(f"kernel: {r[name_col] if name_col is not None else '?'}")
        for key in KEYS:
            if key in idx:
                print(f"  {key:<78} {r[idx[key]]:>22} {units[idx[key]]}")
        print()


def launches(path: str) -> None:
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    k_name, k_metric, k_val = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    unit_col = hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) <= k_val or r[k_metric] != "gpu__time_duration.sum":
            continue
        v = float(r[k_val].replace(",", ""))
        unit = r[unit_col]
        scale = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6,
                 "second": 1e3, "s": 1e3}.get(unit, 1.0)
        name = re.sub(r"\(.*", "", r[k_name])[:90]
        tot[name] += v * scale
        cnt[name] += 1
    total = sum(tot.values())
    print(f"{'kernel':<92}{'launches':>9}{'total ms':>12}{'share':>8}")
    for name in sorted(tot, key=tot.get, reverse=True):
        print(f"{name:<92}{cnt[name]:>9}{tot[name]:>12.3f}{tot[name] / total:>8.1%}")
    print(f"{'TOTAL':<92}{sum(cnt.values()):>9}{total:>12.3f}")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2])
