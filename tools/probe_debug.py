"""Which planted duplicate-edge deletions does probe pruning lose?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2109_06042_b200 import _native, plant_twins  # noqa: E402

ctx = _native.context()
base, _ = ctx.generate_random(30000, 30000, 0.01, 3, 81)
csr = plant_twins(base, 0.002, 0.002, 82)
res = {}
for fp4 in (1, 0):
    for probe in (0, 1):
        ctx.set_option("fp4", fp4)
        ctx.set_option("probe", probe)
        va, ea, st = ctx.kernelize(csr, "dp", max_rounds=1) if False else ctx.kernelize(csr, "dp")
        res[fp4, probe] = (va, ea, st)
        print(fp4, probe, "del_e", st["deleted_edges"], "pruned", st["pruned_tiles"], "rounds", st["rounds"])
rows = {}
for e in range(csr.m):
    key = tuple(csr.edge_vtx[csr.edge_ptr[e]:csr.edge_ptr[e + 1]])
    rows.setdefault(key, []).append(e)
pairs = [v for v in rows.values() if len(v) > 1]
for fp4 in (1, 0):
    ref, got = res[fp4, 0][1], res[fp4, 1][1]
    missed = [(v[0], v[1]) for v in pairs if ref[v[1]] == 0 and got[v[1]] == 1]
    print("fp4", fp4, "pairs", len(pairs), "missed", len(missed))
    for i, j in missed[:20]:
        print("   i", i, "j", j, "i%256", i % 256, "j%256", j % 256, "P", i // 256, "J", j // 256)
