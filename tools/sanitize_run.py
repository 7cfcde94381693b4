"""Workload for compute-sanitizer (memcheck / racecheck / synccheck): the
default path with every stage engaged -- FP4 probe pruning, candidate
verification, lazy X_E / X_V, vertex candidates from the CSR, incremental
rounds, capacity overflows -- on a planted instance (deletions of both phases
over 5 rounds), checked against its by-construction deletion sets; plus the
int8 operands, the other backends, the single-phase entry points and an FE
pipeline on small instances.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [N]

N = instance side (default 20000; racecheck / synccheck are ~100x slower).
Exits 1 on a wrong result; the sanitizer's own exit code reports hazards."""

from __future__ import annotations

import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    side = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
    from paper_2109_06042_b200 import _native, interval_trains, nested_chains, plant_twins, random_csr
    from paper_2109_06042_b200.generate import plant_deletions

    ctx = _native.context()
    base, _ = ctx.generate_random(side, side, 0.02, 3, 71)
    scale = max(1, side // 20000)
    csr, planted = plant_deletions(base, 72, dominated=20 * scale, twin_groups=10 * scale,
                                   dp_pairs=20 * scale, duplicates=20 * scale, chains=4, chain_len=3)
    runs = [{}, {"fp4": 0}, {"cand_cap": 37}, {"vcand_table_log2": 6}]
    for opts in runs:
        for k, v in opts.items():
            ctx.set_option(k, v)
        for rule in ("dp", "se"):
            va, ea, st = ctx.kernelize(csr, rule)
            ok = ({int(i) for i in np.nonzero(ea == 0)[0]} == set(planted.edges[rule])
                  and {int(i) for i in np.nonzero(va == 0)[0]} == set(planted.vertices)
                  and st["rounds"] == planted.rounds[rule])
            print(opts, rule, "rounds", st["rounds"], "pruned", st["pruned_tiles"], "verified",
                  st["verified_pairs"], "ok" if ok else "WRONG", flush=True)
            if not ok:
                sys.exit(1)
        ctx.set_option("fp4", 1)
        ctx.set_option("cand_cap", 1 << 20)
        ctx.set_option("vcand_table_log2", 17)
    # vertex deletions only on a 70k x 70k instance (n m > 2^32: dense mode,
    # nnz > 2^24: streamed upload): round 1's edge phase deletes nothing, so
    # the call adopts its speculative vertex probe and decides the planted
    # vertices from its marks and candidates
    base2, _ = ctx.generate_random(70000, 70000, 0.01, 3, 74)
    csr2, planted2 = plant_deletions(base2, 73, dominated=60, twin_groups=30, dp_pairs=0, duplicates=0, chains=0)
    va, ea, st = ctx.kernelize(csr2, "dp")
    ok = (ea.all() and {int(i) for i in np.nonzero(va == 0)[0]} == set(planted2.vertices))
    print("vertex-only plants (70k): spec_vertex", st["spec_vertex"], "rounds", st["rounds"],
          "ok" if ok and st["spec_vertex"] == 1 else "WRONG", flush=True)
    if not ok or st["spec_vertex"] != 1:
        sys.exit(1)
    for b in ("tc", "tc1", "simt"):
        ctx.set_backend(b)
        for small in (interval_trains(3000, 1200, 1, 1), plant_twins(random_csr(700, 900, 0.03, 2, 2), 0.03, 0.03, 3),
                      nested_chains(12, 30, 3, 4)):
            ctx.kernelize(small)
            ctx.reduce_edges(small, "se")
            ctx.reduce_vertices(small)
            ctx.run_pipeline(small, ("fe", "dp", "md"), True)
    ctx.set_backend("tc")
    print("done", flush=True)


if __name__ == "__main__":
    main()
