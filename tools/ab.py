"""A/B timing of library options on one GPU (CUDA-event device time of one
full kernelization, instance resident in HBM, L2 flushed between steps).

    python tools/ab.py CONFIG[,CONFIG...] [OPTSET ...] [--steps K] [--rule dp]

OPTSET is "key=value,key=value" (library options, include/mhsk.h) or "-" for
the defaults.  Prints one JSON line per (config, optset)."""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs")
    ap.add_argument("optsets", nargs="*", default=["-"])
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--rule", default="dp")
    args = ap.parse_args()

    import torch

    from bench import make_instance
    from paper_2109_06042_b200 import _native

    ctx = _native.Context(0)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for name in args.configs.split(","):
        csr, _ = make_instance(name, 0, ctx)
        d = [torch.from_numpy(a).cuda() for a in (csr.edge_ptr, csr.edge_vtx, csr.demand)]
        va = torch.empty(csr.n, dtype=torch.uint8, device="cuda")
        ea = torch.empty(csr.m, dtype=torch.uint8, device="cuda")
        ref = None
        for optset in args.optsets:
            opts = {} if optset == "-" else dict(kv.split("=") for kv in optset.split(","))
            for k, v in opts.items():
                ctx.set_option(k, int(v))
            stats = []
            for i in range(args.steps + 1):
                flush.fill_(1)
                torch.cuda.synchronize()
                st = ctx.kernelize_device(csr.n, csr.m, d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(),
                                          va.data_ptr(), ea.data_ptr(), rule=args.rule)
                if i:
                    stats.append(st)
            out = (va.cpu().numpy().copy(), ea.cpu().numpy().copy())
            same = ref is None or (np.array_equal(out[0], ref[0]) and np.array_equal(out[1], ref[1]))
            ref = ref or out
            s0 = stats[-1]
            print(json.dumps({"config": name, "opts": opts, "ms": statistics.mean(s["ms_total"] for s in stats),
                              "ms_min": min(s["ms_total"] for s in stats), "gram_ms": s0["ms_gram"],
                              "rounds": s0["rounds"], "del_e": s0["deleted_edges"],
                              "del_v": s0["deleted_vertices"], "executed_ops": s0["executed_ops"],
                              "pruned_tiles": s0["pruned_tiles"], "verified": s0["verified_pairs"],
                              "launches": s0["kernel_launches"], "same_as_first": same}), flush=True)
            defaults = {"incremental": 1, "fast_loop": 1, "sparse": -1, "fp4": 1, "probe": 1, "verify": 1,
                        "lazy": 1, "lazy_e": 1, "vcsr": 1, "probe_entries": 0, "probe_entries_e": 14,
                        "cand_cap": 1 << 20, "vcand_max": 1 << 15, "vcand_table_log2": 17,
                        "raster_gp": 4, "raster_gj": 9, "throttle_slack": 4, "throttle_chunk_log2": 4,
                        "spec_vertex": 1, "pdl": 1}
            for k in opts:   # back to the library defaults
                if k in defaults:
                    ctx.set_option(k, defaults[k])


if __name__ == "__main__":
    main()
