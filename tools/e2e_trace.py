"""e2e (host API, pinned buffers) timing of config 4 under streaming options,
all on one box (PCIe bandwidth varies between boxes): prints the e2e ms of
each option set and the box's plain H2D bandwidth.
    python tools/e2e_trace.py [OPTSET ...]   OPTSET = key=value,... | -"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2109_06042_b200 import _native  # noqa: E402
from paper_2109_06042_b200.instance import CSRInstance  # noqa: E402

ctx = _native.Context(0)
csr, _ = ctx.generate_random(100000, 100000, 0.01, 3, 0)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
h = CSRInstance(csr.n, pin(csr.edge_ptr), pin(csr.edge_vtx), pin(csr.demand), validate=False)
x = torch.empty(csr.nnz, dtype=torch.int32, device="cuda")
src = torch.from_numpy(h.edge_vtx)
for optset in (sys.argv[1:] or ["-"]):
    opts = {} if optset == "-" else dict(kv.split("=") for kv in optset.split(","))
    for k, v in opts.items():
        ctx.set_option(k, int(v))
    ctx.kernelize(h)
    ms = [ctx.kernelize(h)[2]["ms_total"] for _ in range(5)]
    torch.cuda.synchronize()
    t0 = time.time()
    for _ in range(3):
        x.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    print(opts, "e2e ms", round(statistics.median(ms), 3), "min", round(min(ms), 3),
          "| H2D GB/s", round(3 * csr.nnz * 4 / (time.time() - t0) / 1e9, 1), flush=True)
    for k in opts:
        ctx.set_option(k, {"stream_chunks": 16, "stream_sqrt": 1, "spec_vertex": 1, "pdl": 1}.get(k, 0))
