"""Three host-API (streamed, pinned buffers) kernelizations of config 4, for
an ncu launch list of the e2e path (the last third of the list is one call):
    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/e2e_launches.csv python tools/e2e_once.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2109_06042_b200 import _native  # noqa: E402
from paper_2109_06042_b200.instance import CSRInstance  # noqa: E402

ctx = _native.Context(0)
csr, _ = ctx.generate_random(100000, 100000, 0.01, 3, 0)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
h = CSRInstance(csr.n, pin(csr.edge_ptr), pin(csr.edge_vtx), pin(csr.demand), validate=False)
for _ in range(3):
    st = ctx.kernelize(h)[2]
print("launches per call", st["kernel_launches"], "ms", st["ms_total"], "spec_vertex", st["spec_vertex"])
