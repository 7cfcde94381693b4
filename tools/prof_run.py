"""One kernelization of a BASELINE config through the device C ABI -- the
short command profiled under ncu (tools/gpu_profile.sh)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2109_06042_b200 import _native, config_instance  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--backend", default="tc")
a = ap.parse_args()
csr = config_instance(a.config, 0)
ctx = _native.Context(0, backend=a.backend)
d = [torch.from_numpy(x).cuda() for x in (csr.edge_ptr, csr.edge_vtx, csr.demand)]
va = torch.empty(csr.n, dtype=torch.uint8, device="cuda")
ea = torch.empty(csr.m, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
for _ in range(a.reps):
    st = ctx.kernelize_device(csr.n, csr.m, d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(),
                              va.data_ptr(), ea.data_ptr())
print({k: st[k] for k in ("rounds", "ms_total", "ms_gram", "gram_ops", "kernel_launches")})
