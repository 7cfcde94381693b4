"""Counter-based generator: device (mhsk_generate_random) == host C
(mhsk_generate_random_host) == numpy (generate.counter_random), bit for bit."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2109_06042_b200 import _native
from paper_2109_06042_b200.generate import counter_random

pytestmark = pytest.mark.gpu

ARGS = [(3000, 2000, 0.01, 3, 7), (50, 40, 1e-4, 2, 1), (5, 3, 1.0, 2, 1), (1, 4, 0.3, 1, 2),
        (777, 1, 0.5, 5, 3), (300, 0, 0.5, 1, 4), (4097, 1500, 0.002, 4, 9)]


@pytest.mark.parametrize("args", ARGS, ids=[str(a) for a in ARGS])
def test_device_generator_matches_host(args):
    want = counter_random(*args)
    got, dev = _native.context().generate_random(*args)
    assert np.array_equal(got.edge_ptr, want.edge_ptr)
    assert np.array_equal(got.edge_vtx, want.edge_vtx)
    assert np.array_equal(got.demand, want.demand)
    host = _native.generate_random_host(*args)
    assert np.array_equal(host.edge_vtx, want.edge_vtx)
    got.validate()


def test_device_generated_instance_kernelizes_in_place():
    ctx = _native.context()
    csr, (d_ptr, d_vtx, d_dem) = ctx.generate_random(4000, 3000, 0.004, 2, 11)
    import torch

    va = torch.empty(csr.n, dtype=torch.uint8, device="cuda")
    ea = torch.empty(csr.m, dtype=torch.uint8, device="cuda")
    st = ctx.kernelize_device(csr.n, csr.m, d_ptr, d_vtx, d_dem, va.data_ptr(), ea.data_ptr())
    hva, hea, hst = ctx.kernelize(csr)
    assert np.array_equal(va.cpu().numpy(), hva) and np.array_equal(ea.cpu().numpy(), hea)
    assert st["rounds"] == hst["rounds"]
