"""The sharded (multi-rank) CUDA path on one device: `world` ranks as threads,
each with its own libmhsk context running its slice of every phase's tile
list, deleter counts summed by a host-side all-reduce between the Gram
product and the commit (dist.InProcessAllreduce).  No kernel waits on
another rank's kernel.  Results must be bit-identical to the oracle on every
rank (the analogue of the reference's worker-count test,
test_parallel.py:111-117)."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_2109_06042_b200 import interval_trains, nested_chains, plant_twins, random_csr
from paper_2109_06042_b200.dist import kernelize_in_process

pytestmark = pytest.mark.gpu

INSTANCES = [
    ("trains", lambda: interval_trains(6000, 2500, 1, 3)),
    ("twins", lambda: plant_twins(random_csr(1500, 1800, 0.03, 2, 4), 0.02, 0.02, 5)),
    ("chains", lambda: nested_chains(30, 40, 3, 6)),
]


@pytest.mark.parametrize("name,make", INSTANCES, ids=[n for n, _ in INSTANCES])
@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("backend", ["tc", "tc1"])
def test_sharded_ranks_match_oracle(name, make, world, backend):
    csr = make()
    va, ea, rounds, de, dv = oracle.kernelize(csr, "dp")
    results = kernelize_in_process(csr, world, backend=backend)
    total_exec = sum(r[2]["executed_ops"] for r in results)
    for rva, rea, st in results:
        assert np.array_equal(rva, va) and np.array_equal(rea, ea)
        assert st["rounds"] == rounds
        assert st["deleted_edges"] == de and st["deleted_vertices"] == dv
    # the ranks split the work: each executed about 1/world of it
    for _, _, st in results:
        assert st["executed_ops"] <= total_exec / world * 1.5 + 1


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("options", [{"sparse": 1}, {"sparse": 2}, {"incremental": 1, "sparse": 0},
                                     {"fast_loop": 0}, {"sparse": 0, "fp4": 0}, {"sparse": 0, "fp4": 1}],
                         ids=["sparse", "components", "incremental", "host_loop", "int8", "fp4"])
def test_sharded_variants_match_oracle(world, options):
    csr = interval_trains(9000, 4000, 2, 51)
    va, ea, rounds, de, dv = oracle.kernelize(csr, "dp")
    for rva, rea, st in kernelize_in_process(csr, world, options=options):
        assert np.array_equal(rva, va) and np.array_equal(rea, ea)
        assert st["rounds"] == rounds
