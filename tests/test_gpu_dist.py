"""The sharded (multi-rank) CUDA path on one device: `world` ranks as threads,
each with its own libmhsk context running its slice of every phase's tile
list, deleter counts summed by a host-side all-reduce between the Gram
product and the commit (dist.InProcessAllreduce).  No kernel waits on
another rank's kernel.  Results must be bit-identical to the oracle on every
rank (the analogue of the reference's worker-count test,
test_parallel.py:111-117)."""

from __future__ import annotations

import os

import numpy as np
import pytest

import oracle
from paper_2109_06042_b200 import interval_trains, nested_chains, plant_twins, random_csr
from conftest import planted_40k
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


# ------------------------------------------- the headline path, sharded
@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_headline_path_matches_planted_sets(world):
    """World 2/4/8 on a 40k x 40k planted instance where the default path
    engages fully -- FP4 probe pruning, candidate verification, lazy X_E /
    X_V, vertex candidates from the CSR, incremental rounds -- on every rank:
    bit-identical to world 1 and to the by-construction deletion sets
    (which tests/test_oracle.py pins against both oracles)."""
    from paper_2109_06042_b200 import _native

    csr, planted = planted_40k()
    ref_va, ref_ea, ref_st = _native.context().kernelize(csr, "dp")
    assert {int(i) for i in np.nonzero(ref_ea == 0)[0]} == set(planted.edges["dp"])
    assert {int(i) for i in np.nonzero(ref_va == 0)[0]} == set(planted.vertices)
    assert ref_st["rounds"] == planted.rounds["dp"]
    results = kernelize_in_process(csr, world, options={"shard_upload": 2})
    for r, (va, ea, st) in enumerate(results):
        assert np.array_equal(va, ref_va) and np.array_equal(ea, ref_ea), r
        assert st["rounds"] == ref_st["rounds"], r
        assert st["deleted_edges"] == ref_st["deleted_edges"], r
        assert st["deleted_vertices"] == ref_st["deleted_vertices"], r
        assert st["pruned_tiles"] > 0, (r, st)
        assert st["verified_pairs"] > 0, (r, st)
        assert st["fp4_gram_launches"] > 0, (r, st)
    # the probe work is split: the ranks' pruned tiles add up to world 1's
    assert sum(st["pruned_tiles"] for _, _, st in results) == ref_st["pruned_tiles"]
    # ... and the upload (shard_upload 2: also below its 2^24-member default
    # threshold): each rank copied its slice of the member array, the
    # all-reduce hook assembled the rest
    per = -(-csr.nnz // world)
    for _, _, st in results:
        assert st["h2d_bytes"] <= 4 * per + 12 * (csr.m + 1), st["h2d_bytes"]


def _torch_dist_rank(rank, world, port, path, out_dir):
    import pickle

    import torch
    import torch.distributed as dist

    from paper_2109_06042_b200 import _native
    from paper_2109_06042_b200.dist import TorchDistAllreduce

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    with open(path, "rb") as f:
        csr = pickle.load(f)
    ctx = _native.Context(0)
    ctx.set_shard(rank, world, TorchDistAllreduce(0))
    ctx.set_option("shard_upload", 2)   # the member array through the hook too
    va, ea, st = ctx.kernelize(csr, "dp")
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), va=va, ea=ea,
             st=np.array([st["rounds"], st["pruned_tiles"], st["verified_pairs"]]))
    dist.barrier()
    dist.destroy_process_group()


def test_torch_distributed_allreduce_drives_the_library(tmp_path):
    """Two processes, one libmhsk context each (both on cuda:0), exchanging
    the per-phase deleter counts through the real TorchDistAllreduce
    callback (torch.distributed, here the gloo backend on CUDA tensors; NCCL
    on a multi-GPU box) installed with mhsk_set_shard: both ranks commit the
    world-1 result on the planted 40k instance."""
    import pickle
    import socket

    import torch.multiprocessing as mp

    from paper_2109_06042_b200 import _native

    csr, planted = planted_40k()
    ref_va, ref_ea, ref_st = _native.context().kernelize(csr, "dp")
    path = tmp_path / "inst.pkl"
    with open(path, "wb") as f:
        pickle.dump(csr, f)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.start_processes(_torch_dist_rank, args=(2, port, str(path), str(tmp_path)), nprocs=2,
                       join=True, start_method="spawn")
    for r in range(2):
        got = np.load(tmp_path / f"rank{r}.npz")
        assert np.array_equal(got["va"], ref_va) and np.array_equal(got["ea"], ref_ea), r
        rounds, pruned, verified = got["st"].tolist()
        assert rounds == ref_st["rounds"] and pruned > 0 and verified > 0, r
