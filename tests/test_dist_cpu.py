"""The multi-rank path on CPU (world_size 2, gloo).

Each rank runs a host model of the sharded device algorithm -- the library's
own tile list (mhsk_tile_list) shared out by dist.shard_share, the epilogue's
pair predicates evaluated once per unordered pair inside the rank's tiles, a
SUM all-reduce of the per-item deleter counts over torch.distributed, then
the commit -- and the result must equal the single-rank CPU oracle bit for
bit.  This covers the partitioning and exchange logic that the GPU path runs
with NCCL (paper_2109_06042_b200/dist.py); the CUDA kernels themselves are
covered by the -m gpu tests (including a multi-rank run on one device).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2109_06042_b200 import _native, interval_trains, nested_chains, plant_twins, random_csr
from paper_2109_06042_b200.dist import shard_share


def pair_predicates(phase: str, c, ai, bi, aj, bj):
    """numpy restatement of csrc/epilogue.cuh (pairs i < j)."""
    if phase == "dp":
        rij = bi - ai + c >= bj
        rji = bj - aj + c >= bi
        return rij, rji & ~rij
    if phase == "se":
        rij = (c == ai) & (bi >= bj)
        rji = (c == aj) & (bj >= bi)
        return rij, rji & ~rij
    return c == aj, (c == ai) & (c != aj)


def phase_hits(X: np.ndarray, a: np.ndarray, b: np.ndarray, phase: str, rank: int, world: int,
               cols: int = 240):
    """cols: tile columns (240 = the default FP4 kernel, 256 = int8)."""
    M = X.shape[0]
    tiles = _native.tile_list(M, 256, tile_cols=cols)
    hits = np.zeros(M, dtype=np.int64)
    G = X.astype(np.int64) @ X.T.astype(np.int64)
    for I, J in tiles[list(shard_share(len(tiles), rank, world))]:
        i = np.arange(I * 256, min(M, I * 256 + 256))
        j = np.arange(J * cols, min(M, J * cols + cols))
        if len(i) == 0 or len(j) == 0:
            continue
        ii, jj = np.meshgrid(i, j, indexing="ij")
        mask = ii < jj
        ii, jj = ii[mask], jj[mask]
        c = G[ii, jj]
        i_del_j, j_del_i = pair_predicates(phase, c, a[ii], b[ii], a[jj], b[jj])
        np.add.at(hits, jj[i_del_j], 1)
        np.add.at(hits, ii[j_del_i], 1)
    return hits


def sharded_kernelize(csr, rule: str, rank: int, world: int, allreduce):
    """Host model of kernelize_device (mhsk_capi.cu) on one rank."""
    n, m = csr.n, csr.m
    dense = np.zeros((m, n), dtype=np.int8)
    rows = np.repeat(np.arange(m), np.diff(csr.edge_ptr))
    dense[rows, csr.edge_vtx] = 1
    va = np.ones(n, bool)
    ea = np.ones(m, bool)
    rounds = 0
    while True:
        rounds += 1
        X = dense[np.ix_(ea, va)]
        eids = np.nonzero(ea)[0]
        if len(eids):
            hits = allreduce(phase_hits(X, X.sum(1), csr.demand[eids].astype(np.int64), rule, rank, world))
            del_e = eids[hits > 0]
            ea[del_e] = False
        else:
            del_e = []
        XV = dense[np.ix_(ea, va)].T
        vids = np.nonzero(va)[0]
        if len(vids):
            dem = csr.demand[np.nonzero(ea)[0]].astype(np.int64)
            need = np.where(XV.any(1), (XV * dem[None, :]).max(1) if XV.shape[1] else 0, 0)
            hits = allreduce(phase_hits(XV, XV.sum(1), np.zeros(len(vids), np.int64), "md", rank, world))
            dele = vids[(need == 0) | (hits >= need)]
            va[dele] = False
        else:
            dele = []
        if len(del_e) == 0 and len(dele) == 0:
            break
    return va.astype(np.uint8), ea.astype(np.uint8), rounds


INSTANCES = [
    lambda: interval_trains(900, 500, 1, 3),
    lambda: plant_twins(random_csr(400, 520, 0.03, 2, 4), 0.05, 0.05, 5),
    lambda: nested_chains(6, 20, 3, 6),
]


def _worker(rank: int, world: int, port: int, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def allreduce(h: np.ndarray) -> np.ndarray:
        t = torch.from_numpy(h.astype(np.int64))
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t.numpy()

    out = []
    for make in INSTANCES:
        csr = make()
        for rule in ("dp", "se"):
            va, ea, rounds = sharded_kernelize(csr, rule, rank, world, allreduce)
            out.append((va.tolist(), ea.tolist(), rounds))
    results[rank] = out
    dist.destroy_process_group()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2])
def test_two_rank_gloo_sharding_matches_oracle(world):
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    expected = []
    for make in INSTANCES:
        csr = make()
        for rule in ("dp", "se"):
            va, ea, rounds, *_ = oracle.kernelize(csr, rule)
            expected.append((va.tolist(), ea.tolist(), rounds))
    for r in range(world):
        assert results[r] == expected, f"rank {r} diverged"


def test_single_rank_model_matches_oracle():
    csr = interval_trains(700, 400, 3, 11)
    ident = lambda h: h  # noqa: E731
    va, ea, rounds = sharded_kernelize(csr, "dp", 0, 1, ident)
    ova, oea, orounds, *_ = oracle.kernelize(csr, "dp")
    assert np.array_equal(va, ova) and np.array_equal(ea, oea) and rounds == orounds


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_shares_partition_the_tile_list(world):
    for M in (1, 300, 5000, 100000):
        total = len(_native.tile_list(M, 256))
        covered = sorted(i for r in range(world) for i in shard_share(total, r, world))
        assert covered == list(range(total))
        # balanced for every shrunken M: tiles inside M split evenly
        tiles = _native.tile_list(M, 256)
        for M2 in (M // 2, M // 7):
            inside = tiles[:, 1] < -(-M2 // 256)
            per_rank = [int(inside[list(shard_share(total, r, world))].sum()) for r in range(world)]
            assert max(per_rank) - min(per_rank) <= max(2, sum(per_rank) // (4 * world) + 1)
