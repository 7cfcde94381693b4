"""CPU oracle for the kernelization hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this package.  The product path
(``paper_2109_06042_b200``) never does.

``mhsk_oracle.c`` restates the reference's ``parallel.py:80-214`` in C
(bitset AND + popcount, OpenMP over the decided index); this module is its
ctypes wrapper.  Parity of the oracle itself is pinned by
``tests/test_oracle.py`` against ``tests/golden/`` (outputs of the reference
run in this container by ``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libmhsk_oracle.so")
_lib = None

_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_p = ctypes.c_void_p


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.oracle_kernelize.argtypes = [_i32, _i32, _p, _p, _p, _i32, _i32, _i32, _p, _p, _p]
        L.oracle_kernelize.restype = ctypes.c_int
        L.oracle_reduce_edges.argtypes = [_i32, _i32, _p, _p, _p, _i32, _i32, _p]
        L.oracle_reduce_edges.restype = ctypes.c_int
        L.oracle_reduce_vertices.argtypes = [_i32, _i32, _p, _p, _p, _i32, _p]
        L.oracle_reduce_vertices.restype = ctypes.c_int
        L.oracle_decide_sample.argtypes = [_i32, _i32, _p, _p, _p, _i32, _i32, _i32, _i32]
        L.oracle_decide_sample.restype = _i64
        L.oracle_run_pipeline.argtypes = [_i32, _i32, _p, _p, _p, _p, _i32, _i32, _i32, _p, _p, _p]
        L.oracle_run_pipeline.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


_RULES = {"dp": 0, "se": 1}


def _arrays(csr):
    ptr = np.ascontiguousarray(csr.edge_ptr, dtype=np.int64)
    vtx = np.ascontiguousarray(csr.edge_vtx, dtype=np.int32)
    if len(vtx) == 0:
        vtx = np.zeros(1, dtype=np.int32)
    dem = np.ascontiguousarray(csr.demand, dtype=np.int32)
    if len(dem) == 0:
        dem = np.zeros(1, dtype=np.int32)
    return ptr, vtx, dem


def kernelize(csr, rule: str = "dp", max_rounds: int = -1, threads: int = 0):
    """Returns (vertex_alive u8[n], edge_alive u8[m], rounds, edge_deletions,
    vertex_deletions).  Raises ValueError on infeasible / invalid input."""
    ptr, vtx, dem = _arrays(csr)
    n, m = int(csr.n), len(ptr) - 1
    va = np.ones(max(n, 1), dtype=np.uint8)
    ea = np.ones(max(m, 1), dtype=np.uint8)
    stats = np.zeros(3, dtype=np.int64)
    rc = lib().oracle_kernelize(n, m, _ptr(ptr), _ptr(vtx), _ptr(dem), _RULES[rule], max_rounds,
                                threads, _ptr(va), _ptr(ea), _ptr(stats))
    if rc == 1:
        raise ValueError("instance is infeasible")
    if rc:
        raise ValueError(f"oracle error {rc}")
    return va[:n], ea[:m], int(stats[0]), int(stats[1]), int(stats[2])


def reduce_edges(csr, rule: str = "dp", threads: int = 0) -> list[bool]:
    ptr, vtx, dem = _arrays(csr)
    n, m = int(csr.n), len(ptr) - 1
    keep = np.zeros(max(m, 1), dtype=np.uint8)
    rc = lib().oracle_reduce_edges(n, m, _ptr(ptr), _ptr(vtx), _ptr(dem), _RULES[rule], threads,
                                   _ptr(keep))
    if rc:
        raise ValueError(f"oracle error {rc}")
    return [bool(x) for x in keep[:m]]


def reduce_vertices(csr, threads: int = 0) -> list[bool]:
    ptr, vtx, dem = _arrays(csr)
    n, m = int(csr.n), len(ptr) - 1
    keep = np.zeros(max(n, 1), dtype=np.uint8)
    rc = lib().oracle_reduce_vertices(n, m, _ptr(ptr), _ptr(vtx), _ptr(dem), threads, _ptr(keep))
    if rc:
        raise ValueError(f"oracle error {rc}")
    return [bool(x) for x in keep[:n]]


def decide_sample(csr, which: str, j_count: int, rule: str = "dp", threads: int = 0) -> int:
    """Run the reference's per-item decision for the first j_count items of
    round 1's edge ("edges") or vertex ("vertices") phase; returns the number
    of deletions among them."""
    ptr, vtx, dem = _arrays(csr)
    n, m = int(csr.n), len(ptr) - 1
    r = lib().oracle_decide_sample(n, m, _ptr(ptr), _ptr(vtx), _ptr(dem),
                                   0 if which == "edges" else 1, _RULES[rule], j_count, threads)
    if r < 0:
        raise ValueError("oracle sample failed")
    return int(r)


PHASE_CODES = {"fe": 0, "dp": 1, "se": 2, "md": 3}


def run_pipeline(csr, phases, loop: bool, threads: int = 0):
    """Generic phase loop (pipeline.py:130-161) incl. fe_pass's sequential
    cascade.  Returns (vertex_alive, edge_alive, demand, passes,
    {phase: deletions}, forced_vertices, infeasible)."""
    ptr, vtx, dem = _arrays(csr)
    dem = dem.copy()
    n, m = int(csr.n), len(ptr) - 1
    va = np.ones(max(n, 1), dtype=np.uint8)
    ea = np.ones(max(m, 1), dtype=np.uint8)
    codes = np.array([PHASE_CODES[p] for p in phases], dtype=np.int32)
    out = np.zeros(7, dtype=np.int64)
    rc = lib().oracle_run_pipeline(n, m, _ptr(ptr), _ptr(vtx), _ptr(dem), _ptr(codes), len(codes),
                                   int(loop), threads, _ptr(va), _ptr(ea), _ptr(out))
    if rc:
        raise ValueError(f"oracle error {rc}")
    deleted = {p: int(out[1 + c]) for p, c in PHASE_CODES.items()}
    return va[:n], ea[:m], dem[:m], int(out[0]), deleted, int(out[5]), bool(out[6])


def threads_available() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count() or 1
