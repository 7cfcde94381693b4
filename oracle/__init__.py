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
        L.oracle_csr_decide.argtypes = [_i32, _i32, _p, _p, _p, _p, _p, _i32, _i32, _p, _i64, _i32, _p]
        L.oracle_csr_decide.restype = ctypes.c_int
        L.oracle_csr_new.argtypes = [_i32, _i32, _p, _p, _p]
        L.oracle_csr_new.restype = _p
        L.oracle_csr_free.argtypes = [_p]
        L.oracle_csr_free.restype = None
        L.oracle_csr_decide_h.argtypes = [_p, _p, _p, _i32, _i32, _p, _i64, _i32, _p]
        L.oracle_csr_decide_h.restype = ctypes.c_int
        L.oracle_csr_kernelize.argtypes = [_i32, _i32, _p, _p, _p, _i32, _i32, _i32, _p, _p, _p, _p]
        L.oracle_csr_kernelize.restype = ctypes.c_int
        L.oracle_generate_random.argtypes = [_i32, _i32, ctypes.c_double, _i32, ctypes.c_uint64,
                                             _p, _p, _i64, _p, _p]
        L.oracle_generate_random.restype = _i64
        L.oracle_sample_new.argtypes = [_i32, _i32, _p, _p, _p, _i32, _i32]
        L.oracle_sample_new.restype = _p
        L.oracle_sample_decide.argtypes = [_p, _i32, _i64, _i64, _i32]
        L.oracle_sample_decide.restype = _i64
        L.oracle_sample_free.argtypes = [_p]
        L.oracle_sample_free.restype = None
        L.oracle_simd.argtypes = [ctypes.c_int]
        L.oracle_simd.restype = ctypes.c_int
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


class PhaseSample:
    """One round-1 phase of the bitset oracle with its operand built once
    (``build_s``): ``decide(j_lo, j_hi)`` runs the reference's per-item
    decisions for items [j_lo, j_hi) and returns the deletion count."""

    def __init__(self, csr, which: str, threads: int = 0):
        import time

        self._arr = _arrays(csr)
        ptr, vtx, dem = self._arr
        self.n, self.m = int(csr.n), len(ptr) - 1
        self.items = self.m if which == "edges" else self.n
        self.threads = threads
        t0 = time.perf_counter()
        self._h = lib().oracle_sample_new(self.n, self.m, _ptr(ptr), _ptr(vtx), _ptr(dem),
                                          0 if which == "edges" else 1, threads)
        self.build_s = time.perf_counter() - t0
        if not self._h:
            raise ValueError("oracle_sample_new failed")

    def decide(self, j_lo: int, j_hi: int, rule: str = "dp") -> int:
        r = lib().oracle_sample_decide(self._h, _RULES[rule], j_lo, min(j_hi, self.items), self.threads)
        if r < 0:
            raise ValueError("oracle sample failed")
        return int(r)

    def close(self):
        if getattr(self, "_h", None):
            lib().oracle_sample_free(self._h)
            self._h = None

    def __del__(self):
        self.close()


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


def simd(mode: int = -1) -> bool:
    """Select the AND+popcount kernel of the bitset oracle: -1 auto (AVX-512
    VPOPCNTDQ when the CPU has it), 0 scalar, 1 AVX-512 if available.
    Returns True when the AVX-512 kernel is in use."""
    return bool(lib().oracle_simd(mode))


def _mask(a, size):
    if a is None:
        return None
    out = np.ascontiguousarray(a, dtype=np.uint8)
    if len(out) < max(size, 1):
        out = np.concatenate([out, np.ones(max(size, 1) - len(out), np.uint8)])
    return out


def csr_decide(csr, which: str, items, rule: str = "dp", vertex_alive=None, edge_alive=None,
               threads: int = 0) -> np.ndarray:
    """Phase decisions (oracle_csr.c) for arbitrary items at full width:
    ``which`` "edges" (rule dp/se, parallel.py:80-116) or "vertices"
    (parallel.py:119-161), on the alive sub-instance given by the masks
    (None = all alive).  ``items`` are 0-based original ids; returns a bool
    keep array aligned with them."""
    ptr, vtx, dem = _arrays(csr)
    n, m = int(csr.n), len(ptr) - 1
    it = np.ascontiguousarray(items, dtype=np.int32)
    if len(it) == 0:
        return np.zeros(0, dtype=bool)
    keep = np.zeros(len(it), dtype=np.uint8)
    va, ea = _mask(vertex_alive, n), _mask(edge_alive, m)
    rc = lib().oracle_csr_decide(n, m, _ptr(ptr), _ptr(vtx), _ptr(dem),
                                 None if va is None else _ptr(va), None if ea is None else _ptr(ea),
                                 0 if which == "edges" else 1, _RULES[rule], _ptr(it), len(it),
                                 threads, _ptr(keep))
    if rc:
        raise ValueError(f"oracle error {rc}")
    return keep.astype(bool)


class CSROracle:
    """Persistent form of :func:`csr_decide` for many calls on one instance
    (the vertex -> edge index is built once)."""

    def __init__(self, csr):
        self._arr = _arrays(csr)
        self.n, self.m = int(csr.n), len(self._arr[0]) - 1
        ptr, vtx, dem = self._arr
        self._h = lib().oracle_csr_new(self.n, self.m, _ptr(ptr), _ptr(vtx), _ptr(dem))
        if not self._h:
            raise ValueError("oracle_csr_new failed (invalid CSR or out of memory)")

    def close(self):
        if getattr(self, "_h", None):
            lib().oracle_csr_free(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def decide(self, which: str, items, rule: str = "dp", vertex_alive=None, edge_alive=None,
               threads: int = 0) -> np.ndarray:
        it = np.ascontiguousarray(items, dtype=np.int32)
        if len(it) == 0:
            return np.zeros(0, dtype=bool)
        keep = np.zeros(len(it), dtype=np.uint8)
        va, ea = _mask(vertex_alive, self.n), _mask(edge_alive, self.m)
        rc = lib().oracle_csr_decide_h(self._h, None if va is None else _ptr(va),
                                       None if ea is None else _ptr(ea),
                                       0 if which == "edges" else 1, _RULES[rule], _ptr(it), len(it),
                                       threads, _ptr(keep))
        if rc:
            raise ValueError(f"oracle error {rc}")
        return keep.astype(bool)


def csr_kernelize(csr, rule: str = "dp", max_rounds: int = -1, threads: int = 0,
                  vertex_alive=None, edge_alive=None, round_log: bool = False):
    """Full fixpoint with CSR-counted phases (oracle_csr.c); same return as
    :func:`kernelize`, plus the per-item deletion round (edges then
    vertices, 0 = survived) when ``round_log``."""
    ptr, vtx, dem = _arrays(csr)
    n, m = int(csr.n), len(ptr) - 1
    va = np.ones(max(n, 1), dtype=np.uint8) if vertex_alive is None else _mask(vertex_alive, n).copy()
    ea = np.ones(max(m, 1), dtype=np.uint8) if edge_alive is None else _mask(edge_alive, m).copy()
    stats = np.zeros(3, dtype=np.int64)
    log = np.zeros(max(n + m, 1), dtype=np.int32) if round_log else None
    rc = lib().oracle_csr_kernelize(n, m, _ptr(ptr), _ptr(vtx), _ptr(dem), _RULES[rule], max_rounds,
                                    threads, _ptr(va), _ptr(ea), _ptr(stats),
                                    None if log is None else _ptr(log))
    if rc == 1:
        raise ValueError("instance is infeasible")
    if rc:
        raise ValueError(f"oracle error {rc}")
    out = (va[:n], ea[:m], int(stats[0]), int(stats[1]), int(stats[2]))
    return out + ((log[:m], log[m:m + n]),) if round_log else out


def generate_random(n: int, m: int, p: float, alpha: int, seed: int):
    """Counter-based instance of configs 4/5 on the host (oracle_gen.c):
    bit-identical to ``generate.counter_random`` and the device generator.
    Returns a ``CSRInstance``."""
    from paper_2109_06042_b200.instance import CSRInstance

    L = lib()
    ptr = np.zeros(m + 1, dtype=np.int64)
    attempt = np.zeros(max(m, 1), dtype=np.int32)
    nnz = L.oracle_generate_random(n, m, p, alpha, seed, _ptr(ptr), None, 0, None, _ptr(attempt))
    if nnz < 0:
        raise ValueError("invalid generator arguments")
    vtx = np.zeros(max(nnz, 1), dtype=np.int32)
    dem = np.zeros(max(m, 1), dtype=np.int32)
    r = L.oracle_generate_random(n, m, p, alpha, seed, _ptr(ptr), _ptr(vtx), len(vtx), _ptr(dem),
                                 _ptr(attempt))
    if r != nnz:
        raise ValueError("oracle generator failed")
    return CSRInstance(n, ptr, vtx[:nnz], dem[:m], validate=False)


def threads_available() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count() or 1
