"""ctypes binding of libmhsk.so (the C ABI declared in include/mhsk.h).

There is no fallback: if the shared library is missing or no B200 is
visible, every entry point raises :class:`NativeUnavailable`.  The library
is built in-tree by ``__graft_entry__.build()`` (``make -C
paper_2109_06042_b200/csrc``).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MHSK_LIB=checked selects the bounds-checked build (make -C csrc checked:
# device assertions, tools/sanitize_run.py), MHSK_LIB=timing the Gram role
# counter build (make -C csrc timing, with MHSK_GRAM_TIMING=1); any other
# value is a path
_LIB_ENV = os.environ.get("MHSK_LIB", "")
LIB_PATH = (os.path.join(_HERE, f"libmhsk_{_LIB_ENV}.so") if _LIB_ENV in ("checked", "timing")
            else _LIB_ENV or os.path.join(_HERE, "libmhsk.so"))

MHSK_OK, MHSK_INFEASIBLE, MHSK_INVALID, MHSK_CUDA_ERROR, MHSK_OOM = 0, 1, 2, 3, 4
ABI_VERSION = 2   # include/mhsk.h MHSK_ABI_VERSION
RULES = {"dp": 0, "se": 1}
BACKENDS = {"tc": 0, "simt": 1, "tc1": 2}

EXPORTED = (
    "mhsk_create", "mhsk_destroy", "mhsk_set_backend", "mhsk_set_shard", "mhsk_kernelize",
    "mhsk_kernelize_device", "mhsk_reduce_edges", "mhsk_reduce_vertices", "mhsk_last_error",
    "mhsk_abi_version", "mhsk_device_sms", "mhsk_tile_list", "mhsk_tile_list_cols", "mhsk_run_pipeline",
    "mhsk_generate_random", "mhsk_generated_device", "mhsk_generated_copy",
    "mhsk_generate_random_host", "mhsk_parse_instance", "mhsk_instance_dims", "mhsk_instance_copy",
    "mhsk_instance_free", "mhsk_serialize_instance", "mhsk_set_option",
)
PHASE_CODES = {"fe": 0, "dp": 1, "se": 2, "md": 3}


class NativeUnavailable(RuntimeError):
    """libmhsk.so could not be loaded or has no usable device."""


class NativeError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"libmhsk error {code}: {message}")
        self.code = code


class Stats(ctypes.Structure):
    _fields_ = [
        ("rounds", ctypes.c_int64),
        ("deleted_edges", ctypes.c_int64),
        ("deleted_vertices", ctypes.c_int64),
        ("gram_launches", ctypes.c_int64),
        ("kernel_launches", ctypes.c_int64),
        ("gram_ops", ctypes.c_int64),
        ("executed_ops", ctypes.c_int64),
        ("h2d_bytes", ctypes.c_int64),
        ("d2h_bytes", ctypes.c_int64),
        ("ms_total", ctypes.c_double),
        ("ms_gram", ctypes.c_double),
        ("ms_pack", ctypes.c_double),
        ("ms_copy", ctypes.c_double),
        ("fp4_gram_launches", ctypes.c_int64),
        ("pruned_tiles", ctypes.c_int64),
        ("verified_pairs", ctypes.c_int64),
        ("spec_vertex", ctypes.c_int64),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class PipelineResult(ctypes.Structure):
    _fields_ = [
        ("passes", ctypes.c_int64),
        ("deleted", ctypes.c_int64 * 4),
        ("forced_vertices", ctypes.c_int64),
        ("infeasible", ctypes.c_int32),
        ("infeasible_edge", ctypes.c_int32),
        ("ms_by_phase", ctypes.c_double * 4),
    ]


ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                ctypes.c_void_p)

_lib = None
_lock = threading.Lock()


def load_library():
    """Load libmhsk.so and declare its signatures (no device needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(f"{LIB_PATH} is not built (run __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        p, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        L.mhsk_create.argtypes = [ctypes.c_int, ctypes.POINTER(p)]
        L.mhsk_destroy.argtypes = [p]
        L.mhsk_destroy.restype = None
        L.mhsk_set_backend.argtypes = [p, ctypes.c_int]
        L.mhsk_set_option.argtypes = [p, ctypes.c_char_p, i64]
        L.mhsk_set_shard.argtypes = [p, ctypes.c_int, ctypes.c_int, ALLREDUCE_FN, p]
        L.mhsk_kernelize.argtypes = [p, i32, i32, p, p, p, i32, i32, p, p, ctypes.POINTER(Stats)]
        L.mhsk_kernelize_device.argtypes = [p, i32, i32, p, p, p, i32, i32, p, p,
                                            ctypes.POINTER(Stats)]
        L.mhsk_reduce_edges.argtypes = [p, i32, i32, p, p, p, i32, p]
        L.mhsk_reduce_vertices.argtypes = [p, i32, i32, p, p, p, p]
        L.mhsk_last_error.restype = ctypes.c_char_p
        L.mhsk_abi_version.restype = ctypes.c_int
        L.mhsk_device_sms.argtypes = [p]
        L.mhsk_tile_list.argtypes = [i32, i32, i32, i32, p, i64]
        L.mhsk_tile_list.restype = i64
        L.mhsk_tile_list_cols.argtypes = [i32, i32, i32, i32, i32, p, i64]
        L.mhsk_tile_list_cols.restype = i64
        L.mhsk_generate_random.argtypes = [p, i32, i32, ctypes.c_double, i32, ctypes.c_uint64,
                                           ctypes.POINTER(i64)]
        L.mhsk_generated_device.argtypes = [p, ctypes.POINTER(p), ctypes.POINTER(p), ctypes.POINTER(p)]
        L.mhsk_generated_copy.argtypes = [p, p, p, p]
        L.mhsk_generate_random_host.argtypes = [i32, i32, ctypes.c_double, i32, ctypes.c_uint64, p, p,
                                                i64, p, p]
        L.mhsk_generate_random_host.restype = i64
        L.mhsk_parse_instance.argtypes = [ctypes.c_char_p, i64, ctypes.POINTER(p)]
        L.mhsk_instance_dims.argtypes = [p, ctypes.POINTER(i32), ctypes.POINTER(i32),
                                         ctypes.POINTER(i64), ctypes.POINTER(i32), ctypes.POINTER(i64)]
        L.mhsk_instance_copy.argtypes = [p, p, p, p]
        L.mhsk_instance_free.argtypes = [p]
        L.mhsk_instance_free.restype = None
        L.mhsk_serialize_instance.argtypes = [i32, i32, p, p, p, i32, i64, p, i64]
        L.mhsk_serialize_instance.restype = i64
        L.mhsk_run_pipeline.argtypes = [p, i32, i32, p, p, p, p, i32, i32, p, p, p,
                                        ctypes.POINTER(PipelineResult), ctypes.POINTER(Stats)]
        if L.mhsk_abi_version() != ABI_VERSION:   # Stats / PipelineResult layouts above
            raise NativeUnavailable(f"{LIB_PATH} has ABI {L.mhsk_abi_version()}, this binding {ABI_VERSION}"
                                    " (rebuild: __graft_entry__.build())")
        _lib = L
        return L


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _err(L) -> str:
    msg = L.mhsk_last_error()
    return msg.decode() if msg else ""


class Context:
    """One libmhsk context (CUDA stream + device buffers) on one device."""

    def __init__(self, device: int = 0, backend: str | None = None):
        L = load_library()
        self._L = L
        h = ctypes.c_void_p()
        rc = L.mhsk_create(int(device), ctypes.byref(h))
        if rc != MHSK_OK:
            raise NativeUnavailable(f"mhsk_create(device={device}) failed: {_err(L)}")
        self._h = h
        self.device = device
        self._allreduce_ref = None
        self.backend = backend or os.environ.get("MHSK_BACKEND", "tc")
        self.set_backend(self.backend)

    def close(self):
        if getattr(self, "_h", None):
            self._L.mhsk_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_backend(self, backend: str):
        if backend not in BACKENDS:
            raise ValueError(f"unknown backend {backend!r}; expected one of {sorted(BACKENDS)}")
        self._check(self._L.mhsk_set_backend(self._h, BACKENDS[backend]))
        self.backend = backend

    def set_option(self, key: str, value: int):
        """mhsk_set_option: A/B switches that never change results."""
        self._check(self._L.mhsk_set_option(self._h, key.encode(), int(value)))

    def set_shard(self, rank: int, world: int, allreduce=None):
        """allreduce(dev_ptr:int, count:int, stream:int) -> None sums int32s in place."""
        if world > 1 and allreduce is None:
            raise ValueError("world > 1 needs an allreduce callable")

        def _cb(buf, count, stream, user):
            try:
                allreduce(int(buf or 0), int(count), int(stream or 0))
                return 0
            except Exception:  # surfaced as MHSK_CUDA_ERROR by the library
                return 1

        self._allreduce_ref = ALLREDUCE_FN(_cb) if allreduce else ALLREDUCE_FN(0)
        self._check(self._L.mhsk_set_shard(self._h, rank, world, self._allreduce_ref, None))

    @property
    def sms(self) -> int:
        return int(self._L.mhsk_device_sms(self._h))

    def _check(self, rc: int):
        if rc == MHSK_OK:
            return
        msg = _err(self._L)
        if rc in (MHSK_INFEASIBLE, MHSK_INVALID):
            raise NativeError(rc, msg)
        raise NativeError(rc, msg)

    @staticmethod
    def _csr_arrays(csr):
        ptr = np.ascontiguousarray(csr.edge_ptr, dtype=np.int64)
        vtx = np.ascontiguousarray(csr.edge_vtx, dtype=np.int32)
        dem = np.ascontiguousarray(csr.demand, dtype=np.int32)
        if vtx.size == 0:
            vtx = np.zeros(1, dtype=np.int32)
        if dem.size == 0:
            dem = np.zeros(1, dtype=np.int32)
        return ptr, vtx, dem

    def kernelize(self, csr, rule: str = "dp", max_rounds: int = -1):
        ptr, vtx, dem = self._csr_arrays(csr)
        n, m = int(csr.n), len(ptr) - 1
        va = np.empty(max(n, 1), dtype=np.uint8)
        ea = np.empty(max(m, 1), dtype=np.uint8)
        st = Stats()
        rc = self._L.mhsk_kernelize(self._h, n, m, _ptr(ptr), _ptr(vtx), _ptr(dem), RULES[rule],
                                    int(max_rounds), _ptr(va), _ptr(ea), ctypes.byref(st))
        self._check(rc)
        return va[:n], ea[:m], st.as_dict()

    def kernelize_device(self, n: int, m: int, d_ptr: int, d_vtx: int, d_dem: int, d_valive: int,
                         d_ealive: int, rule: str = "dp", max_rounds: int = -1) -> dict:
        """Device-pointer variant (inputs resident in HBM, e.g. torch tensors'
        data_ptr()); fills the device alive arrays."""
        st = Stats()
        rc = self._L.mhsk_kernelize_device(self._h, int(n), int(m), ctypes.c_void_p(d_ptr),
                                           ctypes.c_void_p(d_vtx), ctypes.c_void_p(d_dem),
                                           RULES[rule], int(max_rounds), ctypes.c_void_p(d_valive),
                                           ctypes.c_void_p(d_ealive), ctypes.byref(st))
        self._check(rc)
        return st.as_dict()

    def generate_random(self, n: int, m: int, p: float, alpha: int, seed: int,
                        host: bool = True, pinned: bool = False):
        """Counter-based instance generated on the device (csrc/generate.cuh).
        Returns (CSRInstance on the host or None, (d_ptr, d_vtx, d_dem) device
        pointers owned by this context)."""
        nnz = ctypes.c_int64()
        self._check(self._L.mhsk_generate_random(self._h, int(n), int(m), float(p), int(alpha),
                                                 int(seed), ctypes.byref(nnz)))
        dp, dv, dd = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        self._check(self._L.mhsk_generated_device(self._h, ctypes.byref(dp), ctypes.byref(dv),
                                                  ctypes.byref(dd)))
        csr = None
        if host:
            from .instance import CSRInstance

            if pinned:
                import torch

                alloc = lambda k, dt: torch.empty(max(k, 1), dtype=dt).pin_memory().numpy()  # noqa: E731
                ptr, vtx, dem = alloc(m + 1, torch.int64), alloc(nnz.value, torch.int32), alloc(m, torch.int32)
            else:
                ptr = np.empty(m + 1, np.int64)
                vtx = np.empty(max(nnz.value, 1), np.int32)
                dem = np.empty(max(m, 1), np.int32)
            self._check(self._L.mhsk_generated_copy(self._h, _ptr(ptr), _ptr(vtx), _ptr(dem)))
            csr = CSRInstance(n, ptr[:m + 1], vtx[:nnz.value], dem[:m], validate=False)
        return csr, (dp.value or 0, dv.value or 0, dd.value or 0)

    def run_pipeline(self, csr, phases, loop: bool):
        """Generic phase loop on the device (mhsk_run_pipeline).  Returns
        (vertex_alive, edge_alive, adjusted demand, result dict, stats)."""
        ptr, vtx, dem = self._csr_arrays(csr)
        n, m = int(csr.n), len(ptr) - 1
        codes = np.array([PHASE_CODES[p] for p in phases], dtype=np.int32)
        va = np.empty(max(n, 1), dtype=np.uint8)
        ea = np.empty(max(m, 1), dtype=np.uint8)
        dem_out = np.empty(max(m, 1), dtype=np.int32)
        res = PipelineResult()
        st = Stats()
        rc = self._L.mhsk_run_pipeline(self._h, n, m, _ptr(ptr), _ptr(vtx), _ptr(dem), _ptr(codes),
                                       len(codes), int(bool(loop)), _ptr(va), _ptr(ea),
                                       _ptr(dem_out), ctypes.byref(res), ctypes.byref(st))
        self._check(rc)
        out = {"passes": res.passes,
               "deleted": {p: int(res.deleted[c]) for p, c in PHASE_CODES.items()},
               "forced_vertices": res.forced_vertices, "infeasible": bool(res.infeasible),
               "infeasible_edge": res.infeasible_edge,
               "ms_by_phase": {p: float(res.ms_by_phase[c]) for p, c in PHASE_CODES.items()}}
        return va[:n], ea[:m], dem_out[:m], out, st.as_dict()

    def reduce_edges(self, csr, rule: str = "dp") -> np.ndarray:
        ptr, vtx, dem = self._csr_arrays(csr)
        n, m = int(csr.n), len(ptr) - 1
        keep = np.empty(max(m, 1), dtype=np.uint8)
        self._check(self._L.mhsk_reduce_edges(self._h, n, m, _ptr(ptr), _ptr(vtx), _ptr(dem),
                                              RULES[rule], _ptr(keep)))
        return keep[:m]

    def reduce_vertices(self, csr) -> np.ndarray:
        ptr, vtx, dem = self._csr_arrays(csr)
        n, m = int(csr.n), len(ptr) - 1
        keep = np.empty(max(n, 1), dtype=np.uint8)
        self._check(self._L.mhsk_reduce_vertices(self._h, n, m, _ptr(ptr), _ptr(vtx), _ptr(dem),
                                                 _ptr(keep)))
        return keep[:n]


def tile_list(M: int, tile_rows: int = 256, gp: int = 4, gj: int = 9, tile_cols: int = 256) -> np.ndarray:
    """The library's Gram tile schedule for M items as an (T, 2) array of
    (I, J) block indices (tile_rows x tile_cols tiles -- 256 columns on int8
    operands, 240 on FP4; no device needed)."""
    L = load_library()
    total = L.mhsk_tile_list_cols(int(M), tile_rows, tile_cols, gp, gj, None, 0)
    if total < 0:
        raise ValueError(_err(L))
    buf = np.zeros(max(total, 1), dtype=np.uint32)
    L.mhsk_tile_list_cols(int(M), tile_rows, tile_cols, gp, gj, _ptr(buf), total)
    buf = buf[:total]
    return np.stack([buf & 0xFFFF, buf >> 16], axis=1).astype(np.int64)


def generate_random_host(n: int, m: int, p: float, alpha: int, seed: int):
    """Counter-based instance on the host (OpenMP C, libmhsk.so; no device
    needed) -- bit-identical to Context.generate_random and
    generate.counter_random."""
    from .instance import CSRInstance

    L = load_library()
    ptr = np.empty(m + 1, np.int64)
    attempt = np.empty(max(m, 1), np.int32)
    nnz = L.mhsk_generate_random_host(int(n), int(m), float(p), int(alpha), int(seed), _ptr(ptr),
                                      None, 0, None, _ptr(attempt))
    if nnz < 0:
        raise ValueError(_err(L))
    vtx = np.empty(max(nnz, 1), np.int32)
    dem = np.empty(max(m, 1), np.int32)
    if L.mhsk_generate_random_host(int(n), int(m), float(p), int(alpha), int(seed), _ptr(ptr),
                                   _ptr(vtx), int(nnz), _ptr(dem), _ptr(attempt)) < 0:
        raise ValueError(_err(L))
    return CSRInstance(n, ptr, vtx[:nnz], dem[:m], validate=False)


def parse_instance_text(text: str | bytes):
    """Native parser (mhsk_parse_instance).  Returns (CSRInstance, None) or
    (None, error message) -- the caller maps the message to InstanceError."""
    from .instance import CSRInstance

    L = load_library()
    data = text.encode() if isinstance(text, str) else bytes(text)
    h = ctypes.c_void_p()
    if L.mhsk_parse_instance(data, len(data), ctypes.byref(h)) != MHSK_OK:
        return None, _err(L)
    try:
        n, m, hb = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        nnz, budget = ctypes.c_int64(), ctypes.c_int64()
        L.mhsk_instance_dims(h, ctypes.byref(n), ctypes.byref(m), ctypes.byref(nnz), ctypes.byref(hb),
                             ctypes.byref(budget))
        ptr = np.empty(m.value + 1, np.int64)
        vtx = np.empty(max(nnz.value, 1), np.int32)
        dem = np.empty(max(m.value, 1), np.int32)
        L.mhsk_instance_copy(h, _ptr(ptr), _ptr(vtx), _ptr(dem))
    finally:
        L.mhsk_instance_free(h)
    return CSRInstance(n.value, ptr, vtx[:nnz.value], dem[:m.value],
                       budget.value if hb.value else None, validate=False), None


def serialize_instance_text(csr) -> str:
    L = load_library()
    ptr = np.ascontiguousarray(csr.edge_ptr, np.int64)
    vtx = np.ascontiguousarray(csr.edge_vtx, np.int32)
    dem = np.ascontiguousarray(csr.demand, np.int32)
    if vtx.size == 0:
        vtx = np.zeros(1, np.int32)
    if dem.size == 0:
        dem = np.zeros(1, np.int32)
    hb = csr.budget is not None
    args = (int(csr.n), int(csr.m), _ptr(ptr), _ptr(vtx), _ptr(dem), int(hb), int(csr.budget or 0))
    size = L.mhsk_serialize_instance(*args, None, 0)
    buf = ctypes.create_string_buffer(size + 1)
    L.mhsk_serialize_instance(*args, buf, size)
    return buf.raw[:size].decode()


_contexts: dict[int, Context] = {}


def context(device: int | None = None) -> Context:
    """Process-wide context for ``device`` (default: $MHSK_DEVICE or 0)."""
    if device is None:
        device = int(os.environ.get("MHSK_DEVICE", "0"))
    ctx = _contexts.get(device)
    if ctx is None:
        ctx = Context(device)
        _contexts[device] = ctx
    return ctx
