"""The B200 engine behind the reference's data-parallel API.

Same signatures, return types and error texts as the reference
(``pkg/src/mhskernel/parallel.py``):

* :func:`par_kernelize`        parallel.py:164-214
* :func:`par_reduce_edges`     parallel.py:80-116
* :func:`par_reduce_vertices`  parallel.py:119-161

``workers`` and ``use_matrix_product`` are accepted for drop-in
compatibility and do not change the result (the reference guarantees both
are result-neutral: test_parallel.py:111-129); every phase runs as a
tensor-core Gram product with the rule predicates fused into its epilogue
(libmhsk.so, include/mhsk.h).  There is no CPU fallback.
"""

from __future__ import annotations

import dataclasses
import importlib
import time
from typing import Sequence

import numpy as np

from . import _native
from .bitmatrix import matrix_csr
from .instance import CSRInstance, Hypergraph, as_csr, instance_size, validate_feasibility
from .report import KernelReport, KernelRun


def _check_rule(rule: str) -> None:
    if rule not in ("dp", "se"):
        raise ValueError(f"unknown edge rule {rule!r}")


def caller_types(h):
    """(Hypergraph, KernelRun, KernelReport) classes of the caller's own
    package when ``h`` is a foreign hypergraph -- e.g. the reference's
    ``mhskernel.Hypergraph`` (instance.py:32) -- so results compare equal
    with the caller's objects (test_parallel.py:87 checks
    ``run.hypergraph == Hypergraph(3, ((1, 2), (2, 3)), (2, 2))``).  The
    classes are looked up as ``<package>.report.KernelRun`` /
    ``KernelReport`` next to ``<package>.instance.Hypergraph``; None for this
    package's own types and CSR input, or when the caller's package has no
    such module."""
    cls = type(h)
    if isinstance(h, (Hypergraph, CSRInstance)) or not dataclasses.is_dataclass(cls):
        return None
    pkg = cls.__module__.rpartition(".")[0]
    try:
        rep = importlib.import_module(f"{pkg}.report") if pkg else None
    except ImportError:
        rep = None
    run_cls = getattr(rep, "KernelRun", None) if rep else None
    report_cls = getattr(rep, "KernelReport", None) if rep else None
    if not (dataclasses.is_dataclass(run_cls) and dataclasses.is_dataclass(report_cls)):
        run_cls = report_cls = None
    return cls, run_cls, report_cls


def to_caller_report(report: KernelReport, report_cls):
    """This package's report as the caller's KernelReport (same fields)."""
    if report_cls is None:
        return report
    names = {f.name for f in dataclasses.fields(report_cls)}
    out = report_cls(**{f.name: getattr(report, f.name) for f in dataclasses.fields(report)
                        if f.name in names})
    try:
        out.device_stats = report.device_stats
    except (AttributeError, dataclasses.FrozenInstanceError):
        pass
    return out


def to_caller_hypergraph(reduced: CSRInstance, h, types):
    """The compacted remainder in the input's kind: CSR for CSR input, the
    caller's Hypergraph class for a foreign hypergraph, else this package's."""
    if isinstance(h, CSRInstance):
        return reduced
    hg = reduced.to_hypergraph(trusted=True)
    if types is None:
        return hg
    return types[0](hg.n, hg.edges, hg.demand, hg.budget)


def extract(csr: CSRInstance, vertex_alive: np.ndarray, edge_alive: np.ndarray):
    """Order-preserving compaction of the survivors (ActiveInstance.extract,
    rules.py:88-103): returns (sub CSRInstance, vertex_ids, edge_ids) with
    1-based original ids."""
    va = np.asarray(vertex_alive, dtype=bool)
    ea = np.asarray(edge_alive, dtype=bool)
    vertex_ids = np.nonzero(va)[0]
    edge_ids = np.nonzero(ea)[0]
    new_id = np.full(csr.n, -1, dtype=np.int64)
    new_id[vertex_ids] = np.arange(len(vertex_ids))
    sizes = np.diff(csr.edge_ptr)
    owner = np.repeat(np.arange(csr.m), sizes)
    keep = ea[owner] & va[csr.edge_vtx] if csr.nnz else np.zeros(0, dtype=bool)
    new_vtx = new_id[csr.edge_vtx[keep]].astype(np.int32)
    counts = np.bincount(owner[keep], minlength=csr.m)[edge_ids] if csr.m else np.zeros(0, np.int64)
    ptr = np.zeros(len(edge_ids) + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr[1:])
    sub = CSRInstance(len(vertex_ids), ptr, new_vtx, csr.demand[edge_ids], csr.budget,
                      validate=False)
    return sub, vertex_ids + 1, edge_ids + 1


def kernelize_csr(csr: CSRInstance, *, rule: str = "dp", max_rounds: int = -1,
                  device: int | None = None):
    """CSR-level entry: returns (vertex_alive, edge_alive, stats dict)."""
    _check_rule(rule)
    ctx = _native.context(device)
    try:
        return ctx.kernelize(csr, rule, max_rounds)
    except _native.NativeError as exc:
        if exc.code == _native.MHSK_INFEASIBLE:
            raise ValueError(str(exc)) from None
        raise


def par_kernelize(h, *, rule: str = "dp", workers: int = 1, use_matrix_product: bool = False,
                  device: int | None = None) -> KernelRun:
    """Alternate edge and vertex phases on compacted matrices until a full
    round deletes nothing (reference parallel.py:164-214).  Demands are never
    modified.  Accepts a :class:`Hypergraph`, a :class:`CSRInstance`, or a
    reference ``mhskernel.Hypergraph``; the compacted result has the input's
    kind (CSR for CSR; for a foreign hypergraph the caller's own
    Hypergraph / KernelRun / KernelReport classes, see :func:`caller_types`)."""
    check = validate_feasibility(h)
    if not check:
        raise ValueError(f"instance is infeasible: {check.reason}")
    _check_rule(rule)
    csr = as_csr(h)
    report = KernelReport(n_before=csr.n, m_before=csr.m, size_before=instance_size(csr))
    started = time.perf_counter()
    va, ea, stats = kernelize_csr(csr, rule=rule, device=device)
    report.wall_times_ms["parallel-engine"] = (time.perf_counter() - started) * 1e3
    report.rounds = int(stats["rounds"])
    report.deleted_by_rule[rule] += int(stats["deleted_edges"])
    report.deleted_by_rule["md"] += int(stats["deleted_vertices"])
    report.device_stats = stats
    sub, vertex_ids, edge_ids = extract(csr, va, ea)
    report.n_after, report.m_after = sub.n, sub.m
    report.size_after = instance_size(sub)
    types = caller_types(h)
    reduced = to_caller_hypergraph(sub, h, types)
    run_cls = types[1] if types and types[1] else KernelRun
    return run_cls(reduced, to_caller_report(report, types[2] if types else None),
                   tuple(int(x) for x in vertex_ids), tuple(int(x) for x in edge_ids))


def par_reduce_edges(matrix, demand: Sequence[int], *, rule: str = "dp", workers: int = 1,
                     use_matrix_product: bool = False, device: int | None = None) -> list[bool]:
    """Keep-vector of one exhaustive edge phase (reference parallel.py:80-116)."""
    _check_rule(rule)
    if len(demand) != matrix.rows:
        raise ValueError("one demand per matrix row required")
    csr = matrix_csr(matrix, demand)
    keep = _native.context(device).reduce_edges(csr, rule)
    return [bool(k) for k in keep]


def par_reduce_vertices(matrix, demand: Sequence[int], *, workers: int = 1,
                        use_matrix_product: bool = False, device: int | None = None) -> list[bool]:
    """Keep-vector of one exhaustive vertex phase (reference parallel.py:119-161)."""
    if len(demand) != matrix.rows:
        raise ValueError("one demand per matrix row required")
    csr = matrix_csr(matrix, demand)
    keep = _native.context(device).reduce_vertices(csr)
    return [bool(k) for k in keep]
