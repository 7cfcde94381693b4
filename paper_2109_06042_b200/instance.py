"""Multiple Hitting Set instances: the hot path's input type.

Mirrors the reference's instance model (reference
``pkg/src/mhskernel/instance.py:32-212``) so that results compare field by
field: a :class:`Hypergraph` is ``n`` vertices ``1..n``, a tuple of edges
(each a strictly increasing tuple of 1-based vertex ids), one demand per edge
(``>= 1``) and an optional budget.  On top of that it exposes the CSR form the
native library consumes (:meth:`Hypergraph.csr`), and :class:`CSRInstance`
carries an instance that is too large for Python tuples (configs 3-5).
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property
from typing import Iterable

import numpy as np


class InstanceError(ValueError):
    """Malformed instance text; ``line_no`` is the 1-based offending line
    (reference instance.py:22-29)."""

    def __init__(self, message: str, line_no: int | None = None):
        super().__init__(message if line_no is None else f"line {line_no}: {message}")
        self.line_no = line_no


@dataclass(frozen=True)
class Hypergraph:
    """Immutable hypergraph with per-edge demands (reference instance.py:32-61)."""

    n: int
    edges: tuple[tuple[int, ...], ...]
    demand: tuple[int, ...]
    budget: int | None = None

    def __post_init__(self):
        if self.n < 0:
            raise ValueError("vertex count must be non-negative")
        if len(self.edges) != len(self.demand):
            raise ValueError("one demand per edge required")
        for idx, members in enumerate(self.edges, start=1):
            f = self.demand[idx - 1]
            if f < 1:
                raise ValueError(f"edge {idx}: demand must be positive, got {f}")
            if not all(a < b for a, b in zip(members, members[1:])):
                raise ValueError(f"edge {idx}: vertices must be strictly increasing")
            if members and (members[0] < 1 or members[-1] > self.n):
                raise ValueError(f"edge {idx}: vertex id out of range 1..{self.n}")

    @classmethod
    def from_edges(cls, n: int, edges: Iterable[Iterable[int]], demand: Iterable[int],
                   budget: int | None = None) -> "Hypergraph":
        """Sort each edge; reject repeated vertices inside an edge (duplicate
        edges are fine: the rules tie-break them)."""
        canon = []
        for idx, members in enumerate(edges, start=1):
            mem = tuple(sorted(members))
            if len(set(mem)) != len(mem):
                raise ValueError(f"edge {idx}: duplicate vertex")
            canon.append(mem)
        return cls(n, tuple(canon), tuple(demand), budget)

    @classmethod
    def from_csr(cls, n: int, edge_ptr, edge_vtx, demand, budget: int | None = None,
                 *, trusted: bool = False) -> "Hypergraph":
        """Build from 0-based CSR arrays (each edge's slice sorted ascending).
        ``trusted`` skips re-validation (engine outputs are valid by
        construction)."""
        ptr = np.asarray(edge_ptr, dtype=np.int64)
        vtx = (np.asarray(edge_vtx, dtype=np.int64) + 1).tolist()
        bounds = ptr.tolist()
        edges = tuple(tuple(vtx[a:b]) for a, b in zip(bounds, bounds[1:]))
        dem = tuple(np.asarray(demand).tolist())
        if not trusted:
            return cls(n, edges, dem, budget)
        h = object.__new__(cls)
        for k, v in (("n", int(n)), ("edges", edges), ("demand", dem), ("budget", budget)):
            object.__setattr__(h, k, v)
        return h

    @property
    def m(self) -> int:
        return len(self.edges)

    @cached_property
    def alpha(self) -> int:
        return max(self.demand, default=0)

    @cached_property
    def csr(self) -> "CSRInstance":
        """CSR arrays: ``edge_ptr`` int64[m+1], ``edge_vtx`` int32[nnz]
        (0-based), ``demand`` int32[m]."""
        sizes = np.fromiter((len(e) for e in self.edges), dtype=np.int64, count=self.m)
        ptr = np.zeros(self.m + 1, dtype=np.int64)
        np.cumsum(sizes, out=ptr[1:])
        flat = np.fromiter((v for e in self.edges for v in e), dtype=np.int32, count=int(ptr[-1]))
        return CSRInstance(self.n, ptr, flat - 1, np.asarray(self.demand, dtype=np.int32),
                           self.budget, validate=False)

    @cached_property
    def edge_bits(self) -> tuple[int, ...]:
        """Per edge, a Python-int bitset of its vertices (vertex j -> bit j-1)."""
        out = []
        for members in self.edges:
            bits = 0
            for v in members:
                bits |= 1 << (v - 1)
            out.append(bits)
        return tuple(out)

    @cached_property
    def vertex_edges(self) -> tuple[tuple[int, ...], ...]:
        """Per vertex, the increasing tuple of 1-based edge ids containing it."""
        inc: list[list[int]] = [[] for _ in range(self.n)]
        for i, members in enumerate(self.edges, start=1):
            for v in members:
                inc[v - 1].append(i)
        return tuple(tuple(x) for x in inc)


class CSRInstance:
    """An instance held as CSR numpy arrays (no per-edge Python objects).

    This is what the native library consumes; at configs 3-5 (up to 4e8
    incidences) it is the only practical host representation.
    """

    __slots__ = ("n", "edge_ptr", "edge_vtx", "demand", "budget")

    def __init__(self, n: int, edge_ptr, edge_vtx, demand, budget: int | None = None,
                 *, validate: bool = True):
        self.n = int(n)
        self.edge_ptr = np.ascontiguousarray(edge_ptr, dtype=np.int64)
        self.edge_vtx = np.ascontiguousarray(edge_vtx, dtype=np.int32)
        self.demand = np.ascontiguousarray(demand, dtype=np.int32)
        self.budget = budget
        if validate:
            self.validate()

    @property
    def m(self) -> int:
        return len(self.edge_ptr) - 1

    @property
    def nnz(self) -> int:
        return int(self.edge_ptr[-1]) if len(self.edge_ptr) else 0

    def sizes(self) -> np.ndarray:
        return np.diff(self.edge_ptr)

    def validate(self) -> None:
        if self.n < 0:
            raise ValueError("vertex count must be non-negative")
        if len(self.edge_ptr) < 1 or self.edge_ptr[0] != 0:
            raise ValueError("edge_ptr must start at 0")
        if len(self.demand) != self.m:
            raise ValueError("one demand per edge required")
        if np.any(np.diff(self.edge_ptr) < 0) or self.edge_ptr[-1] != len(self.edge_vtx):
            raise ValueError("edge_ptr must be non-decreasing and end at nnz")
        if self.m and np.any(self.demand < 1):
            bad = int(np.argmax(self.demand < 1))
            raise ValueError(f"edge {bad + 1}: demand must be positive, got {int(self.demand[bad])}")
        if len(self.edge_vtx) and (self.edge_vtx.min() < 0 or self.edge_vtx.max() >= self.n):
            raise ValueError(f"vertex id out of range 1..{self.n}")
        if len(self.edge_vtx) > 1:
            step = np.diff(self.edge_vtx.astype(np.int64))
            inner = np.ones(len(step), dtype=bool)
            inner[self.edge_ptr[1:-1][self.edge_ptr[1:-1] > 0] - 1] = False
            if np.any(step[inner] <= 0):
                raise ValueError("edge vertices must be strictly increasing")

    def to_hypergraph(self, trusted: bool = False) -> Hypergraph:
        return Hypergraph.from_csr(self.n, self.edge_ptr, self.edge_vtx, self.demand, self.budget,
                                   trusted=trusted)


def as_csr(h) -> CSRInstance:
    """CSR view of a :class:`Hypergraph`, a :class:`CSRInstance`, or any
    object with the reference Hypergraph's ``n``/``edges``/``demand``."""
    if isinstance(h, CSRInstance):
        return h
    if isinstance(h, Hypergraph):
        return h.csr
    return Hypergraph(h.n, tuple(tuple(e) for e in h.edges), tuple(h.demand),
                      getattr(h, "budget", None)).csr


def instance_size(h) -> int:
    """|H| = n + sum of edge sizes (reference instance.py:177-179)."""
    if isinstance(h, CSRInstance):
        return h.n + h.nnz
    return h.n + sum(len(e) for e in h.edges)


@dataclass(frozen=True)
class FeasibilityReport:
    feasible: bool
    reason: str | None = None
    edge: int | None = None

    def __bool__(self) -> bool:
        return self.feasible


def validate_feasibility(h) -> FeasibilityReport:
    """No edge may demand more hits than it has vertices; a negative budget
    is infeasible too (reference instance.py:199-212, same reason texts)."""
    budget = getattr(h, "budget", None)
    if budget is not None and budget < 0:
        return FeasibilityReport(False, reason=f"budget {budget} is negative")
    if isinstance(h, CSRInstance):
        sizes = h.sizes()
        bad = np.nonzero(h.demand > sizes)[0]
        if len(bad):
            i = int(bad[0])
            return FeasibilityReport(
                False, reason=f"edge {i + 1} demands {int(h.demand[i])} hits but has "
                              f"{int(sizes[i])} vertices", edge=i + 1)
        return FeasibilityReport(True)
    for i, (members, f) in enumerate(zip(h.edges, h.demand), start=1):
        if f > len(members):
            return FeasibilityReport(
                False, reason=f"edge {i} demands {f} hits but has {len(members)} vertices", edge=i)
    return FeasibilityReport(True)


def parse_instance(text: str) -> Hypergraph:
    """Parse ``p mhs <n> <m> [k]`` / ``e <demand> <v>...`` text (reference
    instance.py:114-165; same error texts and line numbers)."""
    header = None
    header_line = 0
    edges: list[tuple[int, ...]] = []
    demand: list[int] = []
    for line_no, raw in enumerate(text.splitlines(), start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        tok = line.split()
        if header is None:
            if tok[0] != "p" or not 4 <= len(tok) <= 5 or tok[1] != "mhs":
                raise InstanceError("expected header 'p mhs <n> <m> [k]'", line_no)
            try:
                nums = [int(t) for t in tok[2:]]
            except ValueError:
                raise InstanceError("non-integer field in header", line_no) from None
            if nums[0] < 0 or nums[1] < 0:
                raise InstanceError("vertex/edge counts must be non-negative", line_no)
            if len(nums) == 3 and nums[2] < 0:
                raise InstanceError("budget must be non-negative", line_no)
            header = (nums[0], nums[1], nums[2] if len(nums) == 3 else None)
            header_line = line_no
            continue
        if tok[0] != "e":
            raise InstanceError(f"expected edge line 'e <demand> <v1> ...', got {tok[0]!r}", line_no)
        if len(tok) < 2:
            raise InstanceError("edge line missing demand", line_no)
        try:
            vals = [int(t) for t in tok[1:]]
        except ValueError:
            raise InstanceError("non-integer field in edge line", line_no) from None
        if vals[0] < 1:
            raise InstanceError(f"demand must be positive, got {vals[0]}", line_no)
        seen: set[int] = set()
        for v in vals[1:]:
            if not 1 <= v <= header[0]:
                raise InstanceError(f"vertex {v} out of range 1..{header[0]}", line_no)
            if v in seen:
                raise InstanceError(f"duplicate vertex {v} in edge", line_no)
            seen.add(v)
        edges.append(tuple(sorted(vals[1:])))
        demand.append(vals[0])
    if header is None:
        raise InstanceError("missing header line")
    if len(edges) != header[1]:
        raise InstanceError(f"header declares {header[1]} edges but {len(edges)} found", header_line)
    return Hypergraph(header[0], tuple(edges), tuple(demand), header[2])


def parse_instance_csr(text: str) -> CSRInstance:
    """Native parser (libmhsk ``mhsk_parse_instance``):
    the reference format and error texts (instance.py:114-165), straight to
    CSR with no per-edge Python objects -- for instances too large for
    :func:`parse_instance`.  Raises :class:`InstanceError` with the line."""
    import re

    from ._native import parse_instance_text

    csr, err = parse_instance_text(text)
    if csr is None:
        m = re.match(r"line (\d+): (.*)$", err, re.S)
        if m:
            raise InstanceError(m.group(2), int(m.group(1)))
        raise InstanceError(err)
    return csr


def serialize_instance(h: Hypergraph) -> str:
    head = f"p mhs {h.n} {h.m}" + ("" if h.budget is None else f" {h.budget}")
    body = [f"e {f} " + " ".join(map(str, e)) if e else f"e {f}" for e, f in zip(h.edges, h.demand)]
    return "\n".join([head, *body]) + "\n"
