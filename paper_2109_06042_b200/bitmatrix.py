"""Bit-packed 0/1 incidence matrices (host-side format of the reference).

Same storage contract as the reference's ``IncidenceMatrix``
(``pkg/src/mhskernel/bitmatrix.py:21-130``): bit (i, j) is set iff vertex j
lies in edge i; words are little-endian 64-bit, packed along the larger
dimension ("column" orientation, one line of m edge bits per vertex, iff
n >= m; otherwise "row").  ``par_reduce_edges``/``par_reduce_vertices``
accept such a matrix and hand it to the device as CSR (:func:`matrix_csr`);
on the device the matrix is rebuilt as int8 K-major operand tiles.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property

import numpy as np

from .instance import CSRInstance, as_csr

WORD_BITS = 64


@dataclass(frozen=True)
class IncidenceMatrix:
    rows: int
    cols: int
    orientation: str  # "row" or "column"
    words: tuple[int, ...]

    def __post_init__(self):
        if self.orientation not in ("row", "column"):
            raise ValueError(f"unknown orientation {self.orientation!r}")

    @property
    def lines(self) -> int:
        return self.rows if self.orientation == "row" else self.cols

    @property
    def line_width(self) -> int:
        return self.cols if self.orientation == "row" else self.rows

    @property
    def words_per_line(self) -> int:
        return -(-self.line_width // WORD_BITS)

    def bit(self, i: int, j: int) -> bool:
        """Whether vertex ``j`` lies in edge ``i`` (both 1-based)."""
        if not (1 <= i <= self.rows and 1 <= j <= self.cols):
            raise IndexError(f"bit ({i}, {j}) outside {self.rows}x{self.cols} matrix")
        return bool(self.dense[i - 1, j - 1])

    @cached_property
    def dense(self) -> np.ndarray:
        """The matrix as a (rows, cols) uint8 0/1 array."""
        return dense_of(self)

    @cached_property
    def row_bitsets(self) -> tuple[int, ...]:
        return tuple(_to_int(r) for r in self.dense)

    @cached_property
    def col_bitsets(self) -> tuple[int, ...]:
        return tuple(_to_int(c) for c in self.dense.T)

    def row_popcount(self, i: int) -> int:
        return int(self.dense[i - 1].sum())

    def col_popcount(self, j: int) -> int:
        return int(self.dense[:, j - 1].sum())

    def total_bits(self) -> int:
        return int(self.dense.sum())


def _to_int(bits01: np.ndarray) -> int:
    packed = np.packbits(bits01.astype(np.uint8), bitorder="little")
    return int.from_bytes(packed.tobytes(), "little")


def dense_of(matrix) -> np.ndarray:
    """(rows, cols) uint8 0/1 array of any object with the reference
    IncidenceMatrix attributes (``rows``, ``cols``, ``orientation``, ``words``)."""
    rows, cols = int(matrix.rows), int(matrix.cols)
    lines = rows if matrix.orientation == "row" else cols
    width = cols if matrix.orientation == "row" else rows
    wpl = -(-width // WORD_BITS)
    if lines == 0 or width == 0:
        return np.zeros((rows, cols), dtype=np.uint8)
    words = np.array([int(w) for w in matrix.words], dtype=np.uint64).reshape(lines, wpl)
    bits = np.unpackbits(words.view(np.uint8), axis=1, bitorder="little")[:, :width]
    return np.ascontiguousarray(bits if matrix.orientation == "row" else bits.T)


def matrix_csr(matrix, demand) -> CSRInstance:
    """CSR instance (edges = matrix rows) of a packed incidence matrix."""
    d = dense_of(matrix)
    ptr = np.zeros(d.shape[0] + 1, dtype=np.int64)
    np.cumsum(d.sum(axis=1, dtype=np.int64), out=ptr[1:])
    vtx = np.nonzero(d)[1].astype(np.int32)
    return CSRInstance(d.shape[1], ptr, vtx, np.asarray(demand, dtype=np.int32), validate=False)


def incidence_matrix(h) -> IncidenceMatrix:
    """Packed incidence matrix of an instance (orientation rule of
    reference bitmatrix.py:113-130)."""
    c = as_csr(h)
    n, m = c.n, c.m
    d = np.zeros((m, n), dtype=np.uint8)
    if c.nnz:
        rows = np.repeat(np.arange(m), np.diff(c.edge_ptr))
        d[rows, c.edge_vtx] = 1
    orientation = "column" if n >= m else "row"
    lines = d if orientation == "row" else d.T
    width = lines.shape[1]
    wpl = -(-width // WORD_BITS)
    if lines.shape[0] == 0 or wpl == 0:
        return IncidenceMatrix(m, n, orientation, ())
    padded = np.zeros((lines.shape[0], wpl * WORD_BITS), dtype=np.uint8)
    padded[:, :width] = lines
    words = np.packbits(padded, axis=1, bitorder="little").view("<u8").reshape(-1)
    return IncidenceMatrix(m, n, orientation, tuple(int(w) for w in words))
