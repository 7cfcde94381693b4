"""Checksums that tie regenerated config instances to the golden outputs."""

from __future__ import annotations

import hashlib

import numpy as np


def csr_checksum(c) -> str:
    """Same digest as tests/golden/make_golden.py:csr_checksum."""
    h = hashlib.sha256()
    h.update(np.int64(c.n).tobytes())
    h.update(np.ascontiguousarray(c.edge_ptr, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(c.edge_vtx, dtype=np.int32).tobytes())
    h.update(np.ascontiguousarray(c.demand, dtype=np.int32).tobytes())
    return h.hexdigest()
