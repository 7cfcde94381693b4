"""Shared test plumbing: markers, golden fixtures, instance builders."""

from __future__ import annotations

import gzip
import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C-ABI)")
    config.addinivalue_line("markers", "slow: multi-second CPU case")


def load_golden(name: str) -> list[dict]:
    with gzip.open(os.path.join(GOLDEN, f"{name}.json.gz"), "rt") as f:
        return json.load(f)["cases"]


def case_csr(case: dict):
    from paper_2109_06042_b200.instance import CSRInstance

    edges = case["edges"]
    ptr = np.zeros(len(edges) + 1, dtype=np.int64)
    np.cumsum([len(e) for e in edges], out=ptr[1:])
    vtx = np.array([v - 1 for e in edges for v in e], dtype=np.int32)
    return CSRInstance(case["n"], ptr, vtx, np.array(case["demand"], dtype=np.int32),
                       case.get("budget"), validate=False)


def case_hypergraph(case: dict):
    from paper_2109_06042_b200.instance import Hypergraph

    return Hypergraph(case["n"], tuple(tuple(e) for e in case["edges"]), tuple(case["demand"]),
                      case.get("budget"))


def small_cases() -> list[dict]:
    return load_golden("hand") + load_golden("sweeps") + load_golden("structured")


def pytest_collection_modifyitems(config, items):
    # GPU tests cannot run without a device: skip them loudly on CPU-only hosts
    # only when explicitly deselected is not the case (the driver selects -m gpu
    # on a B200 box and -m "not gpu" here).
    pass
