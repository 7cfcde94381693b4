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
    return (load_golden("hand") + load_golden("sweeps") + load_golden("structured")
            + load_golden("acceptance"))


_PLANTED: dict = {}


def planted_40k():
    """40k x 40k, p = 0.01, alpha = 3 (deg ~400) with planted deletions of
    both phases over 5 rounds (generate.plant_deletions): large enough for
    the default path to engage fully (FP4 probe, candidate verification,
    lazy operands, vertex candidates from the CSR, incremental rounds).
    Generated on the device; cached per process."""
    if "p40" not in _PLANTED:
        from paper_2109_06042_b200 import _native
        from paper_2109_06042_b200.generate import plant_deletions

        base, _ = _native.context().generate_random(40000, 40000, 0.01, 3, 71)
        _PLANTED["p40"] = plant_deletions(base, 72, dominated=60, twin_groups=30, dp_pairs=60,
                                          duplicates=60, chains=8, chain_len=3)
    return _PLANTED["p40"]


def pytest_collection_modifyitems(config, items):
    # GPU tests cannot run without a device: skip them loudly on CPU-only hosts
    # only when explicitly deselected is not the case (the driver selects -m gpu
    # on a B200 box and -m "not gpu" here).
    pass


STANDIN_INSTANCE = '''
from dataclasses import dataclass


@dataclass(frozen=True)
class Hypergraph:
    n: int
    edges: tuple
    demand: tuple
    budget: int | None = None
'''

STANDIN_REPORT = '''
from dataclasses import dataclass, field

from .instance import Hypergraph


@dataclass
class KernelReport:
    n_before: int = 0
    m_before: int = 0
    size_before: int = 0
    n_after: int = 0
    m_after: int = 0
    size_after: int = 0
    rounds: int = 0
    deleted_by_rule: dict = field(default_factory=lambda: dict.fromkeys(("fe", "dp", "se", "md", "lp"), 0))
    budget_delta: int = 0
    infeasible: bool = False
    bound_2_alpha_nabla: int | None = None
    matching_bound: int | None = None
    wall_times_ms: dict = field(default_factory=dict)


@dataclass
class KernelRun:
    hypergraph: Hypergraph
    report: KernelReport
    alive_vertices: tuple
    alive_edges: tuple
'''


def standin_package(tmp_path, monkeypatch, name: str = "refstandin"):
    """A stand-in for a foreign caller package shaped like the reference's
    mhskernel (instance.Hypergraph, report.KernelRun / KernelReport
    dataclasses); returns (instance module, report module)."""
    import importlib

    pkg = tmp_path / name
    pkg.mkdir()
    (pkg / "__init__.py").write_text("")
    (pkg / "instance.py").write_text(STANDIN_INSTANCE)
    (pkg / "report.py").write_text(STANDIN_REPORT)
    monkeypatch.syspath_prepend(str(tmp_path))
    return importlib.import_module(f"{name}.instance"), importlib.import_module(f"{name}.report")
