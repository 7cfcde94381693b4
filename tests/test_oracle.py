"""The CPU oracle (oracle/mhsk_oracle.c) against the reference's own outputs.

Pins the oracle before it is trusted as the at-scale parity checker and CPU
baseline: every golden case in tests/golden/ was produced by running the
reference (mhskernel.parallel, parallel.py:80-214) in the build container.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from conftest import case_csr, load_golden, small_cases

CASES = small_cases()


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_phases_match_reference(case):
    csr = case_csr(case)
    assert oracle.reduce_edges(csr, "dp") == case["keep_edges_dp"]
    assert oracle.reduce_edges(csr, "se") == case["keep_edges_se"]
    assert oracle.reduce_vertices(csr) == case["keep_vertices"]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
@pytest.mark.parametrize("rule", ["dp", "se"])
def test_oracle_kernelize_matches_reference(case, rule):
    csr = case_csr(case)
    want = case[f"kernelize_{rule}"]
    if "error" in want:
        if "budget" in want["error"]:
            pytest.skip("negative budget is checked by the host shim, not the oracle")
        with pytest.raises(ValueError):
            oracle.kernelize(csr, rule)
        return
    va, ea, rounds, de, dv = oracle.kernelize(csr, rule)
    assert [i + 1 for i in np.nonzero(va)[0]] == want["alive_vertices"]
    assert [i + 1 for i in np.nonzero(ea)[0]] == want["alive_edges"]
    assert rounds == want["rounds"]
    assert de == want["deleted_by_rule"][rule]
    assert dv == want["deleted_by_rule"]["md"]


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_oracle_thread_count_is_irrelevant(threads):
    # analogue of test_parallel.py:111-117 (worker counts agree)
    for case in load_golden("structured")[:6]:
        csr = case_csr(case)
        assert oracle.kernelize(csr, "dp", threads=threads)[2] == case["kernelize_dp"]["rounds"]


@pytest.mark.slow
def test_oracle_config1_matches_reference():
    from paper_2109_06042_b200.generate import generate_random
    from golden_io import csr_checksum

    case = load_golden("configs")[0]
    csr = generate_random(2000, 2000, 0.05, 1, 0).csr
    assert csr_checksum(csr) == case["checksum"]
    assert oracle.reduce_edges(csr, "dp") == case["keep_edges_dp"]
    assert oracle.reduce_vertices(csr) == case["keep_vertices"]
    va, ea, rounds, de, dv = oracle.kernelize(csr, "dp")
    want = case["kernelize_dp"]
    assert rounds == want["rounds"] and de == 0 and dv == 0
    assert [i + 1 for i in np.nonzero(va)[0]] == want["alive_vertices"]


@pytest.mark.slow
def test_oracle_config2_matches_reference():
    from paper_2109_06042_b200.generate import nested_chains
    from golden_io import csr_checksum

    case = load_golden("configs")[1]
    csr = nested_chains(100, 100, 3, 0)
    assert csr_checksum(csr) == case["checksum"]
    va, ea, rounds, de, dv = oracle.kernelize(csr, "dp")
    want = case["kernelize_dp"]
    assert rounds == want["rounds"]
    assert (de, dv) == (want["deleted_by_rule"]["dp"], want["deleted_by_rule"]["md"])
    assert [i + 1 for i in np.nonzero(va)[0]] == want["alive_vertices"]
    assert [i + 1 for i in np.nonzero(ea)[0]] == want["alive_edges"]


def test_decide_sample_counts_deletions():
    case = [c for c in load_golden("structured") if c["name"] == "c3_small"][0]
    csr = case_csr(case)
    keep = case["keep_edges_dp"]
    assert oracle.decide_sample(csr, "edges", 300) == sum(1 for k in keep[:300] if not k)
    keepv = case["keep_vertices"]
    assert oracle.decide_sample(csr, "vertices", 500) == sum(1 for k in keepv[:500] if not k)


PIPES = load_golden("pipelines")


@pytest.mark.parametrize("case", PIPES, ids=[c["name"] for c in PIPES])
def test_oracle_pipelines_match_reference(case):
    """oracle_run_pipeline (sequential fe cascade + phase loop) against the
    reference's run_pipeline (pipeline.py:95-171)."""
    from paper_2109_06042_b200.engine import extract

    csr = case_csr(case)
    for want in case["pipelines"]:
        rep = want["report"]
        if not case["edges"] and case["n"] == 0:
            continue
        if rep["infeasible"] and rep["rounds"] == 0:
            continue  # rejected up front by validate_feasibility (host)
        va, ea, dem, passes, deleted, forced, infeasible = oracle.run_pipeline(
            csr, want["phases"], want["loop"])
        assert passes == rep["rounds"], want["phases"]
        for k in ("fe", "dp", "se", "md"):
            assert deleted[k] == rep["deleted_by_rule"][k], (want["phases"], k)
        assert forced == rep["budget_delta"]
        from paper_2109_06042_b200.instance import CSRInstance

        adj = CSRInstance(csr.n, csr.edge_ptr, csr.edge_vtx, dem, csr.budget, validate=False)
        sub, _, _ = extract(adj, va, ea)
        red = sub.to_hypergraph()
        assert red.n == want["reduced_n"]
        assert [list(e) for e in red.edges] == want["reduced_edges"]
        assert list(red.demand) == want["reduced_demand"]
        budget = None if csr.budget is None else csr.budget - forced
        assert budget == want["reduced_budget"]
        assert (infeasible or (budget is not None and budget < 0)) == rep["infeasible"]
