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


# ------------------------------------------- CSR-counting oracle (at size)
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_csr_oracle_matches_reference(case):
    """oracle_csr.c (pair counts from the CSR, the reference's predicates)
    against the reference's own phase outputs and fixpoints."""
    csr = case_csr(case)
    assert oracle.csr_decide(csr, "edges", np.arange(csr.m), "dp").tolist() == case["keep_edges_dp"]
    assert oracle.csr_decide(csr, "edges", np.arange(csr.m), "se").tolist() == case["keep_edges_se"]
    assert oracle.csr_decide(csr, "vertices", np.arange(csr.n)).tolist() == case["keep_vertices"]
    for rule in ("dp", "se"):
        want = case[f"kernelize_{rule}"]
        if "error" in want:
            continue
        va, ea, rounds, de, dv = oracle.csr_kernelize(csr, rule)
        assert [i + 1 for i in np.nonzero(va)[0]] == want["alive_vertices"]
        assert [i + 1 for i in np.nonzero(ea)[0]] == want["alive_edges"]
        assert (rounds, de, dv) == (want["rounds"], want["deleted_by_rule"][rule],
                                    want["deleted_by_rule"]["md"])


def _masked_states(csr, rule):
    """The state before every phase of the bitset oracle's fixpoint."""
    states = []
    va = np.ones(csr.n, np.uint8)
    ea = np.ones(csr.m, np.uint8)
    for r in range(1, 8):
        va_r, ea_r, *_ = oracle.kernelize(csr, rule, max_rounds=r)
        states.append(("edges", va.copy(), ea.copy(), ea_r))
        states.append(("vertices", va.copy(), ea_r.copy(), va_r))
        if np.array_equal(va_r, va) and np.array_equal(ea_r, ea):
            break
        va, ea = va_r, ea_r
    return states


def test_csr_oracle_masked_phases_match_bitset_oracle():
    """Decisions on alive sub-instances (masks, original ids) equal the
    bitset oracle's phase-by-phase outcomes of a multi-round fixpoint."""
    from paper_2109_06042_b200 import plant_twins, random_csr

    for seed in range(3):
        csr = plant_twins(random_csr(600, 500, 0.03, 2, seed), 0.03, 0.03, seed + 9)
        chk = oracle.CSROracle(csr)
        for rule in ("dp", "se"):
            for which, va, ea, after in _masked_states(csr, rule):
                alive = np.nonzero((ea if which == "edges" else va))[0]
                keep = chk.decide(which, alive, rule, vertex_alive=va, edge_alive=ea)
                assert np.array_equal(keep, after[alive].astype(bool)), (seed, rule, which)


def test_oracle_generator_matches_numpy_statement():
    from paper_2109_06042_b200.generate import counter_random

    for args in [(300, 250, 0.03, 3, 7), (50, 400, 0.002, 2, 1), (1, 5, 0.5, 1, 3)]:
        a, b = oracle.generate_random(*args), counter_random(*args)
        assert np.array_equal(a.edge_ptr, b.edge_ptr) and np.array_equal(a.edge_vtx, b.edge_vtx)
        assert np.array_equal(a.demand, b.demand)


def test_simd_and_scalar_popcount_agree():
    from paper_2109_06042_b200 import plant_twins, random_csr

    csr = plant_twins(random_csr(900, 700, 0.04, 3, 4), 0.03, 0.03, 5)
    try:
        oracle.simd(0)
        scalar = oracle.kernelize(csr, "dp")
        oracle.simd(1)
        vec = oracle.kernelize(csr, "dp")
    finally:
        oracle.simd(-1)
    assert np.array_equal(scalar[0], vec[0]) and np.array_equal(scalar[1], vec[1])
    assert scalar[2:] == vec[2:]


# ----------------------------------------- planted deletions are exact
PLANTS = [(4000, 0.015, 3, 1), (5000, 0.012, 5, 2), (3000, 0.02, 1, 3), (4000, 0.015, 2, 4)]


@pytest.mark.parametrize("n,p,alpha,seed", PLANTS)
def test_planted_deletions_are_exact(n, p, alpha, seed):
    """generate.plant_deletions' by-construction deletion sets and rounds
    equal both oracles' fixpoints (so the GPU tests at configs 4/5 can assert
    them exactly)."""
    from paper_2109_06042_b200.generate import plant_deletions

    base = oracle.generate_random(n, n, p, alpha, seed)
    inst, planted = plant_deletions(base, seed + 10, dominated=20, twin_groups=10, dp_pairs=20,
                                    duplicates=20, chains=4, chain_len=3)
    inst.validate()
    assert (inst.n, inst.m) == (n, n)
    for rule in ("dp", "se"):
        va, ea, rounds, de, dv, (elog, vlog) = oracle.csr_kernelize(inst, rule, round_log=True)
        assert {int(i): int(elog[i]) for i in np.nonzero(elog)[0]} == planted.edges[rule]
        assert {int(i): int(vlog[i]) for i in np.nonzero(vlog)[0]} == planted.vertices
        assert rounds == planted.rounds[rule] == 5
        bva, bea, brounds, *_ = oracle.kernelize(inst, rule)
        assert np.array_equal(bva, va) and np.array_equal(bea, ea) and brounds == rounds
    assert len(planted.edges["dp"]) > len(planted.edges["se"]) or alpha == 1
