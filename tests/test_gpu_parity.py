"""Parity of the CUDA path (through the C ABI) with the reference.

Small cases compare against the golden outputs of the reference itself
(tests/golden/, parallel.py:80-214); larger cases compare against the CPU
oracle (oracle/mhsk_oracle.c, itself pinned to the reference by
test_oracle.py) on the same seeded inputs; BASELINE-size runs check
size-independent properties (idempotence, exhaustiveness of the kernel,
determinism).  Bit-exact on every item: this is integer work.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from conftest import case_csr, case_hypergraph, load_golden, small_cases
from golden_io import csr_checksum
from paper_2109_06042_b200 import (
    CSRInstance,
    PipelineSpec,
    config_instance,
    generate_random,
    incidence_matrix,
    interval_trains,
    nested_chains,
    par_kernelize,
    par_reduce_edges,
    par_reduce_vertices,
    plant_twins,
    random_csr,
    run_pipeline,
)
from paper_2109_06042_b200 import _native

pytestmark = pytest.mark.gpu

CASES = small_cases()
FEASIBLE = [c for c in CASES if "error" not in c["kernelize_dp"]]


# function scope: a module-scoped parametrized fixture is torn down lazily, so
# the tests after the last "simt" user would silently run on the SIMT backend
@pytest.fixture(params=["tc", "tc1", "simt"])
def backend(request):
    ctx = _native.context()
    ctx.set_backend(request.param)
    yield request.param
    ctx.set_backend("tc")


def alive_ids(mask) -> list[int]:
    return [int(i) + 1 for i in np.nonzero(mask)[0]]


# ----------------------------------------------------- reference golden data
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_phase_keep_vectors_match_reference(case, backend):
    h = case_hypergraph(case)
    A = incidence_matrix(h)
    assert par_reduce_edges(A, h.demand) == case["keep_edges_dp"]
    assert par_reduce_edges(A, h.demand, rule="se") == case["keep_edges_se"]
    keep = par_reduce_vertices(A, h.demand)
    assert keep == case["keep_vertices"]
    assert all(type(k) is bool for k in keep)


@pytest.mark.parametrize("case", FEASIBLE, ids=[c["name"] for c in FEASIBLE])
@pytest.mark.parametrize("rule", ["dp", "se"])
def test_kernelize_matches_reference(case, rule, backend):
    h = case_hypergraph(case)
    run = par_kernelize(h, rule=rule)
    want = case[f"kernelize_{rule}"]
    assert list(run.alive_vertices) == want["alive_vertices"]
    assert list(run.alive_edges) == want["alive_edges"]
    assert run.report.rounds == want["rounds"]
    assert run.report.deleted_by_rule == want["deleted_by_rule"]
    assert run.hypergraph.n == want["reduced_n"]
    assert [list(e) for e in run.hypergraph.edges] == want["reduced_edges"]
    assert list(run.hypergraph.demand) == want["reduced_demand"]
    assert run.hypergraph.budget == want["reduced_budget"]
    assert (run.report.n_after, run.report.m_after, run.report.size_after) == \
        (want["n_after"], want["m_after"], want["size_after"])


def test_reference_known_answers():
    # test_parallel.py:75-92 fixpoints, restated
    ce = case_hypergraph([c for c in CASES if c["name"] == "ce"][0])
    run = par_kernelize(ce)
    assert run.alive_vertices == (1, 2, 3) and run.alive_edges == (1, 2)
    assert run.report.rounds == 3
    assert run.report.deleted_by_rule["md"] == 2 and run.report.deleted_by_rule["dp"] == 1
    assert run.hypergraph.edges == ((1, 2), (2, 3)) and run.hypergraph.demand == (2, 2)


@pytest.mark.parametrize("which", [0, 1])
def test_baseline_configs_1_and_2_match_reference(which):
    case = load_golden("configs")[which]
    csr = generate_random(2000, 2000, 0.05, 1, 0).csr if which == 0 else nested_chains(100, 100, 3, 0)
    assert csr_checksum(csr) == case["checksum"]
    run = par_kernelize(csr)
    want = case["kernelize_dp"]
    assert list(run.alive_vertices) == want["alive_vertices"]
    assert list(run.alive_edges) == want["alive_edges"]
    assert run.report.rounds == want["rounds"]
    assert run.report.deleted_by_rule == want["deleted_by_rule"]
    assert list(run.hypergraph.demand) == want["reduced_demand"]
    if "keep_edges_dp" in case:
        A = incidence_matrix(csr)
        assert par_reduce_edges(A, csr.demand.tolist()) == case["keep_edges_dp"]
        assert par_reduce_vertices(A, csr.demand.tolist()) == case["keep_vertices"]


# ------------------------------------------------------ oracle, larger sizes
def mixed_demand(inst: CSRInstance, seed: int) -> CSRInstance:
    """Demands drawn from 1..min(alpha, |e|): non-uniform over the packed
    rows, so the edge pack takes its need-array path instead of the
    uniform-demand seen map (mhsk_kernels.cuh pack_rows_csr)."""
    rng = np.random.default_rng(seed)
    sizes = np.diff(inst.edge_ptr)
    dem = np.minimum(rng.integers(1, 4, size=inst.m), np.maximum(sizes, 1)).astype(np.int32)
    return CSRInstance(inst.n, inst.edge_ptr, inst.edge_vtx, dem)


LARGER = [
    ("c1_mixed_demand", lambda: plant_twins(mixed_demand(random_csr(2000, 2000, 0.05, 3, 31), 32), 0.01, 0.01, 33)),
    ("sparse_mixed_demand", lambda: plant_twins(mixed_demand(random_csr(3000, 2500, 0.003, 3, 34), 35), 0.02, 0.05, 36)),
    ("c1_uniform_demand", lambda: plant_twins(random_csr(2000, 2000, 0.05, 3, 31), 0.01, 0.01, 33)),
    ("c1_twins", lambda: plant_twins(random_csr(2000, 2000, 0.05, 1, 5), 0.01, 0.01, 6)),
    ("c2_twins_a2", lambda: nested_chains(40, 60, 2, 3, dup_frac=0.1)),
    ("c3_quarter", lambda: interval_trains(12500, 5000, 1, 7)),
    ("c3a3_quarter", lambda: interval_trains(12500, 5000, 3, 7)),
    ("dense_small", lambda: random_csr(700, 900, 0.6, 5, 3)),
    ("tall", lambda: plant_twins(random_csr(300, 5000, 0.02, 2, 8), 0.02, 0.02, 9)),
    ("wide", lambda: plant_twins(random_csr(6000, 400, 0.01, 3, 10), 0.02, 0.05, 11)),
    ("ragged_tiles", lambda: plant_twins(random_csr(257, 383, 0.1, 2, 12), 0.05, 0.05, 13)),
]


@pytest.mark.parametrize("name,make", LARGER, ids=[n for n, _ in LARGER])
@pytest.mark.parametrize("rule", ["dp", "se"])
def test_kernelize_matches_oracle(name, make, rule):
    csr = make()
    va, ea, rounds, de, dv = oracle.kernelize(csr, rule)
    run = par_kernelize(csr, rule=rule)
    assert list(run.alive_vertices) == alive_ids(va)
    assert list(run.alive_edges) == alive_ids(ea)
    assert run.report.rounds == rounds
    assert run.report.deleted_by_rule[rule] == de and run.report.deleted_by_rule["md"] == dv


@pytest.mark.parametrize("name,make", LARGER[:4], ids=[n for n, _ in LARGER[:4]])
def test_phases_match_oracle(name, make):
    csr = make()
    ctx = _native.context()
    for rule in ("dp", "se"):
        assert ctx.reduce_edges(csr, rule).astype(bool).tolist() == oracle.reduce_edges(csr, rule)
    assert ctx.reduce_vertices(csr).astype(bool).tolist() == oracle.reduce_vertices(csr)


def test_backends_agree_on_structured_instance():
    csr = interval_trains(4000, 1600, 1, 21)
    ctx = _native.context()
    out = {}
    for b in ("tc", "tc1", "simt"):
        ctx.set_backend(b)
        out[b] = ctx.kernelize(csr)
    ctx.set_backend("tc")
    for b in ("tc1", "simt"):
        assert np.array_equal(out["tc"][0], out[b][0]) and np.array_equal(out["tc"][1], out[b][1])
        assert out["tc"][2]["rounds"] == out[b][2]["rounds"]


# ------------------------------------------- size-independent properties
@pytest.mark.parametrize("name", ["c3", "c3a3", "c2"])
def test_kernel_is_idempotent_at_config_size(name):
    csr = config_instance(name, seed=1)
    run = par_kernelize(csr)
    again = par_kernelize(run.hypergraph)
    assert again.report.rounds == 1
    assert again.report.deleted_by_rule["dp"] == 0 and again.report.deleted_by_rule["md"] == 0
    # deterministic: a second run is bit-identical
    run2 = par_kernelize(csr)
    assert run2.alive_vertices == run.alive_vertices and run2.alive_edges == run.alive_edges


def test_config3_matches_oracle():
    csr = config_instance("c3", seed=0)
    va, ea, rounds, de, dv = oracle.kernelize(csr, "dp")
    run = par_kernelize(csr)
    assert list(run.alive_vertices) == alive_ids(va)
    assert list(run.alive_edges) == alive_ids(ea)
    assert run.report.rounds == rounds


def test_pipeline_b200_engine():
    csr = interval_trains(3000, 1200, 1, 4)
    red, rep = run_pipeline(csr, PipelineSpec(("dp", "md"), loop=True))
    run = par_kernelize(csr)
    assert rep.rounds == run.report.rounds and red.n == run.hypergraph.n
    # generic phase loop (one native phase per step) reaches the same kernel
    red2, rep2 = run_pipeline(csr, PipelineSpec(("dp", "md", "dp"), loop=True))
    va, ea, *_ = oracle.kernelize(csr, "dp")
    assert red.m == int(ea.sum())
    assert rep2.deleted_by_rule["dp"] + rep2.deleted_by_rule["md"] >= 1


def test_device_pointer_entry_point():
    import torch

    csr = nested_chains(20, 30, 3, 2)
    d_ptr = torch.from_numpy(csr.edge_ptr).cuda()
    d_vtx = torch.from_numpy(csr.edge_vtx).cuda()
    d_dem = torch.from_numpy(csr.demand).cuda()
    va = torch.empty(csr.n, dtype=torch.uint8, device="cuda")
    ea = torch.empty(csr.m, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    st = _native.context().kernelize_device(csr.n, csr.m, d_ptr.data_ptr(), d_vtx.data_ptr(),
                                            d_dem.data_ptr(), va.data_ptr(), ea.data_ptr())
    ova, oea, rounds, *_ = oracle.kernelize(csr)
    assert np.array_equal(va.cpu().numpy(), ova) and np.array_equal(ea.cpu().numpy(), oea)
    assert st["rounds"] == rounds and st["gram_launches"] == 2 * rounds


def test_invalid_csr_is_rejected():
    bad = CSRInstance(3, np.array([0, 2]), np.array([2, 1], np.int32), np.array([1], np.int32),
                      validate=False)
    with pytest.raises(_native.NativeError):
        _native.context().kernelize(bad)
    infeasible = CSRInstance(3, np.array([0, 1]), np.array([1], np.int32), np.array([2], np.int32),
                             validate=False)
    with pytest.raises(ValueError, match="infeasible"):
        from paper_2109_06042_b200 import kernelize_csr

        kernelize_csr(infeasible)


def test_large_instance_validation():
    """validate_csr on a host CSR of >= 2^24 members: the host-pointer call
    equals the device-pointer call, and a defect anywhere (first, middle,
    last edge; an offset beyond nnz) is reported with the reference's codes
    and the first infeasible edge, without reading outside the CSR."""
    import torch

    csr = random_csr(12000, 12000, 0.12, 3, 5)
    assert int(csr.edge_ptr[-1]) >= 1 << 24
    ctx = _native.context()
    va, ea, st = ctx.kernelize(csr)
    assert st["h2d_bytes"] == 12 * 12001 - 4 + 4 * int(csr.edge_ptr[-1])
    d_ptr = torch.from_numpy(np.asarray(csr.edge_ptr, np.int64)).cuda()
    d_vtx = torch.from_numpy(np.asarray(csr.edge_vtx, np.int32)).cuda()
    d_dem = torch.from_numpy(np.asarray(csr.demand, np.int32)).cuda()
    dva = torch.empty(csr.n, dtype=torch.uint8, device="cuda")
    dea = torch.empty(csr.m, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    dst = ctx.kernelize_device(csr.n, csr.m, d_ptr.data_ptr(), d_vtx.data_ptr(), d_dem.data_ptr(),
                               dva.data_ptr(), dea.data_ptr())
    assert np.array_equal(dva.cpu().numpy(), va) and np.array_equal(dea.cpu().numpy(), ea)
    assert dst["rounds"] == st["rounds"]
    ptr = np.asarray(csr.edge_ptr, np.int64)
    for e in (0, csr.m // 2 + 7, csr.m - 1):          # first, middle, last chunk
        vtx = np.array(csr.edge_vtx, np.int32)
        vtx[ptr[e] + 1] = vtx[ptr[e]]                  # not strictly increasing
        bad = CSRInstance(csr.n, ptr, vtx, csr.demand, validate=False)
        with pytest.raises(_native.NativeError, match="malformed") as ei:
            ctx.kernelize(bad)
        assert ei.value.code == _native.MHSK_INVALID
        dem = np.array(csr.demand, np.int32)
        dem[e] = ptr[e + 1] - ptr[e] + 1               # demands more than |e|
        dem[-1] = ptr[-1] - ptr[-2] + 1                # a later infeasible edge too
        inf = CSRInstance(csr.n, ptr, csr.edge_vtx, dem, validate=False)
        with pytest.raises(_native.NativeError, match=f"edge {e + 1} demands") as ei:
            ctx.kernelize(inf)
        assert ei.value.code == _native.MHSK_INFEASIBLE
    wild = ptr.copy()
    wild[csr.m // 3] = ptr[-1] + 10**9                 # offset beyond nnz: never dereferenced
    with pytest.raises(_native.NativeError, match="malformed"):
        ctx.kernelize(CSRInstance(csr.n, wild, csr.edge_vtx, csr.demand, validate=False))
    va2, ea2, _ = ctx.kernelize(csr)                   # the context is still usable
    assert np.array_equal(va2, va) and np.array_equal(ea2, ea)


# ------------------------------------------------------------ pipelines + FE
PIPES = load_golden("pipelines")


@pytest.mark.parametrize("case", PIPES, ids=[c["name"] for c in PIPES])
def test_pipelines_match_reference(case):
    """run_pipeline(engine="b200") == the reference's run_pipeline
    (pipeline.py:95-171, fe_pass rules.py:138-181) on every spec."""
    h = case_hypergraph(case)
    for want in case["pipelines"]:
        red, rep = run_pipeline(h, PipelineSpec(tuple(want["phases"]), loop=want["loop"]))
        got = rep.to_dict()
        got.pop("wall_times_ms")
        assert got == want["report"], want["phases"]
        assert red.n == want["reduced_n"]
        assert [list(e) for e in red.edges] == want["reduced_edges"]
        assert list(red.demand) == want["reduced_demand"]
        assert red.budget == want["reduced_budget"]


FE_LARGER = [
    ("trains_a3", lambda: interval_trains(12000, 5000, 3, 31)),
    ("chains_a3", lambda: nested_chains(50, 40, 3, 32)),
    ("twins_a2", lambda: plant_twins(random_csr(1500, 1200, 0.004, 2, 33), 0.03, 0.03, 34)),
]


@pytest.mark.parametrize("name,make", FE_LARGER, ids=[n for n, _ in FE_LARGER])
@pytest.mark.parametrize("phases", [("fe", "dp", "md"), ("fe",), ("dp", "md", "fe"), ("fe", "se", "md")])
def test_pipeline_fe_matches_oracle(name, make, phases):
    csr = make()
    va, ea, dem, passes, deleted, forced, infeasible = oracle.run_pipeline(csr, phases, True)
    gva, gea, gdem, res, _ = _native.context().run_pipeline(csr, phases, True)
    assert np.array_equal(gva, va) and np.array_equal(gea, ea)
    alive = ea.astype(bool)
    assert np.array_equal(gdem[alive], dem[alive])
    assert res["passes"] == passes and res["deleted"] == deleted
    assert res["forced_vertices"] == forced and res["infeasible"] == infeasible


# ------------------------------------------------ round-loop variants agree
VARIANT_INSTANCES = [
    ("trains_a1", lambda: interval_trains(12000, 5000, 1, 41)),
    ("trains_small", lambda: interval_trains(700, 300, 2, 46)),
    ("trains_ragged", lambda: interval_trains(2049, 1025, 1, 47, min_len=1, max_len=200)),
    ("trains_a3", lambda: interval_trains(12000, 5000, 3, 42)),
    ("chains", lambda: nested_chains(40, 50, 3, 43)),
    ("twins", lambda: plant_twins(random_csr(3000, 2600, 0.02, 2, 44), 0.02, 0.02, 45)),
]


@pytest.mark.parametrize("name,make", VARIANT_INSTANCES, ids=[n for n, _ in VARIANT_INSTANCES])
@pytest.mark.parametrize("rule", ["dp", "se"])
def test_incremental_and_fast_loop_match_oracle(name, make, rule):
    """Incremental rounds (affected x all rectangles), the device-resident
    loop and the host-driven loop all reproduce the oracle bit for bit."""
    csr = make()
    va, ea, rounds, de, dv = oracle.kernelize(csr, rule)
    ctx = _native.context()
    try:
        for inc, fast, sparse, fp4 in [(1, 1, -1, 1), (0, 1, 0, 1), (0, 0, 0, 1), (1, 0, 0, 1), (1, 1, 1, 1),
                                       (0, 1, 1, 1), (1, 1, 0, 1), (1, 1, 2, 1), (0, 1, 2, 1), (1, 1, 0, 0),
                                       (0, 1, 0, 0)]:
            ctx.set_option("incremental", inc)
            ctx.set_option("fast_loop", fast)
            ctx.set_option("sparse", sparse)
            ctx.set_option("fp4", fp4)
            gva, gea, st = ctx.kernelize(csr, rule)
            assert np.array_equal(gva, va) and np.array_equal(gea, ea), (inc, fast, sparse, fp4)
            assert st["rounds"] == rounds and st["deleted_edges"] == de and st["deleted_vertices"] == dv
        ctx.set_option("rect_rule", 1)   # rectangles up to half the items (dense)
        ctx.set_option("sparse", 0)
        gva, gea, st = ctx.kernelize(csr, rule)
        assert np.array_equal(gva, va) and np.array_equal(gea, ea), "rect_rule"
    finally:
        ctx.set_option("incremental", 1)
        ctx.set_option("fast_loop", 1)
        ctx.set_option("sparse", -1)
        ctx.set_option("fp4", 1)
        ctx.set_option("rect_rule", 0)


@pytest.mark.parametrize("name", ["c3", "c3a3"])
def test_sparse_mode_matches_dense_at_config_size(name):
    """Block-sparse mode (auto-selected for the interval configs) against the
    dense path and the CSR-counting oracle on the full-size instance."""
    csr = config_instance(name, seed=2)
    ctx = _native.context()
    try:
        ctx.set_option("sparse", 1)
        sva, sea, sst = ctx.kernelize(csr)
        ctx.set_option("sparse", 0)
        dva, dea, dst = ctx.kernelize(csr)
    finally:
        ctx.set_option("sparse", -1)
    assert np.array_equal(sva, dva) and np.array_equal(sea, dea)
    assert sst["rounds"] == dst["rounds"]
    assert_matches_csr_oracle(csr, "dp", (sva, sea, sst))


@pytest.mark.parametrize("name", ["c2", "c2-twins"])
def test_component_ordering_matches_dense_at_config_size(name):
    """Config 2 (shuffled nested chains) is block-diagonal by connected
    component: auto mode orders it by component and runs block-sparse (a
    fraction of the dense tensor work), with results identical to the dense
    path and the first-vertex sparse order."""
    csr = config_instance(name, seed=3)
    ctx = _native.context()
    out = {}
    try:
        for mode in (-1, 0, 1, 2):
            ctx.set_option("sparse", mode)
            out[mode] = ctx.kernelize(csr)
    finally:
        ctx.set_option("sparse", -1)
    for mode in (-1, 1, 2):
        assert np.array_equal(out[mode][0], out[0][0]) and np.array_equal(out[mode][1], out[0][1]), mode
        assert out[mode][2]["rounds"] == out[0][2]["rounds"]
    assert out[-1][2]["executed_ops"] * 4 < out[0][2]["executed_ops"]


@pytest.mark.parametrize("rule", ["dp", "se"])
def test_probe_pruning_matches_full_products(rule):
    """Probe pruning stops a dense tile after 1/16 of K when no pair can still
    fire.  Random 30k x 30k (p = 0.01) with planted duplicate edges / twin
    vertices: most tiles are pruned, the planted ones are not; results equal
    the unpruned products for FP4 and int8 operands, and the oracle's."""
    ctx = _native.context()
    base, _ = ctx.generate_random(30000, 30000, 0.01, 3, 81)
    csr = plant_twins(base, 0.002, 0.002, 82)
    out = {}
    try:
        for fp4 in (1, 0):
            for probe in (1, 0):
                ctx.set_option("fp4", fp4)
                ctx.set_option("probe", probe)
                out[fp4, probe] = ctx.kernelize(csr, rule)
    finally:
        ctx.set_option("fp4", 1)
        ctx.set_option("probe", 1)
    ref = out[1, 0]
    for key, (va, ea, st) in out.items():
        assert np.array_equal(va, ref[0]) and np.array_equal(ea, ref[1]), key
        assert st["rounds"] == ref[2]["rounds"], key
        if key[1]:
            assert st["pruned_tiles"] > 0, key
        else:
            assert st["pruned_tiles"] == 0, key
    assert ref[2]["deleted_edges"] > 0
    assert out[1, 1][2]["executed_ops"] < out[1, 0][2]["executed_ops"] / 3
    # and the CSR-counting oracle's full kernelization (~5 s on the box)
    assert_matches_csr_oracle(csr, rule, ref)


def assert_matches_csr_oracle(csr, rule, result):
    """The whole kernelization against oracle/oracle_csr.c (the reference's
    phases, parallel.py:80-214, counted from the CSR): alive sets and rounds."""
    va, ea, rounds, de, dv = oracle.csr_kernelize(csr, rule)
    assert np.array_equal(result[0].astype(bool), va.astype(bool))
    assert np.array_equal(result[1].astype(bool), ea.astype(bool))
    assert result[2]["rounds"] == rounds
    assert result[2]["deleted_edges"] == de and result[2]["deleted_vertices"] == dv


@pytest.mark.parametrize("rule", ["dp", "se"])
def test_candidate_verification_matches_full_tiles(rule):
    """Tiles whose probe leaves a few candidate pairs (planted duplicate edges
    / twin vertices) are decided by row-pair popcounts (verify.cuh) instead
    of a full-K tile: same results as full tiles (verify off) and as the
    unpruned products, for FP4 and int8 operands; vertex twins exercise the
    MD phase (need <= 1 via alpha = 1 edges)."""
    ctx = _native.context()
    base, _ = ctx.generate_random(20000, 20000, 0.01, 2, 91)
    csr = plant_twins(base, 0.003, 0.003, 92)
    out = {}
    try:
        for fp4 in (1, 0):
            ctx.set_option("fp4", fp4)
            for probe, verify in ((1, 1), (1, 0), (0, 0)):
                ctx.set_option("probe", probe)
                ctx.set_option("verify", verify)
                out[fp4, probe, verify] = ctx.kernelize(csr, rule)
    finally:
        ctx.set_option("fp4", 1)
        ctx.set_option("probe", 1)
        ctx.set_option("verify", 1)
    ref = out[1, 0, 0]
    for key, (va, ea, st) in out.items():
        assert np.array_equal(va, ref[0]) and np.array_equal(ea, ref[1]), key
        assert st["rounds"] == ref[2]["rounds"], key
        assert (st["verified_pairs"] > 0) == (key[2] == 1), key
    assert ref[2]["deleted_edges"] > 0
    # verified tiles skip their full-K pass
    assert out[1, 1, 1][2]["executed_ops"] < out[1, 1, 0][2]["executed_ops"]


def test_candidate_verification_matches_oracle():
    """Oracle check at a size where the probe runs in both phases and the
    planted pairs are verified, with vertex deletions (alpha = 1: need = 1)."""
    ctx = _native.context()
    base, _ = ctx.generate_random(8000, 8000, 0.02, 1, 93)
    csr = plant_twins(base, 0.004, 0.004, 94)
    va, ea, rounds, de, dv = oracle.kernelize(csr, "dp")
    for fp4 in (1, 0):
        try:
            ctx.set_option("fp4", fp4)
            gva, gea, st = ctx.kernelize(csr, "dp")
        finally:
            ctx.set_option("fp4", 1)
        assert np.array_equal(gva, va) and np.array_equal(gea, ea), fp4
        assert st["rounds"] == rounds and st["verified_pairs"] > 0, fp4
    assert de > 0 and dv > 0


@pytest.mark.parametrize("alpha", [1, 3])
def test_lazy_vertex_operand_matches_oracle(alpha):
    """Lazy operands (X_V -- and X_E -- packed only in their probe columns,
    undecided panels packed after the probe pass, need from the edge phase's
    CSR pass minus its deletions): equal to the eager operands and to the
    oracle, with and without candidate verification, FP4 and int8.  alpha = 1
    makes vertex twins deletable (need = 1); duplicate edges exercise the
    deleted-edge fix-up of degrees and need."""
    ctx = _native.context()
    base, _ = ctx.generate_random(9000, 9000, 0.02, alpha, 95 + alpha)
    csr = plant_twins(base, 0.004, 0.004, 97 + alpha)
    va, ea, rounds, de, dv = oracle.kernelize(csr, "dp")
    try:
        for fp4 in (1, 0):
            ctx.set_option("fp4", fp4)
            for lazy, lazy_e in ((1, 1), (1, 0), (0, 0)):   # lazy_e: X_E in probe columns too
                for verify in (1, 0):
                    ctx.set_option("lazy", lazy)
                    ctx.set_option("lazy_e", lazy_e)
                    ctx.set_option("verify", verify)
                    gva, gea, st = ctx.kernelize(csr, "dp")
                    key = (fp4, lazy, lazy_e, verify)
                    assert np.array_equal(gva, va) and np.array_equal(gea, ea), key
                    assert st["rounds"] == rounds, key
    finally:
        ctx.set_option("fp4", 1)
        ctx.set_option("lazy", 1)
        ctx.set_option("lazy_e", 1)
        ctx.set_option("verify", 1)
    assert de > 0 and (dv > 0 or alpha > 1)


@pytest.mark.parametrize("alpha", [1, 2])
def test_vertex_candidates_from_csr_match_oracle(alpha):
    """Vertex-phase candidate pairs counted from the CSR (vcand_*: hash of the
    pairs, one pass over the surviving edges) instead of transposing their
    panels: equal to the panel path and to the oracle; alpha = 1 makes twin
    vertices deletable, so the counted pairs decide deletions."""
    ctx = _native.context()
    base, _ = ctx.generate_random(9000, 9000, 0.02, alpha, 101 + alpha)
    csr = plant_twins(base, 0.004, 0.006, 103 + alpha)
    va, ea, rounds, de, dv = oracle.kernelize(csr, "dp")
    try:
        for fp4 in (1, 0):
            ctx.set_option("fp4", fp4)
            for vcsr in (1, 0):
                ctx.set_option("vcsr", vcsr)
                gva, gea, st = ctx.kernelize(csr, "dp")
                assert np.array_equal(gva, va) and np.array_equal(gea, ea), (fp4, vcsr)
                assert st["rounds"] == rounds and st["verified_pairs"] > 0, (fp4, vcsr)
    finally:
        ctx.set_option("fp4", 1)
        ctx.set_option("vcsr", 1)
    assert de > 0 and (dv > 0 or alpha > 1)


def test_probe_pruning_matches_oracle():
    """Oracle check with the edge phase probing (K = 12000: 94 int8 k-blocks,
    probe = the first 640 columns)."""
    ctx = _native.context()
    csr = plant_twins(random_csr(12000, 3000, 0.02, 3, 83), 0.01, 0.01, 84)
    va, ea, rounds, de, dv = oracle.kernelize(csr, "dp")
    try:
        ctx.set_option("fp4", 0)
        gva, gea, st = ctx.kernelize(csr, "dp")
    finally:
        ctx.set_option("fp4", 1)
    assert np.array_equal(gva, va) and np.array_equal(gea, ea)
    assert st["rounds"] == rounds and st["pruned_tiles"] > 0


def _prefix_rows(n, count, seed):
    from paper_2109_06042_b200.instance import CSRInstance

    rng = np.random.default_rng(seed)
    sizes = np.sort(rng.choice(np.arange(n // 20, n + 1), size=count, replace=False))
    rows = [np.arange(s, dtype=np.int32) for s in sizes]
    rows += [np.arange(int(s) - 1, dtype=np.int32) for s in sizes[::7]]   # one shorter
    ptr = np.zeros(len(rows) + 1, np.int64)
    ptr[1:] = np.cumsum([len(r) for r in rows])
    dem = np.minimum(3, [len(r) for r in rows]).astype(np.int32)
    return CSRInstance(n, ptr, np.concatenate(rows), dem, 10)


def test_fp4_counts_exact_for_long_rows():
    """FP4 operands accumulate in f32: counts stay exact (< 2^24).  Edges of
    up to 60k members nest as prefixes, so co-occurrence counts reach ~60k and
    pairs differ by one -- the DP / SE predicates hinge on exact equality.
    FP4 == int8 there; FP4 == the oracle on a 6k-vertex instance of the same
    shape."""
    csr = _prefix_rows(60000, 300, 5)
    ctx = _native.context()
    out = {}
    try:
        for fp4 in (1, 0):
            ctx.set_option("fp4", fp4)
            for rule in ("dp", "se"):
                out[fp4, rule] = ctx.kernelize(csr, rule)
    finally:
        ctx.set_option("fp4", 1)
    for rule in ("dp", "se"):
        a, b = out[1, rule], out[0, rule]
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), rule
        assert a[2]["rounds"] == b[2]["rounds"]
    small = _prefix_rows(6000, 200, 6)
    for rule in ("dp", "se"):
        va, ea, rounds, de, dv = oracle.kernelize(small, rule)
        gva, gea, st = ctx.kernelize(small, rule)
        assert np.array_equal(gva, va) and np.array_equal(gea, ea), rule
        assert st["rounds"] == rounds


def test_component_ordering_small_components_match_oracle():
    """Many tiny components plus isolated vertices, forced
    component order, both rules."""
    from paper_2109_06042_b200.instance import CSRInstance

    t = plant_twins(nested_chains(300, 7, 2, 71), 0.05, 0.05, 72)
    csr = CSRInstance(t.n + 5, t.edge_ptr, t.edge_vtx, t.demand, t.budget)   # + isolated vertices
    ctx = _native.context()
    try:
        ctx.set_option("sparse", 2)
        for rule in ("dp", "se"):
            va, ea, rounds, de, dv = oracle.kernelize(csr, rule)
            gva, gea, st = ctx.kernelize(csr, rule)
            assert np.array_equal(gva, va) and np.array_equal(gea, ea), rule
            assert st["rounds"] == rounds and st["deleted_edges"] == de and st["deleted_vertices"] == dv
    finally:
        ctx.set_option("sparse", -1)


def test_large_planted_instance_backends_agree_and_idempotent():
    """30k x 30k, p = 0.01 (9e6 incidences) with planted twins: the pair
    kernel (FP4 and int8 operands) and the single-CTA tensor-core kernel
    agree with each other and with the CSR-counting oracle, deletions are
    non-vacuous, and the kernel is a fixpoint."""
    from paper_2109_06042_b200.generate import counter_random

    ctx = _native.context()
    base, _ = ctx.generate_random(30000, 30000, 0.01, 3, 61)
    csr = plant_twins(base, 0.01, 0.01, 62)
    out = {}
    try:
        for b in ("tc", "tc1"):
            ctx.set_backend(b)
            out[b] = ctx.kernelize(csr)
        ctx.set_backend("tc")
        ctx.set_option("fp4", 0)
        out["i8"] = ctx.kernelize(csr)
    finally:
        ctx.set_backend("tc")
        ctx.set_option("fp4", 1)
    for other in ("tc1", "i8"):
        assert np.array_equal(out["tc"][0], out[other][0]) and np.array_equal(out["tc"][1], out[other][1])
    st = out["tc"][2]
    assert st["deleted_edges"] >= 290            # the planted duplicate edges
    assert_matches_csr_oracle(csr, "dp", out["tc"])
    from paper_2109_06042_b200 import extract

    sub, _, _ = extract(csr, out["tc"][0], out["tc"][1])
    va, ea, st2 = ctx.kernelize(sub)
    assert st2["rounds"] == 1 and st2["deleted_edges"] == 0 and st2["deleted_vertices"] == 0


def test_config3a3_half_size_matches_oracle():
    # the bitset oracle (oracle/mhsk_oracle.c) at half size (full size takes
    # it ~3 minutes on the box's CPU); the CSR-counting oracle checks the full
    # size in test_sparse_mode_matches_dense_at_config_size
    csr = interval_trains(25000, 10000, 3, 0)
    va, ea, rounds, de, dv = oracle.kernelize(csr, "dp")
    run = par_kernelize(csr)
    assert list(run.alive_vertices) == alive_ids(va)
    assert list(run.alive_edges) == alive_ids(ea)
    assert run.report.rounds == rounds


# ------------------------------------------ capacity overflows are exact
CAPS = [
    ({"cand_cap": 0}, "no candidate slots: every sparsely-firing tile runs full K"),
    ({"cand_cap": 37}, "the buffer overflows mid-launch: straddling warps mark their tiles"),
    ({"vcand_max": 0}, "vertex candidates always take the panel path"),
    ({"vcand_max": 16}, "CSR counting only for the short late-round lists"),
    ({"vcand_table_log2": 6}, "64-slot hash table at up to 50% load (long probe chains)"),
    ({"vcand_table_log2": 1}, "2-slot table: one pair at most"),
]


@pytest.mark.parametrize("opts,why", CAPS, ids=[next(iter(o)) + str(next(iter(o.values()))) for o, _ in CAPS])
@pytest.mark.parametrize("rule", ["dp", "se"])
def test_candidate_capacity_overflows_match_planted_sets(opts, why, rule):
    """Result-neutral capacity options force the overflow paths of the
    candidate buffer (gram_tc2.cuh cand_reserve: overflowing warps mark
    their tiles for the full-K pass) and of the vertex-candidate hash table
    / gate (verify.cuh: lists over the limit take the panel path): the
    kernelization still deletes exactly the planted sets (pinned against
    both oracles), round for round."""
    from conftest import planted_40k

    csr, planted = planted_40k()
    ctx = _native.context()
    base = ctx.kernelize(csr, rule)
    try:
        for k, v in opts.items():
            ctx.set_option(k, v)
        va, ea, st = ctx.kernelize(csr, rule)
    finally:
        ctx.set_option("cand_cap", 1 << 20)
        ctx.set_option("vcand_max", 1 << 15)
        ctx.set_option("vcand_table_log2", 17)
    assert {int(i) for i in np.nonzero(ea == 0)[0]} == set(planted.edges[rule]), why
    assert {int(i) for i in np.nonzero(va == 0)[0]} == set(planted.vertices), why
    assert st["rounds"] == planted.rounds[rule], why
    assert np.array_equal(va, base[0]) and np.array_equal(ea, base[1])
    if opts.get("cand_cap") == 0:
        assert st["verified_pairs"] == 0 and st["executed_ops"] > base[2]["executed_ops"]
    elif "cand_cap" in opts:
        assert 0 < st["verified_pairs"] < base[2]["verified_pairs"]


def test_capacity_options_are_validated():
    ctx = _native.context()
    for key, bad in (("cand_cap", -1), ("cand_cap", (1 << 20) + 1), ("vcand_max", 1 << 16),
                     ("vcand_table_log2", 0), ("vcand_table_log2", 18)):
        with pytest.raises(_native.NativeError):
            ctx.set_option(key, bad)


def test_device_api_rejects_null_members_and_bad_offsets():
    """mhsk_kernelize_device with a null member array under non-empty edges,
    or edge_ptr[0] != 0, returns MHSK_INVALID (validate_csr) instead of
    faulting; the context stays usable."""
    import torch

    csr = nested_chains(5, 6, 2, 1)
    ctx = _native.context()
    d_ptr = torch.from_numpy(csr.edge_ptr).cuda()
    d_vtx = torch.from_numpy(csr.edge_vtx).cuda()
    d_dem = torch.from_numpy(csr.demand).cuda()
    va = torch.empty(csr.n, dtype=torch.uint8, device="cuda")
    ea = torch.empty(csr.m, dtype=torch.uint8, device="cuda")
    with pytest.raises(_native.NativeError, match="malformed") as ei:
        ctx.kernelize_device(csr.n, csr.m, d_ptr.data_ptr(), 0, d_dem.data_ptr(), va.data_ptr(),
                             ea.data_ptr())
    assert ei.value.code == _native.MHSK_INVALID
    shifted = torch.from_numpy(csr.edge_ptr + 1).cuda()
    with pytest.raises(_native.NativeError, match="malformed"):
        ctx.kernelize_device(csr.n, csr.m, shifted.data_ptr(), d_vtx.data_ptr(), d_dem.data_ptr(),
                             va.data_ptr(), ea.data_ptr())
    st = ctx.kernelize_device(csr.n, csr.m, d_ptr.data_ptr(), d_vtx.data_ptr(), d_dem.data_ptr(),
                              va.data_ptr(), ea.data_ptr())
    ova, oea, rounds, *_ = oracle.kernelize(csr)
    assert np.array_equal(va.cpu().numpy(), ova) and np.array_equal(ea.cpu().numpy(), oea)
    assert st["rounds"] == rounds


def test_foreign_hypergraph_gets_the_callers_result_types(tmp_path, monkeypatch):
    """par_kernelize / run_pipeline on a foreign (reference-shaped)
    Hypergraph return the caller's own KernelRun / KernelReport /
    Hypergraph, so the reference's own assertion
    ``run.hypergraph == Hypergraph(3, ((1, 2), (2, 3)), (2, 2))``
    (test_parallel.py:87) holds when its tests are rebound to this engine."""
    from conftest import standin_package

    ri, rr = standin_package(tmp_path, monkeypatch)
    ce = ri.Hypergraph(5, ((1, 2), (2, 3, 4), (2, 3, 5)), (2, 2, 2))
    run = par_kernelize(ce)
    assert type(run) is rr.KernelRun and type(run.report) is rr.KernelReport
    assert run.hypergraph == ri.Hypergraph(3, ((1, 2), (2, 3)), (2, 2))
    assert run.alive_vertices == (1, 2, 3) and run.alive_edges == (1, 2) and run.report.rounds == 3
    red, rep = run_pipeline(ce, PipelineSpec(("dp", "md"), loop=True))
    assert red == run.hypergraph and type(rep) is rr.KernelReport
    red2, rep2 = run_pipeline(ce, PipelineSpec(("fe", "dp", "md"), loop=True))
    assert type(red2) is ri.Hypergraph and type(rep2) is rr.KernelReport


def test_fused_validation_at_scale():
    """Dense instances beyond 2^32 cells validate inside round 1's edge pack
    (scan_members + pack_rows_csr, one pass over the members) instead of a
    separate validate_csr pass -- through the host API with the member array
    streamed up in chunks (>= 2^24 members) that round 1 consumes as they
    land, and through the device API in one piece: the same codes, messages
    and first infeasible edge for every defect, without reading out of
    bounds; the context stays usable."""
    import torch

    ctx = _native.context()
    good, _ = ctx.generate_random(70000, 70000, 0.004, 3, 23)
    assert good.n * good.m > 1 << 32 and good.nnz / (good.n * good.m) > 1e-3
    assert good.nnz >= 2 << 23   # >= 2 upload chunks (STREAM_CHUNK)
    va, ea, st = ctx.kernelize(good)
    ptr = np.asarray(good.edge_ptr, np.int64)

    def expect(csr, code, match):
        with pytest.raises(_native.NativeError, match=match) as ei:
            ctx.kernelize(csr)
        assert ei.value.code == code
        d = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (csr.edge_ptr, csr.edge_vtx, csr.demand)]
        dva = torch.empty(csr.n, dtype=torch.uint8, device="cuda")
        dea = torch.empty(csr.m, dtype=torch.uint8, device="cuda")
        with pytest.raises(_native.NativeError, match=match) as ei:
            ctx.kernelize_device(csr.n, csr.m, d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(),
                                 dva.data_ptr(), dea.data_ptr())
        assert ei.value.code == code

    for e in (0, good.m // 2 + 3, good.m - 1):
        for kind in ("equal", "swap", "range", "far", "negative"):
            vtx = np.array(good.edge_vtx, np.int32)
            k = ptr[e] + 1
            if kind == "equal":
                vtx[k] = vtx[k - 1]
            elif kind == "swap":
                vtx[k], vtx[k - 1] = vtx[k - 1], vtx[k]
            elif kind == "range":
                vtx[ptr[e + 1] - 1] = good.n
            elif kind == "far":   # (edge 0: read by the speculative vertex probe before validation)
                vtx[ptr[e + 1] - 1] = 1 << 30
            else:
                vtx[ptr[e]] = -1
            expect(CSRInstance(good.n, ptr, vtx, good.demand, validate=False), _native.MHSK_INVALID, "malformed")
        dem = np.array(good.demand, np.int32)
        dem[e] = 0
        expect(CSRInstance(good.n, ptr, good.edge_vtx, dem, validate=False), _native.MHSK_INVALID, "malformed")
        dem = np.array(good.demand, np.int32)
        dem[e] = ptr[e + 1] - ptr[e] + 1
        dem[-1] = ptr[-1] - ptr[-2] + 1
        expect(CSRInstance(good.n, ptr, good.edge_vtx, dem, validate=False), _native.MHSK_INFEASIBLE,
               f"edge {e + 1} demands")
    # an empty edge (its start position is the next edge's): infeasible, not malformed
    e = good.m // 3
    keep = np.ones(good.nnz, bool)
    keep[ptr[e]:ptr[e + 1]] = False
    sizes = np.diff(ptr)
    sizes[e] = 0
    ptr2 = np.concatenate([[0], np.cumsum(sizes)])
    expect(CSRInstance(good.n, ptr2, good.edge_vtx[keep], good.demand, validate=False),
           _native.MHSK_INFEASIBLE, f"edge {e + 1} demands")
    for at in (1, good.m // 4):   # an offset beyond nnz is never dereferenced (edge 1: speculation)
        wild = ptr.copy()
        wild[at] = ptr[-1] + 10**9
        with pytest.raises(_native.NativeError, match="malformed"):
            ctx.kernelize(CSRInstance(good.n, wild, good.edge_vtx, good.demand, validate=False))
    va2, ea2, st2 = ctx.kernelize(good)
    assert np.array_equal(va2, va) and np.array_equal(ea2, ea) and st2["rounds"] == st["rounds"]
