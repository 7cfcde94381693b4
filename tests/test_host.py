"""CPU tests of the host side: instance model, packing, compaction, the
reference-facing error behaviour, generators, and the C-ABI library's
exported symbols.  No GPU compute is called here."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from conftest import REPO, case_csr, case_hypergraph, load_golden, small_cases
from paper_2109_06042_b200 import (
    CSRInstance,
    Hypergraph,
    IncidenceMatrix,
    InstanceError,
    KernelReport,
    PipelineSpec,
    extract,
    generate_random,
    incidence_matrix,
    instance_size,
    interval_trains,
    nested_chains,
    par_kernelize,
    par_reduce_edges,
    par_reduce_vertices,
    parse_instance,
    plant_twins,
    random_csr,
    serialize_instance,
    validate_feasibility,
)
from paper_2109_06042_b200 import _native
from paper_2109_06042_b200.bitmatrix import dense_of, matrix_csr

REF_SRC = "/root/reference/pkg/src"


def reference():
    """The reference package, importable only in the build container."""
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference not present (GPU box)")
    import sys

    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import mhskernel

    return mhskernel


CE_TEXT = "p mhs 5 3\ne 2 1 2\ne 2 2 3 4\ne 2 2 3 5\n"


# ------------------------------------------------------------ instance model
def test_hypergraph_validation_messages():
    with pytest.raises(ValueError, match="demand must be positive"):
        Hypergraph(2, ((1,),), (0,))
    with pytest.raises(ValueError, match="strictly increasing"):
        Hypergraph(3, ((2, 1),), (1,))
    with pytest.raises(ValueError, match="out of range"):
        Hypergraph(2, ((1, 3),), (1,))
    with pytest.raises(ValueError, match="one demand per edge"):
        Hypergraph(2, ((1,),), ())
    with pytest.raises(ValueError, match="duplicate vertex"):
        Hypergraph.from_edges(3, [[1, 1]], [1])


def test_parse_serialize_roundtrip_and_errors():
    h = parse_instance(CE_TEXT)
    assert h.n == 5 and h.edges == ((1, 2), (2, 3, 4), (2, 3, 5)) and h.demand == (2, 2, 2)
    assert parse_instance(serialize_instance(h)) == h
    with pytest.raises(InstanceError, match="line 1"):
        parse_instance("q mhs 1 1\n")
    with pytest.raises(InstanceError, match="out of range"):
        parse_instance("p mhs 2 1\ne 1 3\n")
    with pytest.raises(InstanceError, match="declares 2 edges"):
        parse_instance("p mhs 2 2\ne 1 1\n")


def test_csr_roundtrip():
    h = parse_instance(CE_TEXT)
    c = h.csr
    assert c.edge_ptr.tolist() == [0, 2, 5, 8]
    assert c.edge_vtx.tolist() == [0, 1, 1, 2, 3, 1, 2, 4]
    assert c.to_hypergraph() == h
    c.validate()
    with pytest.raises(ValueError):
        CSRInstance(3, [0, 2], [1, 1], [1])
    assert instance_size(h) == instance_size(c) == 5 + 8


def test_feasibility_reasons():
    assert validate_feasibility(parse_instance(CE_TEXT))
    bad = Hypergraph(1, ((1,),), (2,))
    r = validate_feasibility(bad)
    assert not r and r.reason == "edge 1 demands 2 hits but has 1 vertices"
    assert not validate_feasibility(bad.csr)
    assert validate_feasibility(Hypergraph(1, (), (), -1)).reason == "budget -1 is negative"


# -------------------------------------------------------------- bit packing
@pytest.mark.parametrize("case", load_golden("hand") + load_golden("sweeps")[:60],
                         ids=lambda c: c["name"])
def test_incidence_matrix_matches_reference_packing(case):
    ref = reference()
    h = case_hypergraph(case)
    mine = incidence_matrix(h)
    theirs = ref.incidence_matrix(ref.Hypergraph(h.n, h.edges, h.demand, h.budget))
    assert (mine.rows, mine.cols, mine.orientation) == (theirs.rows, theirs.cols, theirs.orientation)
    assert mine.words == theirs.words
    assert mine.row_bitsets == theirs.row_bitsets and mine.col_bitsets == theirs.col_bitsets


def test_wide_packing_and_matrix_csr():
    # > 64-bit lines (reference test_bitmatrix.py:45-55 analogue)
    h = generate_random(150, 90, 0.2, 2, 3)
    A = incidence_matrix(h)
    assert A.orientation == "column" and A.words_per_line == 2
    d = dense_of(A)
    for i, e in enumerate(h.edges):
        assert np.nonzero(d[i])[0].tolist() == [v - 1 for v in e]
        assert A.row_popcount(i + 1) == len(e)
    c = matrix_csr(A, h.demand)
    assert c.to_hypergraph() == h


# ---------------------------------------------------------------- compaction
@pytest.mark.parametrize("case", [c for c in small_cases() if "error" not in c["kernelize_dp"]],
                         ids=lambda c: c["name"])
def test_extract_reproduces_reference_reduced_instance(case):
    csr = case_csr(case)
    va, ea, *_ = oracle.kernelize(csr, "dp")
    sub, vids, eids = extract(csr, va, ea)
    want = case["kernelize_dp"]
    assert vids.tolist() == want["alive_vertices"] and eids.tolist() == want["alive_edges"]
    red = sub.to_hypergraph()
    assert red.n == want["reduced_n"]
    assert [list(e) for e in red.edges] == want["reduced_edges"]
    assert list(red.demand) == want["reduced_demand"]
    assert red.budget == want["reduced_budget"]
    assert instance_size(sub) == want["size_after"]


# ------------------------------------------------- reference error behaviour
def test_errors_raised_before_any_device_work():
    # infeasible / unknown rule / demand length (parallel.py:95-99,134-135,173-175)
    with pytest.raises(ValueError, match="instance is infeasible: edge 1 demands 2"):
        par_kernelize(Hypergraph(1, ((1,),), (2,)))
    with pytest.raises(ValueError, match="budget -1 is negative"):
        par_kernelize(Hypergraph(2, ((1, 2),), (1,), -1))
    h = Hypergraph.from_edges(3, [[1, 2], [1, 2, 3]], [1, 2])
    with pytest.raises(ValueError, match="unknown edge rule 'w2'"):
        par_reduce_edges(incidence_matrix(h), h.demand, rule="w2")
    with pytest.raises(ValueError, match="unknown edge rule"):
        par_kernelize(h, rule="w2")
    with pytest.raises(ValueError, match="one demand per matrix row required"):
        par_reduce_edges(incidence_matrix(h), (1,))
    with pytest.raises(ValueError, match="one demand per matrix row required"):
        par_reduce_vertices(incidence_matrix(h), (1, 2, 3))


def test_pipeline_spec_engine_names():
    assert PipelineSpec(("dp", "md"), loop=True).engine == "b200"
    with pytest.raises(ValueError):
        PipelineSpec(("dp",), engine="gpu")  # must stay invalid (test_pipeline.py:22-23)
    with pytest.raises(ValueError):
        PipelineSpec(())
    assert PipelineSpec(("fe", "dp", "md"), loop=True).phases == ("fe", "dp", "md")
    with pytest.raises(ValueError):
        PipelineSpec(("lp",))  # exact-oracle LP rule: out of scope for this engine


def test_report_key_order():
    r = KernelReport(wall_times_ms={"b": 1.0, "a": 2.0})
    d = r.to_dict()
    assert list(d) == ["n_before", "m_before", "size_before", "n_after", "m_after", "size_after",
                       "rounds", "deleted_by_rule", "budget_delta", "infeasible",
                       "bound_2_alpha_nabla", "matching_bound", "wall_times_ms"]
    assert list(d["deleted_by_rule"]) == ["fe", "dp", "se", "md", "lp"]
    assert list(d["wall_times_ms"]) == ["a", "b"]


# ----------------------------------------------------------------- generators
def test_generate_random_is_draw_identical_to_reference():
    ref = reference()
    for args in [(12, 9, 0.3, 2, 5), (40, 30, 0.05, 3, 11), (3, 8, 0.01, 1, 2)]:
        mine = generate_random(*args)
        theirs = ref.generate_random(*args)
        assert mine.edges == theirs.edges and mine.demand == theirs.demand


def test_structured_generators_are_valid_and_deterministic():
    for make in (lambda: nested_chains(7, 9, 3, 1), lambda: interval_trains(300, 120, 3, 2),
                 lambda: random_csr(400, 300, 0.03, 5, 4),
                 lambda: plant_twins(random_csr(200, 150, 0.05, 2, 1), 0.05, 0.05, 2)):
        a, b = make(), make()
        a.validate()
        assert np.array_equal(a.edge_ptr, b.edge_ptr) and np.array_equal(a.edge_vtx, b.edge_vtx)
        assert np.all(a.demand >= 1) and validate_feasibility(a)


def test_random_csr_density():
    c = random_csr(5000, 400, 0.01, 3, 9)
    assert abs(c.nnz / (5000 * 400) - 0.01) < 0.001
    assert np.all(c.demand == np.minimum(3, np.diff(c.edge_ptr)))


# ---------------------------------------------------------------- the C ABI
def header_symbols() -> list[str]:
    text = open(os.path.join(REPO, "include", "mhsk.h")).read()
    return sorted(set(re.findall(r"\b(mhsk_[a-z_]+)\s*\(", text)))


def test_c_abi_library_exports_every_header_symbol():
    L = _native.load_library()
    syms = header_symbols()
    assert set(syms) == set(_native.EXPORTED)
    for s in syms:
        assert hasattr(L, s), s
    assert L.mhsk_abi_version() == 2


def test_c_abi_without_device_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is present")
    with pytest.raises(_native.NativeUnavailable):
        _native.Context(0)


# ------------------------------------------------------------ the schedule
@pytest.mark.parametrize("M", [1, 239, 240, 241, 256, 480, 481, 1000, 5000, 40001])
@pytest.mark.parametrize("gp,gj", [(1 << 20, 1), (4, 9), (1, 1), (3, 5)])
def test_fp4_tile_list_covers_each_unordered_pair_once(M, gp, gj):
    """256 x 240 FP4 tiles (non-square): tile (I, J) is scheduled iff it holds
    a pair i < j, each exactly once, and every pair lies in one tile."""
    t = _native.tile_list(M, 256, gp, gj, tile_cols=240)
    MI, NJ = -(-M // 256), -(-M // 240)
    want = {(I, J) for J in range(NJ) for I in range(MI) if I * 256 <= J * 240 + 238}
    got = [tuple(x) for x in t.tolist()]
    assert len(got) == len(set(got)) and set(got) == want
    rng = np.random.default_rng(M)
    for i, j in [(0, M - 1), (M // 3, M // 2)] + [tuple(sorted(rng.integers(0, M, 2))) for _ in range(50)]:
        if i < j:
            hits = [(I, J) for I, J in got if I * 256 <= i < I * 256 + 256 and J * 240 <= j < J * 240 + 240]
            assert len(hits) == 1, (i, j)


@pytest.mark.parametrize("M", [1, 127, 128, 129, 255, 256, 257, 1000, 5000, 40001])
@pytest.mark.parametrize("rows", [128, 256])
@pytest.mark.parametrize("gp,gj", [(1 << 20, 1), (8, 9), (1, 1), (3, 5)])
def test_tile_list_covers_each_unordered_pair_once(M, rows, gp, gj):
    t = _native.tile_list(M, rows, gp, gj)
    R = 256 // rows
    MI, NJ = -(-M // rows), -(-M // 256)
    want = {(I, J) for J in range(NJ) for I in range(min(MI, R * J + R))}
    got = [tuple(x) for x in t.tolist()]
    assert len(got) == len(set(got)) and set(got) == want
    # every unordered pair {i<j} lies in exactly one scheduled tile
    for i, j in [(0, M - 1), (M // 3, M // 2), (max(0, M - 2), M - 1)]:
        if i < j:
            hits = [(I, J) for I, J in got if I * rows <= i < I * rows + rows and J * 256 <= j < J * 256 + 256]
            assert len(hits) == 1


def test_counter_generator_host_c_matches_numpy():
    from paper_2109_06042_b200.generate import counter_random

    for args in [(3000, 2000, 0.01, 3, 7), (50, 40, 1e-4, 2, 1), (5, 3, 1.0, 2, 1), (300, 0, 0.5, 1, 4)]:
        a, b = counter_random(*args), _native.generate_random_host(*args)
        assert np.array_equal(a.edge_ptr, b.edge_ptr) and np.array_equal(a.edge_vtx, b.edge_vtx)
        assert np.array_equal(a.demand, b.demand)
        b.validate()
    dense = counter_random(2000, 300, 0.05, 2, 3)
    assert abs(dense.nnz / (2000 * 300) - 0.05) < 0.005


# ------------------------------------------------------- native text parser
@pytest.mark.parametrize("case", load_golden("parse"), ids=lambda c: repr(c["text"])[:40])
def test_native_parser_matches_reference(case):
    from paper_2109_06042_b200.instance import parse_instance_csr

    if "error" in case:
        with pytest.raises(InstanceError) as exc:
            parse_instance_csr(case["text"])
        assert str(exc.value) == case["error"]
        assert exc.value.line_no == case["line_no"]
        with pytest.raises(InstanceError) as exc2:   # the Python restatement agrees too
            parse_instance(case["text"])
        assert str(exc2.value) == case["error"]
    else:
        csr = parse_instance_csr(case["text"])
        h = csr.to_hypergraph()
        assert (h.n, [list(e) for e in h.edges], list(h.demand), h.budget) == \
            (case["n"], case["edges"], case["demand"], case["budget"])
        assert parse_instance(case["text"]) == h


def test_native_serializer_roundtrip():
    from paper_2109_06042_b200._native import serialize_instance_text
    from paper_2109_06042_b200.instance import parse_instance_csr

    for h in [parse_instance(CE_TEXT), generate_random(40, 30, 0.2, 3, 4),
              Hypergraph(3, ((1, 2), ()), (1, 1), 5), Hypergraph(0, (), ())]:
        text = serialize_instance_text(h.csr)
        assert text == serialize_instance(h)
        back = parse_instance_csr(text)
        assert back.to_hypergraph() == h


def test_stats_struct_matches_header():
    """The ctypes mirror of mhsk_stats lists the header's fields in order with
    the same widths (the C ABI writes the whole struct)."""
    import re

    from paper_2109_06042_b200._native import Stats

    hdr = open(os.path.join(REPO, "include", "mhsk.h")).read()
    body = re.search(r"typedef struct mhsk_stats \{(.*?)\} mhsk_stats;", hdr, re.S).group(1)
    fields = re.findall(r"^\s*(int64_t|double)\s+(\w+);", body, re.M)
    ours = [(name, ctypes.sizeof(t)) for name, t in Stats._fields_]
    assert ours == [(name, 8) for _, name in fields]


def test_caller_types_of_a_foreign_hypergraph(tmp_path, monkeypatch):
    """Results are built in the caller's own classes for a foreign
    hypergraph (the reference's mhskernel.Hypergraph in a drop-in), so
    test_parallel.py:87's dataclass equality holds; this package's own and
    CSR inputs keep this package's types."""
    from conftest import standin_package
    from paper_2109_06042_b200.engine import caller_types, to_caller_hypergraph, to_caller_report
    from paper_2109_06042_b200.instance import CSRInstance, Hypergraph
    from paper_2109_06042_b200.report import KernelReport

    ri, rr = standin_package(tmp_path, monkeypatch)
    h = ri.Hypergraph(3, ((1, 2), (2, 3)), (2, 2))
    types = caller_types(h)
    assert types == (ri.Hypergraph, rr.KernelRun, rr.KernelReport)
    assert caller_types(Hypergraph(3, ((1, 2),), (1,))) is None
    csr = CSRInstance(3, np.array([0, 2, 4]), np.array([0, 1, 1, 2], np.int32), np.array([2, 2], np.int32))
    assert caller_types(csr) is None
    back = to_caller_hypergraph(csr, h, types)
    assert type(back) is ri.Hypergraph and back == h
    assert to_caller_hypergraph(csr, csr, None) is csr
    rep = KernelReport(n_before=5, rounds=3, device_stats={"x": 1})
    rep.deleted_by_rule["md"] = 2
    out = to_caller_report(rep, rr.KernelReport)
    assert type(out) is rr.KernelReport and out.rounds == 3 and out.deleted_by_rule["md"] == 2
    assert out.device_stats == {"x": 1}
    assert to_caller_report(rep, None) is rep
