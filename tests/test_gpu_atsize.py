"""At-size parity for BASELINE configs 4 and 5 (n = m = 1e5 / 2e5, 1e8 /
4e8 incidences) and their planted variants, through the C ABI.

The headline path (FP4 probe, candidate verification, lazy operands, vertex
candidates from the CSR, incremental rounds) runs only at these sizes, and on
the plain random configs it deletes nothing.  So:

* ``-planted`` variants (generate.plant_deletions) carry deletions of both
  phases over several rounds whose sets are exact by construction (pinned
  against both oracles by tests/test_oracle.py): the GPU must delete exactly
  them, round by round (``max_rounds``), under both rules;
* each round's two phases are checked item by item against the CSR-counting
  oracle (oracle/oracle_csr.c, the reference's predicates,
  parallel.py:80-161) on every planted item, its partners, every item the GPU
  deleted and a random sample of the rest;
* the single-phase entry points (par_reduce_edges / par_reduce_vertices)
  are checked the same way at full size;
* the kernel is a fixpoint (idempotence, test_sequential.py:169-176) and
  exhaustive: the oracle keeps sampled survivors (test_parallel.py:154-164).
"""

from __future__ import annotations

import functools

import numpy as np
import pytest

import oracle
from paper_2109_06042_b200 import _native, extract
from paper_2109_06042_b200.generate import COUNTER_CONFIGS, plant_deletions, plant_twins

pytestmark = pytest.mark.gpu

NAMES = ["c4-planted", "c5-planted"]


@functools.lru_cache(maxsize=None)
def instance(name: str):
    base, _, variant = name.partition("-")
    csr, _ = _native.context().generate_random(*COUNTER_CONFIGS[base], 0)
    if variant == "planted":
        return plant_deletions(csr, 1)
    if variant == "twins":   # bench.py's c4-twins: 1% duplicated edges and twin vertices
        return plant_twins(csr, 0.01, 0.01, 1), None
    if variant == "vplanted":   # vertex deletions only: round 1's edge phase deletes nothing
        return plant_deletions(csr, 2, dp_pairs=0, duplicates=0, chains=0)
    return csr, None


@functools.lru_cache(maxsize=None)
def checker(name: str) -> oracle.CSROracle:
    return oracle.CSROracle(instance(name)[0])


def sample(rng, alive: np.ndarray, count: int) -> np.ndarray:
    ids = np.nonzero(alive)[0]
    return rng.choice(ids, size=min(count, len(ids)), replace=False) if len(ids) else ids


def check_phase(chk, which, rule, before_v, before_e, after, items):
    """GPU decisions of one phase (the items that died between `before` and
    `after`) against the oracle on the state before the phase."""
    items = np.unique(items)
    keep = chk.decide(which, items, rule, vertex_alive=before_v, edge_alive=before_e)
    gpu_keep = after[items].astype(bool)
    bad = items[keep != gpu_keep]
    assert len(bad) == 0, (which, rule, bad[:20].tolist(), int(len(bad)))


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("rule", ["dp", "se"])
def test_planted_round_by_round(name, rule):
    """Every round of the headline path deletes exactly the planted sets, and
    both of its phases agree with the oracle on >= 2,000 items (round 1)."""
    csr, planted = instance(name)
    ctx = _native.context()
    chk = checker(name)
    rng = np.random.default_rng(7)
    want_e = planted.edges[rule]
    want_v = planted.vertices
    rounds = planted.rounds[rule]
    assert rounds >= 3 and want_v and want_e
    va_prev = np.ones(csr.n, np.uint8)
    ea_prev = np.ones(csr.m, np.uint8)
    for r in range(1, rounds + 1):
        va, ea, st = ctx.kernelize(csr, rule, max_rounds=r)
        dead_e = {int(i) for i in np.nonzero(ea == 0)[0]}
        dead_v = {int(i) for i in np.nonzero(va == 0)[0]}
        assert dead_e == {e for e, k in want_e.items() if k <= r}, r
        assert dead_v == {v for v, k in want_v.items() if k <= r}, r
        assert st["rounds"] == r
        # round r's edge phase on the state after round r - 1, then its vertex
        # phase on that state minus the edges it deleted
        n_rand = 1500 if r == 1 else 300
        e_items = np.concatenate([planted.item_ids("edges"), sample(rng, ea_prev, n_rand),
                                  np.nonzero(ea_prev & ~ea)[0]])
        e_items = e_items[ea_prev[e_items] == 1]
        check_phase(chk, "edges", rule, va_prev, ea_prev, ea, e_items)
        v_items = np.concatenate([planted.item_ids("vertices"), sample(rng, va_prev, n_rand),
                                  np.nonzero(va_prev & ~va)[0]])
        v_items = v_items[va_prev[v_items] == 1]
        check_phase(chk, "vertices", rule, va_prev, ea, va, v_items)
        if r == 1:
            assert len(e_items) >= 2000 and len(v_items) >= 2000
        va_prev, ea_prev = va, ea
    va, ea, st = ctx.kernelize(csr, rule)
    assert st["rounds"] == rounds
    assert np.array_equal(va, va_prev) and np.array_equal(ea, ea_prev)
    assert st["deleted_edges"] == len(want_e) and st["deleted_vertices"] == len(want_v)
    assert st["pruned_tiles"] > 0 and st["verified_pairs"] > 0


@pytest.mark.parametrize("name", NAMES)
def test_planted_kernel_is_fixpoint_and_exhaustive(name):
    """Idempotence at full size (a second run: 1 round, 0 deletions) and
    exhaustiveness: the oracle keeps 1,000 sampled survivors of each kind on
    the kernel, in both phases."""
    csr, planted = instance(name)
    ctx = _native.context()
    va, ea, st = ctx.kernelize(csr, "dp")
    sub, _, _ = extract(csr, va, ea)
    va2, ea2, st2 = ctx.kernelize(sub, "dp")
    assert st2["rounds"] == 1 and st2["deleted_edges"] == 0 and st2["deleted_vertices"] == 0
    assert va2.all() and ea2.all()
    rng = np.random.default_rng(11)
    chk = checker(name)
    e_items = sample(rng, ea, 1000)
    assert chk.decide("edges", e_items, "dp", vertex_alive=va, edge_alive=ea).all()
    v_items = sample(rng, va, 1000)
    assert chk.decide("vertices", v_items, "dp", vertex_alive=va, edge_alive=ea).all()


@pytest.mark.parametrize("name", ["c4", "c4-planted", "c5", "c5-planted"])
def test_single_phase_entry_points_at_size(name):
    """mhsk_reduce_edges (dp, se) / mhsk_reduce_vertices on the whole
    instance: every deletion and >= 2,000 sampled items per phase equal the
    oracle's decisions."""
    csr, planted = instance(name)
    ctx = _native.context()
    chk = checker(name)
    rng = np.random.default_rng(13)
    ones_v, ones_e = np.ones(csr.n, np.uint8), np.ones(csr.m, np.uint8)
    extra_e = planted.item_ids("edges") if planted else np.zeros(0, np.int64)
    extra_v = planted.item_ids("vertices") if planted else np.zeros(0, np.int64)
    for rule in ("dp", "se"):
        keep = ctx.reduce_edges(csr, rule)
        items = np.concatenate([extra_e, sample(rng, ones_e, 2000), np.nonzero(keep == 0)[0]])
        check_phase(chk, "edges", rule, None, None, keep, items)
        if planted:
            assert {int(i) for i in np.nonzero(keep == 0)[0]} == \
                {e for e, k in planted.edges[rule].items() if k == 1}
        else:
            assert keep.all()
    keep = ctx.reduce_vertices(csr)
    items = np.concatenate([extra_v, sample(rng, ones_v, 2000), np.nonzero(keep == 0)[0]])
    check_phase(chk, "vertices", "dp", None, None, keep, items)
    if not planted:
        assert keep.all()


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_random_config_at_size(name):
    """The BASELINE instance itself: one round, nothing deleted (the probe
    proves every tile empty), and the oracle agrees on 2,000 items per
    phase."""
    csr, _ = instance(name)
    ctx = _native.context()
    va, ea, st = ctx.kernelize(csr, "dp")
    assert st["rounds"] == 1 and va.all() and ea.all()
    assert st["deleted_edges"] == 0 and st["deleted_vertices"] == 0
    rng = np.random.default_rng(17)
    chk = checker(name)
    assert chk.decide("edges", sample(rng, ea, 2000), "dp").all()
    assert chk.decide("vertices", sample(rng, va, 2000), "dp").all()


def test_config4_every_decision_matches_oracle():
    """The headline instance item by item: the oracle decides all 100,000
    edges (dp) and all 100,000 vertices on the GPU's final state and keeps
    every one -- the GPU's kernelization (one round, nothing deleted) is the
    reference's, bit for bit (~1 minute of CPU on the box)."""
    csr, _ = instance("c4")
    va, ea, st = _native.context().kernelize(csr, "dp")
    assert st["rounds"] == 1 and va.all() and ea.all()
    chk = checker("c4")
    assert chk.decide("edges", np.arange(csr.m), "dp", vertex_alive=va, edge_alive=ea).all()
    assert chk.decide("vertices", np.arange(csr.n), "dp", vertex_alive=va, edge_alive=ea).all()


@pytest.mark.parametrize("name", ["c4-twins", "c4-planted"])
def test_config4_variant_round1_every_decision_matches_oracle(name):
    """C4-scale variants with deletions, item by item: round 1's edge phase
    on every edge and its vertex phase on every vertex equal the oracle's
    decisions (c4-twins: bench's 1,000 duplicated edges; c4-planted: both
    phases delete); the final state is a fixpoint on sampled survivors."""
    csr, _ = instance(name)
    ctx = _native.context()
    va1, ea1, st1 = ctx.kernelize(csr, "dp", max_rounds=1)
    assert st1["deleted_edges"] > 0
    chk = checker(name)
    keep_e = chk.decide("edges", np.arange(csr.m), "dp")
    assert np.array_equal(keep_e, ea1.astype(bool))
    keep_v = chk.decide("vertices", np.arange(csr.n), "dp", edge_alive=ea1)
    assert np.array_equal(keep_v, va1.astype(bool))
    if name == "c4-planted":
        assert st1["deleted_vertices"] > 0
    va, ea, st = ctx.kernelize(csr, "dp")
    rng = np.random.default_rng(19)
    assert chk.decide("edges", sample(rng, ea, 2000), "dp", vertex_alive=va, edge_alive=ea).all()
    assert chk.decide("vertices", sample(rng, va, 2000), "dp", vertex_alive=va, edge_alive=ea).all()


@pytest.mark.parametrize("name", ["c5", "c5-planted"])
def test_short_vertex_probe_at_config5(name):
    """Config 5 with the 6-k-block vertex probe (probe_entries 15; the auto
    rule keeps 16 there): ~2,300 vertex candidate pairs, counted from the
    CSR with partner lists, and edges holding more than 512 candidate
    members (vcand_count_heavy).  Same kernelization as the default, and the
    oracle keeps sampled survivors."""
    csr, _ = instance(name)
    ctx = _native.context()
    va, ea, st = ctx.kernelize(csr, "dp")
    try:
        ctx.set_option("probe_entries", 15)
        va2, ea2, st2 = ctx.kernelize(csr, "dp")
    finally:
        ctx.set_option("probe_entries", 0)
    assert np.array_equal(va, va2) and np.array_equal(ea, ea2)
    assert st2["rounds"] == st["rounds"] and st2["verified_pairs"] > st["verified_pairs"]
    rng = np.random.default_rng(23)
    chk = checker(name)
    assert chk.decide("edges", sample(rng, ea2, 500), "dp", vertex_alive=va2, edge_alive=ea2).all()
    assert chk.decide("vertices", sample(rng, va2, 500), "dp", vertex_alive=va2, edge_alive=ea2).all()


def test_reference_arm_instance_is_the_gpu_instance():
    """bench.py's reference arm builds config 4 with the oracle's host
    generator (it must not load libmhsk.so): bit-identical to the device
    generator the GPU arm uses."""
    csr, _ = instance("c4")
    host = oracle.generate_random(*COUNTER_CONFIGS["c4"], 0)
    assert np.array_equal(host.edge_ptr, csr.edge_ptr)
    assert np.array_equal(host.edge_vtx, csr.edge_vtx)
    assert np.array_equal(host.demand, csr.demand)


@pytest.mark.parametrize("name", ["c4-planted", "c5"])
def test_streamed_upload_matches_resident_instance(name):
    """The host API streams the member array up in chunks and runs round 1's
    scan, pack and edge probe band by band as they land (overlapped with the
    copy); the device API gets the instance resident.  Same kernelization;
    at one probe length (the automatic one differs: a streamed round 1 keeps
    the longer vertex probe) also the same probe statistics."""
    import torch

    csr, _ = instance(name)
    ctx = _native.context()
    d = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (csr.edge_ptr, csr.edge_vtx, csr.demand)]
    dva = torch.empty(csr.n, dtype=torch.uint8, device="cuda")
    dea = torch.empty(csr.m, dtype=torch.uint8, device="cuda")
    try:
        for entries in (0, 16):
            ctx.set_option("probe_entries", entries)
            va, ea, st = ctx.kernelize(csr, "dp")
            dst = ctx.kernelize_device(csr.n, csr.m, d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(),
                                       dva.data_ptr(), dea.data_ptr())
            assert np.array_equal(dva.cpu().numpy(), va) and np.array_equal(dea.cpu().numpy(), ea)
            for k in ("rounds", "deleted_edges", "deleted_vertices"):
                assert st[k] == dst[k], k
    finally:
        ctx.set_option("probe_entries", 0)
    for k in ("pruned_tiles", "verified_pairs", "executed_ops"):
        assert st[k] == dst[k], k
    assert st["h2d_bytes"] >= 4 * csr.nnz
    # the speculative vertex probe: adopted on c5 (no edge deleted in round
    # 1), discarded on c4-planted; the resident call never speculates
    assert st["spec_vertex"] == (2 if name == "c4-planted" else 1) and dst["spec_vertex"] == 0


@pytest.mark.parametrize("name", ["c4-vplanted", "c4", "c4-planted"])
def test_speculative_vertex_probe(name):
    """Round 1 of the streamed host call runs the vertex phase's probe during
    the upload, assuming the edge phase deletes nothing (mhsk_capi.cu
    spec_vertex_probe).  It is adopted iff that holds -- c4, and c4-vplanted,
    whose round-1 vertex deletions (dominated vertices, twins) then come from
    the adopted probe's marks and candidates -- and discarded on c4-planted
    (round 1 deletes edges).  Either way the kernelization equals the one
    with the speculation off (same rounds, deletions and probe statistics),
    deletes exactly the planted sets, and round 1's vertex phase agrees with
    the oracle."""
    csr, planted = instance(name)
    ctx = _native.context()
    va, ea, st = ctx.kernelize(csr, "dp")
    assert st["spec_vertex"] == (2 if name == "c4-planted" else 1)
    ctx.set_option("spec_vertex", 0)
    try:
        va0, ea0, st0 = ctx.kernelize(csr, "dp")
        va1, ea1, _ = ctx.kernelize(csr, "dp", max_rounds=1)
    finally:
        ctx.set_option("spec_vertex", 1)
    assert st0["spec_vertex"] == 0
    assert np.array_equal(va, va0) and np.array_equal(ea, ea0)
    for k in ("rounds", "deleted_edges", "deleted_vertices", "pruned_tiles", "verified_pairs", "executed_ops"):
        assert st[k] == st0[k], k
    sv1, se1, st1 = ctx.kernelize(csr, "dp", max_rounds=1)
    assert np.array_equal(sv1, va1) and np.array_equal(se1, ea1)
    if planted is None:
        assert va.all() and ea.all()
        return
    assert {int(i) for i in np.nonzero(ea == 0)[0]} == set(planted.edges["dp"])
    assert {int(i) for i in np.nonzero(va == 0)[0]} == set(planted.vertices)
    if name == "c4-vplanted":
        assert st1["deleted_edges"] == 0 and st1["deleted_vertices"] > 0 and st1["verified_pairs"] > 0
    rng = np.random.default_rng(19)
    v_items = np.concatenate([planted.item_ids("vertices"), sample(rng, np.ones(csr.n, np.uint8), 1500),
                              np.nonzero(sv1 == 0)[0]])
    check_phase(checker(name), "vertices", "dp", np.ones(csr.n, np.uint8), se1, sv1,
                v_items)


@pytest.mark.parametrize("chunks", [2, 5, 32])
def test_stream_chunk_counts_agree(chunks):
    """The streamed call's chunking (band-major tile list, the speculative
    vertex probe's first chunk, sqrt-spaced bounds) is result-neutral: any
    chunk count gives the default run's kernelization and probe statistics,
    and still adopts the speculation on c4-vplanted."""
    csr, planted = instance("c4-vplanted")
    ctx = _native.context()
    va, ea, st = ctx.kernelize(csr, "dp")
    ctx.set_option("stream_chunks", chunks)
    try:
        va2, ea2, st2 = ctx.kernelize(csr, "dp")
    finally:
        ctx.set_option("stream_chunks", 16)
    assert np.array_equal(va, va2) and np.array_equal(ea, ea2)
    for k in ("rounds", "deleted_edges", "deleted_vertices", "pruned_tiles", "verified_pairs", "executed_ops"):
        assert st[k] == st2[k], k
    assert st2["spec_vertex"] == 1
    assert {int(i) for i in np.nonzero(va2 == 0)[0]} == set(planted.vertices)


@pytest.mark.parametrize("name", ["c4-planted", "c4-vplanted"])
def test_programmatic_dependent_launch_is_result_neutral(name):
    """Every fast-path kernel is launched with programmatic stream
    serialization (mhsk_capi.cu launch_pdl) and opens with griddepcontrol.wait:
    the same kernelization with the option off, streamed and resident."""
    import torch

    csr, _ = instance(name)
    ctx = _native.context()
    va, ea, st = ctx.kernelize(csr, "dp")
    ctx.set_option("pdl", 0)
    try:
        va0, ea0, st0 = ctx.kernelize(csr, "dp")
        d = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (csr.edge_ptr, csr.edge_vtx, csr.demand)]
        dva = torch.empty(csr.n, dtype=torch.uint8, device="cuda")
        dea = torch.empty(csr.m, dtype=torch.uint8, device="cuda")
        ctx.kernelize_device(csr.n, csr.m, d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(),
                             dva.data_ptr(), dea.data_ptr())
    finally:
        ctx.set_option("pdl", 1)
    assert np.array_equal(va, va0) and np.array_equal(ea, ea0)
    assert np.array_equal(dva.cpu().numpy(), va) and np.array_equal(dea.cpu().numpy(), ea)
    for k in ("rounds", "deleted_edges", "deleted_vertices", "pruned_tiles", "verified_pairs"):
        assert st[k] == st0[k], k
