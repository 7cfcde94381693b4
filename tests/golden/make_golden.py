"""Generate the golden parity fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the reference package ``mhskernel`` read-only, runs its
``par_kernelize`` / ``par_reduce_edges`` / ``par_reduce_vertices``
(parallel.py:80-214) on

  * the hand-computed known-answer instances of the reference's
    test_parallel.py:21-108 and conftest.py:20-35,
  * the reference test suite's seeded ``generate_random`` sweeps
    (test_parallel.py:111-179) plus a wider seeded sweep,
  * the 500 engine-equivalence instances of test_acceptance.py:61-78
    (par_kernelize outputs + seq_kernelize alive sets),
  * structured instances from this repo's generators (nested chains,
    interval trains, planted twins) at sizes the reference finishes in seconds,
  * run_pipeline (pipeline.py:95-171) with fe/dp/se/md phase lists, looped
    and not, with and without budgets, on hand-made and seeded instances,
  * BASELINE config 1 (``generate_random(2000, 2000, 0.05, 1, seed=0)``) and
    config 2 (``nested_chains(100, 100, 3, seed=0)``), stored by checksum
    (the instances are regenerated deterministically by the tests),

and writes the outputs to tests/golden/*.json.gz.  The fixtures travel; the
reference does not.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

import mhskernel as ref  # noqa: E402  (the reference, read-only)

from paper_2109_06042_b200 import generate as gen  # noqa: E402
from paper_2109_06042_b200.instance import CSRInstance  # noqa: E402


def csr_checksum(c: CSRInstance) -> str:
    h = hashlib.sha256()
    h.update(np.int64(c.n).tobytes())
    h.update(np.ascontiguousarray(c.edge_ptr, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(c.edge_vtx, dtype=np.int32).tobytes())
    h.update(np.ascontiguousarray(c.demand, dtype=np.int32).tobytes())
    return h.hexdigest()


def to_ref(c: CSRInstance) -> "ref.Hypergraph":
    ptr = c.edge_ptr.tolist()
    vtx = (c.edge_vtx.astype(np.int64) + 1).tolist()
    edges = tuple(tuple(vtx[ptr[e]:ptr[e + 1]]) for e in range(c.m))
    return ref.Hypergraph(c.n, edges, tuple(int(x) for x in c.demand.tolist()), c.budget)


def run_case(name: str, h, *, store_instance: bool = True, checksum: str | None = None,
             phases: bool = True, rules=("dp", "se")) -> dict:
    case: dict = {"name": name}
    if store_instance:
        case.update(n=h.n, edges=[list(e) for e in h.edges], demand=list(h.demand), budget=h.budget)
    if checksum:
        case["checksum"] = checksum
    A = ref.incidence_matrix(h)
    feasible = bool(ref.validate_feasibility(h))
    if phases:
        for rule in ("dp", "se"):
            case[f"keep_edges_{rule}"] = [bool(x) for x in ref.par_reduce_edges(A, h.demand, rule=rule)]
        case["keep_vertices"] = [bool(x) for x in ref.par_reduce_vertices(A, h.demand)]
    for rule in rules:
        if not feasible:
            try:
                ref.par_kernelize(h, rule=rule)
            except ValueError as exc:
                case[f"kernelize_{rule}"] = {"error": str(exc)}
            continue
        run = ref.par_kernelize(h, rule=rule)
        case[f"kernelize_{rule}"] = {
            "alive_vertices": list(run.alive_vertices),
            "alive_edges": list(run.alive_edges),
            "rounds": run.report.rounds,
            "deleted_by_rule": dict(run.report.deleted_by_rule),
            "n_after": run.report.n_after,
            "m_after": run.report.m_after,
            "size_after": run.report.size_after,
            "reduced_n": run.hypergraph.n,
            "reduced_edges": [list(e) for e in run.hypergraph.edges] if store_instance else None,
            "reduced_demand": list(run.hypergraph.demand),
            "reduced_budget": run.hypergraph.budget,
        }
    return case


def hand_cases() -> list:
    ce = ref.parse_instance("p mhs 5 3\ne 2 1 2\ne 2 2 3 4\ne 2 2 3 5\n")
    H = ref.Hypergraph
    items = [
        ("duplicates", H(1, ((1,), (1,)), (1, 1))),
        ("ce", ce),
        ("one_way_dp", H.from_edges(4, [[1, 2, 3], [3, 4]], [3, 1])),
        ("se_lower_demand", H.from_edges(3, [[1, 2], [1, 2, 3]], [1, 2])),
        ("se_equal_demand", H.from_edges(3, [[1, 2], [1, 2, 3]], [2, 2])),
        ("dominated_tail", H.from_edges(4, [[1, 2, 3], [1, 2, 3, 4]], [2, 2])),
        ("unit_domination", H.from_edges(3, [[1, 2], [1, 3]], [1, 1])),
        ("orphans", H(3, ((2,),), (1,))),
        ("singletons5", H(5, tuple((j,) for j in range(1, 6)), (1,) * 5)),
        ("infeasible", H(1, ((1,),), (2,))),
        ("empty", H(0, (), ())),
        ("vertices_only", H(4, (), ())),
        ("budget_passthrough", H.from_edges(4, [[1, 2], [1, 2], [2, 3, 4]], [1, 1, 2], budget=3)),
        ("negative_budget", H(2, ((1, 2),), (1,), -1)),
    ]
    return [run_case(name, h) for name, h in items]


def sweep_cases() -> list:
    out = []
    specs = []
    for s in range(40):   # test_parallel.py:111-117
        specs.append(("workers", dict(n=3 + s % 20, m=3 + (7 * s) % 20, p=0.4, alpha=1 + s % 3, seed=s)))
    for s in range(30):   # test_parallel.py:120-129
        specs.append(("product", dict(n=2 + s % 15, m=2 + (3 * s) % 15, p=0.5, alpha=2, seed=s)))
    for s in range(40):   # test_parallel.py:154-164
        specs.append(("exhaustive", dict(n=2 + s % 12, m=2 + (5 * s) % 12, p=0.45, alpha=1 + s % 3, seed=s)))
    for s in range(60):   # test_parallel.py:167-172
        specs.append(("optimum", dict(n=1 + s % 14, m=1 + (3 * s) % 12, p=0.4, alpha=1 + s % 3, seed=s)))
    for s in range(40):   # test_parallel.py:175-179
        specs.append(("rounds", dict(n=2 + s % 16, m=2 + (7 * s) % 16, p=0.35, alpha=1 + s % 3, seed=s)))
    for s in range(160):  # wider sweep: sizes to 70, alpha to 5, sparse and dense
        specs.append(("wide", dict(n=1 + (s * 13) % 70, m=1 + (s * 29) % 70,
                                   p=(0.05, 0.15, 0.3, 0.6, 0.9)[s % 5], alpha=1 + s % 5, seed=1000 + s)))
    for tag, kw in specs:
        h = ref.generate_random(**kw)
        out.append(run_case(f"{tag}_{kw['seed']}", h))
    return out


def structured_cases() -> list:
    out = []
    for s in range(4):
        out.append(run_case(f"chains_{s}", to_ref(gen.nested_chains(5, 12, 1 + s % 3, s))))
        out.append(run_case(f"trains_a1_{s}", to_ref(gen.interval_trains(150, 90, 1, s))))
        out.append(run_case(f"trains_a3_{s}", to_ref(gen.interval_trains(150, 90, 3, s))))
        out.append(run_case(f"twins_{s}", to_ref(gen.plant_twins(gen.random_csr(160, 130, 0.05, 2, s),
                                                               0.05, 0.05, 100 + s))))
    # larger, structured: reduced-scale configs 1 and 3 with planted twins
    out.append(run_case("c1_twins_small", to_ref(gen.plant_twins(gen.random_csr(500, 500, 0.05, 1, 7),
                                                                0.02, 0.02, 8))))
    out.append(run_case("c3_small", to_ref(gen.interval_trains(2000, 800, 1, 3))))
    out.append(run_case("c3a3_small", to_ref(gen.interval_trains(2000, 800, 3, 3))))
    return out


def acceptance_cases() -> list:
    """The 500 seeded instances of the reference's acceptance criteria 3/6
    (test_acceptance.py:61-78: n, m <= 40, p in {0.15, 0.3, 0.5}, alpha
    1..3), with par_kernelize's outputs and seq_kernelize's alive sets
    (criterion 3, engine equivalence, test_acceptance.py:114-125)."""
    out = []
    for seed in range(500):
        h = ref.generate_random(n=1 + (7 * seed) % 40, m=1 + (13 * seed) % 40,
                                p=(0.15, 0.3, 0.5)[seed % 3], alpha=1 + seed % 3, seed=seed)
        case = run_case(f"acceptance_{seed}", h)
        seq = ref.seq_kernelize(h)
        case["seq_alive_vertices"] = list(seq.alive_vertices)
        case["seq_alive_edges"] = list(seq.alive_edges)
        out.append(case)
    return out


def config_cases() -> list:
    out = []
    c1 = gen.generate_random(2000, 2000, 0.05, 1, 0)
    out.append(run_case("config1_seed0", to_ref(c1.csr), store_instance=False,
                        checksum=csr_checksum(c1.csr), rules=("dp",)))
    c2 = gen.nested_chains(100, 100, 3, 0)
    out.append(run_case("config2_seed0", to_ref(c2), store_instance=False,
                        checksum=csr_checksum(c2), phases=False, rules=("dp",)))
    return out


PIPELINE_SPECS = [
    (("fe", "dp", "md"), True),
    (("fe",), False),
    (("fe", "se", "md"), True),
    (("md", "dp"), False),
    (("dp", "md", "fe"), True),
    (("se",), True),
    (("dp", "se", "md"), True),
    (("fe", "md"), True),
]


def pipeline_case(name: str, h) -> dict:
    """Reference run_pipeline (pipeline.py:95-171, engine "parallel") for
    every spec in PIPELINE_SPECS."""
    case = {"name": name, "n": h.n, "edges": [list(e) for e in h.edges], "demand": list(h.demand),
            "budget": h.budget, "pipelines": []}
    for phases, loop in PIPELINE_SPECS:
        spec = ref.PipelineSpec(phases, engine="parallel", loop=loop)
        red, rep = ref.run_pipeline(h, spec)
        d = rep.to_dict()
        d.pop("wall_times_ms")
        case["pipelines"].append({
            "phases": list(phases), "loop": loop, "report": d,
            "reduced_n": red.n, "reduced_edges": [list(e) for e in red.edges],
            "reduced_demand": list(red.demand), "reduced_budget": red.budget})
    return case


def pipeline_cases() -> list:
    out = []
    H = ref.Hypergraph
    ce = ref.parse_instance("p mhs 5 3\ne 2 1 2\ne 2 2 3 4\ne 2 2 3 5\n")
    hand = [
        ("ce", ce),
        ("ce_budget3", H(ce.n, ce.edges, ce.demand, 3)),
        ("ce_budget2", H(ce.n, ce.edges, ce.demand, 2)),
        ("full_chain", H.from_edges(5, [[1, 2], [2, 3, 4], [4, 5]], [2, 2, 1], budget=4)),
        ("cascade", H.from_edges(6, [[1], [1, 2, 3], [2, 3], [3, 4, 5, 6], [5, 6]], [1, 2, 1, 3, 2], budget=5)),
        ("infeasible_start", H(1, ((1,),), (2,))),
        ("empty", H(0, (), ())),
        ("vertices_only", H(4, (), ())),
    ]
    for name, h in hand:
        out.append(pipeline_case(name, h))
    for s in range(120):
        g = ref.generate_random(n=2 + (s * 7) % 25, m=2 + (s * 11) % 25,
                                p=(0.1, 0.25, 0.4, 0.6)[s % 4], alpha=1 + s % 4, seed=5000 + s)
        if s % 3 == 0:
            g = H(g.n, g.edges, g.demand, g.n // 2)
        out.append(pipeline_case(f"pipe_{s}", g))
    for s in range(3):
        out.append(pipeline_case(f"pipe_trains_{s}", to_ref(gen.interval_trains(160, 90, 1 + s, s))))
        out.append(pipeline_case(f"pipe_chains_{s}", to_ref(gen.nested_chains(4, 10, 1 + s, s))))
    return out


PARSE_TEXTS = [
    "p mhs 5 3\ne 2 1 2\ne 2 2 3 4\ne 2 2 3 5\n",
    "# comment\n\n  p mhs 4 2 3  \n e 1 4 1 \n\t# x\ne 2 2 3\n",
    "p mhs 3 1\r\ne 1 3 1\r\n",
    "p mhs 3 0\n",
    "p mhs 0 0 0\n",
    "p mhs 2 1\ne 1\n",
    "p mhs 4 1\ne +1 0_2 +3\n",
    "p mhs 4 1\ne 1 004\n",
    "",
    "# only comments\n",
    "q mhs 1 1\n",
    "p mhs 1\n",
    "p mhs 1 1 1 1\n",
    "p mhx 1 1\n",
    "p mhs a 1\n",
    "p mhs -1 1\n",
    "p mhs 1 1 -2\n",
    "p mhs 2 1\nx 1 2\n",
    "p mhs 2 1\nE 1 2\n",
    "p mhs 2 1\ne\n",
    "p mhs 2 1\ne 1 b\n",
    "p mhs 2 1\ne 1 1.5\n",
    "p mhs 2 1\ne 0 1\n",
    "p mhs 2 1\ne -3 1\n",
    "p mhs 2 1\ne 1 3\n",
    "p mhs 2 1\ne 1 0\n",
    "p mhs 3 1\ne 1 2 2\n",
    "p mhs 3 1\ne 1 2 9 2\n",
    "p mhs 3 1\ne 1 2 2 9\n",
    "p mhs 3 2\ne 1 1\n",
    "p mhs 3 1\ne 1 1\ne 1 2\n",
    "p mhs 3 1\n\n\ne 1 1 2 3\n# tail\n",
    "p mhs 2 1\ne 1 1_\n",
    "p mhs 2 1\ne 1 _1\n",
    "p mhs 2 1\ne 1 1__0\n",
    "p mhs 2 1\ne 1 '1'\n",
    "p mhs 2 1\ne' 1 1\n",
    "p mhs 12 1\ne 1 1_0 3\n",
    "p mhs 3 1\ne 2 1 3\x0ce 1 2\n",
]


def parse_cases() -> list:
    """Reference parse_instance (instance.py:114-165) outcomes."""
    out = []
    for text in PARSE_TEXTS:
        try:
            h = ref.parse_instance(text)
            out.append({"text": text, "n": h.n, "edges": [list(e) for e in h.edges],
                        "demand": list(h.demand), "budget": h.budget})
        except ref.InstanceError as exc:
            out.append({"text": text, "error": str(exc), "line_no": exc.line_no})
    return out


def dump(name: str, cases: list) -> None:
    path = os.path.join(HERE, f"{name}.json.gz")
    with gzip.open(path, "wt") as f:
        json.dump({"generator": "tests/golden/make_golden.py", "reference": "mhskernel " + ref.__version__,
                   "cases": cases}, f, separators=(",", ":"))
    print(f"{path}: {len(cases)} cases, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    t = time.time()
    if "--only-acceptance" in sys.argv:
        dump("acceptance", acceptance_cases())
        sys.exit(0)
    dump("hand", hand_cases())
    dump("sweeps", sweep_cases())
    dump("structured", structured_cases())
    dump("pipelines", pipeline_cases())
    dump("parse", parse_cases())
    dump("acceptance", acceptance_cases())
    print(f"small fixtures in {time.time() - t:.1f}s")
    if "--no-configs" not in sys.argv:
        dump("configs", config_cases())
    print(f"done in {time.time() - t:.1f}s")
