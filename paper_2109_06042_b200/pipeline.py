"""Engine dispatch: the reference's ``run_pipeline`` boundary for this engine.

Mirrors ``pkg/src/mhskernel/pipeline.py:34-171`` for the phases on and
next to the hot path (fe, dp, se, md).  The engine is registered as ``"b200"`` -- not ``"gpu"``,
which the reference's own tests require to stay invalid
(test_pipeline.py:22-23).  The pure ``("dp", "md")`` loop is delegated to
:func:`~.engine.par_kernelize` (one native call for the whole fixpoint,
as the reference's fast path does, pipeline.py:117-128); every other
sequence of fe/dp/se/md runs as ONE native call too (``mhsk_run_pipeline``):
the generic loop of pipeline.py:130-161 with the state -- alive flags and
FE-adjusted demands -- resident on the device.  ``lp`` (exact-solver
oracle) is outside this engine's scope and is rejected at spec
validation.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _native
from .engine import caller_types, extract, par_kernelize, to_caller_hypergraph, to_caller_report
from .instance import CSRInstance, as_csr, instance_size, validate_feasibility
from .report import KernelReport

PHASES = ("fe", "dp", "se", "md")
ENGINES = ("b200",)


@dataclass(frozen=True)
class PipelineSpec:
    phases: tuple[str, ...]
    engine: str = "b200"
    loop: bool = False
    workers: int = 1

    def __post_init__(self):
        if not self.phases:
            raise ValueError("pipeline needs at least one phase")
        for p in self.phases:
            if p not in PHASES:
                raise ValueError(f"unknown phase {p!r}; expected one of {PHASES}")
        if self.engine not in ENGINES:
            raise ValueError(f"unknown engine {self.engine!r}")
        if self.workers < 1:
            raise ValueError("worker count must be positive")


def run_pipeline(h, spec: PipelineSpec, *, device: int | None = None):
    """Run the phases in order (looped to the joint fixpoint when flagged);
    returns (reduced instance, KernelReport) like the reference."""
    csr = as_csr(h)
    report = KernelReport(n_before=csr.n, m_before=csr.m, size_before=instance_size(csr))
    types = caller_types(h)
    if not validate_feasibility(h):
        report.infeasible = True
        report.n_after, report.m_after, report.size_after = csr.n, csr.m, instance_size(csr)
        return h, to_caller_report(report, types[2] if types else None)

    if spec.loop and tuple(spec.phases) == ("dp", "md"):
        run = par_kernelize(h, device=device)
        report.rounds = run.report.rounds
        report.deleted_by_rule = run.report.deleted_by_rule
        report.wall_times_ms.update(run.report.wall_times_ms)
        report.n_after, report.m_after = run.report.n_after, run.report.m_after
        report.size_after = run.report.size_after
        return run.hypergraph, to_caller_report(report, types[2] if types else None)

    va, ea, dem, res, _ = _native.context(device).run_pipeline(csr, spec.phases, spec.loop)
    report.rounds = int(res["passes"])
    for phase in PHASES:
        report.deleted_by_rule[phase] += res["deleted"][phase]
    report.budget_delta = int(res["forced_vertices"])
    report.infeasible = res["infeasible"]
    for phase in dict.fromkeys(spec.phases):
        report.wall_times_ms[phase] = res["ms_by_phase"][phase]
    adjusted = CSRInstance(csr.n, csr.edge_ptr, csr.edge_vtx, dem, csr.budget, validate=False)
    reduced, _, _ = extract(adjusted, va, ea)
    if csr.budget is not None:
        reduced.budget = csr.budget - report.budget_delta
        if reduced.budget < 0:
            report.infeasible = True
    report.n_after, report.m_after, report.size_after = reduced.n, reduced.m, instance_size(reduced)
    return (to_caller_hypergraph(reduced, h, types),
            to_caller_report(report, types[2] if types else None))
