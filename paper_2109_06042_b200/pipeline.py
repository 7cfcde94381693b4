"""Engine dispatch: the reference's ``run_pipeline`` boundary for this engine.

Mirrors ``pkg/src/mhskernel/pipeline.py:34-171`` for the phases on the hot
path (dp, se, md).  The engine is registered as ``"b200"`` -- not ``"gpu"``,
which the reference's own tests require to stay invalid
(test_pipeline.py:22-23).  The pure ``("dp", "md")`` loop is delegated to
:func:`~.engine.par_kernelize` (one native call for the whole fixpoint,
as the reference's fast path does, pipeline.py:117-128); other dp/se/md
sequences run one native phase per step on the re-extracted subinstance
(pipeline.py:58-92,130-161).  ``fe`` and ``lp`` are outside this engine's
scope and are rejected at spec validation.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _native
from .engine import extract, par_kernelize
from .instance import CSRInstance, as_csr, instance_size, validate_feasibility
from .report import KernelReport

PHASES = ("dp", "se", "md")
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
    if not validate_feasibility(h):
        report.infeasible = True
        report.n_after, report.m_after, report.size_after = csr.n, csr.m, instance_size(csr)
        return h, report

    if spec.loop and tuple(spec.phases) == ("dp", "md"):
        run = par_kernelize(h, device=device)
        report.rounds = run.report.rounds
        report.deleted_by_rule = run.report.deleted_by_rule
        report.wall_times_ms.update(run.report.wall_times_ms)
        report.n_after, report.m_after = run.report.n_after, run.report.m_after
        report.size_after = run.report.size_after
        return run.hypergraph, report

    ctx = _native.context(device)
    va = np.ones(csr.n, dtype=bool)
    ea = np.ones(csr.m, dtype=bool)
    while True:
        report.rounds += 1
        deletions = 0
        for phase in spec.phases:
            t0 = time.perf_counter()
            sub, vids, eids = extract(csr, va, ea)
            if phase in ("dp", "se"):
                keep = ctx.reduce_edges(sub, phase).astype(bool)
                dead = eids[~keep] - 1
                ea[dead] = False
            else:
                keep = ctx.reduce_vertices(sub).astype(bool)
                dead = vids[~keep] - 1
                va[dead] = False
            report.deleted_by_rule[phase] += len(dead)
            deletions += len(dead)
            report.wall_times_ms[phase] = report.wall_times_ms.get(phase, 0.0) + \
                (time.perf_counter() - t0) * 1e3
        if not spec.loop or deletions == 0:
            break
    reduced, _, _ = extract(csr, va, ea)
    report.n_after, report.m_after, report.size_after = reduced.n, reduced.m, instance_size(reduced)
    return (reduced if isinstance(h, CSRInstance) else reduced.to_hypergraph()), report
