"""B200-native matrix-multiplication kernelization for Multiple Hitting Set.

Drop-in for the data-parallel engine of the reference package ``mhskernel``
(arXiv 2109.06042): ``par_kernelize``, ``par_reduce_edges`` and
``par_reduce_vertices`` keep the reference's signatures, result types and
error texts, and run on sm_100a tensor cores through the C ABI of
``libmhsk.so`` (include/mhsk.h).  See DESIGN.md.
"""

from .bitmatrix import IncidenceMatrix, incidence_matrix
from .engine import extract, kernelize_csr, par_kernelize, par_reduce_edges, par_reduce_vertices
from .generate import (
    config_instance,
    generate_random,
    interval_trains,
    nested_chains,
    plant_twins,
    random_csr,
)
from .instance import (
    CSRInstance,
    FeasibilityReport,
    Hypergraph,
    InstanceError,
    as_csr,
    instance_size,
    parse_instance,
    serialize_instance,
    validate_feasibility,
)
from .pipeline import ENGINES, PipelineSpec, run_pipeline
from .report import RULE_KEYS, KernelReport, KernelRun

__all__ = [
    "CSRInstance",
    "ENGINES",
    "FeasibilityReport",
    "Hypergraph",
    "IncidenceMatrix",
    "InstanceError",
    "KernelReport",
    "KernelRun",
    "PipelineSpec",
    "RULE_KEYS",
    "as_csr",
    "config_instance",
    "extract",
    "generate_random",
    "incidence_matrix",
    "instance_size",
    "interval_trains",
    "kernelize_csr",
    "nested_chains",
    "par_kernelize",
    "par_reduce_edges",
    "par_reduce_vertices",
    "parse_instance",
    "plant_twins",
    "random_csr",
    "run_pipeline",
    "serialize_instance",
    "validate_feasibility",
]

__version__ = "0.1.0"
