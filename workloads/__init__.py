"""Seeded synthetic workloads (programs + input facts) for configs C1-C5.

This module is the ONLY code shared between the oracle side (tests, bench
cpu_baseline) and the CUDA product path.  It produces data, never results: it
holds no join, no semiring arithmetic, no fixpoint.  Recipes follow SURVEY.md
§8.0 (the config sheet); DESIGN.md §"Input recipe" restates them.
"""
from . import gen  # noqa: F401
from .gen import (  # noqa: F401
    Facts, Workload, PROGRAMS, C1_EDGES, PATH_PROGRAM, PATHFINDER_PROGRAM,
    KINSHIP_PROGRAM, REACH_PROGRAM, c1_workload, grid_workload, c2_workload,
    c3_workload, c4_workload, c5_workload, random_digraph_workload,
    random_dag_workload, workload_by_name,
)
