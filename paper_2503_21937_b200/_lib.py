"""ctypes declarations of include/lobster.h (argument marshalling only).

The shared library is built in-tree (paper_2503_21937_b200/liblobster.so); if
it is missing this module raises — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblobster.so")

OK, E_INVALID_ARG, E_PARSE, E_SCHEMA, E_RANGE, E_STATE, E_OOM, E_ITER_CAP, E_CUDA, E_NCCL = range(10)
STATUS_NAMES = ["OK", "INVALID_ARG", "PARSE", "SCHEMA", "RANGE", "STATE", "OOM", "ITER_CAP", "CUDA", "NCCL"]

UNIT, MAX_MIN_PROB, ADD_MULT_PROB, DIFF_MAX_MULT_PROB, DIFF_MAX_MIN_PROB, DIFF_TOP1_PROOFS, DIFF_ADD_MULT_PROB = 0, 1, 2, 3, 4, 5, 6
SEMIRINGS = {"unit": UNIT, "max-min-prob": MAX_MIN_PROB, "add-mult-prob": ADD_MULT_PROB,
             "diff-max-mult-prob": DIFF_MAX_MULT_PROB, "diff-max-min-prob": DIFF_MAX_MIN_PROB,
             "diff-top-1-proofs": DIFF_TOP1_PROOFS, "diff-add-mult-prob": DIFF_ADD_MULT_PROB}


class Options(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("cuda_stream", ctypes.c_void_p), ("batch_size", ctypes.c_int32),
                ("max_iters", ctypes.c_int32), ("arena_bytes", ctypes.c_int64), ("micro_batch", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("world_size", ctypes.c_int32), ("nccl_comm", ctypes.c_void_p)]


class RunStats(ctypes.Structure):
    _fields_ = [("strata", ctypes.c_int32), ("rounds_total", ctypes.c_int32), ("tuples_derived", ctypes.c_int64),
                ("candidates", ctypes.c_int64), ("ms_total", ctypes.c_double), ("ms_join", ctypes.c_double),
                ("ms_sort", ctypes.c_double), ("ms_reduce", ctypes.c_double), ("ms_merge", ctypes.c_double),
                ("ms_grad", ctypes.c_double), ("ms_comm", ctypes.c_double), ("bytes_algorithmic", ctypes.c_int64),
                ("fj_launches", ctypes.c_int64), ("fj_probe_rows", ctypes.c_int64),
                ("fj_candidates", ctypes.c_int64), ("ms_fused_join", ctypes.c_double),
                ("fj_row_bytes", ctypes.c_int32), ("tile_strata", ctypes.c_int32),
                ("fj_timed_launches", ctypes.c_int64), ("fj_timed_probe_rows", ctypes.c_int64),
                ("fj_timed_candidates", ctypes.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Output(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("arity", ctypes.c_int32), ("on_device", ctypes.c_int32),
                ("sample_ids", ctypes.c_void_p), ("columns", ctypes.POINTER(ctypes.c_void_p)),
                ("probs", ctypes.c_void_p), ("sample_offsets", ctypes.c_void_p),
                ("grad_offsets", ctypes.c_void_p), ("grad_fact_ids", ctypes.c_void_p),
                ("grad_values", ctypes.c_void_p)]


EXPORTS = ["lobster_create", "lobster_destroy", "lobster_last_error", "lobster_program_load",
           "lobster_facts_push", "lobster_run", "lobster_output_get", "lobster_output_backward",
           "lobster_num_facts", "lobster_kernel_launches", "lobster_facts_groups", "lobster_group_local",
           "lobster_nccl_id", "lobster_group_nccl", "lobster_group_destroy", "lobster_partition"]

_lib = None


def load():
    """Load liblobster.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2503_21937_b200._build` "
                           "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp = ctypes.c_void_p
    L.lobster_create.argtypes = [ctypes.POINTER(Options), ctypes.POINTER(vp)]
    L.lobster_create.restype = ctypes.c_int
    L.lobster_destroy.argtypes = [vp]
    L.lobster_destroy.restype = None
    L.lobster_last_error.argtypes = [vp]
    L.lobster_last_error.restype = ctypes.c_char_p
    L.lobster_program_load.argtypes = [vp, ctypes.c_char_p, ctypes.c_int]
    L.lobster_program_load.restype = ctypes.c_int
    L.lobster_facts_push.argtypes = [vp, ctypes.c_char_p, ctypes.c_int64, ctypes.POINTER(vp), vp, vp,
                                     ctypes.POINTER(ctypes.c_int64)]
    L.lobster_facts_push.restype = ctypes.c_int
    L.lobster_run.argtypes = [vp, ctypes.POINTER(RunStats)]
    L.lobster_run.restype = ctypes.c_int
    L.lobster_output_get.argtypes = [vp, ctypes.c_char_p, ctypes.c_int32, ctypes.POINTER(Output)]
    L.lobster_output_get.restype = ctypes.c_int
    L.lobster_output_backward.argtypes = [vp, ctypes.c_char_p, vp, vp]
    L.lobster_output_backward.restype = ctypes.c_int
    L.lobster_num_facts.argtypes = [vp]
    L.lobster_num_facts.restype = ctypes.c_int64
    L.lobster_kernel_launches.argtypes = []
    L.lobster_kernel_launches.restype = ctypes.c_int64
    L.lobster_facts_groups.argtypes = [vp, ctypes.c_int64, ctypes.c_int64, vp]
    L.lobster_facts_groups.restype = ctypes.c_int
    L.lobster_group_local.argtypes = [ctypes.c_int32, ctypes.POINTER(vp)]
    L.lobster_group_local.restype = ctypes.c_int
    L.lobster_nccl_id.argtypes = [ctypes.c_char_p]
    L.lobster_nccl_id.restype = ctypes.c_int
    L.lobster_group_nccl.argtypes = [ctypes.c_char_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(vp)]
    L.lobster_group_nccl.restype = ctypes.c_int
    L.lobster_group_destroy.argtypes = [vp]
    L.lobster_group_destroy.restype = None
    L.lobster_partition.argtypes = [vp, vp, ctypes.c_int32]
    L.lobster_partition.restype = ctypes.c_int
    _lib = L
    return L
