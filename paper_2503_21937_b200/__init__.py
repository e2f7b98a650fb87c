"""B200-native semi-naive fixpoint engine for Datalog over tagged relations
(Lobster, arXiv 2503.21937: the APM runtime's hot path).

    from paper_2503_21937_b200 import Engine, DIFF_MAX_MULT_PROB
    eng = Engine(program_text, DIFF_MAX_MULT_PROB, batch_size=64)
    eng.push("edge", [src, dst], sample_ids, probs)
    stats = eng.run()
    out = eng.output("endpoints_connected")

The compute path is the CUDA library liblobster.so (csrc/, include/lobster.h);
this package only marshals arguments.
"""
from ._lib import (ADD_MULT_PROB, DIFF_ADD_MULT_PROB, DIFF_MAX_MIN_PROB, DIFF_MAX_MULT_PROB, DIFF_TOP1_PROOFS, EXPORTS, LIB_PATH, MAX_MIN_PROB,  # noqa: F401
                   SEMIRINGS, UNIT)
from .engine import Engine, Group, LobsterError, RelationOutput  # noqa: F401


def build(force: bool = False, verbose: bool = False) -> str:
    from ._build import build as _b
    return _b(force=force, verbose=verbose)
