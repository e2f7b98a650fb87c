import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
import oracle
from tests.gpu_util import engine_run, assert_parity
for sr in (0, 1, 3):
    w = W.c1_workload(sr)
    eng, st, _ = engine_run(w)
    o = eng.output("path")
    print(sr, o.n, st["rounds_total"], st["candidates"], flush=True)
    res = oracle.run_workload(w)
    try:
        assert_parity(eng, res, "path", sr)
        print("ok", flush=True)
    except AssertionError as e:
        print("FAIL", str(e)[:500], flush=True)
w = W.c2_workload(semiring=1, n=8, batch=3)
eng, st, _ = engine_run(w)
print("c2", st, flush=True)
