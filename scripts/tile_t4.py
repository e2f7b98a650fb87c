import sys; sys.path.insert(0,".")
import workloads as W
from paper_2503_21937_b200 import Engine
w = W.c3_workload(semiring=2, batch=6, entities=10, rtypes=6, skips=5, ncomp=20)
e = Engine(w.program, 2, batch_size=6); e.push_facts(w.facts); st=e.run(); print(st["candidates"])
