"""Write tests/golden/c5_oracle_samples.json: the oracle's endpoints_connected
for C5 samples 0 and 4095 (diff-max-mult-prob).

Calls only oracle/ and the seeded input generator (workloads/): the stored
values are the oracle's, so test_gpu_deep can compare the full-size GPU run
with them without ~10 minutes of oracle time per GPU test pass.
usage: python scripts/golden_c5.py   (~10 min on 2 host threads)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import workloads as W  # noqa: E402

SAMPLES = [0, 4095]


def main():
    oracle.build()
    sub = W.c5_workload(samples=SAMPLES)
    res = oracle.run(sub.program, 3, sub.batch_size, sub.facts, outputs=["endpoints_connected"],
                     samples=SAMPLES, threads=2)
    r = res.relations["endpoints_connected"]
    out = {"source": "scripts/golden_c5.py (oracle.run, diff-max-mult-prob, C5 samples 0 and 4095 pushed alone)",
           "samples": SAMPLES,
           "edges_per_sample": int(sub.facts["edge"].n // len(SAMPLES)),
           "endpoints_per_sample": int(sub.facts["is_endpoint"].n // len(SAMPLES)),
           "sample_ids": [int(x) for x in r.sample_ids],
           "tag_bits": [int(x) for x in np.asarray(r.tags, dtype=np.float32).view(np.uint32)],
           "grad_offsets": [int(x) for x in r.grad_offsets],
           "grad_fact_ids": [int(x) for x in r.grad_fact_ids],
           "grad_values": [float(x) for x in r.grad_values]}
    path = os.path.join(ROOT, "tests", "golden", "c5_oracle_samples.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print("wrote", path, len(out["grad_fact_ids"]), "gradient entries")


if __name__ == "__main__":
    main()
