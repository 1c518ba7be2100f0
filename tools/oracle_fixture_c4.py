"""Oracle containers for full-size config-3/4 fields (GPU parity fixtures).

The reference itself needs ~9 minutes per 2881x5760 field in numpy; the C
oracle (pinned bit-exact to the reference goldens) produces the same bytes,
so these fixtures pin the GPU path at the largest BASELINE.json shape.
Writes tests/golden/oracle_large.json.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from oracle import oracle  # noqa: E402
from paper_2510_22265_b200 import fields  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


cases = []
for v, f in fields.config4_fields(nvars=7):
    if v not in (0, 6):
        continue
    t0 = time.perf_counter()
    blob = oracle.compress(f, 0.01, 1 - 1e-5)
    t = time.perf_counter() - t0
    cases.append({"name": f"config4_var{v}", "input_sha": sha(f), "eps": 0.01, "q": 1 - 1e-5,
                  "container_sha": hashlib.sha256(blob).hexdigest(), "container_len": len(blob),
                  "oracle_seconds": t})
    print(cases[-1], flush=True)
pr = fields.config3_precip(steps=2)
for t_ in range(2):
    a = pr[t_, 0]
    blob = oracle.compress(a, 0.01, 1 - 1e-5)
    cases.append({"name": f"config3_step{t_}", "input_sha": sha(a), "eps": 0.01, "q": 1 - 1e-5,
                  "container_sha": hashlib.sha256(blob).hexdigest(), "container_len": len(blob)})
    print(cases[-1], flush=True)
with open(os.path.join(REPO, "tests", "golden", "oracle_large.json"), "w") as fh:
    json.dump(cases, fh, indent=1)
