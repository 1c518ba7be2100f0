"""Oracle containers for full-size configs[1] levels at the other error
targets of BASELINE.json (0.1% and 10%; GPU parity fixtures for the
incremental / pruned / abortable probe paths at those budgets).
Writes tests/golden/oracle_eps.json.  The C oracle is pinned bit-exact to
the reference's goldens (tests/test_oracle_golden.py)."""
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


oracle.build()
levels = fields.config2_levels()[0]
cases = []
for lev in (0, 36):
    for eps in (0.001, 0.1):
        a = levels[lev]
        t0 = time.perf_counter()
        blob = oracle.compress(a, eps, 1 - 1e-5)
        t = time.perf_counter() - t0
        cases.append({"name": f"config2_level{lev}", "level": lev, "input_sha": sha(a), "eps": eps,
                      "q": 1 - 1e-5, "container_sha": hashlib.sha256(blob).hexdigest(),
                      "container_len": len(blob), "oracle_seconds": round(t, 1)})
        print(cases[-1], flush=True)
with open(os.path.join(REPO, "tests", "golden", "oracle_eps.json"), "w") as fh:
    json.dump(cases, fh, indent=1)
