"""Developer probe: time ebcc_compress phases on the bench workload
(EBCC_PROFILE=1 prints per-phase host wall time from the library)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2510_22265_b200 import _lib  # noqa: E402

levels = int(sys.argv[1]) if len(sys.argv) > 1 else 37
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
host = bench.workload(0)[:levels].copy()
ctx = _lib.context(0)
for it in range(iters):
    t0 = time.perf_counter()
    recs, offs, total, st = ctx.compress(host, levels, 721, 1440, 0.01, 1 - 1e-5, 10.0, 1e-3)
    t1 = time.perf_counter()
    print(f"compress wall {1e3*(t1 - t0):.1f} ms", ctx.stats(), file=sys.stderr)
    t0 = time.perf_counter()
    out = ctx.decompress
    import numpy as np
    pay = np.empty(total, np.uint8)
    ctx.fetch_payload(pay)
    o = np.empty((levels, 721, 1440), np.float32)
    t1 = time.perf_counter()
    ctx.decompress(pay, offs, recs, 721, 1440, 5, o)
    t2 = time.perf_counter()
    print(f"decompress wall {1e3*(t2 - t1):.1f} ms", ctx.stats(), file=sys.stderr)
