"""Developer probe: a custom chunk_shape over the 37-level stack (four chunk
shapes incl. edge chunks) through the public API; containers must equal the
one-group-at-a-time result."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2510_22265_b200 as ebcc  # noqa: E402
from paper_2510_22265_b200 import pipeline  # noqa: E402

host = bench.workload(0)[None]
cs = (1, 1, 256, 512)
blobs = []
for mode in ("concurrent", "serial", "concurrent"):
    if mode == "serial":
        each = pipeline._each_group
        pipeline._each_group = lambda fn, groups, ctx: [fn(it) for it in groups.items()]  # (now the default too)
    for _ in range(2):
        t0 = time.perf_counter()
        blob = ebcc.compress(host, rel_error=0.01, chunk_shape=cs)
        t1 = time.perf_counter()
        out = ebcc.decompress(blob)
        t2 = time.perf_counter()
    if mode == "serial":
        pipeline._each_group = each
    blobs.append(blob)
    print(f"{mode}: compress {1e3*(t1-t0):.1f} ms, decompress {1e3*(t2-t1):.1f} ms, "
          f"{len(blob)} bytes", flush=True)
assert blobs[0] == blobs[1] == blobs[2]
err = np.abs(out.astype(np.float64) - host.astype(np.float64)).max()
print("containers identical; max abs error", err)
