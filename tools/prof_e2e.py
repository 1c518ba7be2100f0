"""Developer probe: where the public-API (host buffers) round trip spends time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2510_22265_b200 as ebcc  # noqa: E402
from paper_2510_22265_b200 import _lib, core  # noqa: E402
from paper_2510_22265_b200.chunk import EbccParams  # noqa: E402
from paper_2510_22265_b200.container import assemble, parse  # noqa: E402
from paper_2510_22265_b200.pipeline import grid_to_records, records_to_grid  # noqa: E402

host = bench.workload(0)
pinned = torch.empty(host.shape, dtype=torch.float32, pin_memory=True)
pinned.numpy()[...] = host
arr = pinned.numpy()
for it in range(3):
    T = {}
    t = time.perf_counter()
    grid = core.grid_from_array(arr)
    T["grid_from_array"] = time.perf_counter() - t
    t = time.perf_counter()
    recs, payload, offs, _ = grid_to_records(grid, EbccParams(0.01))
    T["compress_records"] = time.perf_counter() - t
    t = time.perf_counter()
    blob = assemble(grid.dims, grid.chunk_shape, recs, payload, offs)
    T["assemble"] = time.perf_counter() - t
    t = time.perf_counter()
    dims, cs, r2, o2, data = parse(blob)
    T["parse"] = time.perf_counter() - t
    t = time.perf_counter()
    out = records_to_grid(dims, cs, r2, o2, data)
    T["decompress"] = time.perf_counter() - t
    print({k: round(v * 1e3, 1) for k, v in T.items()}, "total", round(sum(T.values()) * 1e3, 1),
          _lib.context().stats()["ms_total"], file=sys.stderr)

# the public API as bench.py times it
res = []
for it in range(4):
    t = time.perf_counter()
    blob = ebcc.compress(arr, rel_error=0.01)
    t1 = time.perf_counter()
    st1 = dict(_lib.context().stats())
    res.append(ebcc.decompress(blob))
    t2 = time.perf_counter()
    st2 = dict(_lib.context().stats())
    res = res[-2:]
    print(f"api compress {1e3 * (t1 - t):.1f} ms (device {st1['ms_total']:.1f}), "
          f"decompress {1e3 * (t2 - t1):.1f} ms (device {st2['ms_total']:.1f})", file=sys.stderr)

