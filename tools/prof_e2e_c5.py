"""Developer probe: the public-API round trip of the configs[4] sweep
(pageable host input, as bench.py's e2e) split into host phases."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2510_22265_b200 as ebcc  # noqa: E402
from paper_2510_22265_b200 import _lib, fields  # noqa: E402
from paper_2510_22265_b200.container import parse  # noqa: E402
from paper_2510_22265_b200.pipeline import records_to_grid  # noqa: E402

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 2368
host = fields.config5_stack(range(nf)).reshape(-1, 37, 721, 1440)
tag = os.environ.get("TAG", "")
for it in range(4):
    t0 = time.perf_counter()
    blob = ebcc.compress(host, rel_error=0.01)
    t1 = time.perf_counter()
    dc = _lib.context().stats()["ms_total"]
    dims, cs, r2, o2, data = parse(blob)
    t2 = time.perf_counter()
    out = records_to_grid(dims, cs, r2, o2, data)
    t3 = time.perf_counter()
    dd = _lib.context().stats()["ms_total"]
    del out
    print(f"{tag} it{it}: compress {1e3*(t1-t0):.0f} ms (device {dc:.0f}), parse {1e3*(t2-t1):.1f} ms,"
          f" decompress {1e3*(t3-t2):.0f} ms (device {dd:.0f})", flush=True)
