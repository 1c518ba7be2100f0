"""Developer probe: public-API compress of the configs[4] sweep (pageable host
input) split into ebcc_compress and the container fetch; EBCC_TRACE=1 adds
the per-lane timeline."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2510_22265_b200 import _lib, fields  # noqa: E402
from paper_2510_22265_b200.chunk import EbccParams  # noqa: E402
from paper_2510_22265_b200.container import RECORD_DTYPE, pack_header  # noqa: E402
from paper_2510_22265_b200.pipeline import compress_batch  # noqa: E402

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 2368
host = fields.config5_stack(range(nf))
ctx = _lib.context()
p = EbccParams(0.01)
for it in range(3):
    t0 = time.perf_counter()
    recs, offs, total, st = compress_batch(host, p, ctx, fetch=False)
    t1 = time.perf_counter()
    dc = ctx.stats()["ms_total"]
    out = np.zeros(len(recs), dtype=RECORD_DTYPE)
    for k in ("mode", "vmin", "vmax", "base_len", "resid_len"):
        out[k] = recs[k]
    out["eps"], out["q"] = 0.01, p.q
    t2 = time.perf_counter()
    blob = ctx.fetch_container(pack_header((nf, 1, 721, 1440), (1, 1, 721, 1440), nf), out, total)
    t3 = time.perf_counter()
    print(f"it{it}: ebcc_compress {1e3*(t1-t0):.0f} ms (device span {dc:.0f}), records "
          f"{1e3*(t2-t1):.1f} ms, fetch_container {1e3*(t3-t2):.0f} ms ({len(blob)/1e9:.2f} GB)",
          flush=True)
