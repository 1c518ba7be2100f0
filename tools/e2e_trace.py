"""Developer probe: EBCC_TRACE=1 timeline of the public-API round trip of the
configs[4] sweep (pageable host arrays)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2510_22265_b200 as ebcc
from paper_2510_22265_b200 import fields
nf = int(sys.argv[1]) if len(sys.argv) > 1 else 2368
host = fields.config5_stack(range(nf)).reshape(-1, 37, 721, 1440)
for it in range(3):
    t0 = time.perf_counter()
    blob = ebcc.compress(host, rel_error=0.01, q=1 - 1e-5)
    t1 = time.perf_counter()
    out = ebcc.decompress(blob)
    t2 = time.perf_counter()
    print(f"it{it} compress {1e3*(t1-t0):.0f} ms decompress {1e3*(t2-t1):.0f} ms", flush=True)
    del out
