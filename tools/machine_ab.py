"""Developer A/B: compress / decompress wall time of N fields (device input)
for the library variant in EBCC_LIB."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_22265_b200 import _lib, fields  # noqa: E402

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 474
host = fields.config5_stack(range(nf))
x = torch.from_numpy(host).cuda()
pay = torch.empty(host.nbytes, dtype=torch.uint8, device="cuda")
out = torch.empty_like(x)
ctx = _lib.context(0)
F = _lib.INPUT_ON_DEVICE | _lib.OUTPUT_ON_DEVICE
tag = os.path.basename(os.environ.get("EBCC_LIB", "default"))
res = []
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    recs, offs, total, st = ctx.compress(x.data_ptr(), nf, 721, 1440, 0.01, 1 - 1e-5, 10.0, 1e-3,
                                         flags=F, payload=pay.data_ptr(), payload_cap=pay.numel())
    t1 = time.perf_counter()
    cst = ctx.stats()
    ctx.decompress(pay.data_ptr(), offs, recs, 721, 1440, 5, out.data_ptr(), flags=F)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    if it:
        res.append((t1 - t0, t2 - t1))
c = min(r[0] for r in res)
d = min(r[1] for r in res)
print(f"{tag} {nf} fields: compress {1e3*c:.1f} ms ({4*host.size/c/1e9:.2f} GB/s), "
      f"decompress {1e3*d:.1f} ms ({4*host.size/d/1e9:.2f} GB/s), total payload {total}, "
      f"probe steps {cst.get('probe_launches')}", flush=True)
