"""Developer probe: time ebcc_compress / ebcc_decompress on the bench workload
with device-resident inputs (EBCC_PROFILE=1 prints per-phase host wall time)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_22265_b200 import _lib  # noqa: E402

levels = int(sys.argv[1]) if len(sys.argv) > 1 else 37
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
base = bench.workload(0)
host = np.concatenate([base] * ((levels + len(base) - 1) // len(base)))[:levels].copy()
x = torch.from_numpy(host).cuda()
pay = torch.empty(host.nbytes * 2, dtype=torch.uint8, device="cuda")
out = torch.empty_like(x)
ctx = _lib.context(0)
if os.environ.get("TORCH_STREAM") == "1":
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
F = _lib.INPUT_ON_DEVICE | _lib.OUTPUT_ON_DEVICE
for it in range(iters):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    recs, offs, total, st = ctx.compress(x.data_ptr(), levels, 721, 1440, 0.01, 1 - 1e-5, 10.0,
                                         1e-3, flags=F, payload=pay.data_ptr(),
                                         payload_cap=pay.numel())
    t1 = time.perf_counter()
    if st:
        print("compress status", st, ctx.error(), file=sys.stderr)
    print(f"compress wall {1e3*(t1 - t0):.1f} ms", ctx.stats(), file=sys.stderr)
    ctx.decompress(pay.data_ptr(), offs, recs, 721, 1440, 5, out.data_ptr(), flags=F)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"decompress wall {1e3*(t2 - t1):.1f} ms", ctx.stats(), file=sys.stderr)
