"""Developer probe: compress / decompress time of BASELINE configs[3]
(10 variables x 2881x5760, eps 1%) on one GPU, device-resident input."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_22265_b200 import _lib, fields  # noqa: E402

nv = int(sys.argv[1]) if len(sys.argv) > 1 else 10
host = np.stack([fields.config4_field(v) for v in range(nv)])
R, C = host.shape[1:]
x = torch.from_numpy(host).cuda()
pay = torch.empty(host.nbytes * 2, dtype=torch.uint8, device="cuda")
out = torch.empty_like(x)
ctx = _lib.context(0)
F = _lib.INPUT_ON_DEVICE | _lib.OUTPUT_ON_DEVICE
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    recs, offs, total, st = ctx.compress(x.data_ptr(), nv, R, C, 0.01, 1 - 1e-5, 10.0, 1e-3,
                                         flags=F, payload=pay.data_ptr(), payload_cap=pay.numel())
    t1 = time.perf_counter()
    ctx.decompress(pay.data_ptr(), offs, recs, R, C, 5, out.data_ptr(), flags=F)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    gb = host.nbytes / 1e9
    print(f"configs[3] {nv} x {R}x{C}: compress {1e3*(t1-t0):.1f} ms ({gb/(t1-t0):.2f} GB/s), "
          f"decompress {1e3*(t2-t1):.1f} ms ({gb/(t2-t1):.2f} GB/s), ratio "
          f"{host.nbytes / (total + 42 + 25 * nv):.2f}, lanes {ctx.stats()['lanes']}", flush=True)
