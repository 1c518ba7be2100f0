"""Developer probe: host<->device copy bandwidth of page-locked buffers, and
decompress into a page-locked host array vs a device array."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_22265_b200 import _lib  # noqa: E402

nbytes = 37 * 721 * 1440 * 4
d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
for name, fn in (("d2h", lambda: h.copy_(d, non_blocking=True)),
                 ("h2d", lambda: d.copy_(h, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print(f"{name}: {nbytes / dt / 1e9:.1f} GB/s ({dt * 1e3:.2f} ms)", file=sys.stderr)

host = bench.workload(0)
x = torch.from_numpy(host).cuda()
pay = torch.empty(host.nbytes * 2, dtype=torch.uint8, device="cuda")
outd = torch.empty_like(x)
outh = torch.empty(x.shape, dtype=torch.float32, pin_memory=True)
ctx = _lib.context(0)
F = _lib.INPUT_ON_DEVICE | _lib.OUTPUT_ON_DEVICE
recs, offs, total, st = ctx.compress(x.data_ptr(), 37, 721, 1440, 0.01, 1 - 1e-5, 10.0, 1e-3,
                                     flags=F, payload=pay.data_ptr(), payload_cap=pay.numel())
for it in range(3):
    for name, ptr, fl in (("device out", outd.data_ptr(), F), ("pinned host out", outh.data_ptr(), _lib.INPUT_ON_DEVICE)):
        torch.cuda.synchronize()
        t = time.perf_counter()
        ctx.decompress(pay.data_ptr(), offs, recs, 721, 1440, 5, ptr, flags=fl)
        torch.cuda.synchronize()
        print(f"decompress -> {name}: {1e3 * (time.perf_counter() - t):.2f} ms "
              f"(device {ctx.stats()['ms_total']:.2f})", file=sys.stderr)
