"""Developer probe: the configs[4] sweep's first N fields with the SPIHT base
(the reference's) and the opt-in J2 base (base_codec="ebcot"): device-resident
compress / decompress times and the container ratio."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_22265_b200 import _lib, fields  # noqa: E402

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 148
host = fields.config5_stack(range(nf))
x = torch.from_numpy(host).cuda()
pay = torch.empty(host.nbytes, dtype=torch.uint8, device="cuda")
out = torch.empty_like(x)
ctx = _lib.context(0)
F = _lib.INPUT_ON_DEVICE | _lib.OUTPUT_ON_DEVICE
for name, flag in (("spiht", 0), ("ebcot", _lib.BASE_EBCOT)):
    res = []
    for it in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        recs, offs, total, st = ctx.compress(x.data_ptr(), nf, 721, 1440, 0.01, 1 - 1e-5, 10.0,
                                             1e-3, flags=F | flag, payload=pay.data_ptr(),
                                             payload_cap=pay.numel())
        t1 = time.perf_counter()
        assert st == 0, (st, ctx.error())
        ctx.decompress(pay.data_ptr(), offs, recs, 721, 1440, 5, out.data_ptr(), flags=F)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        if it:
            res.append((t1 - t0, t2 - t1))
    c = min(r[0] for r in res)
    d = min(r[1] for r in res)
    err = ((out - x).abs().amax(dim=(1, 2)) / (x.amax(dim=(1, 2)) - x.amin(dim=(1, 2)))).max().item()
    modes = np.bincount(recs["mode"], minlength=3)
    print(f"{name} {nf} fields: compress {1e3*c:.1f} ms ({4*host.size/c/1e9:.2f} GB/s), "
          f"decompress {1e3*d:.1f} ms ({4*host.size/d/1e9:.2f} GB/s), ratio "
          f"{4*host.size/(total + 25*nf + 42):.3f}, max rel err {err:.5f}, modes {modes.tolist()}",
          flush=True)
