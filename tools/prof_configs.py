"""Developer probe: every BASELINE.json config on one GPU (device-resident
input): configs[0] single field, configs[1] at eps 0.1/1/10%, configs[2]
precipitation steps, configs[4] as batches of 296 sweep fields (the first
296 of the 2368, i.e. one GPU's share at 8 GPUs)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_22265_b200 import _lib, fields  # noqa: E402

ctx = _lib.context(0)
F = _lib.INPUT_ON_DEVICE | _lib.OUTPUT_ON_DEVICE


def run(name, host, eps, iters=3):
    host = np.ascontiguousarray(host.reshape(-1, host.shape[-2], host.shape[-1]))
    nf, R, C = host.shape
    x = torch.from_numpy(host).cuda()
    pay = torch.empty(host.nbytes * 2, dtype=torch.uint8, device="cuda")
    out = torch.empty_like(x)
    best = None
    for _ in range(iters):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        recs, offs, total, st = ctx.compress(x.data_ptr(), nf, R, C, eps, 1 - 1e-5, 10.0, 1e-3,
                                             flags=F, payload=pay.data_ptr(),
                                             payload_cap=pay.numel())
        t1 = time.perf_counter()
        ctx.decompress(pay.data_ptr(), offs, recs, R, C, 5, out.data_ptr(), flags=F)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        if best is None or (t2 - t0) < best[0] + best[1]:
            best = (t1 - t0, t2 - t1)
    back = out.cpu().numpy().astype(np.float64)
    h = host.astype(np.float64)
    rng = h.reshape(nf, -1).max(1) - h.reshape(nf, -1).min(1)
    ok = bool(np.all(np.abs(back - h).reshape(nf, -1).max(1) <= eps * rng))
    gb = host.nbytes / 1e9
    modes = np.bincount(recs["mode"], minlength=3)
    print(f"{name}: {nf} x {R}x{C} eps {eps:g}: compress {1e3*best[0]:.1f} ms "
          f"({gb/best[0]:.2f} GB/s), decompress {1e3*best[1]:.1f} ms ({gb/best[1]:.2f} GB/s), "
          f"round trip {gb/(best[0]+best[1]):.2f} GB/s, ratio "
          f"{host.nbytes/(total + 42 + 25*nf):.2f}, modes const/pure/two {modes.tolist()}, "
          f"bound {'ok' if ok else 'VIOLATED'}", flush=True)


run("configs[0]", fields.config1_field()[None], 0.01)
c2 = fields.config2_levels()
for eps in (0.001, 0.01, 0.1):
    run("configs[1]", c2, eps)
run("configs[2]", fields.config3_precip(), 0.01)
c5 = np.stack([fields.config5_field(i) for i in range(296)])
run("configs[4] share", c5, 0.01, iters=2)
