import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
from paper_2510_22265_b200 import _lib, fields
nf = 2368
host = fields.config5_stack(range(nf))
x = torch.from_numpy(host).cuda()
pay = torch.empty(host.nbytes // 2, dtype=torch.uint8, device="cuda")
out = torch.empty_like(x)
ctx = _lib.context(0)
F = _lib.INPUT_ON_DEVICE | _lib.OUTPUT_ON_DEVICE
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    recs, offs, total, st = ctx.compress(x.data_ptr(), nf, 721, 1440, 0.01, 1 - 1e-5, 10.0, 1e-3, flags=F, payload=pay.data_ptr(), payload_cap=pay.numel())
    t1 = time.perf_counter()
    ctx.decompress(pay.data_ptr(), offs, recs, 721, 1440, 5, out.data_ptr(), flags=F)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    free, tot = torch.cuda.mem_get_info()
    print(f"it{it} compress {1e3*(t1-t0):.0f} ms decompress {1e3*(t2-t1):.0f} ms free {free/1e9:.1f} GB", flush=True)
