"""Developer probe: level-0 kernel time of full base probes (37 x 721x1440,
one lane) at a few budgets; EBCC_LIB selects a library variant."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["EBCC_LANES"] = "1"
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_22265_b200 import _lib  # noqa: E402

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 37
host = bench.workload(0)[:nf].copy()
x = torch.from_numpy(host).cuda()
pay = torch.empty(host.nbytes * 2, dtype=torch.uint8, device="cuda")
ctx = _lib.context(0)
F = _lib.INPUT_ON_DEVICE | _lib.OUTPUT_ON_DEVICE
ctx.compress(x.data_ptr(), nf, 721, 1440, 0.01, 1 - 1e-5, 10.0, 1e-3, flags=F,
             payload=pay.data_ptr(), payload_cap=pay.numel())
tag = os.environ.get("EBCC_LIB", "default")
for frac in (0.2, 1.0):
    for early in (0, 1):
        l0, allp = ctx.dev_probe_bench(frac, 30, early)
        print(f"{os.path.basename(tag)} frac {frac} early {early}: level0 {l0:.1f} us, probe {allp:.1f} us")
