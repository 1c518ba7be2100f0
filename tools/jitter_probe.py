"""Developer probe: correlate compress/decompress tail latencies with SM clocks
and clock-event reasons sampled through NVML every few ms."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml as nv  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_22265_b200 import _lib  # noqa: E402

nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
samples = []
stop = threading.Event()


def poll():
    while not stop.is_set():
        t = time.perf_counter()
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        samples.append((t, nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), int(r)))
        time.sleep(0.002)


host = bench.workload(0)
x = torch.from_numpy(host).cuda()
pay = torch.empty(host.nbytes * 2, dtype=torch.uint8, device="cuda")
out = torch.empty_like(x)
ctx = _lib.context(0)
F = _lib.INPUT_ON_DEVICE | _lib.OUTPUT_ON_DEVICE
th = threading.Thread(target=poll, daemon=True)
th.start()
rows = []
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 40):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    recs, offs, total, st = ctx.compress(x.data_ptr(), 37, 721, 1440, 0.01, 1 - 1e-5, 10.0, 1e-3,
                                         flags=F, payload=pay.data_ptr(), payload_cap=pay.numel())
    t1 = time.perf_counter()
    ctx.decompress(pay.data_ptr(), offs, recs, 721, 1440, 5, out.data_ptr(), flags=F)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    rows.append((t0, t1, t2))
stop.set()
th.join()
cs = sorted((t1 - t0) * 1e3 for t0, t1, t2 in rows[1:])
ds = sorted((t2 - t1) * 1e3 for t0, t1, t2 in rows[1:])
medc, medd = cs[len(cs) // 2], ds[len(ds) // 2]
print(f"compress median {medc:.1f} max {cs[-1]:.1f}; decompress median {medd:.1f} max {ds[-1]:.1f}")
for t0, t1, t2 in rows[1:]:
    for name, a, b, med in (("compress", t0, t1, medc), ("decompress", t1, t2, medd)):
        if (b - a) * 1e3 > 1.5 * med:
            win = [s for s in samples if a <= s[0] <= b]
            clk = sorted(s[1] for s in win)
            reasons = sorted({hex(s[2]) for s in win})
            print(f"  slow {name} {1e3 * (b - a):.1f} ms: {len(win)} samples, sm clock "
                  f"min {clk[0] if clk else None} max {clk[-1] if clk else None}, reasons {reasons}")
