"""Developer probe: PCIe copy throughput of page-locked buffers with 1, 2 and
4 concurrent copies (streams) in each direction."""
import sys
import time

import torch

nbytes = 37 * 721 * 1440 * 4
d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
streams = [torch.cuda.Stream() for _ in range(4)]
for direction in ("d2h", "h2d"):
    for k in (1, 2, 4):
        def go():
            step = nbytes // k
            for i in range(k):
                with torch.cuda.stream(streams[i]):
                    a, b = i * step, (i + 1) * step if i < k - 1 else nbytes
                    if direction == "d2h":
                        h[a:b].copy_(d[a:b], non_blocking=True)
                    else:
                        d[a:b].copy_(h[a:b], non_blocking=True)
        go()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            go()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 5
        print(f"{direction} x{k}: {nbytes / dt / 1e9:.1f} GB/s", file=sys.stderr)
