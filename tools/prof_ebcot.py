"""Developer probe: one compress + decompress of N configs[4] fields with the
opt-in J2 base layer (device-resident input), for ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_22265_b200 import _lib, fields  # noqa: E402

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 37
host = fields.config5_stack(range(nf))
x = torch.from_numpy(host).cuda()
pay = torch.empty(host.nbytes, dtype=torch.uint8, device="cuda")
out = torch.empty_like(x)
ctx = _lib.context(0)
F = _lib.INPUT_ON_DEVICE | _lib.OUTPUT_ON_DEVICE
recs, offs, total, st = ctx.compress(x.data_ptr(), nf, 721, 1440, 0.01, 1 - 1e-5, 10.0, 1e-3,
                                     flags=F | _lib.BASE_EBCOT, payload=pay.data_ptr(),
                                     payload_cap=pay.numel())
assert st == 0, ctx.error()
ctx.decompress(pay.data_ptr(), offs, recs, 721, 1440, 5, out.data_ptr(), flags=F)
torch.cuda.synchronize()
print("ok", total)
