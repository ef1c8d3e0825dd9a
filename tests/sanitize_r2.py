"""Small invocations of the round-2 paths for compute-sanitizer (experiment tool, not a test):
tail-split launches, fs_scale_keys, the Gram kernels, the fp16 overflow scan.
    compute-sanitizer --tool memcheck python tests/sanitize_r2.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_09326_b200 import flashsign as fs  # noqa: E402


def r(b, n, h, d, dt, seed, scale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn((b, n, h, d), generator=g, device="cuda") * scale).to(dt)


for dt in (torch.bfloat16, torch.float16):
    for d in (64, 128, 96):
        q, k, v = r(1, 600, 80, d, dt, 1), r(1, 1100, 40, d, dt, 2), r(1, 1100, 40, d, dt, 3)
        fs.fwd(q, k, v, kv_splits=3, split_tail=True, check=False)           # whole waves + tail items
        fs.fwd(r(2, 300, 3, d, dt, 4), r(2, 900, 1, d, dt, 5), r(2, 900, 1, d, dt, 6), kv_splits=2,
               split_tail=True, check=False)                                 # every tile a tail tile
        m = torch.randint(0, 6, (1, 1100), device="cuda").float()
        fs.fwd(q, k, v, key_scale=m, check=False)                            # fs_scale_keys + kernel
        fs.gram_fwd(q, k, v, key_scale=m, check=False)                       # Gram kernels
        fs.gram_fwd(q, k, v, out_dtype=torch.float32, check=False)
    # fp16 P overflow scan (rows whose z reaches the bound) and an empty key stream for the Gram path
q = r(1, 256, 2, 64, torch.float16, 7, scale=300.0)
fs.fwd(q, q, q, check=False)
fs.gram_fwd(r(1, 64, 1, 64, torch.bfloat16, 8), torch.empty((1, 0, 1, 64), dtype=torch.bfloat16, device="cuda"),
            torch.empty((1, 0, 1, 64), dtype=torch.bfloat16, device="cuda"), check=False)
torch.cuda.synchronize()
print("sanitize_r2 ok")
