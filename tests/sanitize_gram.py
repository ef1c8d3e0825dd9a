"""The Gram-form and K' = m K kernels alone, for compute-sanitizer racecheck (experiment tool)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_09326_b200 import flashsign as fs  # noqa: E402

for dt in (torch.bfloat16, torch.float16):
    for d in (64, 128):
        g = torch.Generator(device="cuda").manual_seed(d)
        q, k, v = (torch.randn((2, 700, 4, d), generator=g, device="cuda").to(dt) for _ in range(3))
        m = torch.randint(0, 6, (2, 700), generator=g, device="cuda").float()
        fs.gram_fwd(q, k[:, :, :2], v[:, :, :2], key_scale=m, check=False)
        fs.gram_fwd(q, k, v, out_dtype=torch.float32, check=False)
torch.cuda.synchronize()
print("sanitize_gram ok")
