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
if os.environ.get("SANITIZE_GRAM_BIG") == "1":
    # ~7 query tiles per CTA: the apply kernel's Q ring and accumulator buffers wrap
    g = torch.Generator(device="cuda").manual_seed(7)
    q, k, v = (torch.randn((4, 4096, 8, 128), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
    fs.gram_fwd(q, k, v, check=False)
    if os.environ.get("SANITIZE_GRAM_ONLY") == "1":
        torch.cuda.synchronize()
        print("sanitize_gram ok")
        sys.exit(0)
torch.cuda.synchronize()
print("sanitize_gram ok")
# the float64 mode kernel (fs_exact_fwd) through the drop-in API
import numpy as np  # noqa: E402

from paper_2505_09326_b200 import SPHERICAL, attention  # noqa: E402

attention.set_compute_dtype("f64")
rng = np.random.default_rng(3)
for (y, x, d) in ((70, 100, 32), (130, 70, 64), (65, 33, 128)):
    q, k, v = (rng.standard_normal((n, d)).astype(np.float32) for n in (y, x, x))
    attention.streamed_attention_array(q, k, v, SPHERICAL, 0.5, attention.TileConfig())
torch.cuda.synchronize()
print("sanitize_exact ok")
