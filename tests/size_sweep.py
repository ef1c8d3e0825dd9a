"""Drop-in call time against array size for the three host paths (GPU box; experiment tool):
packed small path, three-stream pipeline with pageable copies, with the pinned staging ring."""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2505_09326_b200 import SPHERICAL, hostpath
    from paper_2505_09326_b200.attention import multi_head_attention_array
    h, d = 8, 64
    rng = np.random.default_rng(0)
    for mb in (0.25, 0.5, 1, 2, 4, 8, 16):
        n = int(mb * (1 << 20) / (h * d * 4))
        q, k, v = (rng.standard_normal((n, h, d)).astype(np.float32) for _ in range(3))
        row = {"mb_per_array": mb, "n": n}
        for name, small, stage_min, mode in (("small", 1 << 40, None, "auto"), ("pageable", 0, None, "pageable"),
                                             ("staged", 0, None, "staged")):
            hostpath._SMALL_BYTES = small
            hostpath._engines.clear()
            os.environ["FLASHSIGN_H2D"] = mode
            for _ in range(3):
                multi_head_attention_array(q, k, v, SPHERICAL, h, h)
            reps = max(3, int(0.3 / max(1e-4, mb * 3e-3)))
            t0 = time.perf_counter()
            for _ in range(reps):
                multi_head_attention_array(q, k, v, SPHERICAL, h, h)
            row[name + "_us"] = round(1e6 * (time.perf_counter() - t0) / reps, 1)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
