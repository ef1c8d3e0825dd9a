"""Where the host time of a small drop-in call goes (GPU box): cProfile over repeated
``multi_head_attention_array`` calls at the GRN demo shape and the C1 shape."""

from __future__ import annotations

import cProfile
import io
import os
import pstats
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2505_09326_b200 import SPHERICAL
    from paper_2505_09326_b200.attention import multi_head_attention_array
    rng = np.random.default_rng(0)
    for (n, h, hkv, d) in ((12, 4, 2, 4), (256, 1, 1, 64), (256, 8, 8, 64)):
        q = rng.standard_normal((n, h, d)).astype(np.float32)
        k = rng.standard_normal((n, hkv, d)).astype(np.float32)
        v = rng.standard_normal((n, hkv, d)).astype(np.float32)
        for _ in range(20):
            multi_head_attention_array(q, k, v, SPHERICAL, h, hkv)
        reps = 300
        t0 = time.perf_counter()
        for _ in range(reps):
            multi_head_attention_array(q, k, v, SPHERICAL, h, hkv)
        us = 1e6 * (time.perf_counter() - t0) / reps
        print(f"shape n{n} h{h} hkv{hkv} d{d}: {us:.1f} us per call", flush=True)
        if (n, h) == (256, 8):
            pr = cProfile.Profile()
            pr.enable()
            for _ in range(reps):
                multi_head_attention_array(q, k, v, SPHERICAL, h, hkv)
            pr.disable()
            s = io.StringIO()
            pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(30)
            print(s.getvalue()[:6000])


if __name__ == "__main__":
    main()
