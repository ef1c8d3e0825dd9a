"""Host-side copy-in study for the numpy drop-in (hostpath staging); GPU box, one process per setting.

  python tests/stage_bench.py            # sweep: threads x slot MB, prints one JSON line per setting
  python tests/stage_bench.py --one      # (internal) one setting from the environment

Per setting: the pageable -> pinned fill alone, the staged H2D pipeline alone (``_Engine._h2d`` on
a 128 MB float32 array), and ``multi_head_attention_array`` on one C3 batch element
(16384 x 16 x 128 float32: 3 x 128 MB in, 128 MB out), wall clock, best of 3.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _best(fn, reps=3):
    b = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        b = min(b, time.perf_counter() - t0)
    return b


def one():
    sys.path.insert(0, ROOT)
    import torch

    from paper_2505_09326_b200 import SPHERICAL, hostpath
    from paper_2505_09326_b200.attention import multi_head_attention_array
    dev = torch.device("cuda", 0)
    n, h, d = 16384, 16, 128
    rng = np.random.default_rng(0)
    q, k, v = (rng.standard_normal((n, h, d), dtype=np.float32) for _ in range(3))
    multi_head_attention_array(q, k, v, SPHERICAL, h, h, scale=1.0)
    e = hostpath.engine(dev)
    nthr = e.pool._max_workers
    slot = e.ring[0][0].numel()
    # fill alone: pageable -> the pinned slot with the engine's threads
    flat = q.reshape(-1).view(np.uint8)[:slot]
    host = e.ring[0][0].numpy()
    step = -(-slot // nthr)

    def fill():
        if e.copy is not None:
            dp, sp = e.ring[0][0].data_ptr(), flat.ctypes.data
            list(e.pool.map(lambda j: e.copy(dp + j, sp + j, min(step, slot - j)), range(0, slot, step)))
        else:
            list(e.pool.map(lambda j: np.copyto(host[j:j + step], flat[j:j + step]), range(0, slot, step)))
    t_fill = _best(fill)
    # staged H2D pipeline alone
    dst = torch.empty((n * h, d), dtype=torch.float32, device=dev)

    def h2d():
        e._h2d(dst, q.reshape(-1, d))
        e.s_h2d.synchronize()
    t_h2d = _best(h2d)

    def call():
        multi_head_attention_array(q, k, v, SPHERICAL, h, h, scale=1.0)
    t_call = _best(call)
    print(json.dumps({"copy": "nt" if e.copy is not None else "numpy", "threads": nthr, "slot_mb": slot >> 20, "fill_gbs": slot / t_fill / 1e9,
                      "staged_h2d_gbs": q.nbytes / t_h2d / 1e9, "call_ms": t_call * 1e3,
                      "call_in_gbs": 3 * q.nbytes / t_call / 1e9, "cpus": os.cpu_count()}), flush=True)


def main():
    for rep in range(2):
        for copy in ("numpy", "nt"):
            for thr in (4, 8, 16):
                for slot in (16, 64):
                    env = dict(os.environ, FLASHSIGN_H2D_THREADS=str(thr), FLASHSIGN_STAGE_MB=str(slot),
                               FLASHSIGN_STAGE_COPY=copy)
                    subprocess.run([sys.executable, __file__, "--one"], env=env, check=False, timeout=300)




def register_study():
    """Pin the caller's pageable array in place (cudaHostRegister) instead of staging it."""
    import torch
    dev = torch.device("cuda", 0)
    cudart = torch.cuda.cudart()
    n = 128 << 20
    out = {}
    for label, alloc in (("fresh", lambda: np.ones(n // 4, dtype=np.float32)),):
        a = alloc()
        dst = torch.empty(n // 4, dtype=torch.float32, device=dev)
        torch.cuda.synchronize()
        regs, unregs, dmas, whole = [], [], [], []
        for _ in range(3):
            t0 = time.perf_counter()
            r = cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
            t1 = time.perf_counter()
            src = torch.from_numpy(a)
            pinned = src.is_pinned()
            dst.copy_(src, non_blocking=True)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            cudart.cudaHostUnregister(a.ctypes.data)
            t3 = time.perf_counter()
            regs.append(t1 - t0); dmas.append(t2 - t1); unregs.append(t3 - t2); whole.append(t3 - t0)
        out[label] = {"register_rc": int(r), "is_pinned_after": bool(pinned), "register_gbs": n / min(regs) / 1e9,
                      "dma_gbs": n / min(dmas) / 1e9, "unregister_gbs": n / min(unregs) / 1e9,
                      "whole_gbs": n / min(whole) / 1e9}
        # chunked: register chunk i+1 while chunk i's DMA runs
        for chunk_mb in (8, 32):
            cb = chunk_mb << 20
            s = torch.cuda.Stream(dev)
            best = float("inf")
            for _ in range(3):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                flat = a.view(np.uint8)
                dflat = dst.view(torch.uint8)
                for lo in range(0, n, cb):
                    hi = min(n, lo + cb)
                    cudart.cudaHostRegister(flat[lo:].ctypes.data, hi - lo, 0)
                    with torch.cuda.stream(s):
                        dflat[lo:hi].copy_(torch.from_numpy(flat[lo:hi]), non_blocking=True)
                s.synchronize()
                for lo in range(0, n, cb):
                    cudart.cudaHostUnregister(flat[lo:].ctypes.data)
                best = min(best, time.perf_counter() - t0)
            out[f"chunked_{chunk_mb}mb_gbs"] = n / best / 1e9
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    if "--one" in sys.argv:
        one()
    elif "--register" in sys.argv:
        register_study()
    else:
        main()
