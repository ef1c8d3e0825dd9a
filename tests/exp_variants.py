"""Kernel-variant timing experiment (not a test): loads _lib/exp/libfs_*.so built with
-DFS_VARIANT=n and times each on C3/C2/C4 shapes.  Results -> gpurun_out/exp_variants.json."""

import ctypes
import glob
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_09326_b200 import _lib  # noqa: E402

CASES = {
    "c3": (8, 16384, 16, 128, torch.bfloat16, _lib.FS_BF16),
    "c2": (16, 4096, 16, 64, torch.float16, _lib.FS_F16),
    "c4": (8, 8192, 16, 128, torch.float8_e4m3fn, _lib.FS_E4M3),
}


def params(q, k, v, o, code, out_code, bad):
    p = _lib.FsFwdParams()
    p.q, p.k, p.v, p.o = q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr()
    for dst, t in ((p.q_stride, q), (p.k_stride, k), (p.v_stride, v), (p.o_stride, o)):
        dst[0], dst[1], dst[2] = t.stride(0), t.stride(1), t.stride(2)
    p.batch, p.heads_q, p.heads_kv = q.shape[0], q.shape[2], k.shape[2]
    p.seqlen_q, p.seqlen_kv, p.head_dim = q.shape[1], k.shape[1], q.shape[3]
    p.in_dtype, p.out_dtype = code, out_code
    p.scale, p.eps, p.p_scale, p.q_descale, p.k_descale, p.v_descale = 1, 0, 1, 1, 1, 1
    p.bad_key = bad.data_ptr()
    return p


def main():
    res = {}
    libs = sorted(glob.glob(os.path.join(os.path.dirname(_lib.LIB_PATH), "exp", "libfs_*.so")))
    for name, (B, N, H, D, dt, code) in CASES.items():
        g = torch.Generator(device="cuda").manual_seed(0)
        q, k, v = (torch.randn((B, N, H, D), generator=g, device="cuda").to(dt) for _ in range(3))
        o = torch.empty((B, N, H, D), dtype=torch.bfloat16 if code == _lib.FS_E4M3 else dt, device="cuda")
        out_code = _lib.FS_BF16 if code != _lib.FS_F16 else _lib.FS_F16
        bad = torch.empty(1, dtype=torch.int64, device="cuda")
        flops = 4.0 * B * H * N * N * D
        for path in libs:
            lib = ctypes.CDLL(path)
            lib.fs_fwd.argtypes = [ctypes.POINTER(_lib.FsFwdParams), ctypes.c_void_p]
            p = params(q, k, v, o, code, out_code, bad)
            s = torch.cuda.current_stream().cuda_stream
            for _ in range(3):
                assert lib.fs_fwd(ctypes.byref(p), ctypes.c_void_p(s)) == 0
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            n = 20
            for _ in range(n):
                lib.fs_fwd(ctypes.byref(p), ctypes.c_void_p(s))
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / n
            try:
                import pynvml
                pynvml.nvmlInit()
                clk = pynvml.nvmlDeviceGetClockInfo(pynvml.nvmlDeviceGetHandleByIndex(0), pynvml.NVML_CLOCK_SM)
            except Exception:
                clk = None
            key = f"{name}/{os.path.basename(path)}"
            res[key] = {"ms": ms, "tflops": flops / ms / 1e9, "sm_mhz_after": clk}
            print(key, res[key], flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(res, open("gpurun_out/exp_variants.json", "w"), indent=1)


if __name__ == "__main__":
    main()
