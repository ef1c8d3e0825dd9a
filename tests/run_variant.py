"""Launch one A/B variant library (paper_2505_09326_b200/_lib/ab/libfs_NAME.so) on one configuration,
a few times -- a target for `ncu` (experiment tool, not a test).   python tests/run_variant.py NAME c5 [launches]"""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_09326_b200 import _lib  # noqa: E402
sys.path.insert(0, os.path.join(ROOT, "tests"))
from ab_variants import AB_DIR, CASES  # noqa: E402

name, cname = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 2
lib = ctypes.CDLL(os.path.join(AB_DIR, f"libfs_{name}.so"))
lib.fs_fwd.argtypes = [ctypes.POINTER(_lib.FsFwdParams), ctypes.c_void_p]
B, N, H, D, dt, eps = CASES[cname]
tdt = {"fp16": torch.float16, "bf16": torch.bfloat16, "e4m3": torch.float8_e4m3fn}[dt]
code = {"fp16": _lib.FS_F16, "bf16": _lib.FS_BF16, "e4m3": _lib.FS_E4M3}[dt]
q, k, v = (torch.randn((B, N, H, D), device="cuda").to(tdt) for _ in range(3))
o = torch.empty((B, N, H, D), dtype=torch.float16 if dt == "fp16" else torch.bfloat16, device="cuda")
bad = torch.empty(1, dtype=torch.int64, device="cuda")
p = _lib.FsFwdParams()
p.q, p.k, p.v, p.o = q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr()
for dst, t in ((p.q_stride, q), (p.k_stride, k), (p.v_stride, v), (p.o_stride, o)):
    dst[0], dst[1], dst[2] = t.stride(0), t.stride(1), t.stride(2)
p.batch, p.heads_q, p.heads_kv, p.seqlen_q, p.seqlen_kv, p.head_dim = B, H, H, N, N, D
p.in_dtype, p.out_dtype = code, (_lib.FS_F16 if dt == "fp16" else _lib.FS_BF16)
p.scale, p.eps, p.p_scale, p.q_descale, p.k_descale, p.v_descale = 1.0, eps, 1.0, 1.0, 1.0, 1.0
p.bad_key = bad.data_ptr()
for _ in range(n):
    assert lib.fs_fwd(ctypes.byref(p), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
torch.cuda.synchronize()
print("ok", name, cname)
