"""A/B of Gram-form builds (experiment tool): python tests/gram_ab.py build NAME=FLAGS ... | run."""

import ctypes
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
AB_DIR = os.path.join(ROOT, "paper_2505_09326_b200", "_lib", "ab")


def build(specs):
    from paper_2505_09326_b200 import build as b
    os.makedirs(AB_DIR, exist_ok=True)
    for spec in specs:
        name, _, flags = spec.partition("=")
        out = os.path.join(AB_DIR, f"libgram_{name}.so")
        srcs = [os.path.join(b.CSRC, f) for f in ("flashsign_fwd.cu", "flashsign_gram.cu", "flashsign_prep.cu",
                                                  "flashsign_exact.cu", "fs_host.cpp")]
        subprocess.run([b._nvcc(), *b.NVCC_FLAGS, *flags.split(), "-o", out, *srcs], check=True, cwd=b.CSRC)


def run():
    import torch
    from paper_2505_09326_b200 import _lib
    libs = {os.path.basename(p)[8:-3]: ctypes.CDLL(p) for p in sorted(glob.glob(os.path.join(AB_DIR, "libgram_*.so")))}
    for cname, (B, N, H, D) in {"c3": (8, 16384, 16, 128), "c5": (64, 20000, 8, 64)}.items():
        g = torch.Generator(device="cuda").manual_seed(0)
        q, k, v = (torch.randn((B, N, H, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
        o = torch.empty_like(q)
        p = _lib.FsFwdParams()
        p.q, p.k, p.v, p.o = q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr()
        for dst, t in ((p.q_stride, q), (p.k_stride, k), (p.v_stride, v), (p.o_stride, o)):
            dst[0], dst[1], dst[2] = t.stride(0), t.stride(1), t.stride(2)
        p.batch, p.heads_q, p.heads_kv, p.seqlen_q, p.seqlen_kv, p.head_dim = B, H, H, N, N, D
        p.in_dtype = p.out_dtype = _lib.FS_BF16
        p.scale, p.eps, p.p_scale, p.q_descale, p.k_descale, p.v_descale = 1.0, 1e-6, 1.0, 1.0, 1.0, 1.0
        s = torch.cuda.current_stream().cuda_stream
        res, outs = {}, {}
        for rnd in range(4):
            for name, lib in libs.items():
                lib.fs_gram_workspace_bytes.restype = ctypes.c_int64
                ws_b = lib.fs_gram_workspace_bytes(ctypes.byref(p))
                ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
                fn = lambda: lib.fs_gram_fwd(ctypes.byref(p), ctypes.c_void_p(ws.data_ptr()), ctypes.c_int64(ws_b),  # noqa: E731
                                             ctypes.c_void_p(s))
                for _ in range(3):
                    assert fn() == 0
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(30):
                    fn()
                e1.record()
                torch.cuda.synchronize()
                if rnd:
                    res.setdefault(name, []).append(e0.elapsed_time(e1) / 30)
                outs[name] = o.clone()
        for name, lib in libs.items():  # -DFS_GRAM_PROF=1 builds: per-role waits of the apply kernel
            if not hasattr(lib, "fs_gram_prof_read"):
                continue
            buf = (ctypes.c_ulonglong * 8)()
            wb = lib.fs_gram_workspace_bytes(ctypes.byref(p))
            ws = torch.empty(wb, dtype=torch.uint8, device="cuda")
            lib.fs_gram_prof_read(buf)
            lib.fs_gram_fwd(ctypes.byref(p), ctypes.c_void_p(ws.data_ptr()), ctypes.c_int64(wb), ctypes.c_void_p(s))
            torch.cuda.synchronize()
            lib.fs_gram_prof_read(buf)
            b = list(buf)
            nt = max(b[3], 1)
            print(cname, name, "per tile (cycles): mma wait q_full", b[0] // nt, "mma wait t_empty", b[1] // nt,
                  "mma loop", b[2] // nt, "producer wait q_empty", b[4] // nt, "epilogue(warp 2) wait t_full",
                  b[5] // nt, "tiles", b[3], flush=True)
        ref = next(iter(outs.values()))
        for name in libs:
            ms = sorted(res[name])[len(res[name]) // 2]
            print(cname, name, f"{ms * 1e3:.1f} us", "max_abs_vs_first", float((outs[name].float() - ref.float()).abs().max()),
                  flush=True)


if __name__ == "__main__":
    build(sys.argv[2:]) if sys.argv[1] == "build" else run()
