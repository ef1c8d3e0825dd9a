"""A/B timing of kernel build variants in one process (experiment tool, not a test).

    python tests/ab_variants.py build base= nwt4=-DFS_NWT=4      # here (nvcc cross-compiles)
    python tests/ab_variants.py run [c2 c3 c4 c5] [--rounds R]   # on the GPU box

``build`` compiles csrc/flashsign_fwd.cu once per NAME=FLAGS into
paper_2505_09326_b200/_lib/ab/libfs_NAME.so.  ``run`` loads every variant and, per
configuration, alternates them round-robin (same thermal/power state), timing
back-to-back launches with CUDA events while NVML samples the SM clock.  Reports the
median TFLOP/s, the median SM clock and TFLOP/s per GHz -> gpurun_out/ab_variants.json.
"""

import ctypes
import glob
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
AB_DIR = os.path.join(ROOT, "paper_2505_09326_b200", "_lib", "ab")

CASES = {  # name: (B, N, H, D, dtype, eps)
    "c2": (16, 4096, 16, 64, "fp16", 0.0),
    "c2b": (16, 4096, 16, 64, "bf16", 0.0),
    "c5h": (64, 20000, 8, 64, "fp16", 1e-6),
    "c3": (8, 16384, 16, 128, "bf16", 0.0),
    "c4": (8, 8192, 16, 128, "e4m3", 0.0),
    "c5": (64, 20000, 8, 64, "bf16", 1e-6),
    "c5m": (64, 20000, 8, 64, "bf16", 1e-6),   # + fused multiplicities m in {0..5} (key_scale)
    "c3m": (8, 16384, 16, 128, "bf16", 1e-6),
}


def build(specs):
    from paper_2505_09326_b200 import build as b
    os.makedirs(AB_DIR, exist_ok=True)
    for spec in specs:
        name, _, flags = spec.partition("=")
        out = os.path.join(AB_DIR, f"libfs_{name}.so")
        cmd = [b._nvcc(), *b.NVCC_FLAGS, *flags.split(), "-o", out, os.path.join(b.CSRC, "flashsign_fwd.cu")]
        print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True, cwd=b.CSRC)


def run(cases, rounds):
    import torch
    from paper_2505_09326_b200 import _lib
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    except Exception:
        pynvml = None
    libs = {}
    for path in sorted(glob.glob(os.path.join(AB_DIR, "libfs_*.so"))):
        lib = ctypes.CDLL(path)
        lib.fs_fwd.argtypes = [ctypes.POINTER(_lib.FsFwdParams), ctypes.c_void_p]
        lib.fs_fwd.restype = ctypes.c_int
        lib.fs_last_error.restype = ctypes.c_char_p
        if hasattr(lib, "fs_prof_timeline"):
            lib.fs_prof_timeline.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
        libs[os.path.basename(path)[6:-3]] = lib
    tdt = {"fp16": torch.float16, "bf16": torch.bfloat16, "e4m3": torch.float8_e4m3fn}
    code = {"fp16": _lib.FS_F16, "bf16": _lib.FS_BF16, "e4m3": _lib.FS_E4M3}
    res = {}
    for cname in cases:
        auto = cname.endswith("a")
        B, N, H, D, dt, eps = CASES[cname[:-1] if auto else cname]
        g = torch.Generator(device="cuda").manual_seed(0)
        q, k, v = (torch.randn((B, N, H, D), generator=g, device="cuda").to(tdt[dt]) for _ in range(3))
        odt = torch.float16 if dt == "fp16" else torch.bfloat16
        o = torch.empty((B, N, H, D), dtype=odt, device="cuda")
        bad = torch.empty(1, dtype=torch.int64, device="cuda")
        p = _lib.FsFwdParams()
        p.q, p.k, p.v, p.o = q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr()
        for dst, t in ((p.q_stride, q), (p.k_stride, k), (p.v_stride, v), (p.o_stride, o)):
            dst[0], dst[1], dst[2] = t.stride(0), t.stride(1), t.stride(2)
        p.batch, p.heads_q, p.heads_kv, p.seqlen_q, p.seqlen_kv, p.head_dim = B, H, H, N, N, D
        p.in_dtype, p.out_dtype = code[dt], (_lib.FS_F16 if dt == "fp16" else _lib.FS_BF16)
        p.scale, p.eps, p.p_scale, p.q_descale, p.k_descale, p.v_descale = 1.0, eps, 1.0, 1.0, 1.0, 1.0
        p.bad_key = bad.data_ptr()
        if auto:  # the library's split plan (tail-wave K/V split + merge), as flashsign.fwd runs it
            lib0 = next(iter(libs.values()))
            lib0.fs_partial_floats.restype = ctypes.c_int64
            p.kv_splits = _lib.FS_SPLITS_AUTO
            nf = lib0.fs_partial_floats(ctypes.byref(p))
            part = torch.empty(max(1, nf), dtype=torch.float32, device="cuda")
            p.partial = part.data_ptr()
        if cname.endswith("m"):
            m = torch.randint(0, 6, (B, N), generator=g, device="cuda").float()
            p.key_scale, p.key_scale_stride = m.data_ptr(), m.stride(0)
        flops = 4.0 * B * H * N * N * D
        s = torch.cuda.current_stream().cuda_stream
        est_ms = flops / 1.2e15 * 1e3
        n = max(5, int(300.0 / est_ms))  # ~300 ms of back-to-back launches per sample
        samples = {name: [] for name in libs}
        outs = {}
        for rnd in range(rounds + 1):
            for name, lib in libs.items():
                for _ in range(2):
                    rc = lib.fs_fwd(ctypes.byref(p), ctypes.c_void_p(s))
                    assert rc == 0, lib.fs_last_error()
                torch.cuda.synchronize()
                clk, pw, stop = [], [], threading.Event()

                def sampler():
                    while not stop.is_set():
                        if pynvml is not None:
                            clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                            try:
                                fv = pynvml.nvmlDeviceGetFieldValues(h, [pynvml.NVML_FI_DEV_POWER_INSTANT])[0]
                                if fv.nvmlReturn == 0:
                                    pw.append(fv.value.uiVal / 1000.0)
                            except Exception:
                                pass
                        time.sleep(0.01)
                th = threading.Thread(target=sampler, daemon=True)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                th.start()
                e0.record()
                for _ in range(n):
                    lib.fs_fwd(ctypes.byref(p), ctypes.c_void_p(s))
                e1.record()
                torch.cuda.synchronize()
                stop.set()
                th.join()
                ms = e0.elapsed_time(e1) / n
                mhz = statistics.median(clk) if clk else float("nan")
                watts = statistics.median(pw) if pw else float("nan")
                if rnd > 0:  # round 0 is a warm-up
                    samples[name].append((flops / ms / 1e9, mhz, watts))
                if rnd == 1:
                    outs[name] = o.float().clone()
        for name, lib in libs.items():  # diagnostic builds (-DFS_PROF=1): per-event latencies, one launch
            if not hasattr(lib, "fs_prof_read"):
                continue
            buf = (ctypes.c_ulonglong * 16)()
            lib.fs_prof_read(buf)
            lib.fs_fwd(ctypes.byref(p), ctypes.c_void_p(s))
            torch.cuda.synchronize()
            lib.fs_prof_read(buf)
            b = list(buf)
            prof = {"norm_cyc_per_tile": b[0] / max(b[1], 1), "norm_wait_s_cyc": b[6] / max(b[1], 1),
                    "mma_wait_p_cyc": b[2] / max(b[3], 1), "mma_wait_kv_cyc": b[4] / max(b[5], 1),
                    "mma_cyc_per_kv_tile": b[7] / max(b[5], 1)}
            if hasattr(lib, "fs_prof_timeline"):  # per-CTA globaltimer: entry, set-up, work done, exit
                tl = (ctypes.c_ulonglong * 6144)()
                lib.fs_prof_timeline(tl)
                rows = [tl[6 * i:6 * i + 6] for i in range(1024)]
                rows = [r for r in rows if r[0] != 0 and r[3] >= r[0]][:148]
                t0 = min(r[0] for r in rows)
                t_end = max(r[3] for r in rows)
                span = t_end - t0
                q = lambda xs, f: sorted(xs)[min(len(xs) - 1, int(f * len(xs)))]  # noqa: E731
                starts = [r[0] - t0 for r in rows]
                dones = [r[2] - t0 for r in rows]
                prof.update({"ctas": len(rows), "span_us": span / 1e3,
                             "start_us_p50_max": [q(starts, 0.5) / 1e3, max(starts) / 1e3],
                             "setup_us_p50": q([r[1] - r[0] for r in rows], 0.5) / 1e3,
                             "work_done_us_min_p50_max": [min(dones) / 1e3, q(dones, 0.5) / 1e3, max(dones) / 1e3],
                             "exit_after_done_us_p50": q([r[3] - r[2] for r in rows], 0.5) / 1e3,
                             "idle_frac": 1.0 - sum(r[3] - r[0] for r in rows) / (len(rows) * span),
                             "per_cta": [[int(r[4]), int(r[5]), round((r[2] - t0) / 1e3, 2)] for r in rows]})
            res[f"{cname}/{name}/prof"] = prof
            print(cname, name, "prof", {k: (round(v, 3) if isinstance(v, float) else v) for k, v in prof.items()
                                        if k != "per_cta"}, flush=True)
        ref = next(iter(outs.values()))
        for name in libs:
            tf = statistics.median(x[0] for x in samples[name])
            mhz = statistics.median(x[1] for x in samples[name])
            diff = float((outs[name] - ref).abs().max())
            watts = statistics.median(x[2] for x in samples[name])
            res[f"{cname}/{name}"] = {"tflops": round(tf, 1), "sm_mhz": mhz, "tflops_per_ghz": round(tf / mhz * 1e3, 1),
                                      "power_w": round(watts, 1), "tflops_per_kw": round(tf / watts * 1e3, 1),
                                      "max_abs_vs_first": diff, "launches_per_sample": n}
            print(cname, name, res[f"{cname}/{name}"], flush=True)
        del q, k, v, o
        torch.cuda.empty_cache()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "ab_variants.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        args = [a for a in sys.argv[2:] if not a.startswith("--")]
        rounds = 3
        if "--rounds" in sys.argv:
            rounds = int(sys.argv[sys.argv.index("--rounds") + 1])
            args = [a for a in args if a != str(rounds)]
        run(args or list(CASES), rounds)
