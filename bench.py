"""FlashSign forward benchmark (BASELINE.json metric: FlashSign fwd TFLOP/s and % of
B200 tensor-core peak, 1-8 GPUs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

A step is one FlashSign forward over the rank's shard of the configuration
(synthetic standard-normal Q/K/V, resident in HBM).  Work is sharded by
(batch, kv-head) units with no collective (strong scaling: the configuration
is fixed, ranks split it).  Timing: W warm-up steps, barrier +
synchronize, CUDA events around exactly K steps on the launching stream,
synchronize + barrier, MAX over ranks.  Rank 0 prints one JSON line.

``--impl reference`` times the reference's own CPU implementation -- ncstream's
``multi_head_attention_array`` from baseline/_ref (baseline/install_ref.sh), else the
oracle port of the same loop -- on this host's cores on a bounded sample of the same
workload (``kind`` says which ran).

Beside the device-timed value the line carries: ``e2e`` (HostPipeline, pinned host
buffers), ``e2e_dropin`` (the reference's call pattern through the numpy drop-in API),
``context`` (SDPA softmax / eager spherical on the full configuration, same window
protocol), ``host_latency`` (per-call host microseconds), ``roofline``, ``cpu_baseline``.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs (C1 is the CPU-runnable correctness case, not a bench line)
CONFIGS = {
    "c2": dict(B=16, H=16, HKV=16, N=4096, D=64, dtype="fp16", eps=0.0, desc="B16 H16 N4096 d64 fp16"),
    "c3": dict(B=8, H=16, HKV=16, N=16384, D=128, dtype="bf16", eps=0.0, desc="B8 H16 N16384 d128 bf16"),
    "c4": dict(B=8, H=16, HKV=16, N=8192, D=128, dtype="e4m3", eps=0.0, desc="B8 H16 N8192 d128 e4m3 (bf16 out)"),
    "c5": dict(B=64, H=8, HKV=8, N=20000, D=64, dtype="bf16", eps=1e-6, mult=True,
               desc="GRN B64 H8 N20000 d64 bf16, eps=1e-6, multiplicity-scaled keys m in {0..5}"),
}
PAPER_A100_TFLOPS = 200.0  # PAPER.md:199 (FlashSign fwd, d=128, FP16, A100) -- BASELINE.md section 1


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"bf16_tflops": 1590.0, "hbm_gbs": 6650.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def measure_fp8_peak(device, n: int = 8192, reps: int = 10):
    """Dense e4m3 tensor-core roofline measured in this run: cuBLASLt
    ``torch._scaled_mm`` n^3, best of ``reps`` (burst, like MEASURED_PEAKS' bf16 figure)."""
    import torch
    try:
        a = torch.randn((n, n), device=device).to(torch.float8_e4m3fn)
        b = torch.randn((n, n), device=device).to(torch.float8_e4m3fn).t()
        one = torch.ones((), device=device)
        torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16)
        torch.cuda.synchronize()
        best = float("inf")
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return 2.0 * n ** 3 / (best * 1e-3) / 1e12
    except Exception:
        return None


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.power_mw, self.limit_w = [], None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            try:
                self.limit_w = pynvml.nvmlDeviceGetEnforcedPowerLimit(self.h) / 1000.0
            except Exception:
                pass
        except Exception:
            self.nvml = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
                try:  # instantaneous board power (GetPowerUsage is a ~1 s average, too slow here)
                    fv = self.nvml.nvmlDeviceGetFieldValues(self.h, [self.nvml.NVML_FI_DEV_POWER_INSTANT])[0]
                    if fv.nvmlReturn == 0:
                        self.power_mw.append(fv.value.uiVal)
                except Exception:
                    pass
                r = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nvml is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        out = {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
               "reasons": sorted(self.reasons), "samples": len(self.samples)}
        if self.power_mw:  # board power during the timed region (clock and power)
            out["power_w"] = statistics.median(self.power_mw) / 1000.0  # NVML_FI_DEV_POWER_INSTANT
            out["power_limit_w"] = self.limit_w
        return out


def make_inputs(cfg, lo, hi, device, seed=1000):
    """Shard [lo, hi) of (batch, kv-head) units as full-batch-row tensors.

    Deterministic per unit: unit u's Q/K/V come from a generator seeded with
    seed+u, so a shard's data equals the same units of a 1-GPU run.
    Returns q, k, v for batch rows [b_lo, b_hi), the per-key multiplicities m
    [rows, N] (GRN configuration, else None) and the unit offset.
    """
    import torch
    B, H, HKV, N, D = cfg["B"], cfg["H"], cfg["HKV"], cfg["N"], cfg["D"]
    b_lo, b_hi = lo // HKV, -(-hi // HKV)
    r = H // HKV
    tdt = {"bf16": torch.bfloat16, "fp16": torch.float16, "e4m3": torch.float8_e4m3fn}[cfg["dtype"]]
    nb = b_hi - b_lo
    q = torch.empty((nb, N, H, D), dtype=tdt, device=device)
    k = torch.empty((nb, N, HKV, D), dtype=tdt, device=device)
    v = torch.empty((nb, N, HKV, D), dtype=tdt, device=device)
    g = torch.Generator(device=device)
    # GRN: one multiplicity per gene (key) and cell (batch row), m in {0..5} (cli.py:296; grn.py:150).
    # Default: the caller's K' = m K (attention.py:381-388) is applied here, outside the timed region,
    # as the reference's grn._layer_qkv does before calling attention.  --fused-mult instead passes m
    # with the call (key_scale): for 16-bit inputs the K' = m K pass (fs_scale_keys) then runs inside
    # the timed step, ahead of the kernel.
    m = torch.empty((nb, N), dtype=torch.float32, device=device) if cfg.get("mult") else None
    for u in range(max(lo, b_lo * HKV), min(hi, b_hi * HKV)):
        b, hk = divmod(u, HKV)
        g.manual_seed(seed + u)
        bl = b - b_lo
        q[bl, :, hk * r:(hk + 1) * r] = torch.randn((N, r, D), generator=g, device=device).to(tdt)
        k[bl, :, hk] = torch.randn((N, D), generator=g, device=device).to(tdt)
        v[bl, :, hk] = torch.randn((N, D), generator=g, device=device).to(tdt)
    if m is not None:
        for bl in range(nb):
            g.manual_seed(seed + 1_000_003 * (b_lo + bl))
            m[bl] = torch.randint(0, 6, (N,), generator=g, device=device).float()
    if m is not None and not cfg.get("fused_mult"):
        k.copy_((k.float() * m[:, :, None, None]).to(tdt))
        m = None
    return q, k, v, m, b_lo * HKV


REF_INSTALL = os.path.join(ROOT, "baseline", "_ref")


def reference_impl():
    """The reference's own batched entry ``ncstream.attention.multi_head_attention_array``
    (attention.py:318-361) from baseline/_ref (``kind`` "reference"), else the oracle port of the
    same loop (oracle/spherical.py, ``kind`` "port")."""
    if os.path.isdir(os.path.join(REF_INSTALL, "ncstream")) and REF_INSTALL not in sys.path:
        sys.path.append(REF_INSTALL)
    try:
        from ncstream.attention import TileConfig, multi_head_attention_array
        from ncstream.normalizers import SPHERICAL

        def call(q, k, v, h, hkv, eps):
            return multi_head_attention_array(q, k, v, SPHERICAL.with_epsilon(eps), h, hkv, scale=1.0,
                                              tile=TileConfig(64, 64))
        return call, "reference", "ncstream.attention.multi_head_attention_array (baseline/_ref, unmodified)"
    except ImportError:
        from oracle.spherical import multi_head_spherical

        def call(q, k, v, h, hkv, eps):
            return multi_head_spherical(q, k, v, h, hkv, 1.0, eps)
        return call, "port", "oracle port of multi_head_attention_array / _streamed_tiles (oracle/spherical.py)"


def reference_rows(cfg) -> int:
    """Query rows per CPU sample: ~4 GFLOP per step (~0.3 s at the reference's ~14 GFLOP/s), a
    multiple of the default 64-row query group."""
    per_row = 4.0 * cfg["H"] * cfg["N"] * cfg["D"]
    return int(max(64, round(4e9 / per_row / 64) * 64))


def _quantised(shape, dtype, seed):
    """float32 arrays holding the configuration dtype's values (SURVEY.md 8(d) CPU baseline)."""
    import torch
    g = torch.Generator().manual_seed(seed)
    t = torch.randn(shape, generator=g)
    tdt = {"bf16": torch.bfloat16, "fp16": torch.float16, "e4m3": torch.float8_e4m3fn}[dtype]
    return t.to(tdt).float().numpy()


def cpu_reference_sample(cfg, rows: int, seed: int = 7):
    """Time the reference CPU path on its own batched call pattern:
    ``multi_head_attention_array(q, k, v, SPHERICAL, H, H_kv)`` on ``rows`` query positions x all
    H heads of one batch element against all N keys, default tile 64x64, float32 inputs holding
    the dtype-quantised values.  Returns (seconds, flops, threads, kind, what)."""
    call, kind, what = reference_impl()
    threads = None
    try:
        from threadpoolctl import threadpool_info
        threads = max((i.get("num_threads", 0) for i in threadpool_info() if i.get("user_api") == "blas"), default=None)
    except Exception:
        pass
    N, D, H, HKV = cfg["N"], cfg["D"], cfg["H"], cfg["HKV"]
    q = _quantised((rows, H, D), cfg["dtype"], seed)
    k = _quantised((N, HKV, D), cfg["dtype"], seed + 1)
    v = _quantised((N, HKV, D), cfg["dtype"], seed + 2)
    call(q[:8], k[:256], v[:256], H, HKV, cfg.get("eps", 0.0))  # warm-up
    t0 = time.perf_counter()
    call(q, k, v, H, HKV, cfg.get("eps", 0.0))
    dt = time.perf_counter() - t0
    return dt, 4.0 * rows * H * N * D, threads or os.cpu_count(), kind, what


def _link_roofline(dev, h2d_bytes, d2h_bytes, step_s):
    """Host<->device copy roofline of the e2e step.  Pinned 256 MiB copies (best of 3): each
    direction alone, and both at once on two streams (the boxes' PCIe + host memory carry less
    than the sum of the two one-way rates).  bound = max(h2d / BW_h2d, d2h / BW_d2h,
    (h2d + d2h) / BW_both)."""
    import torch
    n = 256 << 20
    host = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    devb = [torch.empty(n, dtype=torch.uint8, device=dev) for _ in range(2)]
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def best_of(fn):
        best = float("inf")
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best

    def h2d():
        with torch.cuda.stream(s_in):
            devb[0].copy_(host[0], non_blocking=True)

    def d2h():
        with torch.cuda.stream(s_out):
            host[1].copy_(devb[1], non_blocking=True)

    def both():
        h2d()
        d2h()

    bw_h2d = n / best_of(h2d) / 1e9
    bw_d2h = n / best_of(d2h) / 1e9
    bw_both = 2 * n / best_of(both) / 1e9
    bound = max(h2d_bytes / bw_h2d, d2h_bytes / bw_d2h, (h2d_bytes + d2h_bytes) / bw_both) / 1e9
    return {"h2d_gbs": bw_h2d, "d2h_gbs": bw_d2h, "both_gbs": bw_both, "bound_ms": bound * 1e3,
            "frac": bound / step_s}


def _host_info():
    """CPU model and BLAS backend of the host the CPU baseline ran on."""
    info = {"cpu_model": None, "blas": None, "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS")}
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    info["cpu_model"] = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        from threadpoolctl import threadpool_info
        info["blas"] = ", ".join(f"{i.get('internal_api')} {i.get('version')} x{i.get('num_threads')}"
                                 for i in threadpool_info() if i.get("user_api") == "blas") or None
    except Exception:
        pass
    return info


def _all_host_threads():
    """BLAS thread pool sized to every host core (torchrun sets OMP_NUM_THREADS=1 per rank)."""
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=os.cpu_count(), user_api="blas")
    except Exception:
        import contextlib
        return contextlib.nullcontext()


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # reference arm: rank 0 only
    with _all_host_threads():
        _run_reference(args, cfg)


def _run_reference(args, cfg):
    rows = args.ref_rows or reference_rows(cfg)
    times = []
    for i in range(args.warmup + args.steps):
        dt, fl, threads, kind, what = cpu_reference_sample(cfg, rows, seed=7 + i)
        if i >= args.warmup:
            times.append((dt, fl))
    tot_t = sum(t for t, _ in times)
    # median of the per-step rates: robust to host noise, and the statistic the ours-arm's
    # cpu_baseline reports on the same sample size (so the two CPU numbers are comparable)
    val = statistics.median(f / t for t, f in times) / 1e12
    sample = (f"{rows} query positions x {cfg['H']} heads x {cfg['N']} keys x d{cfg['D']} of one batch element "
              f"per step, float32 holding {cfg['dtype']} values, tile 64x64: {what}")
    line = {
        "impl": "reference", "metric": "FlashSign fwd TFLOP/s", "value": val, "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_t / len(times), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": args.config, "desc": cfg["desc"], "sample": sample},
        "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": threads, "kind": kind, "sample": sample,
                         "cpu_count": os.cpu_count(), **_host_info()},
        "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _timed(fn, steps, device_index):
    """CUDA-event time of ``steps`` back-to-back calls (after one warm-up) with NVML clocks sampled
    over the same window: (ms per call, clock summary)."""
    import torch
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(device_index) as clk:
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps, clk.summary()


def context_baselines(cfg, q, k, v, device, steps, device_index):
    """Same-GPU context on the FULL configuration, timed like FlashSign (CUDA
    events over back-to-back steps, clocks sampled in the same window):
      * SDPA softmax attention, per backend (cuDNN, flash) -- the paper's "within 5 % of
        FlashAttention-2" claim, on B200;
      * PyTorch-eager spherical attention (materialises S per (b, h));
      * the O(N d^2) Gram-form identity through our own kernels (fs_gram_fwd; a
        different algorithm, reported beside, never under the 4 B H N^2 d metric).
    e4m3 configurations run the baselines in bf16 (no fp8 SDPA)."""
    import torch
    import torch.nn.functional as F
    res = {}
    if cfg["dtype"] == "e4m3":
        q, k, v = (t.to(torch.bfloat16) for t in (q, k, v))
    B, N, H, D = q.shape
    HKV = k.shape[2]
    fl = 4.0 * B * H * N * k.shape[1] * D
    qt, kt, vt = (t.transpose(1, 2) for t in (q, k, v))  # BHSD views, as SDPA takes them

    def sdpa():
        F.scaled_dot_product_attention(qt, kt, vt, enable_gqa=HKV != H)

    def eager():  # per (b, h) to bound memory: S = q k^T ; O = (S v) / ||S||_row
        for b in range(B):
            for h in range(H):
                hk = h * HKV // H
                s_ = q[b, :, h] @ k[b, :, hk].T
                z = s_.float().square().sum(-1, keepdim=True).sqrt()
                (s_ @ v[b, :, hk]).float().div_(z)

    from paper_2505_09326_b200 import flashsign
    go = torch.empty(q.shape, dtype=q.dtype, device=q.device)
    gbad = torch.empty(1, dtype=torch.int64, device=q.device)

    def gram():  # our tensor-core Gram-form kernels (fs_gram_fwd), same inputs, same output dtype
        flashsign.gram_fwd(q, k, v, eps=cfg["eps"], out=go, check=False, bad_key=gbad)

    fns = []
    try:
        from torch.nn.attention import SDPBackend, sdpa_kernel

        def pinned(be):
            def run():
                with sdpa_kernel([be]):
                    sdpa()
            return run
        fns += [("sdpa_softmax_cudnn", pinned(SDPBackend.CUDNN_ATTENTION), steps),
                ("sdpa_softmax_flash", pinned(SDPBackend.FLASH_ATTENTION), max(3, steps // 4))]
    except ImportError:
        fns.append(("sdpa_softmax", sdpa, steps))
    fns += [("torch_eager_spherical", eager, 2), ("gram_form_kernel_not_flashsign", gram, max(10, steps))]
    for name, fn, n in fns:
        try:
            ms, clk = _timed(fn, n, device_index)
            if name.startswith("gram"):
                # HBM roofline of the Gram path: Q, K, V read and O written once
                byts = sum(t.numel() * t.element_size() for t in (q, k, v, go))
                res[name] = {"ms_per_step": ms, "steps": n, "clocks": clk, "hbm_gbs": byts / ms / 1e6,
                             "bytes_per_step": byts, "speedup_vs_flashsign_step": None,
                             "note": "fs_gram_fwd: the O(N d^2) moment form of the same spherical "
                                     "contract (SURVEY.md 0 fact 4), not the 4*N^2*d FlashSign work"}
            else:
                res[name] = {"tflops": fl / ms / 1e9, "ms_per_step": ms, "steps": n, "clocks": clk,
                             "dtype": str(q.dtype).replace("torch.", ""), "shape": "full configuration"}
        except Exception as ex:  # OOM etc. recorded, as the paper did
            res[name] = {"error": f"{type(ex).__name__}: {str(ex)[:160]}"}
        torch.cuda.empty_cache()
    return res


def host_latency(device):
    """Host time per call of the torch entry (``flashsign.fwd_async``: extension + C-ABI + cached
    TMA descriptors + launch) and of the numpy drop-in (``multi_head_attention_array``) at the
    C1 shape (B1 H1 N256 d64) and a per-cell GRN call shape (one cell, N=256 genes, H8, d64).
    Launches are queued back to back (no synchronisation inside the timed loop for fwd_async)."""
    import torch

    from paper_2505_09326_b200 import SPHERICAL, flashsign
    from paper_2505_09326_b200.attention import multi_head_attention_array
    out = {}
    for name, (b, n, h, d) in (("c1", (1, 256, 1, 64)), ("grn_cell", (1, 256, 8, 64))):
        qd = torch.randn((b, n, h, d), device=device).to(torch.bfloat16)
        o = torch.empty_like(qd)
        bad = torch.empty(1, dtype=torch.int64, device=device)
        for _ in range(50):
            flashsign.fwd_async(qd, qd, qd, out=o, bad_key=bad)
        torch.cuda.synchronize()
        reps = 2000
        t0 = time.perf_counter()
        for _ in range(reps):
            flashsign.fwd_async(qd, qd, qd, out=o, bad_key=bad)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        qn = np.random.default_rng(0).standard_normal((n, h, d)).astype(np.float32)
        multi_head_attention_array(qn, qn, qn, SPHERICAL, h, h)
        t3 = time.perf_counter()
        for _ in range(50):
            multi_head_attention_array(qn, qn, qn, SPHERICAL, h, h)
        t4 = time.perf_counter()
        out[name] = {"shape_bnhd": [b, n, h, d], "fwd_async_host_us": 1e6 * (t1 - t0) / reps,
                     "fwd_async_incl_gpu_us": 1e6 * (t2 - t0) / reps,
                     "dropin_numpy_call_us": 1e6 * (t4 - t3) / 50}
    return out


def _pageable_link(dev, nbytes=128 << 20):
    """The host link as a numpy caller sees it: pageable host -> device, device -> pinned host, and
    both at once (GB/s, best of 3)."""
    import torch
    src = torch.from_numpy(np.ones(nbytes // 4, dtype=np.float32))   # pageable
    dst = torch.empty(nbytes // 4, dtype=torch.float32, device=dev)
    dsrc = torch.empty(nbytes // 4, dtype=torch.float32, device=dev)
    hdst = torch.empty(nbytes // 4, dtype=torch.float32, pin_memory=True)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def best(fn):
        b = float("inf")
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            b = min(b, time.perf_counter() - t0)
        return b

    def h2d():
        with torch.cuda.stream(s1):
            dst.copy_(src, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            hdst.copy_(dsrc, non_blocking=True)

    def both():
        d2h()
        h2d()

    hsrc = torch.empty(nbytes // 4, dtype=torch.float32, pin_memory=True)

    def h2d_pinned():
        with torch.cuda.stream(s1):
            dst.copy_(hsrc, non_blocking=True)

    def both_pinned():
        d2h()
        h2d_pinned()

    # the staging copy pageable -> pinned as the drop-in does it (hostpath): 8 host threads, each
    # copying its share with non-temporal stores (fs_host_copy)
    import ctypes
    from concurrent.futures import ThreadPoolExecutor

    from paper_2505_09326_b200 import _lib
    cp = _lib.load().fs_host_copy
    cp.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]
    a = np.ones(nbytes, dtype=np.uint8)
    dp, sp = hsrc.data_ptr(), a.ctypes.data
    nthr = 8
    step = -(-nbytes // nthr)
    with ThreadPoolExecutor(nthr) as pool:
        def stage():
            list(pool.map(lambda j: cp(dp + j, sp + j, min(step, nbytes - j)), range(0, nbytes, step)))
        stage()
        t_stage = min(_wall(stage) for _ in range(3))

    # the drop-in's whole staged copy-in (fill + DMA together, sharing host memory): hostpath's
    # own staging ring on a 128 MB array
    from paper_2505_09326_b200 import hostpath
    eng = hostpath.engine(dev)
    mode, eng.mode = eng.mode, "staged"
    src_np = np.ones(nbytes // 4, dtype=np.float32)

    def staged():
        eng._h2d(dst, src_np)
        eng.s_h2d.synchronize()
    try:
        staged()
        t_staged = min(_wall(staged) for _ in range(3))
    finally:
        eng.mode = mode

    return {"h2d_pageable_gbs": nbytes / best(h2d) / 1e9, "d2h_pinned_gbs": nbytes / best(d2h) / 1e9,
            "h2d_staged_gbs": nbytes / t_staged / 1e9,
            "both_gbs": 2 * nbytes / best(both) / 1e9, "h2d_pinned_gbs": nbytes / best(h2d_pinned) / 1e9,
            "both_pinned_gbs": 2 * nbytes / best(both_pinned) / 1e9, "host_stage_gbs": nbytes / t_stage / 1e9}


def _wall(fn):
    t0 = time.perf_counter()
    fn()
    return time.perf_counter() - t0


def dropin_e2e(cfg, q, k, v, device, passes=2):
    """The reference's own call pattern through the drop-in API (grn.py:171-173):
    ``multi_head_attention_array(q[b], k[b], v[b], SPHERICAL, H, H_kv)`` once per batch element, with
    float32 numpy arrays (pageable host memory) in and out.  Wall clock over whole passes of the
    batch; the host link bound uses the measured pageable H2D / pinned D2H bandwidth."""
    import torch

    from paper_2505_09326_b200 import SPHERICAL
    from paper_2505_09326_b200.attention import multi_head_attention_array
    B, N, H, D = q.shape
    HKV = k.shape[2]
    spec = SPHERICAL.with_epsilon(cfg["eps"])
    qs = [q[b].float().cpu().numpy() for b in range(B)]
    ks = [k[b].float().cpu().numpy() for b in range(B)]
    vs = [v[b].float().cpu().numpy() for b in range(B)]
    multi_head_attention_array(qs[0], ks[0], vs[0], spec, H, HKV, scale=1.0)  # warm-up (engine, buffers)
    t0 = time.perf_counter()
    for _ in range(passes):
        for b in range(B):
            multi_head_attention_array(qs[b], ks[b], vs[b], spec, H, HKV, scale=1.0)
    dt = (time.perf_counter() - t0) / passes
    h2d = sum(a.nbytes for a in qs + ks + vs)
    d2h = sum(a.nbytes for a in qs)
    link = _pageable_link(device)
    # the drop-in's copy-in stages large arrays through pinned memory (hostpath, FLASHSIGN_H2D=auto):
    # its DMA bound is the pinned link; the pageable one is what a direct copy of the caller's arrays
    # would be held to
    bound = max(h2d / link["h2d_staged_gbs"], d2h / link["d2h_pinned_gbs"], (h2d + d2h) / link["both_pinned_gbs"]) / 1e9
    bound_pg = max(h2d / link["h2d_pageable_gbs"], d2h / link["d2h_pinned_gbs"], (h2d + d2h) / link["both_gbs"]) / 1e9
    link.update({"bound_ms": bound * 1e3, "frac": bound / dt, "pageable_bound_ms": bound_pg * 1e3,
                 "copy_in": os.environ.get("FLASHSIGN_H2D", "auto") + " (pinned staging for arrays >= 8 MB; "
                            "bound: the staged copy-in, fill and DMA together, h2d_staged_gbs)"})
    fl = 4.0 * B * H * N * k.shape[1] * D
    return {"value": fl / dt / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": dt * 1e3, "passes": passes,
            "api": "paper_2505_09326_b200.attention.multi_head_attention_array per batch element, float32 numpy "
                   "in/out (the reference's call pattern)", "link": link}


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_2505_09326_b200 import flashsign, partition
    from paper_2505_09326_b200.pipeline import HostPipeline

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} != --gpus {args.gpus}", file=sys.stderr)
    # FS_BENCH_BACKEND=gloo runs the multi-rank path on a box with fewer GPUs than ranks (ranks
    # share devices round-robin) -- a functional check of the sharded bench, not a measurement
    backend = os.environ.get("FS_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    B, H, HKV, N, D = cfg["B"], cfg["H"], cfg["HKV"], cfg["N"], cfg["D"]
    n_units = B * HKV
    lo, hi = partition.unit_range(n_units, world, rank)
    q, k, v, mult, u_off = make_inputs(cfg, lo, hi, dev)
    out_dtype = torch.bfloat16 if cfg["dtype"] == "e4m3" else q.dtype
    o = torch.empty(q.shape, dtype=out_dtype, device=dev)
    r = H // HKV
    my_flops = 4.0 * (hi - lo) * r * N * N * D
    total_flops = 4.0 * B * H * N * N * D
    kw = dict(scale=1.0, eps=cfg["eps"])
    bad = torch.empty(1, dtype=torch.int64, device=dev)

    def step():
        return partition.fwd_shard(q, k, v, o, lo - u_off, hi - u_off,
                                   lambda *a, **k2: flashsign.fwd_async(*a, bad_key=bad, **k2), key_scale=mult, **kw)

    pcs = partition.pieces(q.shape[0], HKV, lo - u_off, hi - u_off)
    n_launch_per_step = len(pcs)
    # kernels per step besides the FlashSign kernels: the K' = m K pass per piece (--fused-mult,
    # 16-bit) and the merge kernel of any piece whose automatic plan splits K/V (e.g. C3's tail wave)
    n_prepass = n_launch_per_step if (mult is not None and q.dtype in (torch.bfloat16, torch.float16)) else 0
    n_merge = sum(1 for pc in pcs if flashsign.plan(pc.b1 - pc.b0, (pc.g1 - pc.g0) * r, N, N, dev, D,
                                                    q.dtype).splits > 1)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    flashsign.raise_if_bad(bad, H, N) if cfg["eps"] == 0.0 else None

    # ---------------- device-resident timed region
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # per-step events too (median / min per step); they add no work to the stream
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        e0.record(stream)
        for i in range(args.steps):
            step()
            ev[i].record(stream)
        e1.record(stream)
        torch.cuda.synchronize()
    per_step = [e0.elapsed_time(ev[0])] + [ev[i - 1].elapsed_time(ev[i]) for i in range(1, args.steps)]
    if world > 1:
        dist.barrier()
    ms_total = e0.elapsed_time(e1)
    t = torch.tensor([ms_total], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = total_flops / (ms_step * 1e-3) / 1e12 if world > 1 else my_flops / (ms_step * 1e-3) / 1e12
    kernel_ms = ms_step / n_launch_per_step  # one kernel launch per piece; back-to-back on one stream

    # ---------------- optional O gather onto every rank (NCCL all_gather), timed separately
    gather = None
    if world > 1 and n_units % world == 0 and ((hi - lo) % HKV == 0) and lo % HKV == 0:
        o_mine = o[(lo - u_off) // HKV:(hi - u_off) // HKV]
        for _ in range(2):
            partition.gather_output(o_mine)
        torch.cuda.synchronize()
        dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        for _ in range(3):
            full = partition.gather_output(o_mine)
        g1.record()
        torch.cuda.synchronize()
        tg = torch.tensor([g0.elapsed_time(g1) / 3], device=dev, dtype=torch.float64)
        dist.all_reduce(tg, op=dist.ReduceOp.MAX)
        gather = {"ms": float(tg.item()), "bytes_per_rank_out": int(full.numel() * full.element_size()),
                  "api": "partition.gather_output (all_gather_into_tensor)", "in_timed_region": False}
        del full

    # ---------------- end-to-end through the host-buffer API (pinned host in, host out)
    e2e = None
    if not args.no_e2e:
        qh = q.cpu().pin_memory()
        kh = k.cpu().pin_memory()
        vh = v.cpu().pin_memory()
        oh = torch.empty(o.shape, dtype=o.dtype, pin_memory=True)
        mh = None if mult is None else mult.cpu().pin_memory()
        pipe = HostPipeline(dev)
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        for _ in range(min(args.warmup, 2)):
            pipe.run(qh, kh, vh, oh, check=False, key_scale=mh, **kw)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            pipe.run(qh, kh, vh, oh, check=False, key_scale=mh, **kw)  # run() synchronises: output on the host
        dt = (time.perf_counter() - t0) / e2e_steps
        tt = torch.tensor([dt], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
        elsz = q.element_size()
        h2d = (q.numel() + k.numel() + v.numel()) * elsz + (0 if mh is None else mh.numel() * 4)
        d2h = o.numel() * o.element_size()
        link = _link_roofline(dev, h2d, d2h, dt)
        if world > 1:
            vals = torch.tensor([h2d, d2h], device=dev, dtype=torch.float64)
            dist.all_reduce(vals)
            h2d, d2h = int(vals[0].item()), int(vals[1].item())
        e2e = {"value": (total_flops if world > 1 else my_flops) / dt / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": dt * 1e3,
               "steps": e2e_steps, "api": "paper_2505_09326_b200.pipeline.HostPipeline.run (pinned host bf16 in/out)",
               "link": link}

    e2e_dropin = lat = None
    if world == 1 and not args.no_e2e:
        try:
            e2e_dropin = dropin_e2e(cfg, q, k, v, dev)
        except Exception as ex:  # recorded, never silently dropped
            e2e_dropin = {"error": f"{type(ex).__name__}: {str(ex)[:200]}"}
        try:
            lat = host_latency(dev)
        except Exception as ex:
            lat = {"error": f"{type(ex).__name__}: {str(ex)[:200]}"}

    if rank == 0:
        peaks, peak_src = load_peaks()
        fp8 = cfg["dtype"] == "e4m3"
        peak = peaks.get("fp8_tflops") if fp8 else peaks["bf16_tflops"]
        peak_note = "MEASURED_PEAKS.json bf16_tflops (burst)"
        if fp8 and peak is None:
            peak = measure_fp8_peak(dev)
            peak_src, peak_note = "measured", "this run: cuBLASLt torch._scaled_mm e4m3 8192^3, best of 10 (burst)"
        if fp8 and peak is None:
            peak = 2.0 * peaks["bf16_tflops"]
            peak_note = "2 x MEASURED_PEAKS.json bf16_tflops (FP8 dense = 2x BF16; no measured FP8 peak)"
        per_launch_flops = my_flops / n_launch_per_step
        achieved = per_launch_flops / (kernel_ms * 1e-3) / 1e12
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                traffic = json.load(f).get(args.config)
        except Exception:
            pass
        roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": traffic, "peak_source": f"{peak_src}: {peak_note}",
                    "frac_of_sustained": (achieved / peaks["bf16_tflops_sustained"] / (2.0 if fp8 else 1.0))
                    if "bf16_tflops_sustained" in peaks else None,
                    "flops_per_launch": per_launch_flops, "kernel_ms": kernel_ms}
        if fp8:  # the same against twice the measured dense bf16 burst (FP8 dense = 2x BF16 on B200)
            roofline["frac_of_2x_bf16_burst"] = achieved / (2.0 * peaks["bf16_tflops"])
        cpu = None
        if world == 1 and not args.no_cpu:
            rows = args.cpu_rows or reference_rows(cfg)
            with _all_host_threads():
                tt_, rates = 0.0, []
                cpu_reference_sample(cfg, rows, seed=6)  # warm-up, like the reference arm's
                for rep_ in range(5):  # same sample as one step of the reference arm, five times
                    dt, fl, threads, kind, what = cpu_reference_sample(cfg, rows, seed=7 + rep_)
                    tt_ += dt
                    rates.append(fl / dt)
                host = _host_info()
            cpu = {"value": statistics.median(rates) / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": kind,
                   "sample": f"1 warm-up + 5 x ({rows} query positions x {H} heads x {N} keys x d{D} of one batch "
                             f"element), median rate, float32 holding {cfg['dtype']} values, tile 64x64: {what}; "
                             f"{tt_:.2f} s",
                   "cpu_count": os.cpu_count(), **host}
        ctx = None
        if world == 1 and not args.no_context:
            ctx = context_baselines(cfg, q, k, v, dev, args.steps, local)
            gk = ctx.get("gram_form_kernel_not_flashsign", {})
            if "ms_per_step" in gk:
                gk["speedup_vs_flashsign_step"] = ms_step / gk["ms_per_step"]
        line = {
            "metric": "FlashSign fwd TFLOP/s", "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "ms_per_step_median": statistics.median(per_step), "ms_per_step_min": min(per_step),
            "higher_is_better": True,
            "scaling": "strong", "vs_baseline": value / PAPER_A100_TFLOPS,
            "vs_baseline_ref": "paper's A100 FlashSign fwd ~200 TFLOP/s (PAPER.md:199, BASELINE.md section 1)",
            "dtype": {"bf16": "bf16", "fp16": "fp16", "e4m3": "e4m3"}[cfg["dtype"]], "data": "synthetic",
            "config": {"workload": args.config, "desc": cfg["desc"], "batch": B, "heads": H, "heads_kv": HKV,
                       "seq_len": N, "head_dim": D, "eps": cfg["eps"], "parallelism": f"batchxhead-shard{world}",
                       "l2": "inputs larger than L2 (no flush needed)",
                       "flops_per_step": total_flops},
            "clocks": clk.summary(), "e2e": e2e, "gpu_launches": (n_launch_per_step + n_prepass + n_merge) * args.steps,
            "roofline": roofline, "cpu_baseline": cpu, "gather": gather,
            "e2e_dropin": e2e_dropin, "host_latency": lat,
        }
        if ctx is not None:
            line["context"] = ctx
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-rows", type=int, default=0, help="query positions per CPU reference sample (0: ~4 GFLOP)")
    ap.add_argument("--cpu-rows", type=int, default=0, help="query rows of the cpu_baseline sample (0: one full slice)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-context", action="store_true", help="skip the SDPA / eager / Gram context baselines")
    ap.add_argument("--fused-mult", action="store_true", help="c5: fuse the key multiplicities into the kernel")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = dict(CONFIGS[args.config])
    if args.fused_mult:
        if not cfg.get("mult"):
            ap.error("--fused-mult applies to the GRN configuration (c5) only")
        cfg["fused_mult"] = True
        cfg["desc"] += ", multiplicities with the call (key_scale: K' = m K pass + kernel, both timed)"
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
