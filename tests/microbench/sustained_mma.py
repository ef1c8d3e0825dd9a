"""Sustained (power-capped) tensor throughput of a pure tcgen05 stream -- the QK/PV mix of
FlashSign with no TMA, norm or epilogue -- vs the FlashSign kernel on C3, back to back.
Answers: how close is FlashSign to the power-limited tensor ceiling?  (experiment, not a test)"""
import ctypes, json, os, statistics, sys, threading, time
import torch
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
lib = ctypes.CDLL(os.path.join(HERE, "libmma_bench.so"))
import pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)


def sample(fn, seconds):
    clk, pw, stop = [], [], threading.Event()
    def run():
        while not stop.is_set():
            clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0)
            time.sleep(0.02)
    th = threading.Thread(target=run, daemon=True)
    th.start()
    t0 = time.time()
    flops = 0.0
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < seconds:
        flops += fn()
    e1.record(); torch.cuda.synchronize()
    stop.set(); th.join()
    ms = e0.elapsed_time(e1)
    return {"tflops": flops / ms / 1e9, "sm_mhz": statistics.median(clk[len(clk)//2:]),
            "power_w": statistics.median(pw[len(pw)//2:])}


out = torch.zeros(148, dtype=torch.int64, device="cuda")
groups = 20000
def mma_only():
    ms = ctypes.c_float(0)
    lib.run_mma_bench(3, 1, 1, 2, groups, 148, ctypes.c_void_p(out.data_ptr()), ctypes.byref(ms))
    return 2.0 * 128 * 128 * 16 * 8 * groups * 148 * 2  # two launches per call (warm + timed)

from paper_2505_09326_b200 import flashsign
q, k, v = (torch.randn((8, 16384, 16, 128), device="cuda").to(torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
bad = torch.empty(1, dtype=torch.int64, device="cuda")
def fs():
    flashsign.fwd_async(q, k, v, out=o, bad_key=bad)
    return 4.0 * 8 * 16 * 16384 * 16384 * 128

res = {"mma_only_qk_pv_mix": sample(mma_only, 3.0), "flashsign_c3": sample(fs, 3.0),
       "mma_only_again": sample(mma_only, 3.0)}
for k2, v2 in res.items():
    print(k2, {a: round(b, 1) for a, b in v2.items()}, flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/sustained_mma.json", "w"), indent=1)
