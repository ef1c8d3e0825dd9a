import ctypes, json, os, torch
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmma_bench.so"))
out = torch.zeros(148, dtype=torch.int64, device="cuda")
res = {}
names = {0: ("SS_128x128", 128), 1: ("SS_128x256", 256), 2: ("TS_128x128_Bmn", 128), 3: ("QK/PV_alt", 128),
         4: ("d64: 4xSS_N128 + 8xTS_N64", None), 5: ("8xTS_N64", None)}
combos = [(4,1,0,2),(4,1,1,2),(5,1,0,1),(5,1,1,2),(0,0,0,1),(0,1,0,1),(0,1,1,1),(0,1,1,2),(0,0,1,2),(1,1,0,1),(1,1,1,1),(2,0,0,1),(2,1,0,1),(2,1,1,1),(2,1,1,2),(3,1,0,2),(3,1,1,2),(3,0,1,2)]
for mode, wi, ce, nacc in combos:
    name, n = names[mode]
    ms = ctypes.c_float(0)
    groups = 1024
    rc = lib.run_mma_bench(mode, wi, ce, nacc, groups, 148, ctypes.c_void_p(out.data_ptr()), ctypes.byref(ms))
    torch.cuda.synchronize()
    if mode >= 4:  # per group (one tile's d=64 QK + PV): ideal 4*64 + 8*32 = 512 cycles (mode 5: 256)
        cyc = out.float().mean().item() / groups
        ideal = 512 if mode == 4 else 256
        flops = 2.0 * 128 * 64 * 128 * (2 if mode == 4 else 1) * groups * 148
    else:
        cyc = out.float().mean().item() / (groups * 8)
        ideal = 128 * n / 256
        flops = 2.0 * 128 * n * 16 * groups * 8 * 148
    key = f"{name} warp={wi} commit={ce} nacc={nacc}"
    res[key] = {"cyc_per_mma_or_group": round(cyc, 1), "ideal": ideal, "eff": round(ideal / cyc, 3), "tflops": round(flops / ms.value / 1e9), "rc": rc}
    print(key, res[key], flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/mma_bench.json", "w"), indent=1)
