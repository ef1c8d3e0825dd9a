"""TMEM ld/st throughput per SM (experiment).  Writes gpurun_out/tmem_bench.json."""
import ctypes, json, os, torch
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtmem_bench.so"))
out = torch.zeros(148, dtype=torch.int64, device="cuda")
shapes = {0: "32x32b.x32", 1: "16x256b.x8", 2: "16x128b.x16", 3: "16x64b.x32"}
modes = {0: "ld", 1: "ld+st16", 2: "ld+st32", 3: "2ld/wait", 4: "4ld/wait"}
combos = [(s, 0, 0, nw) for s in range(4) for nw in (4, 8, 16)]
combos += [(0, 1, 0, 4), (0, 1, 0, 8), (0, 2, 0, 8), (1, 1, 0, 8), (0, 3, 0, 4), (0, 3, 0, 8), (0, 4, 0, 4), (0, 4, 0, 8),
           (1, 3, 0, 8), (0, 0, 1, 8), (0, 1, 1, 8), (1, 0, 1, 8), (0, 3, 1, 8)]
res = {}
for s, m, x, nw in combos:
    iters = 2048
    ms = ctypes.c_float(0)
    rc = lib.run_tmem_bench(s, m, x, iters, nw, 148, ctypes.c_void_p(out.data_ptr()), ctypes.byref(ms))
    torch.cuda.synchronize()
    cyc = out.float().max().item()
    lpw = 2 if m == 3 else 4 if m == 4 else 1
    rd = nw * iters * 4096 * lpw
    key = f"{shapes[s]} {modes[m]} nw={nw} mma={x}"
    res[key] = {"read_B_per_clk": round(rd / cyc, 1), "cyc_per_warp_iter": round(cyc / iters, 1), "ms": round(ms.value, 3), "rc": rc}
    print(key, res[key], flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/tmem_bench.json", "w"), indent=1)
