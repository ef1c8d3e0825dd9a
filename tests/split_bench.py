import torch, time, sys
sys.path.insert(0, ".")
from paper_2505_09326_b200 import flashsign as fs
for (b, h, n, d) in [(1, 1, 16384, 128), (1, 2, 32768, 128), (1, 4, 65536, 64), (2, 1, 8192, 128)]:
    q, k, v = (torch.randn((b, n, h, d), device="cuda").to(torch.bfloat16) for _ in range(3))
    fl = 4.0 * b * h * n * n * d
    res = {}
    for sp in (1, None):
        for _ in range(3): fs.fwd_async(q, k, v, kv_splits=sp)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): fs.fwd_async(q, k, v, kv_splits=sp)
        e1.record(); torch.cuda.synchronize()
        res[sp] = fl / (e0.elapsed_time(e1) / 10 * 1e-3) / 1e12
    print((b, h, n, d), "auto splits", fs.auto_splits(b, h, n, n, q.device, d), "TFLOP/s single-pass %.0f  split %.0f" % (res[1], res[None]), flush=True)
