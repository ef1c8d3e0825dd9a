"""Diagnostic run of the FlashSign kernel on a B200 (not a pytest module).

    python tests/gpu_first_light.py

Each case prints max-abs error of the kernel vs the fp64 oracle on the SAME
(dtype-quantised) inputs.  The V = I case exposes S directly (O = S / ||S||),
which separates a QK^T descriptor bug from a PV one.
"""

from __future__ import annotations

import json
import os
import sys
import traceback

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle.spherical import gram_batched  # noqa: E402
from paper_2505_09326_b200 import flashsign  # noqa: E402


def run_case(name, b, nq, nkv, h, hkv, d, dtype, scale=1.0, eps=0.0, vid=False, out_dtype=None, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    q = torch.randn((b, nq, h, d), generator=g, device="cuda").to(dtype)
    k = torch.randn((b, nkv, hkv, d), generator=g, device="cuda").to(dtype)
    if vid:
        assert nkv == d
        v = torch.eye(d, device="cuda")[None, :, None, :].expand(b, nkv, hkv, d).contiguous().to(dtype)
    else:
        v = torch.randn((b, nkv, hkv, d), generator=g, device="cuda").to(dtype)
    o, bad = flashsign.fwd_async(q, k, v, scale=scale, eps=eps, out_dtype=out_dtype)
    torch.cuda.synchronize()
    ref = gram_batched(q.float().cpu().numpy(), k.float().cpu().numpy(), v.float().cpu().numpy(), scale, eps)
    got = o.float().cpu().numpy()
    err = np.abs(got - ref)
    res = {
        "case": name, "max_abs": float(np.nanmax(err)), "mean_abs": float(np.nanmean(err)),
        "frac_within_0.01": float(np.mean(err <= 0.01)),
        "bad_key": hex(int(bad.item()) & 0xFFFFFFFFFFFFFFFF),
        "ref_absmax": float(np.nanmax(np.abs(ref))),
    }
    if vid:
        # O = S/||S|| with V=I: compare direction of first rows
        s = np.einsum("bnhd,bmhd->bhnm", q.float().cpu().numpy().astype(np.float64),
                      k.float().cpu().numpy().astype(np.float64))
        res["S00_ref_first8"] = (s[0, 0, 0, :8] / np.linalg.norm(s[0, 0, 0])).round(4).tolist()
        res["O00_got_first8"] = got[0, 0, 0, :8].round(4).tolist()
    return res


def main():
    torch.cuda.init()
    print(torch.cuda.get_device_name(), torch.cuda.get_device_capability(), flush=True)
    cases = [
        ("vid_bf16_d128", dict(b=1, nq=128, nkv=128, h=1, hkv=1, d=128, dtype=torch.bfloat16, vid=True)),
        ("small_bf16_d128", dict(b=1, nq=128, nkv=128, h=1, hkv=1, d=128, dtype=torch.bfloat16)),
        ("small_bf16_d64", dict(b=1, nq=128, nkv=128, h=1, hkv=1, d=64, dtype=torch.bfloat16)),
        ("small_fp16_d128", dict(b=1, nq=256, nkv=256, h=1, hkv=1, d=128, dtype=torch.float16)),
        ("ragged_bf16", dict(b=2, nq=300, nkv=517, h=4, hkv=2, d=128, dtype=torch.bfloat16)),
        ("ragged_fp16_d64_f32out", dict(b=2, nq=1000, nkv=777, h=2, hkv=1, d=64, dtype=torch.float16,
                                        out_dtype=torch.float32)),
        ("d96_bf16", dict(b=1, nq=200, nkv=300, h=2, hkv=2, d=96, dtype=torch.bfloat16)),
        ("scale_eps", dict(b=1, nq=256, nkv=1024, h=2, hkv=1, d=64, dtype=torch.bfloat16, scale=-0.7, eps=1e-6)),
        ("e4m3_d128", dict(b=1, nq=256, nkv=512, h=2, hkv=2, d=128, dtype=torch.float8_e4m3fn)),
        ("long_bf16", dict(b=1, nq=512, nkv=4096, h=2, hkv=2, d=128, dtype=torch.bfloat16)),
    ]
    results = []
    for name, kw in cases:
        try:
            r = run_case(name, **kw)
        except Exception as e:  # keep going: report every case
            r = {"case": name, "error": f"{type(e).__name__}: {e}", "tb": traceback.format_exc()[-800:]}
        print(json.dumps(r), flush=True)
        results.append(r)
        if "error" in r and "CUDA" in r["error"]:
            break
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/first_light.json", "w") as f:
        json.dump(results, f, indent=1)


if __name__ == "__main__":
    main()
