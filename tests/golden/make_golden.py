"""Generate golden vectors by running the REFERENCE itself (ncstream, pure Python).

Run in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes ``tests/golden/golden.npz`` (committed).  The GPU box never needs the
reference: tests load the fixture and check the oracle (and, on GPU, the
kernel) against it.  Every case names the reference test or spec line it
mirrors.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from ncstream.attention import (  # noqa: E402
    TileConfig,
    apply_multiplicity_array,
    multi_head_attention_array,
    naive_attention_array,
    streamed_attention_array,
)
from ncstream.normalizers import SIGNED_L1, SPHERICAL, DegenerateDenominatorError  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def rand_qkv(rng, y, x, k, dtype=np.float64):
    # test_attention.py:35-38
    return (rng.standard_normal((y, k)).astype(dtype),
            rng.standard_normal((x, k)).astype(dtype),
            rng.standard_normal((x, k)).astype(dtype))


def main():
    g: dict[str, np.ndarray] = {}
    cases: list[str] = []

    def put(name, q, k, v, out, scale=1.0, eps=0.0, extra=None):
        cases.append(name)
        g[f"{name}/q"] = q
        g[f"{name}/k"] = k
        g[f"{name}/v"] = v
        g[f"{name}/out"] = out
        g[f"{name}/scale"] = np.float64(scale)
        g[f"{name}/eps"] = np.float64(eps)
        for key, val in (extra or {}).items():
            g[f"{name}/{key}"] = np.asarray(val)

    # KAT: test_attention.py:46-52 / SPEC.md:273 -> [[22.0]]
    q = np.array([[1.0]]); k = np.array([[3.0], [4.0]]); v = np.array([[10.0], [20.0]])
    put("kat_hand", q, k, v, naive_attention_array(q, k, v, SPHERICAL, 1.0))
    put("kat_hand_streamed11", q, k, v, streamed_attention_array(q, k, v, SPHERICAL, 1.0, TileConfig(1, 1)))
    # float32 version of the same KAT (what the GPU compat path sees)
    put("kat_hand_f32", q.astype(np.float32), k.astype(np.float32), v.astype(np.float32),
        streamed_attention_array(q.astype(np.float32), k.astype(np.float32), v.astype(np.float32),
                                 SPHERICAL, 1.0, TileConfig()))

    # Sign KAT: test_attention.py:60-67
    q = np.array([[2.0]]); v = np.array([[5.0, -7.0]])
    for tag, kk in (("pos", np.array([[1.0]])), ("neg", np.array([[-1.0]]))):
        put(f"kat_sign_{tag}", q, kk, v, naive_attention_array(q, kk, v, SPHERICAL, 1.0))

    # Oracle-equivalence grid: test_attention.py:127-145
    rng = np.random.default_rng(5)
    for (y, x, kd) in [(1, 1, 1), (2, 3, 4), (16, 16, 8), (33, 97, 4)]:
        q, kk, v = rand_qkv(rng, y, x, kd)
        put(f"grid64_{y}_{x}_{kd}", q, kk, v, naive_attention_array(q, kk, v, SPHERICAL, 1.0),
            extra={"streamed_13_7": streamed_attention_array(q, kk, v, SPHERICAL, 1.0, TileConfig(13, 7))})
    rng = np.random.default_rng(6)
    for (y, x, kd) in [(3, 2, 1), (16, 33, 8), (64, 64, 16)]:
        q, kk, v = rand_qkv(rng, y, x, kd, np.float32)
        put(f"grid32_{y}_{x}_{kd}", q, kk, v, naive_attention_array(q, kk, v, SPHERICAL, 1.0),
            extra={"streamed_5_9": streamed_attention_array(q, kk, v, SPHERICAL, 1.0, TileConfig(5, 9))})

    # Prime sizes: test_attention.py:93-98
    rng = np.random.default_rng(3)
    q, kk, v = rand_qkv(rng, 97, 97, 8)
    put("prime97", q, kk, v, streamed_attention_array(q, kk, v, SPHERICAL, 1.0, TileConfig(16, 16)))

    # Negative scale + epsilon + multiplicity-scaled keys (grn.py:146-173 semantics)
    rng = np.random.default_rng(123)
    q, kk, v = rand_qkv(rng, 40, 70, 64, np.float32)
    m = rng.integers(0, 6, 70).astype(np.float32)
    kk = kk * m[:, None]
    spec = SPHERICAL.with_epsilon(1e-6)
    put("scale_eps_mult", q, kk, v, streamed_attention_array(q, kk, v, spec, -0.7, TileConfig()),
        scale=-0.7, eps=1e-6)

    # GQA: test_attention.py:253-273
    rng = np.random.default_rng(18)
    q = rng.standard_normal((4, 4, 3)); k3 = rng.standard_normal((6, 2, 3)); v3 = rng.standard_normal((6, 2, 3))
    put("gqa_4_2", q, k3, v3, multi_head_attention_array(q, k3, v3, SPHERICAL, h=4, h_kv=2),
        extra={"h": 4, "h_kv": 2})
    rng = np.random.default_rng(19)
    q = rng.standard_normal((5, 2, 4)); k3 = rng.standard_normal((8, 1, 4)); v3 = rng.standard_normal((8, 1, 4))
    put("gqa_2_1", q, k3, v3, multi_head_attention_array(q, k3, v3, SPHERICAL, h=2, h_kv=1),
        extra={"h": 2, "h_kv": 1})
    # a larger GQA case in float32 (GPU-sized heads)
    rng = np.random.default_rng(77)
    q = rng.standard_normal((300, 8, 64)).astype(np.float32)
    k3 = rng.standard_normal((300, 2, 64)).astype(np.float32)
    v3 = rng.standard_normal((300, 2, 64)).astype(np.float32)
    put("gqa_8_2_f32", q, k3, v3, multi_head_attention_array(q, k3, v3, SPHERICAL, h=8, h_kv=2),
        extra={"h": 8, "h_kv": 2})

    # f16 emulation: test_attention.py:351-357 (64x64x16) and criterion 4 inputs (seed 44)
    rng = np.random.default_rng(21)
    q, kk, v = rand_qkv(rng, 64, 64, 16, np.float32)
    put("f16_64", q, kk, v, naive_attention_array(q, kk, v, SPHERICAL, 1.0),
        extra={"f16_out": streamed_attention_array(q, kk, v, SPHERICAL, 1.0, TileConfig(16, 16), f16=True)})
    rng = np.random.default_rng(44)  # test_acceptance.py:188-205
    q = rng.standard_normal((1024, 128)).astype(np.float32)
    kk = rng.standard_normal((1024, 128)).astype(np.float32)
    v = rng.standard_normal((1024, 128)).astype(np.float32)
    g["crit4/out"] = naive_attention_array(q, kk, v, SPHERICAL, 1.0)
    g["crit4/seed"] = np.int64(44)

    # C1: B1 H1 N256 d64 fp32 (BASELINE.json configs[0])
    rng = np.random.default_rng(1000)
    q, kk, v = rand_qkv(rng, 256, 256, 64, np.float32)
    put("c1", q, kk, v, streamed_attention_array(q, kk, v, SPHERICAL, 1.0, TileConfig()))

    # Degenerate rows: test_attention.py:69-77 and measured edge cases
    degen = []
    q = np.array([[1.0, 0.0], [0.0, 0.0]]); k = np.random.default_rng(1).standard_normal((3, 2)); v = np.ones((3, 2))
    degen.append(("degen_row1", q, k, v))
    rng = np.random.default_rng(9)
    q, kk, v = rand_qkv(rng, 5, 7, 4)
    qn = q.copy(); qn[2, 1] = np.nan
    degen.append(("degen_nan_row2", qn, kk, v))
    degen.append(("degen_empty_k", q, kk[:0], v[:0]))
    for name, q, k, v in degen:
        try:
            streamed_attention_array(q, k, v, SPHERICAL, 1.0, TileConfig())
            raise SystemExit(f"{name}: expected DegenerateDenominatorError")
        except DegenerateDenominatorError as e:
            msg = str(e)
            row = int(msg.rsplit("row ", 1)[1].rstrip(")"))
            cases.append(name)
            g[f"{name}/q"], g[f"{name}/k"], g[f"{name}/v"] = q, k, v
            g[f"{name}/err_row"] = np.int64(row)
            g[f"{name}/err_z"] = np.float64(e.z)
            g[f"{name}/scale"] = np.float64(1.0)
            g[f"{name}/eps"] = np.float64(0.0)

    # ---- SIGNED_L1 (normalizers.py:111-117): the other exp-free triple the kernel compiles
    q = np.array([[1.0]]); k = np.array([[3.0], [4.0]]); v = np.array([[10.0], [20.0]])
    put("l1_kat_hand", q, k, v, naive_attention_array(q, k, v, SIGNED_L1, 1.0),
        extra={"streamed_1_1": streamed_attention_array(q, k, v, SIGNED_L1, 1.0, TileConfig(1, 1))})
    rng = np.random.default_rng(31)
    for (y, x, kd) in [(2, 3, 4), (16, 16, 8), (33, 97, 4)]:
        q, kk, v = rand_qkv(rng, y, x, kd)
        put(f"l1_grid64_{y}_{x}_{kd}", q, kk, v, naive_attention_array(q, kk, v, SIGNED_L1, 1.0),
            extra={"streamed_13_7": streamed_attention_array(q, kk, v, SIGNED_L1, 1.0, TileConfig(13, 7))})
    rng = np.random.default_rng(32)
    for (y, x, kd) in [(16, 33, 8), (64, 64, 16), (100, 301, 64)]:
        q, kk, v = rand_qkv(rng, y, x, kd, np.float32)
        put(f"l1_grid32_{y}_{x}_{kd}", q, kk, v, naive_attention_array(q, kk, v, SIGNED_L1, 1.0),
            extra={"streamed_5_9": streamed_attention_array(q, kk, v, SIGNED_L1, 1.0, TileConfig(5, 9))})
    rng = np.random.default_rng(33)
    q, kk, v = rand_qkv(rng, 40, 70, 64, np.float32)
    put("l1_scale_eps", q, kk, v, streamed_attention_array(q, kk, v, SIGNED_L1.with_epsilon(1e-3), -0.7,
                                                           TileConfig()), scale=-0.7, eps=1e-3)
    rng = np.random.default_rng(34)
    q = rng.standard_normal((200, 4, 64)).astype(np.float32)
    k3 = rng.standard_normal((200, 2, 64)).astype(np.float32)
    v3 = rng.standard_normal((200, 2, 64)).astype(np.float32)
    put("l1_gqa_4_2_f32", q, k3, v3, multi_head_attention_array(q, k3, v3, SIGNED_L1, h=4, h_kv=2),
        extra={"h": 4, "h_kv": 2})

    # ---- GRN caller: multiplicity-scaled keys (grn.py:146-173): the fixture keeps the UNSCALED keys
    # and m; out = multi_head_attention_array(q, apply_multiplicity_array(k, m), v, ...)
    for tag, spec, seed in (("sph", SPHERICAL, 35), ("l1", SIGNED_L1, 36)):
        rng = np.random.default_rng(seed)
        q = rng.standard_normal((200, 4, 64)).astype(np.float32)
        k3 = rng.standard_normal((200, 2, 64)).astype(np.float32)
        v3 = rng.standard_normal((200, 2, 64)).astype(np.float32)
        m = rng.integers(0, 6, 200).astype(np.float64)
        spec_e = spec.with_epsilon(1e-6)
        put(f"mult_{tag}_gqa_f32", q, k3, v3,
            multi_head_attention_array(q, apply_multiplicity_array(k3, m), v3, spec_e, h=4, h_kv=2, scale=1.0),
            eps=1e-6, extra={"h": 4, "h_kv": 2, "m": m})

    # SIGNED_L1 degenerate row: test_attention.py:69-77 with the L1 triple
    q = np.array([[1.0, 0.0], [0.0, 0.0]]); k = np.random.default_rng(1).standard_normal((3, 2)); v = np.ones((3, 2))
    try:
        streamed_attention_array(q, k, v, SIGNED_L1, 1.0, TileConfig())
        raise SystemExit("l1_degen_row1: expected DegenerateDenominatorError")
    except DegenerateDenominatorError as e:
        cases.append("l1_degen_row1")
        g["l1_degen_row1/q"], g["l1_degen_row1/k"], g["l1_degen_row1/v"] = q, k, v
        g["l1_degen_row1/err_row"] = np.int64(int(str(e).rsplit("row ", 1)[1].rstrip(")")))
        g["l1_degen_row1/err_z"] = np.float64(e.z)
        g["l1_degen_row1/scale"] = np.float64(1.0)
        g["l1_degen_row1/eps"] = np.float64(0.0)

    g["__cases__"] = np.array(cases)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(cases)} cases")


if __name__ == "__main__":
    main()
