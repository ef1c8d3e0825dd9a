"""CPU oracle for the FlashSign (spherical attention) forward -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it.  The shipped path
(``paper_2505_09326_b200``) never imports anything under ``oracle/`` and
fails loudly when its CUDA library is missing.

It is a numpy restatement of the reference's hot path
(``/root/reference/pkg/src/ncstream/attention.py``), not a copy: each
function names the reference lines whose behaviour it restates.

Contract (attention.py:1-11, normalizers.py:94-100):

    s_ij = c * (q_i . k_j)
    O_i  = sum_j s_ij v_j / sqrt(sum_j s_ij^2 + eps)

and the other exp-free triple the kernel compiles, SIGNED_L1 (normalizers.py:111-117):
O_i = sum_j s_ij v_j / (sum_j |s_ij| + eps).  ``norm="signed_l1"`` selects it.

Parity pinning: ``tests/test_oracle.py`` checks every function here against
golden vectors produced by running the reference itself
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``), including the
reference's own known-answer tests (test_attention.py:46-77).
"""

from __future__ import annotations

import math

import numpy as np


class OracleDegenerate(ValueError):
    """First row whose denominator b(z + eps) is zero or non-finite.

    Mirrors ``DegenerateDenominatorError(z, "row i")`` (normalizers.py:29-35)
    as raised by attention.py:136-139 (naive) and :196-199 (streamed).
    """

    def __init__(self, z: float, row: int, head: int | None = None, batch: int | None = None):
        self.z = z
        self.row = row
        self.head = head
        self.batch = batch
        super().__init__(f"degenerate denominator z={z!r} (row {row})")


def _check(q, k, v):
    # attention.py:104-111 (_check_qkv)
    if q.ndim != 2 or k.ndim != 2 or v.ndim != 2:
        raise ValueError(f"expected rank-2 Q/K/V, got {q.shape}, {k.shape}, {v.shape}")
    if q.shape[1] != k.shape[1]:
        raise ValueError(f"Q and K feature dims differ: {q.shape} vs {k.shape}")
    if v.shape[0] != k.shape[0]:
        raise ValueError(f"K and V row counts differ: {k.shape} vs {v.shape}")


_A2 = {"spherical": lambda s: s * s, "signed_l1": np.abs}       # normalizers.py:97, 114
_B = {"spherical": np.sqrt, "signed_l1": lambda z: z}          # normalizers.py:98, 115


def naive_spherical(q: np.ndarray, k: np.ndarray, v: np.ndarray,
                    scale: float = 1.0, eps: float = 0.0, norm: str = "spherical") -> np.ndarray:
    """Materialising oracle, restating ``naive_attention_array`` (attention.py:114-143).

    float32 inputs: scores accumulate in float64 and round to float32
    (124-128), z is summed in float32 (134), the weighted sum runs in
    float64 and rounds to float32 (140-142).  float64 stays float64.
    """
    _check(q, k, v)
    f32 = q.dtype == np.float32
    if f32:
        s = (q.astype(np.float64) @ k.astype(np.float64).T).astype(np.float32)
    else:
        s = q @ k.T
    if scale != 1.0:
        s = s * np.asarray(scale, dtype=s.dtype)
    z = _A2[norm](s).sum(axis=1)
    den = _B[norm](z + eps) if eps else _B[norm](z)
    bad = ~np.isfinite(den) | (den == 0)
    if bad.any():
        row = int(np.argmax(bad))
        raise OracleDegenerate(float(z[row]), row)
    w = s / den[:, None]
    if f32:
        return (w.astype(np.float64) @ v.astype(np.float64)).astype(np.float32)
    return w @ v


def quantize_f16(a: np.ndarray) -> np.ndarray:
    """RNE to binary16, kept float32 (tensor.py:132-139)."""
    with np.errstate(over="ignore"):
        return a.astype(np.float16).astype(np.float32)


def streamed_spherical(q: np.ndarray, k: np.ndarray, v: np.ndarray,
                       scale: float = 1.0, eps: float = 0.0,
                       g_y: int = 64, s_x: int = 64, f16: bool = False, norm: str = "spherical") -> np.ndarray:
    """The FlashSign tile loop, restating ``streamed_attention_array`` +
    ``_streamed_tiles`` non-safe branch (attention.py:252-279, 146-200) for the
    exp-free triples (``norm``: spherical | signed_l1).

    Query groups of ``g_y`` rows; K/V chunks of ``s_x`` keys; per-row (o, z)
    accumulators in float64 (float32 under f16 emulation, 157-158); scores
    rounded to float32 for float32 outputs (163-164), scaled (165-166),
    f16-quantised in f16 mode (167-168); o re-quantised per chunk in f16 mode
    (189-190); finalise o / sqrt(z + eps) with the first-bad-row check
    (195-200).
    """
    _check(q, k, v)
    in_dtype = q.dtype
    if f16:
        if in_dtype != np.float32:
            raise ValueError("f16 emulation requires float32 inputs")
        q, k, v = quantize_f16(q), quantize_f16(k), quantize_f16(v)
    y, x = q.shape[0], k.shape[0]
    d = v.shape[1]  # the reference sizes o by q's width (157) and so rejects d_v != d; the checker allows it
    out = np.empty((y, d), dtype=in_dtype)
    q64, k64, v64 = (a.astype(np.float64, copy=False) for a in (q, k, v))
    kt = np.ascontiguousarray(k64.T)
    out_f32 = in_dtype == np.float32
    acc_t = np.float32 if f16 else np.float64
    for g0 in range(0, y, g_y):
        g1 = min(g0 + g_y, y)
        qg = q64[g0:g1]
        o = np.zeros((g1 - g0, d), dtype=acc_t)
        z = np.zeros(g1 - g0, dtype=acc_t)
        for c0 in range(0, x, s_x):
            c1 = min(c0 + s_x, x)
            st = qg @ kt[:, c0:c1]
            if out_f32:
                st = st.astype(np.float32)
            if scale != 1.0:
                st *= np.asarray(scale, dtype=st.dtype)
            if f16:
                st = quantize_f16(st)
                o += st @ v64[c0:c1].astype(np.float32)
            else:
                o += st.astype(np.float64, copy=False) @ v64[c0:c1]
            z += _A2[norm](st).sum(axis=1, dtype=z.dtype)
            if f16:
                o = quantize_f16(o)
        den = _B[norm](z + eps) if eps else _B[norm](z)
        bad = ~np.isfinite(den) | (den == 0)
        if bad.any():
            i = int(np.argmax(bad))
            raise OracleDegenerate(float(z[i]), g0 + i)
        out[g0:g1] = o / den[:, None]
    return out


def multi_head_spherical(q: np.ndarray, k: np.ndarray, v: np.ndarray, h: int, h_kv: int,
                         scale: float = 1.0, eps: float = 0.0, path: str = "streamed",
                         g_y: int = 64, s_x: int = 64, f16: bool = False, norm: str = "spherical") -> np.ndarray:
    """GQA over ``[n, heads, d]``, restating ``multi_head_attention_array``
    (attention.py:318-361): query head i reads kv head (i*h_kv)//h (352), heads
    run serially (351) so the first degenerate head in loop order raises."""
    if h < 1 or h_kv < 1 or h % h_kv != 0:
        raise ValueError(f"query heads must be a multiple of kv heads, got h={h}, h_kv={h_kv}")
    out = np.empty_like(q)
    for i in range(h):
        kv = (i * h_kv) // h
        try:
            if path == "streamed":
                out[:, i, :] = streamed_spherical(q[:, i], k[:, kv], v[:, kv], scale, eps, g_y, s_x, f16, norm)
            else:
                out[:, i, :] = naive_spherical(q[:, i], k[:, kv], v[:, kv], scale, eps, norm)
        except OracleDegenerate as e:
            e.head = i
            raise
    return out


def gram_spherical(q: np.ndarray, k: np.ndarray, v: np.ndarray,
                   scale: float = 1.0, eps: float = 0.0) -> np.ndarray:
    """Full-size float64 oracle via the exact linear-attention identity
    (SURVEY.md section 0 fact 4):

        O_i = c q_i (K^T V) / sqrt(c^2 q_i (K^T K) q_i^T + eps)

    Algebraically identical to the reference contract because a1 is the
    identity and a2 the square (normalizers.py:94-100); checked against the
    reference-generated golden vectors and ``naive_spherical`` in
    tests/test_oracle.py.  O(N d^2) so every output of a full benchmark
    configuration can be checked.  Never a throughput number for FlashSign.
    Inputs [y, d], [x, d], [x, d]; returns float64.  Degenerate rows are
    reported by returning NaN in that row (callers compare finiteness).
    """
    q64, k64, v64 = (np.asarray(a, dtype=np.float64) for a in (q, k, v))
    kv = k64.T @ v64            # [d, d]
    kk = k64.T @ k64            # [d, d]
    num = q64 @ kv
    z = np.einsum("id,de,ie->i", q64, kk, q64)
    z = np.maximum(z, 0.0)       # roundoff can push an exact 0 slightly negative
    den = np.sqrt(scale * scale * z + eps)
    with np.errstate(divide="ignore", invalid="ignore"):
        out = (scale * num) / den[:, None]
    out[den == 0] = np.nan
    return out


def gram_batched(q: np.ndarray, k: np.ndarray, v: np.ndarray,
                 scale: float = 1.0, eps: float = 0.0, m: np.ndarray | None = None) -> np.ndarray:
    """``gram_spherical`` over BSHD ``[B, N, H, d]`` with GQA (h -> h*H_kv//H).
    ``m`` [B, Nkv]: key multiplicities, K' = m K (attention.py:381-388) in float64."""
    b_, n_q, h_, d = q.shape
    h_kv = k.shape[2]
    out = np.empty(q.shape, dtype=np.float64)
    for b in range(b_):
        for h in range(h_):
            kv = (h * h_kv) // h_
            kb = np.asarray(k[b, :, kv], dtype=np.float64)
            if m is not None:
                kb = kb * np.asarray(m[b], dtype=np.float64)[:, None]
            out[b, :, h] = gram_spherical(q[b, :, h], kb, v[b, :, kv], scale, eps)
    return out


def exact_batched(q: np.ndarray, k: np.ndarray, v: np.ndarray, scale: float = 1.0, eps: float = 0.0,
                  norm: str = "spherical", m: np.ndarray | None = None) -> np.ndarray:
    """float64 oracle over BSHD with GQA for either exp-free triple: the Gram form for
    spherical, the materialised scores (attention.py:114-143 in float64) for signed_l1.
    Degenerate rows come back as NaN."""
    if norm == "spherical":
        return gram_batched(q, k, v, scale, eps, m)
    b_, n_q, h_, d = q.shape
    h_kv = k.shape[2]
    out = np.empty(q.shape, dtype=np.float64)
    for b in range(b_):
        for h in range(h_):
            kv = (h * h_kv) // h_
            kb = np.asarray(k[b, :, kv], dtype=np.float64)
            if m is not None:
                kb = kb * np.asarray(m[b], dtype=np.float64)[:, None]
            s = scale * (np.asarray(q[b, :, h], dtype=np.float64) @ kb.T)
            den = _A2[norm](s).sum(axis=1) + eps
            with np.errstate(divide="ignore", invalid="ignore"):
                o = (s @ np.asarray(v[b, :, kv], dtype=np.float64)) / den[:, None]
            o[den == 0] = np.nan
            out[b, :, h] = o
    return out


def flops(batch: int, heads: int, n_q: int, n_kv: int, d: int) -> int:
    """Algorithmic FLOPs per forward: 4 B H Nq Nkv d (costmodel.py:129)."""
    return 4 * batch * heads * n_q * n_kv * d


def reference_cpu_time_per_slice(n: int, d: int, reps: int = 1, seed: int = 0,
                                 g_y: int = 64, s_x: int = 64) -> float:
    """Median wall time (s) of ``streamed_spherical`` on one (b,h) slice of
    float32 standard normals, mirroring the reference bench harness
    (cli.py:216-223: one warm-up, ``reps`` timed runs, median)."""
    import time
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((n, d)).astype(np.float32)
    k = rng.standard_normal((n, d)).astype(np.float32)
    v = rng.standard_normal((n, d)).astype(np.float32)
    streamed_spherical(q[: min(n, 256)], k, v, 1.0, 0.0, g_y, s_x)  # warm-up (bounded)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        streamed_spherical(q, k, v, 1.0, 0.0, g_y, s_x)
        times.append(time.perf_counter() - t0)
    return float(np.median(times)) if times else math.nan
