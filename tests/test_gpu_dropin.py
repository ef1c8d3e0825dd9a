"""GPU tests of the drop-in (host-array) path: inputs the reference accepts must run, with the
reference's results and errors.

* float32 / float64 inputs of any magnitude (|s| far above 65504, tiny values, eps-dominated
  rows): ``fs_prepare`` chooses power-of-two operand scales and a Cauchy-Schwarz P scale on the
  device, so the default fp16 compute path cannot overflow (reference attention.py:252-279
  computes these in float64 and returns finite results).
* NaN / inf in V only: the reference returns the non-finite column and raises nothing
  (attention.py:183-200); so must the GPU path -- in the drop-in and the torch fp16 entry.
* chunked host streaming (query chunks, pinned ring) is bitwise equal to one chunk.

Tolerances are relative, fp16-operand level: rel-Frobenius <= 2e-3 and
max-abs <= 8e-3 * max|O| against the float64 oracle on the ORIGINAL (unrounded) inputs.
"""

import numpy as np
import pytest
import torch

from oracle.spherical import OracleDegenerate, gram_spherical, naive_spherical

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def att():
    from paper_2505_09326_b200 import attention
    return attention


def check_rel(got, ref, rel_fro=2e-3, rel_max=8e-3, tag=""):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert np.isfinite(got).all(), tag
    scale = max(np.abs(ref).max(), 1e-300)
    fro = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300)
    mx = np.abs(got - ref).max() / scale
    assert fro <= rel_fro and mx <= rel_max, f"{tag}: rel_fro={fro:.3g} rel_max={mx:.3g}"


def _tile():
    return att().TileConfig()


@pytest.mark.parametrize("mag_q,mag_k,mag_v,dtype", [
    (1e3, 1e3, 1.0, np.float32),      # |s| ~ 1e7 >> 65504: fp16 P overflow without the P scale
    (3e4, 2e4, 5e4, np.float32),      # values near / above the fp16 range
    (1e-4, 1e-4, 1e-5, np.float32),   # values in the fp16 subnormal range
    (1e-30, 1e-30, 1e30, np.float64),  # far outside fp16, inside fp32
    (1e20, 1e-20, 1e-3, np.float64),
])
def test_large_and_tiny_magnitudes_match_reference(mag_q, mag_k, mag_v, dtype):
    rng = np.random.default_rng(1)
    q = (rng.standard_normal((300, 64)) * mag_q).astype(dtype)
    k = (rng.standard_normal((517, 64)) * mag_k).astype(dtype)
    v = (rng.standard_normal((517, 64)) * mag_v).astype(dtype)
    from paper_2505_09326_b200 import SPHERICAL
    got = att().streamed_attention_array(q, k, v, SPHERICAL, 1.0, _tile())
    assert got.dtype == dtype
    check_rel(got, gram_spherical(q.astype(np.float64), k.astype(np.float64), v.astype(np.float64)),
              tag=f"{mag_q},{mag_k},{mag_v}")


def test_eps_dominated_tiny_inputs():
    # z << eps: O ~ c sum s v / sqrt(eps); the operand scales are limited so eps / g^2 stays finite
    rng = np.random.default_rng(2)
    q, k, v = (rng.standard_normal((200, 32)) * 1e-12 for _ in range(3))
    from paper_2505_09326_b200 import SPHERICAL
    spec = SPHERICAL.with_epsilon(1e-6)
    got = att().streamed_attention_array(q, k, v, spec, 1.0, _tile())
    check_rel(got, gram_spherical(q, k, v, 1.0, 1e-6), tag="eps")


def test_signed_l1_large_magnitudes():
    rng = np.random.default_rng(3)
    q = (rng.standard_normal((257, 128)) * 500).astype(np.float32)
    k = (rng.standard_normal((300, 128)) * 500).astype(np.float32)
    v = rng.standard_normal((300, 128)).astype(np.float32)
    from paper_2505_09326_b200 import SIGNED_L1
    got = att().streamed_attention_array(q, k, v, SIGNED_L1, 1.0, _tile())
    ref = naive_spherical(q.astype(np.float64), k.astype(np.float64), v.astype(np.float64), norm="signed_l1")
    check_rel(got, ref, rel_fro=3e-3, rel_max=1.5e-2, tag="signed_l1")


@pytest.mark.parametrize("col", [0, 5])
def test_nan_in_v_passes_through_like_reference(col):
    rng = np.random.default_rng(4)
    q = rng.standard_normal((130, 64)).astype(np.float32)
    k = rng.standard_normal((200, 64)).astype(np.float32)
    v = rng.standard_normal((200, 64)).astype(np.float32)
    v[17, col] = np.nan
    from paper_2505_09326_b200 import SPHERICAL
    got = att().streamed_attention_array(q, k, v, SPHERICAL, 1.0, _tile())   # no exception
    assert np.isnan(got[:, col]).all()
    keep = [c for c in range(64) if c != col]
    vv = v.copy()
    vv[17, col] = 0.0
    check_rel(got[:, keep], gram_spherical(q.astype(np.float64), k.astype(np.float64),
                                           vv.astype(np.float64))[:, keep], tag="nan-v")


def test_nan_in_v_torch_fp16_entry_not_flagged():
    # the fp16 overflow detector only flags rows whose O is non-finite in EVERY column and whose
    # z reaches the overflow range; a NaN in one column of V is passed through unflagged
    from paper_2505_09326_b200 import flashsign
    g = torch.Generator(device="cuda").manual_seed(5)
    q = torch.randn((1, 300, 2, 64), generator=g, device="cuda").half() * 25   # z >= 65504^2: the gate passes
    k = torch.randn((1, 400, 2, 64), generator=g, device="cuda").half() * 25
    v = torch.randn((1, 400, 2, 64), generator=g, device="cuda").half()
    v[0, 3, 1, 0] = float("nan")
    o, bad = flashsign.fwd_async(q, k, v, out_dtype=torch.float32)
    assert flashsign.decode_bad_key(int(bad.item()), 2, 300) is None
    assert torch.isnan(o[0, :, 1, 0]).all() and torch.isfinite(o[0, :, 1, 1:]).all()
    assert torch.isfinite(o[0, :, 0]).all()


def test_inf_in_q_row_is_degenerate_like_reference():
    rng = np.random.default_rng(6)
    q = rng.standard_normal((40, 16)).astype(np.float32)
    k = rng.standard_normal((50, 16)).astype(np.float32)
    v = rng.standard_normal((50, 16)).astype(np.float32)
    q[9, 3] = np.inf
    from paper_2505_09326_b200 import SPHERICAL, DegenerateDenominatorError
    with pytest.raises(OracleDegenerate) as ref:
        naive_spherical(q, k, v)
    with pytest.raises(DegenerateDenominatorError, match=f"row {ref.value.row}") as got:
        att().streamed_attention_array(q, k, v, SPHERICAL, 1.0, _tile())
    assert np.isinf(got.value.z) == np.isinf(ref.value.z) and np.isnan(got.value.z) == np.isnan(ref.value.z)


def test_output_dtypes_follow_inputs():
    rng = np.random.default_rng(7)
    from paper_2505_09326_b200 import SPHERICAL
    for dt in (np.float16, np.float32, np.float64):
        q, k, v = (rng.standard_normal((70, 24)).astype(dt) for _ in range(3))
        got = att().streamed_attention_array(q, k, v, SPHERICAL, 1.0, _tile())
        assert got.dtype == dt and got.shape == (70, 24) and got.flags.c_contiguous
        check_rel(got, gram_spherical(*(a.astype(np.float64) for a in (q, k, v))), rel_fro=3e-3,
                  rel_max=1.5e-2 if dt == np.float16 else 8e-3, tag=str(dt))


@pytest.mark.parametrize("mode", ["pageable", "staged"])
def test_chunked_stream_bitwise_equals_single_chunk(monkeypatch, mode):
    from paper_2505_09326_b200 import SPHERICAL, hostpath
    rng = np.random.default_rng(8)
    q = rng.standard_normal((1000, 4, 64)).astype(np.float32)
    k = rng.standard_normal((700, 2, 64)).astype(np.float32)
    v = rng.standard_normal((700, 2, 64)).astype(np.float32)
    whole = att().multi_head_attention_array(q, k, v, SPHERICAL, 4, 2)
    monkeypatch.setattr(hostpath, "_CHUNK_BYTES", 64 * 4 * 64 * 4 + 1000)   # 64 query rows per chunk
    hostpath._engines.clear()
    monkeypatch.setenv("FLASHSIGN_H2D", mode)
    try:
        chunked = att().multi_head_attention_array(q, k, v, SPHERICAL, 4, 2)
    finally:
        hostpath._engines.clear()
    assert np.array_equal(whole, chunked)


def test_first_bad_row_across_chunks_and_heads(monkeypatch):
    from paper_2505_09326_b200 import SPHERICAL, DegenerateDenominatorError, hostpath
    rng = np.random.default_rng(9)
    q = rng.standard_normal((300, 3, 32)).astype(np.float32)
    k = rng.standard_normal((100, 3, 32)).astype(np.float32)
    v = rng.standard_normal((100, 3, 32)).astype(np.float32)
    q[250, 0] = 0   # head 0, row 250 (third chunk) <- first in (head, row) order
    q[10, 1] = 0    # head 1, row 10 (first chunk)
    monkeypatch.setattr(hostpath, "_CHUNK_BYTES", 100 * 3 * 32 * 4)
    hostpath._engines.clear()
    try:
        with pytest.raises(DegenerateDenominatorError, match="row 250"):
            att().multi_head_attention_array(q, k, v, SPHERICAL, 3, 3)
    finally:
        hostpath._engines.clear()


def test_multiplicity_call_large_counts():
    # GRN with large gene counts: K' = m K far above the fp16 range
    rng = np.random.default_rng(10)
    q = rng.standard_normal((200, 2, 64)).astype(np.float32)
    k = rng.standard_normal((300, 2, 64)).astype(np.float32) * 100
    v = rng.standard_normal((300, 2, 64)).astype(np.float32)
    m = rng.integers(0, 5000, 300).astype(np.float64)
    from paper_2505_09326_b200 import SPHERICAL
    got = att().multiplicity_attention_array(q, k, v, m, SPHERICAL.with_epsilon(1e-6), 2, 2, scale=1.0)
    kp = k.astype(np.float64) * m[:, None, None]
    for h in range(2):
        check_rel(got[:, h], gram_spherical(q[:, h].astype(np.float64), kp[:, h], v[:, h].astype(np.float64),
                                            1.0, 1e-6), tag=f"head {h}")


@pytest.mark.parametrize("dt", [np.float32, np.float64, np.float16])
def test_small_call_path_bitwise_equals_pipeline(monkeypatch, dt):
    # the packed single-stream path for small calls against the three-stream chunk pipeline
    from paper_2505_09326_b200 import SPHERICAL, hostpath
    rng = np.random.default_rng(11)
    q = rng.standard_normal((77, 4, 40)).astype(dt)
    k = rng.standard_normal((53, 2, 40)).astype(dt)
    v = rng.standard_normal((53, 2, 40)).astype(dt)
    small = att().multi_head_attention_array(q, k, v, SPHERICAL.with_epsilon(1e-6), 4, 2, scale=0.5)
    monkeypatch.setattr(hostpath, "_SMALL_BYTES", 0)
    piped = att().multi_head_attention_array(q, k, v, SPHERICAL.with_epsilon(1e-6), 4, 2, scale=0.5)
    assert small.dtype == piped.dtype == dt and small.shape == (77, 4, 40)
    assert np.array_equal(small, piped)


def test_small_call_path_bad_row_and_reuse():
    from paper_2505_09326_b200 import SPHERICAL, DegenerateDenominatorError
    rng = np.random.default_rng(12)
    q = rng.standard_normal((30, 2, 8)).astype(np.float32)
    k = rng.standard_normal((20, 2, 8)).astype(np.float32)
    v = rng.standard_normal((20, 2, 8)).astype(np.float32)
    q[7, 1] = 0
    q[9, 0] = 0
    with pytest.raises(DegenerateDenominatorError, match="row 9"):
        att().multi_head_attention_array(q, k, v, SPHERICAL, 2, 2)
    # the reused packed buffers: a larger then a smaller call, each against the float64 oracle
    for n, x in ((300, 500), (5, 3)):
        q = rng.standard_normal((n, 1, 16)).astype(np.float32)
        k = rng.standard_normal((x, 1, 16)).astype(np.float32)
        v = rng.standard_normal((x, 1, 16)).astype(np.float32)
        got = att().multi_head_attention_array(q, k, v, SPHERICAL, 1, 1)
        check_rel(got[:, 0], gram_spherical(*(a[:, 0].astype(np.float64) for a in (q, k, v))), tag=f"n{n}")


# ------------------------------------------------------------------ randomized drop-in sweep

def _dropin_cases():
    # FS_DROPIN_N / FS_SWEEP_SEED widen it for stress runs (default 24 cases)
    import os
    n = int(os.environ.get("FS_DROPIN_N", 24))
    rng = np.random.default_rng(int(os.environ.get("FS_SWEEP_SEED", 31)))
    modes = ["fp16", "bf16", "e4m3", "f64"]
    out = []
    for i in range(n):
        hkv = int(rng.choice([1, 2, 3]))
        out.append(dict(mode=modes[i % 4], n=int(rng.integers(1, 1500)), x=int(rng.integers(16, 1500)),
                        h=hkv * int(rng.choice([1, 2, 4])), hkv=hkv, d=int(rng.integers(1, 129)),
                        dt=[np.float32, np.float64, np.float16][int(rng.integers(0, 3))],
                        norm=str(rng.choice(["spherical", "signed_l1"])),
                        scale=float(rng.choice([1.0, -0.25, 3.0])), eps=float(rng.choice([0.0, 1e-4])),
                        seed=int(rng.integers(1 << 30))))
    return out


@pytest.mark.parametrize("c", _dropin_cases(), ids=lambda c: f"{c['mode']}-{np.dtype(c['dt']).name}-n{c['n']}x{c['x']}"
                                                             f"-h{c['h']}/{c['hkv']}-d{c['d']}-{c['norm']}")
def test_dropin_random_sweep(c):
    from oracle.spherical import multi_head_spherical
    from paper_2505_09326_b200 import SIGNED_L1, SPHERICAL
    A = att()
    rng = np.random.default_rng(c["seed"])
    q = rng.standard_normal((c["n"], c["h"], c["d"])).astype(c["dt"])
    k = rng.standard_normal((c["x"], c["hkv"], c["d"])).astype(c["dt"])
    v = rng.standard_normal((c["x"], c["hkv"], c["d"])).astype(c["dt"])
    spec = (SPHERICAL if c["norm"] == "spherical" else SIGNED_L1).with_epsilon(c["eps"])
    prev = A.get_compute_dtype()
    A.set_compute_dtype(c["mode"])
    try:
        got = A.multi_head_attention_array(q, k, v, spec, c["h"], c["hkv"], scale=c["scale"])
    finally:
        A.set_compute_dtype(prev)
    assert got.dtype == c["dt"] and got.shape == q.shape
    ref = multi_head_spherical(*(a.astype(np.float64) for a in (q, k, v)), c["h"], c["hkv"], c["scale"], c["eps"],
                               path="naive", norm=c["norm"])
    assert np.isfinite(got).all()
    if c["d"] >= 8:
        tol = {"fp16": (4e-3, 3e-2), "bf16": (2e-2, 1e-1), "e4m3": (8e-2, 0.5), "f64": (1e-9, 1e-8)}[c["mode"]]
        if c["dt"] == np.float16:  # the float16 result rounding
            tol = (max(tol[0], 2e-3), max(tol[1], 1e-2))
        elif c["dt"] == np.float32 and c["mode"] == "f64":  # the reference's float32 rounding points
            tol = (1e-5, 1e-4)
        check_rel(got, ref, *tol, tag=str(c))
        return
    # d < 8: a row's output is a handful of cancelling sums (d = 1: every row is the same sum
    # sum_j k_j v_j / |k|), so a relative check fails on unlucky seeds for any 16-bit kernel; the
    # error is held to the first-order condition instead: with M = |Q||K|^T (what one rounding of q
    # and k moves a score by, relative), cond = M |V| / b + |O| * (relative move of b), b = b(z + eps)
    cond = np.empty_like(ref)
    for i in range(c["h"]):
        kv = (i * c["hkv"]) // c["h"]
        qa, ka = q[:, i].astype(np.float64), k[:, kv].astype(np.float64)
        sc = c["scale"] * (qa @ ka.T)
        m = abs(c["scale"]) * (np.abs(qa) @ np.abs(ka).T)
        if c["norm"] == "spherical":
            den = np.sqrt((sc * sc).sum(1) + c["eps"])
            rel_den = (np.abs(sc) * m).sum(1) / den ** 2
        else:
            den = np.abs(sc).sum(1) + c["eps"]
            rel_den = m.sum(1) / den
        cond[:, i] = (m @ np.abs(v[:, kv].astype(np.float64))) / den[:, None] + np.abs(ref[:, i]) * rel_den[:, None]
    tol = {"fp16": 4e-3, "bf16": 3e-2, "e4m3": 0.25, "f64": 1e-9}[c["mode"]]
    if c["dt"] == np.float16:
        tol = max(tol, 2e-3)
    elif c["dt"] == np.float32 and c["mode"] == "f64":
        tol = 1e-5
    worst = float((np.abs(got.astype(np.float64) - ref) / cond).max())
    assert worst <= tol, (c, worst)


@pytest.mark.parametrize("dts", [(np.float32, np.float64, np.float32), (np.float64, np.float32, np.float16),
                                 (np.float16, np.float32, np.float64)])
def test_mixed_dtype_arrays_small_and_pipeline(monkeypatch, dts):
    # the reference accepts q, k, v of different float dtypes (result in q's dtype)
    from paper_2505_09326_b200 import SPHERICAL, hostpath
    rng = np.random.default_rng(13)
    q = rng.standard_normal((40, 2, 16)).astype(dts[0])
    k = rng.standard_normal((60, 1, 16)).astype(dts[1])
    v = rng.standard_normal((60, 1, 16)).astype(dts[2])
    small = att().multi_head_attention_array(q, k, v, SPHERICAL, 2, 1)
    monkeypatch.setattr(hostpath, "_SMALL_BYTES", 0)
    piped = att().multi_head_attention_array(q, k, v, SPHERICAL, 2, 1)
    assert small.dtype == piped.dtype == dts[0]
    assert np.array_equal(small, piped)
    ref = np.stack([gram_spherical(q[:, i].astype(np.float64), k[:, 0].astype(np.float64),
                                   v[:, 0].astype(np.float64)) for i in range(2)], axis=1)
    check_rel(small, ref, 3e-3, 1.5e-2)
