"""GPU parity of the FlashSign kernel against the CPU oracle (run with -m gpu on a B200).

Every comparison uses identical inputs: values quantised to the kernel dtype,
then upcast for the float64 oracle.  Tolerances (GPU vs fp64 oracle on the
same quantised inputs):

    fp16 -> fp16 : max-abs <= 8e-3, >= 99.7% within 0.01
    bf16 -> bf16 : rel-Frobenius <= 5e-3, max-abs <= 5e-2, >= 99.0% within 0.01
    e4m3 -> bf16 : rel-Frobenius <= 4e-2, mean-abs <= 3e-2, max-abs <= 0.3

Known-answer tests whose values are exact in every dtype are checked bitwise.
"""

import os

import numpy as np
import pytest
import torch

from oracle.spherical import gram_batched, gram_spherical, streamed_spherical

pytestmark = pytest.mark.gpu

TOL = {
    torch.float16: dict(max_abs=8e-3, within=0.997),
    torch.bfloat16: dict(rel_fro=5e-3, max_abs=5e-2, within=0.99),
    torch.float8_e4m3fn: dict(rel_fro=4e-2, mean_abs=3e-2, max_abs=0.3),
}


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2505_09326_b200 import build
    build.build()


def fs():
    from paper_2505_09326_b200 import flashsign
    return flashsign


def compat():
    from paper_2505_09326_b200 import attention
    return attention


def check_tol(got, ref, dtype, tag=""):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert np.isfinite(got).all(), f"{tag}: non-finite output"
    err = np.abs(got - ref)
    t = TOL[dtype]
    stats = dict(max_abs=float(err.max()), mean_abs=float(err.mean()),
                 rel_fro=float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)),
                 within=float(np.mean(err <= 0.01)))
    for key, lim in t.items():
        if key == "within":
            assert stats[key] >= lim, f"{tag}: {stats}"
        else:
            assert stats[key] <= lim, f"{tag}: {stats}"
    return stats


def rand_bshd(b, n, h, d, dtype, seed, scale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn((b, n, h, d), generator=g, device="cuda") * scale).to(dtype)


def oracle_of(q, k, v, scale=1.0, eps=0.0):
    return gram_batched(q.float().cpu().numpy(), k.float().cpu().numpy(), v.float().cpu().numpy(), scale, eps)


# ------------------------------------------------------------------ kernel vs oracle (torch-native entry)

SHAPES = [  # (B, Nq, Nkv, H, Hkv, d)
    (1, 128, 128, 1, 1, 128),
    (1, 256, 256, 1, 1, 64),
    (2, 300, 517, 4, 2, 128),   # ragged N, GQA
    (1, 1, 1, 1, 1, 64),        # one query, one key
    (1, 129, 255, 2, 2, 64),    # one row past a tile, one key short of two tiles
    (3, 777, 1000, 2, 1, 64),
    (1, 200, 300, 2, 2, 96),    # head dim zero-padded in SMEM by TMA
    (1, 64, 64, 1, 1, 16),
    (1, 2048, 4096, 2, 2, 128),
]


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16, torch.float8_e4m3fn], ids=["bf16", "fp16", "e4m3"])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_kernel_matches_oracle(shape, dtype):
    b, nq, nkv, h, hkv, d = shape
    if dtype == torch.float8_e4m3fn and d % 16:
        pytest.skip("fp8 head dim must be a multiple of 16")
    q = rand_bshd(b, nq, h, d, dtype, 1)
    k = rand_bshd(b, nkv, hkv, d, dtype, 2)
    v = rand_bshd(b, nkv, hkv, d, dtype, 3)
    o = fs().fwd(q, k, v)
    assert o.dtype == (torch.bfloat16 if dtype == torch.float8_e4m3fn else dtype)
    check_tol(o.float().cpu().numpy(), oracle_of(q, k, v), dtype, f"{shape}")


@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16, torch.float16])
def test_output_dtypes_agree(out_dtype):
    q, k, v = (rand_bshd(1, 333, 2, 128, torch.float16, s) for s in (4, 5, 6))
    ref = fs().fwd(q, k, v, out_dtype=torch.float32)
    o = fs().fwd(q, k, v, out_dtype=out_dtype)
    assert torch.equal(o, ref.to(out_dtype))


@pytest.mark.parametrize("scale,eps", [(-0.7, 1e-6), (3.0, 0.0), (0.125, 0.5), (-1.0, 0.0)])
def test_scale_and_epsilon(scale, eps):
    q, k, v = (rand_bshd(2, 400, 2, 64, torch.float16, s) for s in (7, 8, 9))
    o = fs().fwd(q, k, v, scale=scale, eps=eps, out_dtype=torch.float32)
    check_tol(o.cpu().numpy(), oracle_of(q, k, v, scale, eps), torch.float16, f"scale={scale} eps={eps}")


def test_deterministic_bitwise():
    q, k, v = (rand_bshd(2, 1000, 4, 128, torch.bfloat16, s) for s in (10, 11, 12))
    a = fs().fwd(q, k, v)
    bb = fs().fwd(q, k, v)
    assert torch.equal(a, bb)


def test_gqa_equals_duplicated_kv_heads_bitwise():
    # test_attention.py:264-273 duplication oracle -- same data, same order -> bitwise
    q = rand_bshd(2, 500, 4, 64, torch.bfloat16, 13)
    k = rand_bshd(2, 700, 2, 64, torch.bfloat16, 14)
    v = rand_bshd(2, 700, 2, 64, torch.bfloat16, 15)
    gqa = fs().fwd(q, k, v)
    dup = fs().fwd(q, k.repeat_interleave(2, dim=2).contiguous(), v.repeat_interleave(2, dim=2).contiguous())
    assert torch.equal(gqa, dup)


def test_strided_views_equal_contiguous():
    q = rand_bshd(2, 300, 8, 64, torch.bfloat16, 16)
    k = rand_bshd(2, 300, 8, 64, torch.bfloat16, 17)
    v = rand_bshd(2, 300, 8, 64, torch.bfloat16, 18)
    o_full = fs().fwd(q, k, v)
    o_view = fs().fwd(q[:, :, 2:6], k[:, :, 2:6], v[:, :, 2:6])
    assert torch.equal(o_full[:, :, 2:6], o_view)


def test_sharded_equals_full_bitwise():
    """Batch x head partition (paper_2505_09326_b200.partition): every rank's pieces
    computed separately equal the same slices of one full launch."""
    from paper_2505_09326_b200 import partition
    B, N, H, HKV, D = 3, 640, 8, 4, 64
    q = rand_bshd(B, N, H, D, torch.bfloat16, 19)
    k = rand_bshd(B, N, HKV, D, torch.bfloat16, 20)
    v = rand_bshd(B, N, HKV, D, torch.bfloat16, 21)
    full = fs().fwd(q, k, v)
    for world in (2, 3, 5, 8):
        o = torch.full_like(full, float("nan"))
        for rank in range(world):
            lo, hi = partition.unit_range(B * HKV, world, rank)
            partition.fwd_shard(q, k, v, o, lo, hi, fs().fwd_async)
        assert torch.equal(o, full), world


def test_sharded_c2_with_tail_split():
    # 8-way batch x head shards of C2 (B16 H16 N4096 d64 fp16): each shard's launch is 256 work tiles
    # = 3 waves + 34, so the automatic plan splits the tail wave's K/V (fs_plan, split_tail); the
    # single full launch does not.  Rows of whole-wave tiles are bitwise the full launch's; tail rows
    # differ only by the fp32 summation order of the two halves (one fp16 rounding at most).
    # With kv_splits=1 every shard is bitwise the full launch.
    from paper_2505_09326_b200 import partition
    B, N, H, D = 16, 4096, 16, 64
    q = rand_bshd(B, N, H, D, torch.float16, 25)
    k = rand_bshd(B, N, H, D, torch.float16, 26)
    v = rand_bshd(B, N, H, D, torch.float16, 27)
    full = fs().fwd(q, k, v)
    lo, hi = partition.unit_range(B * H, 8, 0)
    pl = fs().plan(2, H, N, N, q.device, D, torch.float16)
    assert pl.split_tail == 1 and pl.splits == 2 and pl.efficiency > 0.98
    for splits, exact in ((None, False), (1, True)):
        o = torch.full_like(full, float("nan"))
        for rank in range(8):
            lo, hi = partition.unit_range(B * H, 8, rank)
            partition.fwd_shard(q, k, v, o, lo, hi, fs().fwd_async, kv_splits=splits)
        if exact:
            assert torch.equal(o, full)
        else:
            d = (o.float() - full.float()).abs()
            assert bool(torch.isfinite(o).all())
            assert float(d.max()) <= 2.0 ** -10 * max(1.0, float(full.float().abs().max()))
            assert float((d == 0).float().mean()) >= 0.9


def test_negating_k_single_key_flips_exactly():
    # test_attention.py:186-191
    q = rand_bshd(1, 6, 1, 64, torch.bfloat16, 22)
    k = rand_bshd(1, 1, 1, 64, torch.bfloat16, 23)
    v = rand_bshd(1, 1, 1, 64, torch.bfloat16, 24)
    a = fs().fwd(q, k, v, out_dtype=torch.float32)
    bb = fs().fwd(q, -k, v, out_dtype=torch.float32)
    assert torch.equal(bb, -a)


def test_positive_scale_invariance():
    # test_attention.py:177-184 (within tolerance: power-of-two lambdas are exact)
    # bf16 keeps fp32's exponent range, so power-of-two rescaling of q is exact end to end
    q, k, v = (rand_bshd(1, 300, 2, 64, torch.bfloat16, s) for s in (25, 26, 27))
    base = fs().fwd(q, k, v, out_dtype=torch.float32)
    for lam in (0.5, 4.0):
        got = fs().fwd((q.float() * lam).bfloat16(), k, v, out_dtype=torch.float32)
        assert torch.equal(got, base)
    for lam in (3.0, 100.0):
        got = fs().fwd(q, k, v, scale=lam, out_dtype=torch.float32)
        torch.testing.assert_close(got, base, rtol=1e-5, atol=1e-5)


def test_key_permutation_equivariance():
    q, k, v = (rand_bshd(1, 200, 1, 64, torch.float16, s) for s in (28, 29, 30))
    perm = torch.randperm(200, device="cuda")
    base = fs().fwd(q, k, v, out_dtype=torch.float32)
    got = fs().fwd(q, k[:, perm].contiguous(), v[:, perm].contiguous(), out_dtype=torch.float32)
    torch.testing.assert_close(got, base, rtol=0, atol=2e-3)


def test_zero_keys_are_removable():
    # a1(0)=a2(0)=0: zero keys contribute nothing (test_attention.py:219-228)
    q, k, v = (rand_bshd(1, 256, 2, 64, torch.bfloat16, s) for s in (31, 32, 33))
    keep = torch.ones(256, dtype=torch.bool, device="cuda")
    keep[::3] = False
    k0 = k.clone()
    k0[:, ~keep] = 0
    full = fs().fwd(q, k0, v, out_dtype=torch.float32)
    red = fs().fwd(q, k[:, keep].contiguous(), v[:, keep].contiguous(), out_dtype=torch.float32)
    torch.testing.assert_close(full, red, rtol=1e-5, atol=1e-5)


# ------------------------------------------------------------------ degenerate rows and overflow

def test_degenerate_row_first_in_loop_order():
    from paper_2505_09326_b200.normalizers import DegenerateDenominatorError
    q = rand_bshd(2, 300, 4, 64, torch.bfloat16, 34)
    k = rand_bshd(2, 300, 2, 64, torch.bfloat16, 35)
    v = rand_bshd(2, 300, 2, 64, torch.bfloat16, 36)
    q[1, 250, 3] = 0   # batch 1 head 3 row 250
    q[1, 7, 2] = 0     # batch 1 head 2 row 7   <- first in (batch, head, row) order
    q[1, 3, 3] = 0
    o, bad = fs().fwd_async(q, k, v)
    assert fs().decode_bad_key(int(bad.item()), 4, 300) == (1, 2, 7, 0.0)
    with pytest.raises(DegenerateDenominatorError, match="row 7"):
        fs().fwd(q, k, v)
    # eps > 0 turns the zero row into a zero output (normalizers.py:62-66 docstring)
    o = fs().fwd(q, k, v, eps=1e-6, out_dtype=torch.float32)
    assert torch.all(o[1, 7, 2] == 0)


def test_nan_row_reported_with_nan_z():
    q = rand_bshd(1, 50, 1, 64, torch.float16, 37)
    k = rand_bshd(1, 50, 1, 64, torch.float16, 38)
    v = rand_bshd(1, 50, 1, 64, torch.float16, 39)
    q[0, 2, 0, 5] = float("nan")
    _, bad = fs().fwd_async(q, k, v)
    b_, h_, row, z = fs().decode_bad_key(int(bad.item()), 1, 50)
    assert row == 2 and np.isnan(z)


def test_fp16_p_overflow_is_reported_not_silent():
    q = torch.full((1, 4, 1, 64), 200.0, device="cuda", dtype=torch.float16)
    k = torch.full((1, 4, 1, 64), 200.0, device="cuda", dtype=torch.float16)   # s = 64*4e4 > 65504
    v = rand_bshd(1, 4, 1, 64, torch.float16, 40)
    _, bad = fs().fwd_async(q, k, v)
    info = fs().decode_bad_key(int(bad.item()), 1, 4)
    assert info is not None and info[2] == 0 and np.isinf(info[3])
    # bf16 keeps fp32 range: no overflow, correct result
    o = fs().fwd(q.bfloat16(), k.bfloat16(), v.bfloat16(), out_dtype=torch.float32)
    check_tol(o.cpu().numpy(), oracle_of(q.bfloat16(), k.bfloat16(), v.bfloat16()), torch.bfloat16)


def test_empty_inputs():
    q = rand_bshd(1, 0, 2, 64, torch.bfloat16, 41)
    k = rand_bshd(1, 10, 2, 64, torch.bfloat16, 42)
    o = fs().fwd(q, k, k)
    assert o.shape == (1, 0, 2, 64)
    q = rand_bshd(1, 5, 2, 64, torch.bfloat16, 43)
    k0 = torch.zeros((1, 1, 2, 64), dtype=torch.bfloat16, device="cuda")[:, :0]
    _, bad = fs().fwd_async(q, k0, k0)
    assert fs().decode_bad_key(int(bad.item()), 2, 5) == (0, 0, 0, 0.0)
    o = fs().fwd(q, k0, k0, eps=1.0, out_dtype=torch.float32)
    assert torch.all(o == 0)


# ------------------------------------------------------------------ the ncstream-compatible API

def test_compat_kat_hand_exact(golden):
    # test_attention.py:46-52 / 100-106 -> [[22.0]] exactly, through the DenseTensor API
    at = compat()
    from paper_2505_09326_b200.tensor import DenseTensor
    q = DenseTensor([[1.0]])
    k = DenseTensor([[3.0], [4.0]])
    v = DenseTensor([[10.0], [20.0]])
    for dt in ("fp16", "bf16"):
        at.set_compute_dtype(dt)
        try:
            out = at.streamed_attention(q, k, v, at.AttentionConfig(at.SPHERICAL if hasattr(at, "SPHERICAL") else
                                                                     __import__("paper_2505_09326_b200").SPHERICAL,
                                                                     tile=at.TileConfig(1, 1)))
            assert out.tolist() == [[22.0]]
            out = at.naive_generalized_attention(q, k, v, at.AttentionConfig(__import__("paper_2505_09326_b200").SPHERICAL))
            assert out.tolist() == [[22.0]]
        finally:
            at.set_compute_dtype("fp16")
    f32 = golden["kat_hand_f32/q"], golden["kat_hand_f32/k"], golden["kat_hand_f32/v"]
    from paper_2505_09326_b200 import SPHERICAL
    got = at.streamed_attention_array(*f32, SPHERICAL, 1.0, at.TileConfig())
    assert got.dtype == np.float32 and got.tolist() == [[22.0]]


def test_compat_sign_kat_exact():
    # test_attention.py:60-67 (value width = head width for the streamed kernel)
    from paper_2505_09326_b200 import SPHERICAL
    at = compat()
    q = np.array([[2.0]])
    v = np.array([[5.0]])
    assert np.array_equal(at.streamed_attention_array(q, np.array([[1.0]]), v, SPHERICAL, 1.0, at.TileConfig()), v)
    assert np.array_equal(at.streamed_attention_array(q, np.array([[-1.0]]), v, SPHERICAL, 1.0, at.TileConfig()), -v)
    v2 = np.array([[5.0, -7.0]])
    assert np.array_equal(at.naive_attention_array(q, np.array([[-1.0]]), v2, SPHERICAL, 1.0), -v2)


def test_compat_degenerate_rows_match_reference(golden):
    from paper_2505_09326_b200 import SPHERICAL, DegenerateDenominatorError
    at = compat()
    for case in ("degen_row1", "degen_nan_row2", "degen_empty_k"):
        q, k, v = golden[f"{case}/q"], golden[f"{case}/k"], golden[f"{case}/v"]
        row, z = int(golden[f"{case}/err_row"]), float(golden[f"{case}/err_z"])
        for tile in (at.TileConfig(1, 1), at.TileConfig(4, 2), at.TileConfig()):
            with pytest.raises(DegenerateDenominatorError, match=f"row {row}") as ei:
                at.streamed_attention_array(q, k, v, SPHERICAL, 1.0, tile)
            assert (np.isnan(z) and np.isnan(ei.value.z)) or ei.value.z == z


@pytest.mark.parametrize("compute", ["fp16", "bf16"])
def test_compat_grid_against_reference_golden(golden, compute):
    """The reference's oracle-equivalence grid (test_attention.py:127-145) and prime case,
    through the drop-in API, at the compute dtype's tolerance."""
    from paper_2505_09326_b200 import SPHERICAL
    at = compat()
    at.set_compute_dtype(compute)
    try:
        for c in [c for c in golden["__cases__"].tolist() if c.startswith(("grid", "prime97", "c1", "scale_eps"))]:
            q, k, v = golden[f"{c}/q"], golden[f"{c}/k"], golden[f"{c}/v"]
            s, e = float(golden[f"{c}/scale"]), float(golden[f"{c}/eps"])
            spec = SPHERICAL.with_epsilon(e)
            got = at.streamed_attention_array(q, k, v, spec, s, at.TileConfig(13, 7))
            assert got.dtype == q.dtype
            want = golden[f"{c}/out"]
            err = np.abs(got.astype(np.float64) - want)
            # inputs are rounded to the compute dtype: error ~ 2^-11 (fp16) / 2^-8 (bf16) of |O|
            lim = (8e-3 if compute == "fp16" else 5e-2) * max(1.0, float(np.abs(want).max()))
            assert err.max() <= lim, (c, float(err.max()))
    finally:
        at.set_compute_dtype("fp16")


def test_compat_gqa_mapping(golden):
    from paper_2505_09326_b200 import SPHERICAL
    at = compat()
    for c in ("gqa_4_2", "gqa_2_1", "gqa_8_2_f32"):
        q, k, v = golden[f"{c}/q"], golden[f"{c}/k"], golden[f"{c}/v"]
        h, hkv = int(golden[f"{c}/h"]), int(golden[f"{c}/h_kv"])
        got = at.multi_head_attention_array(q, k, v, SPHERICAL, h, hkv)
        assert got.shape == q.shape
        assert np.abs(got - golden[f"{c}/out"]).max() <= 8e-3 * max(1, np.abs(golden[f"{c}/out"]).max())
        nv = at.multi_head_attention_array(q, k, v, SPHERICAL, h, hkv, path="naive")
        np.testing.assert_allclose(nv, golden[f"{c}/out"], rtol=1e-5 if q.dtype == np.float32 else 1e-10,
                                   atol=1e-6 if q.dtype == np.float32 else 1e-12)


def test_compat_f16_mode_matches_f16_inputs(golden):
    """f16=True computes on binary16-rounded inputs: an off-grid input cannot change the
    result (test_attention.py:359-367), and accuracy meets test_attention.py:351-357."""
    from paper_2505_09326_b200 import SPHERICAL
    at = compat()
    q = np.array([[1.0002]], dtype=np.float32)
    k = np.array([[1.0]], dtype=np.float32)
    v = np.array([[4.0]], dtype=np.float32)
    got = at.streamed_attention_array(q, k, v, SPHERICAL, 1.0, at.TileConfig(1, 2), f16=True)
    exact = at.streamed_attention_array(np.ones((1, 1), np.float32), k, v, SPHERICAL, 1.0, at.TileConfig(1, 2),
                                        f16=True)
    assert np.array_equal(got, exact)
    q, k, v = golden["f16_64/q"], golden["f16_64/k"], golden["f16_64/v"]
    got = at.streamed_attention_array(q, k, v, SPHERICAL, 1.0, at.TileConfig(16, 16), f16=True)
    assert np.mean(np.abs(got - golden["f16_64/out"]) <= 0.01) >= 0.99


@pytest.mark.parametrize("compute,frac", [("fp16", 0.997), ("bf16", 0.99)])
def test_compat_criterion4_accuracy(golden, compute, frac):
    """Acceptance criterion 4 (test_acceptance.py:188-205; paper 99.7%)."""
    from paper_2505_09326_b200 import SPHERICAL
    at = compat()
    rng = np.random.default_rng(int(golden["crit4/seed"]))
    q = rng.standard_normal((1024, 128)).astype(np.float32)
    k = rng.standard_normal((1024, 128)).astype(np.float32)
    v = rng.standard_normal((1024, 128)).astype(np.float32)
    at.set_compute_dtype(compute)
    try:
        got = at.streamed_attention_array(q, k, v, SPHERICAL, 1.0, at.TileConfig(64, 64))
    finally:
        at.set_compute_dtype("fp16")
    within = float(np.mean(np.abs(got - golden["crit4/out"]) <= 0.01))
    assert within >= frac, within


def test_compat_meter_records_reference_tile_contract():
    # the reference's contract, min(g_y, y) * min(s_x, x) (test_attention.py:149-157; 1 for the
    # scalar 1x1 path, attention.py:217-218); the kernel's own on-chip tile is reported separately
    from paper_2505_09326_b200 import SPHERICAL, flashsign
    at = compat()
    rng = np.random.default_rng(7)
    for (y, x, g, s) in [(16, 16, 4, 4), (97, 33, 13, 7), (5, 400, 64, 64), (8, 8, 64, 64), (300, 300, 1, 1)]:
        m = at.ScoreBufferMeter()
        at.streamed_attention_array(rng.standard_normal((y, 64)), rng.standard_normal((x, 64)),
                                    rng.standard_normal((x, 64)), SPHERICAL, 1.0, at.TileConfig(g, s), meter=m)
        assert m.peak_elements == (1 if (g, s) == (1, 1) else min(g, y) * min(s, x))
    assert flashsign.kernel_score_tile(64, torch.bfloat16) == 128 * 192
    assert flashsign.kernel_score_tile(128, torch.bfloat16) == 128 * 128


def test_compat_empty_query_returns_empty():
    from paper_2505_09326_b200 import SPHERICAL
    at = compat()
    out = at.streamed_attention_array(np.ones((0, 8)), np.ones((3, 8)), np.ones((3, 8)), SPHERICAL, 1.0,
                                      at.TileConfig())
    assert out.shape == (0, 8)


def test_reference_streamed_oracle_agrees_at_c1(golden):
    """C1 (B1 H1 N256 d64 fp32): kernel (fp16 and bf16 compute) vs the reference's own output."""
    q, k, v = (torch.from_numpy(golden[f"c1/{x}"]).cuda()[None, :, None, :] for x in "qkv")
    for dt in (torch.float16, torch.bfloat16):
        o = fs().fwd(q.to(dt), k.to(dt), v.to(dt), out_dtype=torch.float32)[0, :, 0].cpu().numpy()
        # against the oracle on the same quantised inputs (dtype tolerance) ...
        ref_q = streamed_spherical(*(t.to(dt).float()[0, :, 0].cpu().numpy() for t in (q, k, v)))
        check_tol(o, ref_q, dt, "c1")
        # ... and against the reference's float32 output (adds input rounding)
        assert np.abs(o - golden["c1/out"]).max() < (1e-2 if dt == torch.float16 else 6e-2)


# ------------------------------------------------------------------ full-size configurations (sampled slices)

@pytest.mark.parametrize("cfg", [
    ("c2", 16, 16, 4096, 64, torch.float16),
    ("c3", 8, 16, 16384, 128, torch.bfloat16),
    ("c4", 8, 16, 8192, 128, torch.float8_e4m3fn),
    ("c5", 64, 8, 20000, 64, torch.bfloat16),
], ids=lambda c: c[0])
def test_full_size_config_against_gram_oracle(cfg):
    """BASELINE.json configurations at full N: the kernel runs the whole (reduced-batch)
    problem and every output of a few (b, h) slices is checked against the float64
    Gram-form oracle (exact identity, O(N d^2))."""
    name, B, H, N, D, dt = cfg
    Bs = 2  # two batch rows of the real sequence length and head count
    q = rand_bshd(Bs, N, H, D, dt, 100)
    k = rand_bshd(Bs, N, H, D, dt, 101)
    v = rand_bshd(Bs, N, H, D, dt, 102)
    eps = 1e-6 if name == "c5" else 0.0
    o = fs().fwd(q, k, v, eps=eps)
    for b, h in [(0, 0), (1, H - 1), (1, H // 2)]:
        ref = gram_spherical(q[b, :, h].float().cpu().numpy(), k[b, :, h].float().cpu().numpy(),
                             v[b, :, h].float().cpu().numpy(), 1.0, eps)
        check_tol(o[b, :, h].float().cpu().numpy(), ref, dt, f"{name} b{b} h{h}")


@pytest.mark.parametrize("name,fused", [("c2", False), ("c3", False), ("c4", False), ("c5", False), ("c5", True)],
                         ids=["c2", "c3", "c4", "c5-prescaled", "c5-key_scale"])
def test_full_size_as_benchmarked(name, fused):
    """The configurations exactly as bench.py runs them: full batch, full N, the bench's own
    inputs (bench.make_inputs, seeded per unit), C5 with its multiplicities m in {0..5} and
    eps = 1e-6 -- pre-scaled K' = m K (the default bench line) and fused in-kernel (key_scale,
    --fused-mult).  Slices from the first, middle and LAST batch rows are checked in float64."""
    import bench
    cfg = dict(bench.CONFIGS[name])
    if fused:
        cfg["fused_mult"] = True
    B, H, N, D = cfg["B"], cfg["H"], cfg["N"], cfg["D"]
    q, k, v, m, _ = bench.make_inputs(cfg, 0, B * cfg["HKV"], torch.device("cuda"))
    dt = q.dtype
    o = fs().fwd(q, k, v, eps=cfg["eps"], key_scale=m)
    for b, h in [(0, 0), (B // 2, H // 2), (B - 1, H - 1), (B - 1, 0)]:
        kb = k[b, :, h].float().cpu().numpy().astype(np.float64)
        if m is not None:
            kb = kb * m[b].cpu().numpy().astype(np.float64)[:, None]
        ref = gram_spherical(q[b, :, h].float().cpu().numpy(), kb, v[b, :, h].float().cpu().numpy(), 1.0, cfg["eps"])
        check_tol(o[b, :, h].float().cpu().numpy(), ref, dt, f"{name} b{b} h{h}")
    del q, k, v, o
    torch.cuda.empty_cache()


def test_host_pipeline_equals_device_path():
    from paper_2505_09326_b200.pipeline import HostPipeline
    q = rand_bshd(5, 700, 4, 128, torch.bfloat16, 50)
    k = rand_bshd(5, 900, 2, 128, torch.bfloat16, 51)
    v = rand_bshd(5, 900, 2, 128, torch.bfloat16, 52)
    ref = fs().fwd(q, k, v)
    qh, kh, vh = (t.cpu().pin_memory() for t in (q, k, v))
    oh = torch.empty(q.shape, dtype=torch.bfloat16, pin_memory=True)
    for chunk, qs in ((1, None), (2, None), (1, 3), (2, 2), (None, None), (4, 2)):
        oh.zero_()
        HostPipeline(0, chunk=chunk, q_split=qs).run(qh, kh, vh, oh)
        # chunks are separate launches whose automatic K/V split plans differ from the whole call's
        # (fp32 summation order of the split partials): equal up to one bf16 rounding step
        r = ref.cpu().float()
        assert bool(((oh.float() - r).abs() <= 2.0 ** -7 * r.abs() + 1e-6).all()), (chunk, qs)
    # the first degenerate row in (batch, head, row) order, across batch chunks and query slices
    from paper_2505_09326_b200.normalizers import DegenerateDenominatorError
    qh[3, 650, 1] = 0
    qh[3, 20, 3] = 0
    qh[4, 5, 0] = 0
    with pytest.raises(DegenerateDenominatorError, match="row 650"):
        HostPipeline(0, chunk=1, q_split=3).run(qh, kh, vh, oh)


def test_host_pipeline_with_multiplicities_and_fp8():
    from paper_2505_09326_b200.pipeline import HostPipeline
    q = rand_bshd(3, 600, 4, 64, torch.float16, 53)
    k = rand_bshd(3, 500, 2, 64, torch.float16, 54)
    v = rand_bshd(3, 500, 2, 64, torch.float16, 55)
    g = torch.Generator(device="cuda").manual_seed(56)
    m = torch.randint(0, 6, (3, 500), generator=g, device="cuda").float()
    ref = fs().fwd(q, k, v, eps=1e-6, key_scale=m)
    qh, kh, vh, mh = (t.cpu().pin_memory() for t in (q, k, v, m))
    oh = torch.empty(q.shape, dtype=torch.float16, pin_memory=True)
    for chunk, qs in ((1, None), (2, 2)):
        HostPipeline(0, chunk=chunk, q_split=qs).run(qh, kh, vh, oh, eps=1e-6, key_scale=mh)
        assert torch.equal(oh, ref.cpu()), (chunk, qs)
    # e4m3 inputs, bf16 output
    q8, k8, v8 = (t.to(torch.float8_e4m3fn) for t in (q, k, v))
    ref8 = fs().fwd(q8, k8, v8, out_dtype=torch.bfloat16)
    o8 = torch.empty(q.shape, dtype=torch.bfloat16, pin_memory=True)
    HostPipeline(0).run(q8.cpu().pin_memory(), k8.cpu().pin_memory(), v8.cpu().pin_memory(), o8)
    assert torch.equal(o8, ref8.cpu())


# ------------------------------------------------------------------ SIGNED_L1 and fused key multiplicities

# signed_l1 outputs are weighted means (weights |s|/sum|s|), so they are O(1/sqrt(N)) and the
# tolerance is relative: rel-Frobenius and max-abs relative to max|O_ref|.
TOL_REL = {torch.float16: 3e-3, torch.bfloat16: 1.5e-2, torch.float8_e4m3fn: 8e-2}


def check_rel(got, ref, dtype, tag=""):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert np.isfinite(got).all(), f"{tag}: non-finite output"
    rel_fro = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))
    rel_max = float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))
    assert rel_fro <= TOL_REL[dtype] and rel_max <= 4 * TOL_REL[dtype], f"{tag}: rel_fro={rel_fro} rel_max={rel_max}"
    return rel_fro


def exact_of(q, k, v, scale=1.0, eps=0.0, norm="spherical", m=None):
    from oracle.spherical import exact_batched
    return exact_batched(q.float().cpu().numpy(), k.float().cpu().numpy(), v.float().cpu().numpy(), scale, eps,
                         norm, None if m is None else m.double().cpu().numpy())


@pytest.mark.parametrize("dt", [torch.float16, torch.bfloat16, torch.float8_e4m3fn])
@pytest.mark.parametrize("shape", [(2, 300, 517, 4, 2, 128), (1, 129, 255, 2, 2, 64), (1, 256, 256, 1, 1, 64)])
def test_signed_l1_matches_oracle(dt, shape):
    b, nq, nkv, h, hkv, d = shape
    if dt == torch.float8_e4m3fn and d != 128:
        d = 128
    q = rand_bshd(b, nq, h, d, dt, 50)
    k = rand_bshd(b, nkv, hkv, d, dt, 51)
    v = rand_bshd(b, nkv, hkv, d, dt, 52)
    for scale, eps in ((1.0, 0.0), (-0.7, 1e-3)):
        o = fs().fwd(q, k, v, scale=scale, eps=eps, out_dtype=torch.float32, normalizer="signed_l1")
        check_rel(o.cpu().numpy(), exact_of(q, k, v, scale, eps, "signed_l1"), dt, f"l1 {shape} {dt} {scale}")


def test_signed_l1_kat_and_degenerate_row():
    # (3*10 + 4*20) / (3 + 4): exact inputs, fp32 output within one rounding of 110/7
    q = torch.zeros((1, 1, 1, 64), device="cuda", dtype=torch.bfloat16)
    k = torch.zeros((1, 2, 1, 64), device="cuda", dtype=torch.bfloat16)
    v = torch.zeros((1, 2, 1, 64), device="cuda", dtype=torch.bfloat16)
    q[0, 0, 0, 0] = 1
    k[0, 0, 0, 0], k[0, 1, 0, 0] = 3, 4
    v[0, 0, 0, 0], v[0, 1, 0, 0] = 10, 20
    o = fs().fwd(q, k, v, out_dtype=torch.float32, normalizer="signed_l1")
    assert abs(float(o[0, 0, 0, 0]) - 110.0 / 7.0) <= 2e-6
    q2 = rand_bshd(1, 50, 2, 64, torch.bfloat16, 53)
    k2 = rand_bshd(1, 60, 2, 64, torch.bfloat16, 54)
    q2[0, 17, 1] = 0
    _, bad = fs().fwd_async(q2, k2, k2, normalizer="signed_l1")
    assert fs().decode_bad_key(int(bad.item()), 2, 50) == (0, 1, 17, 0.0)


def test_unknown_normalizer_rejected():
    from paper_2505_09326_b200._errors import ConfigError
    q = rand_bshd(1, 8, 1, 64, torch.bfloat16, 55)
    with pytest.raises(ConfigError, match="normalizer"):
        fs().fwd(q, q, q, normalizer="softmax")


@pytest.mark.parametrize("norm", ["spherical", "signed_l1"])
@pytest.mark.parametrize("dt", [torch.float16, torch.bfloat16, torch.float8_e4m3fn])
def test_key_scale_matches_oracle(norm, dt):
    # fused K' = m K (attention.py:381-388, grn.py:150): integer multiplicities 0..5 as in the GRN demo
    b, nq, nkv, h, hkv, d = 2, 300, 517, 4, 2, (128 if dt == torch.float8_e4m3fn else 64)
    q = rand_bshd(b, nq, h, d, dt, 60)
    k = rand_bshd(b, nkv, hkv, d, dt, 61)
    v = rand_bshd(b, nkv, hkv, d, dt, 62)
    g = torch.Generator(device="cuda").manual_seed(63)
    m = torch.randint(0, 6, (b, nkv), generator=g, device="cuda").float()
    o = fs().fwd(q, k, v, eps=1e-6, out_dtype=torch.float32, normalizer=norm, key_scale=m)
    ref = exact_of(q, k, v, 1.0, 1e-6, norm, m)
    if norm == "spherical":
        check_tol(o.cpu().numpy(), ref, dt, f"ks {norm} {dt}")
    else:
        check_rel(o.cpu().numpy(), ref, dt, f"ks {norm} {dt}")


def test_key_scale_power_of_two_is_bitwise_prescaled_keys():
    # m_j * (q . k_j) in fp32 == q . (m_j k_j) when m_j is a power of two (both exact)
    q = rand_bshd(2, 200, 2, 128, torch.bfloat16, 64)
    k = rand_bshd(2, 333, 2, 128, torch.bfloat16, 65)
    v = rand_bshd(2, 333, 2, 128, torch.bfloat16, 66)
    g = torch.Generator(device="cuda").manual_seed(67)
    m = torch.tensor([0.0, 0.5, 1.0, 2.0, 4.0], device="cuda")[torch.randint(0, 5, (2, 333), generator=g,
                                                                            device="cuda")]
    fused = fs().fwd(q, k, v, eps=1e-6, out_dtype=torch.float32, key_scale=m)
    pre = fs().fwd(q, (k.float() * m[:, :, None, None]).to(k.dtype), v, eps=1e-6, out_dtype=torch.float32)
    assert torch.equal(fused, pre)
    # a strided / unaligned multiplicity view is repacked, same result
    big = torch.zeros((2, 340), device="cuda")
    big[:, 1:334] = m
    assert torch.equal(fs().fwd(q, k, v, eps=1e-6, out_dtype=torch.float32, key_scale=big[:, 1:334]), fused)


@pytest.mark.parametrize("dt,d", [(torch.bfloat16, 64), (torch.bfloat16, 128), (torch.float16, 64),
                                  (torch.float16, 128)])
def test_key_scale_integer_is_bitwise_prescaled_keys(dt, d):
    # 16-bit inputs: the kernel forms K' = m K in shared memory with one rounding (packed HMUL2) --
    # bit for bit what pre-scaling K in fp32 / float64 and casting gives, for integer m (GRN counts,
    # grn.py:150) and for the fp32 fallback path (non-representable m); several work tiles per CTA
    # so ring slots are reused
    g = torch.Generator(device="cuda").manual_seed(69)
    q = rand_bshd(3, 700, 4, d, dt, 70)
    k = rand_bshd(3, 2500, 2, d, dt, 71)
    v = rand_bshd(3, 2500, 2, d, dt, 72)
    for vals in ([0.0, 1.0, 2.0, 3.0, 4.0, 5.0], [0.3, 1.7, 2.9]):
        m = torch.tensor(vals, device="cuda")[torch.randint(0, len(vals), (3, 2500), generator=g, device="cuda")]
        fused = fs().fwd(q, k, v, eps=1e-6, out_dtype=torch.float32, key_scale=m)
        pre = fs().fwd(q, (k.float() * m[:, :, None, None]).to(dt), v, eps=1e-6, out_dtype=torch.float32)
        assert torch.equal(fused, pre), vals


def _abi_fwd(q, k, v, out, key_scale=None, eps=0.0):
    # fs_fwd called directly through the C-ABI (no torch extension): the in-kernel key_scale path
    import ctypes
    from paper_2505_09326_b200 import _lib
    codes = {torch.bfloat16: _lib.FS_BF16, torch.float16: _lib.FS_F16, torch.float32: _lib.FS_F32}
    p = _lib.FsFwdParams()
    p.q, p.k, p.v, p.o = q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr()
    for dst, t in ((p.q_stride, q), (p.k_stride, k), (p.v_stride, v), (p.o_stride, out)):
        dst[0], dst[1], dst[2] = t.stride(0), t.stride(1), t.stride(2)
    p.batch, p.heads_q, p.heads_kv, p.seqlen_q, p.seqlen_kv, p.head_dim = (q.shape[0], q.shape[2], k.shape[2],
                                                                        q.shape[1], k.shape[1], q.shape[3])
    p.in_dtype, p.out_dtype = codes[q.dtype], codes[out.dtype]
    p.scale, p.eps, p.p_scale, p.q_descale, p.k_descale, p.v_descale = 1.0, eps, 1.0, 1.0, 1.0, 1.0
    p.kv_splits = 1
    if key_scale is not None:
        p.key_scale, p.key_scale_stride = key_scale.data_ptr(), key_scale.stride(0)
    st = _lib.load().fs_fwd(ctypes.byref(p), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert st == _lib.FS_OK, _lib.last_error()
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("dt,d", [(torch.bfloat16, 64), (torch.float16, 128)])
def test_key_scale_in_kernel_abi_path(dt, d):
    # C-ABI callers passing key_scale get the in-kernel per-score multiply (fp32 m_j s_ij); the torch
    # entry forms K' = m K first (fs_scale_keys).  Both match the oracle and each other closely.
    g = torch.Generator(device="cuda").manual_seed(73)
    q = rand_bshd(2, 400, 4, d, dt, 74)
    k = rand_bshd(2, 900, 2, d, dt, 75)
    v = rand_bshd(2, 900, 2, d, dt, 76)
    m = torch.randint(0, 6, (2, 900), generator=g, device="cuda").float()
    o_abi = _abi_fwd(q, k, v, torch.empty(q.shape, dtype=torch.float32, device="cuda"), m, 1e-6)
    check_tol(o_abi.cpu().numpy(), exact_of(q, k, v, 1.0, 1e-6, "spherical", m), dt, "abi key_scale")
    o_torch = fs().fwd(q, k, v, eps=1e-6, out_dtype=torch.float32, key_scale=m)
    assert float((o_abi - o_torch).abs().max()) <= 2e-2


def test_scale_keys_pass_matches_torch():
    # fs_scale_keys on a strided BSHD view: RNE(m * k) per element
    import ctypes
    from paper_2505_09326_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(77)
    for dt in (torch.bfloat16, torch.float16):
        kb = rand_bshd(3, 333, 6, 64, dt, 78)
        k = kb[:, :, 1:5]                      # strided heads
        m = torch.rand((3, 336), generator=g, device="cuda")[:, :333] * 7
        out = torch.empty((3, 333, 4, 64), dtype=dt, device="cuda")
        p = _lib.FsFwdParams()
        p.k, p.batch, p.seqlen_kv, p.heads_kv, p.head_dim = k.data_ptr(), 3, 333, 4, 64
        p.k_stride[0], p.k_stride[1], p.k_stride[2] = k.stride(0), k.stride(1), k.stride(2)
        p.in_dtype = _lib.FS_BF16 if dt == torch.bfloat16 else _lib.FS_F16
        p.key_scale, p.key_scale_stride = m.data_ptr(), m.stride(0)
        ost = (ctypes.c_int64 * 3)(out.stride(0), out.stride(1), out.stride(2))
        st = _lib.load().fs_scale_keys(ctypes.byref(p), ctypes.c_void_p(out.data_ptr()), ost,
                                       ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert st == _lib.FS_OK, _lib.last_error()
        torch.cuda.synchronize()
        assert torch.equal(out, (k.float() * m[:, :, None, None]).to(dt))


def test_key_scale_validation():
    q = rand_bshd(1, 8, 1, 64, torch.bfloat16, 68)
    from paper_2505_09326_b200.tensor import ShapeMismatchError
    with pytest.raises(ValueError, match="finite and nonnegative"):
        fs().fwd(q, q, q, key_scale=torch.tensor([[1.0, -1.0] + [1.0] * 6], device="cuda"))
    with pytest.raises(ShapeMismatchError, match="key_scale"):
        fs().fwd(q, q, q, key_scale=torch.ones((1, 7), device="cuda"))


@pytest.mark.parametrize("compute", ["fp16", "bf16"])
def test_compat_signed_l1_against_reference_golden(golden, compute):
    from paper_2505_09326_b200 import SIGNED_L1
    at = compat()
    at.set_compute_dtype(compute)
    tdt = torch.float16 if compute == "fp16" else torch.bfloat16
    try:
        for c in [c for c in golden["__cases__"].tolist() if c.startswith(("l1_grid", "l1_scale_eps", "l1_kat"))]:
            q, k, v = golden[f"{c}/q"], golden[f"{c}/k"], golden[f"{c}/v"]
            s, e = float(golden[f"{c}/scale"]), float(golden[f"{c}/eps"])
            got = at.streamed_attention_array(q, k, v, SIGNED_L1.with_epsilon(e), s, at.TileConfig(13, 7))
            assert got.dtype == q.dtype
            check_rel(got, golden[f"{c}/out"], tdt, c)
        c = "l1_gqa_4_2_f32"
        got = at.multi_head_attention_array(golden[f"{c}/q"], golden[f"{c}/k"], golden[f"{c}/v"], SIGNED_L1, 4, 2)
        check_rel(got, golden[f"{c}/out"], tdt, c)
        with pytest.raises(__import__("paper_2505_09326_b200").DegenerateDenominatorError, match="row 1"):
            at.streamed_attention_array(golden["l1_degen_row1/q"], golden["l1_degen_row1/k"],
                                        golden["l1_degen_row1/v"], SIGNED_L1, 1.0, at.TileConfig())
    finally:
        at.set_compute_dtype("fp16")


@pytest.mark.parametrize("tag", ["sph", "l1"])
def test_compat_fused_multiplicity_against_reference_golden(golden, tag):
    # the GRN caller's multi_head_attention_array(q, apply_multiplicity_array(k, m), v, ...) in one launch
    from paper_2505_09326_b200 import SIGNED_L1, SPHERICAL
    at = compat()
    c = f"mult_{tag}_gqa_f32"
    spec = (SPHERICAL if tag == "sph" else SIGNED_L1).with_epsilon(float(golden[f"{c}/eps"]))
    got = at.multiplicity_attention_array(golden[f"{c}/q"], golden[f"{c}/k"], golden[f"{c}/v"], golden[f"{c}/m"],
                                          spec, 4, 2, scale=1.0)
    want = golden[f"{c}/out"]
    if tag == "sph":
        assert np.abs(got.astype(np.float64) - want).max() <= 8e-3 * max(1.0, float(np.abs(want).max()))
    else:
        check_rel(got, want, torch.float16, c)


# ------------------------------------------------------------------ split K/V and context parallelism

@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16, torch.float8_e4m3fn])
@pytest.mark.parametrize("splits", [2, 3, 7])
def test_kv_splits_match_oracle(dt, splits):
    d = 128 if dt == torch.float8_e4m3fn else 64
    q = rand_bshd(1, 300, 2, d, dt, 70)
    k = rand_bshd(1, 1000, 1, d, dt, 71)
    v = rand_bshd(1, 1000, 1, d, dt, 72)
    o1 = fs().fwd(q, k, v, eps=1e-6, out_dtype=torch.float32, kv_splits=1)
    os_ = fs().fwd(q, k, v, eps=1e-6, out_dtype=torch.float32, kv_splits=splits)
    ref = oracle_of(q, k, v, 1.0, 1e-6)
    check_tol(os_.cpu().numpy(), ref, dt, f"splits={splits}")
    # only the summation order of the split partials differs from the single pass
    assert float((os_ - o1).abs().max()) <= 2e-5 * max(1.0, float(o1.abs().max()))


def test_kv_splits_signed_l1_and_degenerate_rows():
    q = rand_bshd(2, 200, 2, 128, torch.bfloat16, 73)
    k = rand_bshd(2, 900, 2, 128, torch.bfloat16, 74)
    v = rand_bshd(2, 900, 2, 128, torch.bfloat16, 75)
    o = fs().fwd(q, k, v, out_dtype=torch.float32, normalizer="signed_l1", kv_splits=4)
    check_rel(o.cpu().numpy(), exact_of(q, k, v, 1.0, 0.0, "signed_l1"), torch.bfloat16, "l1 split")
    q[1, 33, 0] = 0  # batch 1 head 0 row 33 -> z = 0 after the merge
    q[1, 150, 1] = 0
    _, bad = fs().fwd_async(q, k, v, kv_splits=4)
    assert fs().decode_bad_key(int(bad.item()), 2, 200) == (1, 0, 33, 0.0)


def test_auto_splits_small_batch_long_sequence():
    # B*H*ceil(N/256) = 16 work tiles < 148 SMs -> the launch is split automatically
    q = rand_bshd(1, 1024, 4, 128, torch.bfloat16, 76)
    k = rand_bshd(1, 16384, 4, 128, torch.bfloat16, 77)
    v = rand_bshd(1, 16384, 4, 128, torch.bfloat16, 78)
    assert fs().auto_splits(1, 4, 1024, 16384, q.device) > 1
    o = fs().fwd(q, k, v, out_dtype=torch.float32)
    check_tol(o.cpu().numpy(), oracle_of(q, k, v), torch.bfloat16, "auto split")


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16, torch.float8_e4m3fn])
@pytest.mark.parametrize("shape,splits", [((1, 600, 2000, 80, 80), 2),    # 160 tiles: whole waves + a tail
                                          ((1, 600, 2000, 80, 40), 5),    # GQA, ragged query blocks
                                          ((2, 700, 1500, 3, 1), 3)])     # 12 tiles < one wave: all tail
def test_tail_splits_match_oracle(dt, shape, splits):
    # split_tail: only the last partial wave's work tiles are cut into K/V ranges; their partials are
    # merged by the combine kernel, the whole-wave tiles write O directly
    b, nq, nkv, h, hkv = shape
    d = 128 if dt == torch.float8_e4m3fn else 64
    q = rand_bshd(b, nq, h, d, dt, 90)
    k = rand_bshd(b, nkv, hkv, d, dt, 91)
    v = rand_bshd(b, nkv, hkv, d, dt, 92)
    pl = fs().plan(b, h, nq, nkv, q.device, d, dt, kv_splits=splits, split_tail=True)
    o1 = fs().fwd(q, k, v, eps=1e-6, out_dtype=torch.float32, kv_splits=1)
    ot = fs().fwd(q, k, v, eps=1e-6, out_dtype=torch.float32, kv_splits=splits, split_tail=True)
    check_tol(ot.cpu().numpy(), oracle_of(q, k, v, 1.0, 1e-6), dt, f"tail splits={splits}")
    assert float((ot - o1).abs().max()) <= 2e-5 * max(1.0, float(o1.abs().max()))
    # rows of the whole-wave tiles come from the unsplit path: bitwise equal to the single pass
    tiles_per_bh = -(-nq // 512)
    for u in range(min(pl.n_whole, b * h * tiles_per_bh)):
        bh, qc = divmod(u, tiles_per_bh)
        bb, hh = divmod(bh, h)
        rows = slice(qc * 512, min(nq, qc * 512 + 512))
        assert torch.equal(ot[bb, rows, hh], o1[bb, rows, hh]), u


def test_tail_splits_degenerate_rows_and_auto_plan():
    # a zero query row inside a tail tile and one inside a whole-wave tile: the first in the
    # reference's (batch, head, row) order is reported, from either path
    b, nq, nkv, h, d = 1, 1024, 4096, 80, 128
    q = rand_bshd(b, nq, h, d, torch.bfloat16, 93)
    k = rand_bshd(b, nkv, h, d, torch.bfloat16, 94)
    v = rand_bshd(b, nkv, h, d, torch.bfloat16, 95)
    pl = fs().plan(b, h, nq, nkv, q.device, d)
    assert pl.split_tail == 1 and pl.splits > 1, (pl.splits, pl.split_tail, pl.clusters)
    assert pl.efficiency > fs().plan(b, h, nq, nkv, q.device, d, kv_splits=1).efficiency
    o = fs().fwd(q, k, v, out_dtype=torch.float32)  # automatic plan: tail split
    check_tol(o.cpu().numpy(), oracle_of(q, k, v), torch.bfloat16, "auto tail split")
    q[0, 700, h - 1] = 0      # last head: a tail tile
    _, bad = fs().fwd_async(q, k, v)
    assert fs().decode_bad_key(int(bad.item()), h, nq) == (0, h - 1, 700, 0.0)
    q[0, 5, 3] = 0            # head 3: a whole-wave tile, earlier in loop order
    _, bad = fs().fwd_async(q, k, v)
    assert fs().decode_bad_key(int(bad.item()), h, nq) == (0, 3, 5, 0.0)
    with pytest.raises(Exception, match="row 5"):
        fs().fwd(q, k, v)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_context_parallel_emulated_on_one_gpu(world):
    # the all_reduce(SUM) of the per-shard partial workspaces, done here by adding them
    from paper_2505_09326_b200 import partition
    q = rand_bshd(2, 257, 4, 128, torch.bfloat16, 79)
    k = rand_bshd(2, 2000, 2, 128, torch.bfloat16, 80)
    v = rand_bshd(2, 2000, 2, 128, torch.bfloat16, 81)
    total, n_parts = None, None
    for r in range(world):
        lo, hi = partition.kv_shard_range(k.shape[1], world, r)
        part, n = fs().fwd_partial(q, k[:, lo:hi], v[:, lo:hi], eps=1e-6)
        total = part.clone() if total is None else total + part
        assert n_parts in (None, n)
        n_parts = n
    o = fs().combine(total, n_parts, q, eps=1e-6, out_dtype=torch.float32)
    check_tol(o.cpu().numpy(), oracle_of(q, k, v, 1.0, 1e-6), torch.bfloat16, f"cp world={world}")
    full = fs().fwd(q, k, v, eps=1e-6, out_dtype=torch.float32)
    assert float((o - full).abs().max()) <= 2e-5 * max(1.0, float(full.abs().max()))
    # single process: context_parallel_fwd without a process group is the plain partial + combine
    o2 = partition.context_parallel_fwd(q, k, v, eps=1e-6, out_dtype=torch.float32)
    assert float((o2 - full).abs().max()) <= 2e-5 * max(1.0, float(full.abs().max()))


def test_combine_validates_workspace_and_output():
    from paper_2505_09326_b200.tensor import ShapeMismatchError
    q = rand_bshd(1, 300, 2, 64, torch.float16, 85)
    k = rand_bshd(1, 600, 2, 64, torch.float16, 86)
    part, n = fs().fwd_partial(q, k, k)
    with pytest.raises(ShapeMismatchError, match="partial"):
        fs().combine(part[:-1], n, q)
    with pytest.raises(ShapeMismatchError, match="partial"):
        fs().combine(part, n + 1, q)
    with pytest.raises(ShapeMismatchError, match="out tensor"):
        fs().combine(part, n, q, out=torch.empty((1, 299, 2, 64), dtype=torch.float16, device="cuda"))
    o = fs().combine(part, n, q)
    assert torch.equal(o, fs().fwd(q, k, k, kv_splits=1))


def test_cuda_graph_capture_and_replay():
    # fs_fwd is capturable (memset node + kernel node); replays see new input data
    q = rand_bshd(2, 300, 4, 128, torch.bfloat16, 90)
    k = rand_bshd(2, 517, 2, 128, torch.bfloat16, 91)
    v = rand_bshd(2, 517, 2, 128, torch.bfloat16, 92)
    cap = fs().CapturedFwd(q, k, v, out_dtype=torch.float32)
    o1 = cap.replay().clone()
    assert torch.equal(o1, fs().fwd(q, k, v, out_dtype=torch.float32))
    q.copy_(rand_bshd(2, 300, 4, 128, torch.bfloat16, 93))
    o2 = cap.replay().clone()
    assert torch.equal(o2, fs().fwd(q, k, v, out_dtype=torch.float32))
    assert not torch.equal(o1, o2)
    torch.cuda.synchronize()
    assert fs().decode_bad_key(int(cap.bad_key.item()), 4, 300) is None


# ------------------------------------------------------------------ per-tensor scales (FP8 quantisation recipe)

def test_fp8_descales_and_p_scale():
    # real q, k, v stored as e4m3 codes x / s with per-tensor descales s; P = p_scale * s_ij before
    # the PV MMA (kept inside the e4m3 range), output divided by p_scale again (include/flashsign.h)
    g = torch.Generator(device="cuda").manual_seed(94)
    q, k, v = (torch.randn((2, 300, 2, 128), generator=g, device="cuda") for _ in range(3))
    sq, sk, sv, ps = 0.25, 0.25, 0.5, 0.2
    q8, k8, v8 = ((t / s).to(torch.float8_e4m3fn) for t, s in ((q, sq), (k, sk), (v, sv)))
    o = fs().fwd(q8, k8, v8, q_descale=sq, k_descale=sk, v_descale=sv, p_scale=ps, out_dtype=torch.float32)
    deq = [t.float() * s for t, s in ((q8, sq), (k8, sk), (v8, sv))]
    check_tol(o.cpu().numpy(), oracle_of(*deq), torch.float8_e4m3fn, "fp8 descales")
    # same P range without p_scale saturates e4m3 (|q8 . k8| > 448): reported as z = +inf
    _, bad = fs().fwd_async(q8, k8, v8, q_descale=sq, k_descale=sk, v_descale=sv, p_scale=1.0)
    info = fs().decode_bad_key(int(bad.item()), 2, 300)
    assert info is not None and np.isinf(info[3])


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16])
def test_16bit_descales_and_p_scale(dt):
    q = rand_bshd(1, 256, 2, 64, dt, 95)
    k = rand_bshd(1, 300, 2, 64, dt, 96)
    v = rand_bshd(1, 300, 2, 64, dt, 97)
    o = fs().fwd(q, k, v, scale=0.5, q_descale=2.0, k_descale=0.5, v_descale=4.0, p_scale=0.25,
                 out_dtype=torch.float32)
    ref = oracle_of(q.float() * 2.0, k.float() * 0.5, v.float() * 4.0, 0.5)
    check_tol(o.cpu().numpy() / 4.0, ref / 4.0, dt, f"{dt} descales")


# ------------------------------------------------------------------ randomized sweep over the feature matrix

def _sweep_cases(n=None, seed=None):
    # FS_SWEEP_N / FS_SWEEP_SEED widen the sweep for stress runs (default: 48 cases, seed 2024)
    n = int(os.environ.get("FS_SWEEP_N", 48)) if n is None else n
    seed = int(os.environ.get("FS_SWEEP_SEED", 2024)) if seed is None else seed
    wide = os.environ.get("FS_SWEEP_WIDE", "0") == "1"  # stress runs: all widths, longer sequences
    rng = np.random.default_rng(seed)
    dts = [torch.bfloat16, torch.float16, torch.float8_e4m3fn]
    out = []
    for i in range(n):
        dt = dts[i % 3]
        if wide:  # every width the C-ABI takes (16-byte rows: d % 8 == 0, d % 16 == 0 for e4m3)
            d = int(rng.choice(list(range(16 if dt == torch.float8_e4m3fn else 8, 129,
                                          16 if dt == torch.float8_e4m3fn else 8))))
        else:
            d = int(rng.choice([16, 32, 48, 64, 80, 96, 112, 128] if dt != torch.float8_e4m3fn else [16, 32, 64, 96, 128]))
        hkv = int(rng.choice([1, 2, 3, 8]))
        h = hkv * int(rng.choice([1, 2, 4]))
        out.append(dict(dt=dt, b=int(rng.integers(1, 4)), nq=int(rng.integers(1, 3000 if wide else 700)),
                        nkv=int(rng.integers(1, 4000 if wide else 900)),
                        h=h, hkv=hkv, d=d, norm=str(rng.choice(["spherical", "signed_l1"])),
                        ks=bool(rng.integers(0, 2)), splits=int(rng.choice([1, 1, 2, 3])),
                        scale=float(rng.choice([1.0, -0.5, 2.0])), eps=float(rng.choice([0.0, 1e-3])),
                        out=[torch.float32, torch.bfloat16][int(rng.integers(0, 2))], seed=int(rng.integers(1 << 30)),
                        tail=bool(rng.integers(0, 2))))
    return out


@pytest.mark.parametrize("case", _sweep_cases(), ids=lambda c: f"{str(c['dt'])[6:]}-d{c['d']}-n{c['nq']}x{c['nkv']}-"
                                                                f"h{c['h']}/{c['hkv']}-{c['norm']}-ks{int(c['ks'])}-s{c['splits']}{'t' if c['tail'] else ''}")
def test_random_feature_sweep(case):
    c = case
    g = torch.Generator(device="cuda").manual_seed(c["seed"])
    q = torch.randn((c["b"], c["nq"], c["h"], c["d"]), generator=g, device="cuda").to(c["dt"])
    k = torch.randn((c["b"], c["nkv"], c["hkv"], c["d"]), generator=g, device="cuda").to(c["dt"])
    v = torch.randn((c["b"], c["nkv"], c["hkv"], c["d"]), generator=g, device="cuda").to(c["dt"])
    m = torch.randint(0, 4, (c["b"], c["nkv"]), generator=g, device="cuda").float() if c["ks"] else None
    eps = c["eps"] if not c["ks"] else max(c["eps"], 1e-3)  # zero multiplicities can empty a row
    # (split_tail: only the last partial wave's work tiles take the K/V split; with few tiles every
    # tile is a tail tile, with > 74 cluster tiles whole-wave and tail tiles mix)
    o = fs().fwd(q, k, v, scale=c["scale"], eps=eps, out_dtype=c["out"], normalizer=c["norm"], key_scale=m,
                 kv_splits=c["splits"], split_tail=c.get("tail", False), check=False)
    if m is not None and c["dt"] != torch.float8_e4m3fn:
        # 16-bit keys: the kernel's operand is K' = rn(m K) in the input dtype (fs_scale_keys), one
        # rounding of the scaled key as in the reference's own f16 mode (grn.py:150 then
        # attention.py:268-270); the oracle takes that K', since rows whose scores cancel (|s| <<
        # |q||k'|) amplify the rounding (FS_SWEEP_WIDE seed 777: s = -0.05 against |q||k'| = 48)
        ref = exact_of(q, (k.float() * m[:, :, None, None]).to(c["dt"]), v, c["scale"], eps, c["norm"], None)
    else:
        ref = exact_of(q, k, v, c["scale"], eps, c["norm"], m)
    got = o.float().cpu().numpy()
    finite = np.isfinite(ref).all(axis=-1)
    assert finite.mean() > 0.5
    got, ref = got[finite], ref[finite]
    err = np.abs(got - ref)
    scale_ref = np.abs(ref).max()
    # per-dtype tolerance relative to the output scale (the input dtype's rounding dominates)
    tol = {torch.float16: 0.01, torch.bfloat16: 0.05, torch.float8_e4m3fn: 0.35}[c["dt"]]
    if c["out"] == torch.bfloat16:
        tol = max(tol, 0.02)
    assert err.max() <= tol * max(scale_ref, 1e-3) + 1e-6, (c, float(err.max()), float(scale_ref))
    rel = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
    assert rel <= {torch.float16: 4e-3, torch.bfloat16: 1.5e-2, torch.float8_e4m3fn: 8e-2}[c["dt"]], (c, rel)


# ------------------------------------------------------------------ maximum extents

@pytest.mark.parametrize("b,h,n,d,dt", [
    (65535, 1, 3, 16, torch.bfloat16),    # largest batch the C-ABI accepts: 65535 work tiles
    (1, 65535, 3, 16, torch.float16),     # largest head count (GQA 65535 -> 5 kv heads)
])
def test_maximum_batch_and_heads(b, h, n, d, dt):
    hkv = 5 if h > 1 else 1
    q = rand_bshd(b, n, h, d, dt, 120)
    k = rand_bshd(b, n + 2, hkv, d, dt, 121)
    v = rand_bshd(b, n + 2, hkv, d, dt, 122)
    o = fs().fwd(q, k, v, out_dtype=torch.float32)
    # every row against the exact float64 oracle: S = q K^T directly (tiny N), O = S V / |S|
    qd, kd, vd = (t.double() for t in (q, k, v))
    grp = h // hkv
    kd = kd.repeat_interleave(grp, dim=2)
    vd = vd.repeat_interleave(grp, dim=2)
    s = torch.einsum("bnhd,bmhd->bhnm", qd, kd)
    ref = torch.einsum("bhnm,bmhd->bnhd", s, vd) / s.pow(2).sum(-1).sqrt().permute(0, 2, 1)[..., None]
    check_tol(o.cpu().numpy(), ref.cpu().numpy(), dt, f"b{b} h{h}")


def test_long_sequence_million_keys():
    # N = 2^20 queries and keys in one (b, h): 5462 K/V tiles per work tile, 4096 work tiles
    n, d = 1 << 20, 64
    q = rand_bshd(1, n, 1, d, torch.bfloat16, 130)
    k = rand_bshd(1, n, 1, d, torch.bfloat16, 131)
    v = rand_bshd(1, n, 1, d, torch.bfloat16, 132)
    o = fs().fwd(q, k, v, kv_splits=1)
    rows = torch.tensor([0, 1, 4095, 4096, 777777, n - 1])
    ref = gram_spherical(q[0, rows.cuda(), 0].float().cpu().numpy(), k[0, :, 0].float().cpu().numpy(),
                         v[0, :, 0].float().cpu().numpy(), 1.0, 0.0)
    check_tol(o[0, rows.cuda(), 0].float().cpu().numpy(), ref, torch.bfloat16, "N=2^20")
    # and split into 4 K/V ranges of 2^18 keys (partials + merge kernel)
    o2 = fs().fwd(q, k, v, kv_splits=4)
    check_tol(o2[0, rows.cuda(), 0].float().cpu().numpy(), ref, torch.bfloat16, "N=2^20 split 4")


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_full_size_repeat_launches_bitwise(name):
    # a race between the kernel's roles shows up as launch-to-launch differences at full size
    # (many work tiles per CTA, the tail-split merge, the K' pass for C5's multiplicities)
    b, n, h, d, dt = {"c3": (8, 16384, 16, 128, torch.bfloat16), "c4": (8, 8192, 16, 128, torch.float8_e4m3fn),
                      "c5": (64, 20000, 8, 64, torch.bfloat16)}[name]
    g = torch.Generator(device="cuda").manual_seed(1)
    q, k, v = (torch.randn((b, n, h, d), generator=g, device="cuda").to(dt) for _ in range(3))
    m = torch.randint(0, 6, (b, n), generator=g, device="cuda").float() if name == "c5" else None
    eps = 1e-6 if name == "c5" else 0.0
    ref = fs().fwd(q, k, v, out_dtype=torch.bfloat16, key_scale=m, eps=eps)
    for _ in range(6):
        o = fs().fwd(q, k, v, out_dtype=torch.bfloat16, key_scale=m, eps=eps)
        assert torch.equal(o.view(torch.int16), ref.view(torch.int16))
