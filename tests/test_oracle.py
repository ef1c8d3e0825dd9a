"""Pin the CPU oracle (oracle/spherical.py) against golden vectors produced by
running the reference itself (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle.spherical import (
    OracleDegenerate,
    exact_batched,
    gram_batched,
    gram_spherical,
    multi_head_spherical,
    naive_spherical,
    streamed_spherical,
)


def _args(g, c):
    return g[f"{c}/q"], g[f"{c}/k"], g[f"{c}/v"], float(g[f"{c}/scale"]), float(g[f"{c}/eps"])


def test_golden_has_cases(golden):
    assert len(golden["__cases__"]) >= 20


def test_kat_hand_exact(golden):
    # test_attention.py:46-52 -- weights (0.6, 0.8): 0.6*10 + 0.8*20 = 22
    for c in ("kat_hand", "kat_hand_streamed11", "kat_hand_f32"):
        q, k, v, s, e = _args(golden, c)
        assert golden[f"{c}/out"].tolist() == [[22.0]]
        assert naive_spherical(q, k, v, s, e).tolist() == [[22.0]]
        assert streamed_spherical(q, k, v, s, e, 1, 1).tolist() == [[22.0]]
        assert streamed_spherical(q, k, v, s, e).tolist() == [[22.0]]


def test_kat_sign_exact(golden):
    for tag, sign in (("pos", 1.0), ("neg", -1.0)):
        q, k, v, s, e = _args(golden, f"kat_sign_{tag}")
        want = golden[f"kat_sign_{tag}/out"]
        assert np.array_equal(want, sign * v)
        assert np.array_equal(naive_spherical(q, k, v, s, e), want)
        assert np.array_equal(streamed_spherical(q, k, v, s, e, 1, 1), want)


@pytest.mark.parametrize("prefix", ["grid64", "grid32", "prime97", "c1", "scale_eps_mult"])
def test_streamed_and_naive_match_reference(golden, prefix):
    cases = [c for c in golden["__cases__"].tolist() if c.startswith(prefix)]
    assert cases
    for c in cases:
        q, k, v, s, e = _args(golden, c)
        want = golden[f"{c}/out"]
        f32 = q.dtype == np.float32
        rtol, atol = (1e-5, 1e-6) if f32 else (1e-12, 1e-14)
        np.testing.assert_allclose(naive_spherical(q, k, v, s, e), want, rtol=rtol, atol=atol)
        np.testing.assert_allclose(streamed_spherical(q, k, v, s, e), want, rtol=rtol, atol=atol)
        for key, tile in (("streamed_13_7", (13, 7)), ("streamed_5_9", (5, 9))):
            if f"{c}/{key}" in golden:
                got = streamed_spherical(q, k, v, s, e, *tile)
                # same tile + same precision policy as the reference -> tight agreement
                np.testing.assert_allclose(got, golden[f"{c}/{key}"], rtol=rtol, atol=atol)


@pytest.mark.parametrize("case", ["gqa_4_2", "gqa_2_1", "gqa_8_2_f32"])
def test_multi_head_gqa_matches_reference(golden, case):
    q, k, v, s, e = _args(golden, case)
    h, hkv = int(golden[f"{case}/h"]), int(golden[f"{case}/h_kv"])
    want = golden[f"{case}/out"]
    f32 = q.dtype == np.float32
    rtol, atol = (1e-5, 1e-6) if f32 else (1e-12, 1e-14)
    np.testing.assert_allclose(multi_head_spherical(q, k, v, h, hkv, s, e), want, rtol=rtol, atol=atol)
    # batched Gram oracle with the same GQA map (what the GPU tests use at full size)
    got = gram_batched(q[None], k[None], v[None], s, e)[0]
    np.testing.assert_allclose(got, want, rtol=1e-4 if f32 else 1e-10, atol=1e-5 if f32 else 1e-12)


def test_f16_emulation_matches_reference(golden):
    q, k, v, s, e = _args(golden, "f16_64")
    got = streamed_spherical(q, k, v, s, e, 16, 16, f16=True)
    np.testing.assert_array_equal(got, golden["f16_64/f16_out"])
    # reference's own accuracy criterion (test_attention.py:351-357)
    assert np.mean(np.abs(got - golden["f16_64/out"]) <= 0.01) >= 0.99


def test_gram_identity_matches_reference_float64(golden):
    for c in [c for c in golden["__cases__"].tolist() if c.startswith("grid64") or c == "prime97"]:
        q, k, v, s, e = _args(golden, c)
        np.testing.assert_allclose(gram_spherical(q, k, v, s, e), golden[f"{c}/out"], rtol=1e-9, atol=1e-12)


def test_gram_criterion4(golden):
    rng = np.random.default_rng(int(golden["crit4/seed"]))
    q = rng.standard_normal((1024, 128)).astype(np.float32)
    k = rng.standard_normal((1024, 128)).astype(np.float32)
    v = rng.standard_normal((1024, 128)).astype(np.float32)
    got = gram_spherical(q, k, v)
    np.testing.assert_allclose(got, golden["crit4/out"], rtol=1e-4, atol=2e-6)


@pytest.mark.parametrize("case", ["degen_row1", "degen_nan_row2", "degen_empty_k"])
def test_degenerate_rows_match_reference(golden, case):
    q, k, v, s, e = golden[f"{case}/q"], golden[f"{case}/k"], golden[f"{case}/v"], 1.0, 0.0
    row = int(golden[f"{case}/err_row"])
    z = float(golden[f"{case}/err_z"])
    for fn in (lambda: naive_spherical(q, k, v, s, e), lambda: streamed_spherical(q, k, v, s, e),
               lambda: streamed_spherical(q, k, v, s, e, 1, 1)):
        with pytest.raises(OracleDegenerate) as ei:
            fn()
        assert ei.value.row == row
        assert (np.isnan(z) and np.isnan(ei.value.z)) or ei.value.z == z


REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not __import__("os").path.isdir(REF_SRC), reason="reference not mounted (GPU box)")
def test_oracle_port_bitwise_equals_live_reference():
    """The CPU baseline (oracle port of _streamed_tiles) is the reference's algorithm:
    bitwise-identical outputs to ncstream.attention.streamed_attention_array, run live."""
    import sys
    sys.path.insert(0, REF_SRC)
    try:
        from ncstream.attention import TileConfig, multi_head_attention_array, streamed_attention_array
        from ncstream.normalizers import SPHERICAL
    finally:
        sys.path.remove(REF_SRC)
    rng = np.random.default_rng(11)
    for (y, x, d, dt, tile, scale, eps) in [(300, 517, 64, np.float32, (64, 64), 1.0, 0.0),
                                           (97, 33, 8, np.float64, (13, 7), -0.7, 1e-6),
                                           (128, 256, 128, np.float32, (16, 32), 2.0, 0.0)]:
        q, k, v = (rng.standard_normal(s).astype(dt) for s in ((y, d), (x, d), (x, d)))
        want = streamed_attention_array(q, k, v, SPHERICAL.with_epsilon(eps), scale, TileConfig(*tile))
        got = streamed_spherical(q, k, v, scale, eps, *tile)
        assert np.array_equal(got, want)
    q = rng.standard_normal((50, 4, 16)).astype(np.float32)
    k = rng.standard_normal((70, 2, 16)).astype(np.float32)
    v = rng.standard_normal((70, 2, 16)).astype(np.float32)
    assert np.array_equal(multi_head_spherical(q, k, v, 4, 2),
                          multi_head_attention_array(q, k, v, SPHERICAL, 4, 2))
    f = rng.standard_normal((64, 16)).astype(np.float32)
    assert np.array_equal(streamed_spherical(f, f, f, 1.0, 0.0, 16, 16, f16=True),
                          streamed_attention_array(f, f, f, SPHERICAL, 1.0, TileConfig(16, 16), f16=True))


# ---------------------------------------------------------------- SIGNED_L1 and fused multiplicities

def test_l1_kat_hand_exact(golden):
    # signed_l1 on the hand KAT: (3*10 + 4*20) / (3 + 4) = 110/7 (normalizers.py:111-117)
    q, k, v, s, e = _args(golden, "l1_kat_hand")
    assert golden["l1_kat_hand/out"][0, 0] == 110.0 / 7.0
    assert naive_spherical(q, k, v, s, e, norm="signed_l1")[0, 0] == 110.0 / 7.0
    assert streamed_spherical(q, k, v, s, e, 1, 1, norm="signed_l1").tolist() == golden["l1_kat_hand/streamed_1_1"].tolist()


@pytest.mark.parametrize("prefix", ["l1_grid64", "l1_grid32", "l1_scale_eps"])
def test_l1_streamed_and_naive_match_reference(golden, prefix):
    cases = [c for c in golden["__cases__"].tolist() if c.startswith(prefix)]
    assert cases
    for c in cases:
        q, k, v, s, e = _args(golden, c)
        want = golden[f"{c}/out"]
        f32 = q.dtype == np.float32
        rtol, atol = (1e-5, 1e-6) if f32 else (1e-12, 1e-14)
        np.testing.assert_allclose(naive_spherical(q, k, v, s, e, norm="signed_l1"), want, rtol=rtol, atol=atol)
        np.testing.assert_allclose(streamed_spherical(q, k, v, s, e, norm="signed_l1"), want, rtol=rtol, atol=atol)
        for key, tile in (("streamed_13_7", (13, 7)), ("streamed_5_9", (5, 9))):
            if f"{c}/{key}" in golden:
                got = streamed_spherical(q, k, v, s, e, *tile, norm="signed_l1")
                np.testing.assert_allclose(got, golden[f"{c}/{key}"], rtol=rtol, atol=atol)
        ex = exact_batched(q[None, :, None], k[None, :, None], v[None, :, None], s, e, norm="signed_l1")[0, :, 0]
        np.testing.assert_allclose(ex, want, rtol=1e-4 if f32 else 1e-10, atol=1e-5 if f32 else 1e-12)


def test_l1_gqa_matches_reference(golden):
    c = "l1_gqa_4_2_f32"
    q, k, v, s, e = _args(golden, c)
    want = golden[f"{c}/out"]
    np.testing.assert_allclose(multi_head_spherical(q, k, v, 4, 2, s, e, norm="signed_l1"), want, rtol=1e-5, atol=1e-6)
    got = exact_batched(q[None], k[None], v[None], s, e, norm="signed_l1")[0]
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-5)


@pytest.mark.parametrize("tag,norm", [("sph", "spherical"), ("l1", "signed_l1")])
def test_fused_multiplicity_oracle_matches_reference(golden, tag, norm):
    # grn.py:150 + 171-173: multi_head_attention_array(q, apply_multiplicity_array(k, m), v, ...)
    c = f"mult_{tag}_gqa_f32"
    q, k, v, s, e = _args(golden, c)
    m = golden[f"{c}/m"]
    want = golden[f"{c}/out"]
    got = exact_batched(q[None], k[None], v[None], s, e, norm=norm, m=m[None])[0]
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-5)
    km = k * m.astype(np.float32)[:, None, None]
    np.testing.assert_allclose(multi_head_spherical(q, km, v, 4, 2, s, e, norm=norm), want, rtol=1e-5, atol=1e-6)


def test_l1_degenerate_row_matches_reference(golden):
    c = "l1_degen_row1"
    q, k, v = golden[f"{c}/q"], golden[f"{c}/k"], golden[f"{c}/v"]
    for fn in (lambda: naive_spherical(q, k, v, norm="signed_l1"), lambda: streamed_spherical(q, k, v, norm="signed_l1")):
        with pytest.raises(OracleDegenerate) as ei:
            fn()
        assert ei.value.row == int(golden[f"{c}/err_row"]) and ei.value.z == float(golden[f"{c}/err_z"])
