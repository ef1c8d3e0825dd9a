"""The drop-in API's ``f64`` compute mode (C-ABI ``fs_exact_fwd``, csrc/flashsign_exact.cu): the
reference's streamed loop (attention.py:146-200) with its rounding points on the FP64 units.

Checked against the golden vectors the reference itself produced (tests/golden/make_golden.py) at
the reference's OWN float tolerances: float64 inputs rtol 1e-12, float32 inputs within one float32
rounding of the reference's output (rtol 2e-7 / atol 1e-7); degenerate rows raise the same
exception with the same row and z.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GOLDEN = __import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "golden.npz")


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2505_09326_b200 import build
    build.build()


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


@pytest.fixture()
def at():
    from paper_2505_09326_b200 import attention
    attention.set_compute_dtype("f64")
    yield attention
    attention.set_compute_dtype("fp16")


def close(got, want):
    got = np.asarray(got)
    if want.dtype == np.float32:
        np.testing.assert_allclose(got.astype(np.float64), want.astype(np.float64), rtol=2e-7, atol=1e-7)
    else:
        np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-13)


def test_exact_single_head_cases_match_reference(golden, at):
    from paper_2505_09326_b200 import SIGNED_L1, SPHERICAL
    cases = [c for c in golden["__cases__"].tolist()
             if c.startswith(("kat_", "grid", "prime97", "c1", "scale_eps", "l1_")) and f"{c}/out" in golden.files]
    assert len(cases) >= 20
    for c in cases:
        q, k, v = golden[f"{c}/q"], golden[f"{c}/k"], golden[f"{c}/v"]
        if q.ndim != 2 or v.shape[1] != q.shape[1]:  # (d_v != d: a naive-path KAT; the streamed path rejects it)
            continue
        spec = (SIGNED_L1 if c.startswith("l1_") else SPHERICAL).with_epsilon(float(golden[f"{c}/eps"]))
        got = at.streamed_attention_array(q, k, v, spec, float(golden[f"{c}/scale"]), at.TileConfig(13, 7))
        assert got.dtype == q.dtype, c
        close(got, golden[f"{c}/out"])
    # the hand KAT is exact: [[22.0]]
    assert at.streamed_attention_array(golden["kat_hand/q"], golden["kat_hand/k"], golden["kat_hand/v"], SPHERICAL,
                                       1.0, at.TileConfig(1, 1)).tolist() == [[22.0]]


@pytest.mark.parametrize("c", ["gqa_4_2", "gqa_2_1", "gqa_8_2_f32"])
def test_exact_multi_head_matches_reference(golden, at, c):
    from paper_2505_09326_b200 import SPHERICAL
    q, k, v = golden[f"{c}/q"], golden[f"{c}/k"], golden[f"{c}/v"]
    got = at.multi_head_attention_array(q, k, v, SPHERICAL, int(golden[f"{c}/h"]), int(golden[f"{c}/h_kv"]))
    close(got, golden[f"{c}/out"])


@pytest.mark.parametrize("c", ["degen_row1", "degen_nan_row2", "degen_empty_k", "l1_degen_row1"])
def test_exact_degenerate_rows_like_reference(golden, at, c):
    from paper_2505_09326_b200 import SIGNED_L1, SPHERICAL
    from paper_2505_09326_b200.normalizers import DegenerateDenominatorError
    spec = (SIGNED_L1 if c.startswith("l1_") else SPHERICAL).with_epsilon(float(golden[f"{c}/eps"]))
    with pytest.raises(DegenerateDenominatorError, match=f"row {int(golden[f'{c}/err_row'])}") as ei:
        at.streamed_attention_array(golden[f"{c}/q"], golden[f"{c}/k"], golden[f"{c}/v"], spec,
                                    float(golden[f"{c}/scale"]), at.TileConfig())
    want = float(golden[f"{c}/err_z"])
    got = float(ei.value.z) if hasattr(ei.value, "z") else None
    if got is not None:
        assert (np.isnan(want) and np.isnan(got)) or got == pytest.approx(want, rel=1e-12, abs=0.0)


def test_exact_zero_score_key_deletion_is_bitwise(at):
    # keys are accumulated strictly in order: appending / inserting a key with score 0 everywhere
    # leaves every output bit-identical (the reference's own claim, test_attention.py:219-228)
    from paper_2505_09326_b200 import SPHERICAL
    rng = np.random.default_rng(5)
    q = rng.standard_normal((37, 8))
    q[:, 0] = 0.0
    k = rng.standard_normal((50, 8))
    v = rng.standard_normal((50, 8))
    zero = np.zeros((1, 8))
    zero[0, 0] = 3.0  # orthogonal to every query
    k2 = np.concatenate([k[:20], zero, k[20:]])
    v2 = np.concatenate([v[:20], rng.standard_normal((1, 8)), v[20:]])
    a = at.streamed_attention_array(q, k, v, SPHERICAL, 1.0, at.TileConfig())
    b = at.streamed_attention_array(q, k2, v2, SPHERICAL, 1.0, at.TileConfig())
    assert np.array_equal(a, b)


def test_exact_multiplicities_and_large_shape(golden, at):
    from paper_2505_09326_b200 import SPHERICAL
    c = "mult_sph_gqa_f32"
    got = at.multiplicity_attention_array(golden[f"{c}/q"], golden[f"{c}/k"], golden[f"{c}/v"], golden[f"{c}/m"],
                                          SPHERICAL.with_epsilon(float(golden[f"{c}/eps"])), 4, 2, scale=1.0)
    np.testing.assert_allclose(got.astype(np.float64), golden[f"{c}/out"].astype(np.float64), rtol=1e-5, atol=1e-6)
    # a C1-sized and a d=128 case against the float64 oracle
    from oracle.spherical import gram_spherical
    rng = np.random.default_rng(9)
    for (y, x, d) in ((256, 256, 64), (300, 1000, 128), (5, 3000, 96)):
        q, k, v = (rng.standard_normal((n, d)) for n in (y, x, x))
        got = at.streamed_attention_array(q, k, v, SPHERICAL, 0.125, at.TileConfig())
        np.testing.assert_allclose(got, gram_spherical(q, k, v, 0.125, 0.0), rtol=1e-10, atol=1e-12)
