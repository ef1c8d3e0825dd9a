"""CPU-only tests of the drop-in boundary: the C-ABI library loads and exports every
symbol include/flashsign.h declares, its struct layout matches the header, host
validation maps to the reference's exception types, and the ncstream-compatible
API rejects bad input exactly like the reference -- all without a GPU."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2505_09326_b200 import _lib, flashsign
from paper_2505_09326_b200.attention import (
    AttentionConfig,
    ConfigError,
    TileConfig,
    default_score_scale,
    multi_head_attention_array,
    streamed_attention,
    streamed_attention_array,
)
from paper_2505_09326_b200.normalizers import SIGNED_L1, SOFTMAX, SPHERICAL, DegenerateDenominatorError
from paper_2505_09326_b200.tensor import DenseTensor, ShapeMismatchError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "flashsign.h")


def header_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*[a-z0-9_ ]+\**\s*\*?\s*(fs_[a-z_]+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    names = header_functions()
    assert set(names) == set(_lib.EXPORTED_SYMBOLS)
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}$", out, re.M), f"{n} not exported"


def test_library_is_sm100a_with_tcgen05():
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in sass
    for mnem in ("UTCHMMA", "UTCQMMA", "UTMALDG", "LDTM", "STTM"):
        assert mnem in sass, mnem
    assert "HMMA" not in re.sub(r"UTC[HQ]MMA", "", sass)  # no legacy mma.sync path


@pytest.mark.parametrize("cname,cls", [("fs_fwd_params", _lib.FsFwdParams), ("fs_peer_params", _lib.FsPeerParams),
                                       ("fs_prep_tensor", _lib.FsPrepTensor), ("fs_prep_params", _lib.FsPrepParams),
                                       ("fs_plan_info", _lib.FsPlanInfo), ("fs_exact_params", _lib.FsExactParams)])
def test_struct_layout_matches_header(tmp_path, cname, cls):
    fields = [f[0] for f in cls._fields_]
    prog = tmp_path / "layout.c"
    body = "\n".join(f'printf("{f} %zu\\n", offsetof({cname}, {f}));' for f in fields)
    prog.write_text(f'#include <stdio.h>\n#include <stddef.h>\n#include "{HEADER}"\nint main(void){{\n'
                    f'printf("size %zu\\n", sizeof({cname}));\n{body}\nreturn 0;}}\n')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c99", str(prog), "-o", str(exe)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    assert int(got["size"]) == ctypes.sizeof(cls)
    for f in fields:
        assert int(got[f]) == getattr(cls, f).offset, f


def test_peer_validation_without_gpu():
    # fs_fwd_peer / fs_combine_peer reject bad rank layouts before touching the device
    lib = _lib.load()
    prm = _params()
    for world, rank, rows in ((0, 0, 64), (2, 2, 64), (2, 0, 63), (2, -1, 64)):
        pp = _lib.FsPeerParams()
        pp.world, pp.rank, pp.rows_per_rank = world, rank, rows
        pp.peer_partial, pp.local_partial = 1 << 20, 1 << 20
        assert lib.fs_fwd_peer(ctypes.byref(prm), ctypes.byref(pp), None) == _lib.FS_ERR_CONFIG
        assert lib.fs_combine_peer(ctypes.byref(prm), ctypes.byref(pp), None) == _lib.FS_ERR_CONFIG
    pp = _lib.FsPeerParams()
    pp.world, pp.rank, pp.rows_per_rank = 2, 1, 64
    assert lib.fs_fwd_peer(ctypes.byref(prm), ctypes.byref(pp), None) == _lib.FS_ERR_CONFIG  # no workspaces
    pp.peer_partial, pp.local_partial = 1 << 20, 1 << 20
    # numerators [2][B=1][H=4][64][64] + z [2][1][4][64]
    assert lib.fs_peer_floats(ctypes.byref(prm), ctypes.byref(pp)) == 2 * 4 * 64 * 65
    from paper_2505_09326_b200.peer import peer_rows
    assert [peer_rows(10, 3, r) for r in range(3)] == [(0, 4), (4, 8), (8, 10)]
    assert [peer_rows(2, 3, r) for r in range(3)] == [(0, 1), (1, 2), (2, 2)]


def _params(**kw):
    p = _lib.FsFwdParams()
    p.batch, p.heads_q, p.heads_kv, p.seqlen_q, p.seqlen_kv, p.head_dim = 1, 4, 2, 128, 128, 64
    p.in_dtype, p.out_dtype = _lib.FS_BF16, _lib.FS_BF16
    p.scale, p.eps, p.p_scale, p.q_descale, p.k_descale, p.v_descale = 1.0, 0.0, 1.0, 1.0, 1.0, 1.0
    p.q = p.k = p.v = p.o = 1 << 20
    for s in (p.q_stride, p.k_stride, p.v_stride, p.o_stride):
        s[0], s[1], s[2] = 128 * 4 * 64, 4 * 64, 64
    for k, v in kw.items():
        setattr(p, k, v)
    return p


@pytest.mark.parametrize("kw,status,needle", [
    (dict(heads_q=3, heads_kv=2), _lib.FS_ERR_CONFIG, "multiple"),
    (dict(head_dim=200), _lib.FS_ERR_UNSUPPORTED, "head_dim"),
    (dict(head_dim=4), _lib.FS_ERR_UNSUPPORTED, "multiple of 16"),
    (dict(in_dtype=_lib.FS_F32), _lib.FS_ERR_DTYPE, "in_dtype"),
    (dict(scale=float("nan")), _lib.FS_ERR_CONFIG, "finite"),
    (dict(eps=-1.0), _lib.FS_ERR_CONFIG, "epsilon"),
    (dict(p_scale=0.0), _lib.FS_ERR_CONFIG, "positive"),
    (dict(heads_q=0), _lib.FS_ERR_SHAPE, "extents"),
    (dict(q=(1 << 20) + 8), _lib.FS_ERR_UNSUPPORTED, "aligned"),
    (dict(normalizer=7), _lib.FS_ERR_CONFIG, "normalizer"),
    (dict(key_scale=(1 << 20) + 4), _lib.FS_ERR_UNSUPPORTED, "key_scale must be 16-byte aligned"),
    (dict(batch=2, key_scale=1 << 20, key_scale_stride=130), _lib.FS_ERR_UNSUPPORTED, "key_scale_stride"),
    (dict(batch=2, key_scale=1 << 20, key_scale_stride=64), _lib.FS_ERR_UNSUPPORTED, "key_scale_stride"),
    (dict(batch=65535, heads_q=65535, heads_kv=65535, seqlen_q=2), _lib.FS_ERR_UNSUPPORTED, "2^32"),
    (dict(heads_q=70000, heads_kv=70000), _lib.FS_ERR_UNSUPPORTED, "65535"),
])
def test_fs_fwd_validation(kw, status, needle):
    lib = _lib.load()
    st = lib.fs_fwd(ctypes.byref(_params(**kw)), None)
    assert st == status
    assert needle in _lib.last_error()


def test_query_tile():
    assert _lib.query_tile(64, _lib.FS_BF16) == (128, 192)   # d=64 16-bit: 192-key K/V tiles
    assert _lib.query_tile(128, _lib.FS_BF16) == (128, 128)
    assert _lib.query_tile(128, _lib.FS_E4M3) == (128, 128)
    with pytest.raises(ValueError):
        _lib.query_tile(0, _lib.FS_BF16)


def test_bad_key_decoding():
    lin = (2 * 8 + 5) * 300 + 17  # batch 2, head 5 of 8, row 17 of 300
    z = np.float32(0.0)
    key = (lin << 32) | int(np.array([z]).view(np.uint32)[0])
    assert flashsign.decode_bad_key(key, 8, 300) == (2, 5, 17, 0.0)
    assert flashsign.decode_bad_key(_lib.FS_BAD_NONE, 8, 300) is None
    key_nan = (3 << 32) | 0x7FC00000
    b, h, row, zz = flashsign.decode_bad_key(key_nan, 1, 10)
    assert (b, h, row) == (0, 0, 3) and np.isnan(zz)
    # ordering of packed keys == reference loop order (batch, head, row)
    keys = [((bb * 4 + hh) * 10 + rr) << 32 for bb in range(2) for hh in range(4) for rr in range(10)]
    assert keys == sorted(keys)


# ---------------------------------------------------------------- compat API (validation paths only)

def test_compat_shape_errors_match_reference():
    with pytest.raises(ShapeMismatchError):
        streamed_attention_array(np.ones((2, 3)), np.ones((2, 4)), np.ones((2, 4)), SPHERICAL, 1.0, TileConfig())
    with pytest.raises(ShapeMismatchError):
        streamed_attention_array(np.ones((2, 3, 1)), np.ones((2, 3)), np.ones((2, 3)), SPHERICAL, 1.0, TileConfig())
    with pytest.raises(ShapeMismatchError):
        streamed_attention_array(np.ones((2, 3)), np.ones((4, 3)), np.ones((5, 3)), SPHERICAL, 1.0, TileConfig())


def test_compat_config_errors_match_reference():
    # test_attention.py:275-278
    with pytest.raises(ConfigError, match="multiple"):
        multi_head_attention_array(np.ones((2, 3, 2)), np.ones((2, 2, 2)), np.ones((2, 2, 2)), SPHERICAL, h=3, h_kv=2)
    with pytest.raises(ConfigError):
        multi_head_attention_array(np.ones((2, 2, 2)), np.ones((2, 1, 2)), np.ones((2, 1, 2)), SPHERICAL, 2, 1,
                                   path="bogus")
    with pytest.raises(ShapeMismatchError):
        multi_head_attention_array(np.ones((2, 2)), np.ones((2, 1, 2)), np.ones((2, 1, 2)), SPHERICAL, 2, 1)
    with pytest.raises(ConfigError):
        TileConfig(0, 4)
    with pytest.raises(ConfigError):
        AttentionConfig(SPHERICAL, score_scale=0.0)
    with pytest.raises(ConfigError):
        AttentionConfig(SPHERICAL, score_scale=float("nan"))
    # test_attention.py:340-344: f16 emulation needs float32
    q = DenseTensor(np.ones((2, 2)))
    with pytest.raises(ConfigError, match="float32"):
        streamed_attention(q, q, q, AttentionConfig(SPHERICAL, f16_emulation=True))


def test_compat_softmax_rejected_on_streamed_path():
    # softmax is not an exp-free FlashSign triple: ConfigError before any device work (no CPU fallback)
    with pytest.raises(ConfigError, match="exp-free"):
        streamed_attention_array(np.ones((2, 8), np.float32), np.ones((2, 8), np.float32),
                                 np.ones((2, 8), np.float32), SOFTMAX, 1.0, TileConfig())


def test_multiplicity_validation_matches_reference():
    # attention.py:381-388: length mismatch -> ShapeMismatchError, negative/non-finite -> ValueError,
    # raised before any device work
    from paper_2505_09326_b200.attention import multiplicity_attention_array
    q = np.ones((4, 2, 8), np.float32)
    k = np.ones((4, 1, 8), np.float32)
    with pytest.raises(ShapeMismatchError, match="multiplicity length"):
        multiplicity_attention_array(q, k, k, np.ones(3), SPHERICAL, 2, 1)
    for bad in ([1, -1, 0, 2], [1, np.nan, 0, 2], [1, np.inf, 0, 2]):
        with pytest.raises(ValueError, match="finite and nonnegative"):
            multiplicity_attention_array(q, k, k, np.array(bad, float), SPHERICAL, 2, 1)
    with pytest.raises(ConfigError, match="exp-free"):
        multiplicity_attention_array(q, k, k, np.ones(4), SOFTMAX, 2, 1)


def test_default_scales_match_reference():
    # test_attention.py:321-325
    assert default_score_scale(SOFTMAX, 64) == 64 ** -0.5
    assert default_score_scale(SPHERICAL, 64) == 1.0
    assert default_score_scale(SIGNED_L1, 64) == 1.0
    assert AttentionConfig(SOFTMAX).resolve_scale(16) == 0.25
    assert AttentionConfig(SOFTMAX, score_scale=2.0).resolve_scale(16) == 2.0


def test_degenerate_error_message_matches_reference():
    e = DegenerateDenominatorError(0.0, "row 1")
    assert "row 1" in str(e) and e.z == 0.0 and isinstance(e, ValueError)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="CUDA"):
        streamed_attention_array(np.ones((4, 8), np.float32), np.ones((4, 8), np.float32),
                                 np.ones((4, 8), np.float32), SPHERICAL, 1.0, TileConfig())


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2505_09326_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|\"\"\".*?\"\"\"", "", src, flags=re.S).replace(
                    "oracle/", ""), f"{f} references the oracle"


def test_split_plan_host_functions():
    # fs_kv_splits / fs_partial_floats are host-only: effective splits clamp to [1, K/V tiles] and
    # leave no empty range; the workspace holds S x rows x (Dk + 1) floats
    lib = _lib.load()
    p = _params(head_dim=128, seqlen_kv=1000, seqlen_q=300, batch=2, heads_q=4, heads_kv=2)
    for req in (0, 1, 2, 3, 7, 100):
        p.kv_splits = req
        got = lib.fs_kv_splits(ctypes.byref(p))
        assert 1 <= got <= 8 and (req <= 1 and got == 1 or req > 1)
    p.kv_splits = 7   # 8 tiles of 128 keys, ceil(8/7)=2 per split -> 4 non-empty splits
    assert lib.fs_kv_splits(ctypes.byref(p)) == 4
    assert lib.fs_partial_floats(ctypes.byref(p)) == 4 * 2 * 4 * 300 * (128 + 1)
    p.head_dim, p.in_dtype = 64, _lib.FS_BF16   # d=64 16-bit: 192-key tiles -> 6 tiles
    p.kv_splits = 100
    assert lib.fs_kv_splits(ctypes.byref(p)) == 6
    assert lib.fs_partial_floats(ctypes.byref(p)) == 6 * 2 * 4 * 300 * (64 + 1)
    p.kv_splits, p.partial = 2, None
    assert lib.fs_fwd(ctypes.byref(p), None) == _lib.FS_ERR_CONFIG and "partial" in _lib.last_error()


def test_auto_splits_wave_model():
    # FS_SPLITS_AUTO planned for 74 co-resident clusters (148-SM B200), host only
    def plan(b, h, n, d=128, dt=_lib.FS_BF16):
        p = _params(head_dim=d, seqlen_kv=n, seqlen_q=n, batch=b, heads_q=h, heads_kv=h)
        p.in_dtype = dt
        p.kv_splits = _lib.FS_SPLITS_AUTO
        return _lib.plan(p, 74)
    assert plan(1, 1, 16384).splits > 1 and plan(1, 1, 16384).split_tail == 0   # 32 tiles: uniform split
    assert plan(1, 1, 300, 128).splits == 1                                    # too few K/V tiles (3)
    c3 = plan(8, 16, 16384)      # 4096 tiles = 55 waves + 26: the tail wave is split in two
    assert (c3.splits, c3.split_tail, c3.n_whole, c3.tail_tiles) == (2, 1, 55 * 74, 26)
    assert c3.items == 55 * 74 + 52 and c3.efficiency > 0.995
    assert plan(16, 16, 4096, 64, _lib.FS_F16).splits == 1   # C2 on one GPU: 27.7 waves, a split would not pay


def test_plan_edge_cases():
    # host-only fs_plan: empty launches, short K/V streams, partial_only (context parallelism wants
    # every row's partial: never a tail split), explicit split_tail, whole waves (nothing to balance)
    def params(b, h, nq, nkv, d=128):
        p = _params(head_dim=d, seqlen_kv=nkv, seqlen_q=nq, batch=b, heads_q=h, heads_kv=h)
        p.in_dtype = _lib.FS_BF16
        return p
    p = params(0, 4, 256, 256)
    p.kv_splits = _lib.FS_SPLITS_AUTO
    assert _lib.plan(p, 74).splits == 1 and _lib.plan(p, 74).items == 0
    p = params(1, 80, 1024, 4096)                      # 160 tiles = 2 waves + 12
    p.kv_splits = _lib.FS_SPLITS_AUTO
    auto = _lib.plan(p, 74)
    assert auto.split_tail == 1 and auto.n_whole == 148 and auto.tail_tiles == 12
    assert auto.partial_floats == auto.splits * 12 * 512 * 129
    p.partial_only = 1
    cp = _lib.plan(p, 74)
    assert cp.split_tail == 0 and cp.splits == 1
    p.partial_only, p.kv_splits, p.split_tail = 0, 3, 1
    ex = _lib.plan(p, 74)
    assert (ex.splits, ex.split_tail, ex.items) == (3, 1, 148 + 36)
    ex80 = _lib.plan(p, 80)                            # 160 = 2 whole waves of 80: no tail to split
    assert (ex80.splits, ex80.split_tail, ex80.items) == (1, 0, 160)
    p.kv_splits = -2
    with pytest.raises(ValueError):
        _lib.plan(p, 74)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_wave_efficiency_of_sharded_configs(world):
    # batch x head shards of C2-C5 (BASELINE.json configs) on `world` GPUs: each rank's launch
    # keeps >= 95 % of the persistent grid's clusters busy (static-stride wave model, 74 clusters)
    from paper_2505_09326_b200 import partition
    cfgs = {"c2": (16, 16, 4096, 64, _lib.FS_F16), "c3": (8, 16, 16384, 128, _lib.FS_BF16),
            "c4": (8, 16, 8192, 128, _lib.FS_E4M3), "c5": (64, 8, 20000, 64, _lib.FS_BF16)}
    for name, (b, h, n, d, dt) in cfgs.items():
        for rank in range(world):
            lo, hi = partition.unit_range(b * h, world, rank)
            for pc in partition.pieces(b, h, lo, hi):
                p = _params(head_dim=d, seqlen_kv=n, seqlen_q=n, batch=pc.b1 - pc.b0, heads_q=pc.g1 - pc.g0,
                            heads_kv=pc.g1 - pc.g0)
                p.in_dtype = dt
                p.kv_splits = _lib.FS_SPLITS_AUTO
                info = _lib.plan(p, 74)
                assert info.efficiency >= 0.95, (name, world, rank, info.splits, info.split_tail, info.efficiency)
                p.kv_splits = 1
                unsplit = _lib.plan(p, 74).efficiency
                assert info.efficiency >= unsplit - 1e-9


def test_integration_c_snippet_compiles(tmp_path):
    # the C example in INTEGRATION.md builds against include/flashsign.h as written
    text = open(os.path.join(os.path.dirname(HEADER), "..", "INTEGRATION.md")).read()
    block = text.split("C/C++ callers include the header")[1].split("```c")[1].split("```")[0]
    lines = [ln for ln in block.splitlines() if not ln.startswith("#include")]
    prog = tmp_path / "snippet.c"
    prog.write_text('#include <stdio.h>\n#include <stdint.h>\n#include "' + HEADER + '"\n'
                    "void run(void *dq, void *dk, void *dv, void *dout, uint64_t *d_bad, int B, int H, int Hkv,"
                    " int N, fs_stream_t stream) {\n" + "\n".join(lines) + "\n}\n")
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-c", str(prog), "-o", str(tmp_path / "snippet.o")],
                   check=True)


@pytest.mark.parametrize("n", [0, 1, 63, 64, 65, 255, 256, 4097, 1 << 20, (1 << 20) + 37])
@pytest.mark.parametrize("dst_off,src_off", [(0, 0), (1, 0), (0, 3), (17, 41)])
def test_host_copy_bitwise(n, dst_off, src_off):
    # the drop-in staging fill (fs_host_copy, non-temporal stores): host only, any size / alignment
    import ctypes
    lib = _lib.load()
    lib.fs_host_copy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]
    lib.fs_host_copy.restype = ctypes.c_int
    rng = np.random.default_rng(n + dst_off)
    src = rng.integers(0, 256, n + src_off + 64, dtype=np.uint8)
    dst = np.zeros(n + dst_off + 64, dtype=np.uint8)
    width = lib.fs_host_copy(dst[dst_off:].ctypes.data, src[src_off:].ctypes.data, n)
    assert width in (0, 256, 512)
    assert np.array_equal(dst[dst_off:dst_off + n], src[src_off:src_off + n])
    assert not dst[:dst_off].any() and not dst[dst_off + n:].any()  # nothing outside the range
