"""Torch-native FlashSign forward: CUDA tensors in, CUDA tensor out, one launch.

Normalisers (``normalizer=``): ``"spherical"`` (the FlashSign contract,
normalizers.py:94-100) and ``"signed_l1"`` (normalizers.py:111-117, a2 = |u|,
b = identity) -- both exp-free, compiled into the same kernel.  ``key_scale``
fuses the GRN caller's ``apply_multiplicity_array(K, m)`` (attention.py:381-388,
grn.py:150) into the score: s_ij -> m_j s_ij.

``fwd(q, k, v)`` takes BSHD tensors ``q [B, Nq, H, d]``, ``k, v [B, Nkv, H_kv, d]``
(d contiguous, ``H % H_kv == 0``) in bf16 / fp16 / float8_e4m3fn and calls the
C-ABI ``fs_fwd`` (include/flashsign.h) on the caller's current CUDA stream.
It is the batched, device-resident form of the reference's
``multi_head_attention_array`` (attention.py:318-361): every (batch, head,
query tile) runs in one launch; query head h reads kv head h*H_kv//H
(attention.py:352).

Degenerate rows (b(z+eps) zero or non-finite, attention.py:196-199) are
flagged on the device; ``check=True`` synchronises and raises
``DegenerateDenominatorError`` for the first (batch, head, row) in the
reference's loop order.  ``fwd_async`` returns the flag tensor instead of
synchronising (benchmarks).
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._errors import ConfigError
from .normalizers import DegenerateDenominatorError
from .tensor import ShapeMismatchError

_IN_CODES = {torch.bfloat16: _lib.FS_BF16, torch.float16: _lib.FS_F16}
if hasattr(torch, "float8_e4m3fn"):
    _IN_CODES[torch.float8_e4m3fn] = _lib.FS_E4M3
_OUT_CODES = {torch.float32: _lib.FS_F32, torch.bfloat16: _lib.FS_BF16, torch.float16: _lib.FS_F16}
NORMALIZERS = {"spherical": _lib.FS_NORM_SPHERICAL, "signed_l1": _lib.FS_NORM_SIGNED_L1}

_STATUS_EXC = {
    _lib.FS_ERR_SHAPE: ShapeMismatchError,
    _lib.FS_ERR_DTYPE: ShapeMismatchError,
    _lib.FS_ERR_CONFIG: ConfigError,
    _lib.FS_ERR_UNSUPPORTED: ConfigError,
    _lib.FS_ERR_CUDA: RuntimeError,
}

BAD_NONE = _lib.FS_BAD_NONE
_ext = None  # the torch extension, bound on first use


def torch_ext():
    """The torch extension over the C-ABI (csrc/fs_torch.cpp), loaded on first use."""
    global _ext
    if _ext is None:
        _ext = _lib.load_torch_ext()
    return _ext


def _check_inputs(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor):
    for name, t in (("q", q), ("k", k), ("v", v)):
        if not t.is_cuda:
            raise RuntimeError(f"flashsign: {name} must be a CUDA tensor (no CPU fallback)")
        if t.dim() != 4:
            raise ShapeMismatchError(f"flashsign: {name} must be BSHD rank-4, got shape {tuple(t.shape)}")
        if t.stride(-1) != 1:
            raise ShapeMismatchError(f"flashsign: {name} head dim must be contiguous")
    if not (q.dtype == k.dtype == v.dtype):
        raise ShapeMismatchError(f"dtype mismatch: {q.dtype}, {k.dtype}, {v.dtype}")
    if q.dtype not in _IN_CODES:
        raise ShapeMismatchError(f"flashsign: unsupported input dtype {q.dtype} (bf16, fp16, float8_e4m3fn)")
    b, _, _, d = q.shape
    if k.shape[0] != b or v.shape[0] != b:
        raise ShapeMismatchError(f"batch mismatch: {tuple(q.shape)}, {tuple(k.shape)}, {tuple(v.shape)}")
    if k.shape[3] != d:
        raise ShapeMismatchError(f"Q and K feature dims differ: {tuple(q.shape)} vs {tuple(k.shape)}")
    if v.shape[1] != k.shape[1] or v.shape[2] != k.shape[2]:
        raise ShapeMismatchError(f"K and V shapes differ: {tuple(k.shape)} vs {tuple(v.shape)}")
    if v.shape[3] != d:
        raise ShapeMismatchError(f"flashsign: value dim must equal head dim ({v.shape[3]} vs {d})")
    if q.device != k.device or q.device != v.device:
        raise RuntimeError("flashsign: q, k, v must be on the same device")


def fwd_async(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *, scale: float = 1.0, eps: float = 0.0,
              out: torch.Tensor | None = None, out_dtype: torch.dtype | None = None, p_scale: float = 1.0,
              q_descale: float = 1.0, k_descale: float = 1.0, v_descale: float = 1.0,
              bad_key: torch.Tensor | None = None, stream: torch.cuda.Stream | None = None,
              tile_hint: tuple[int, int] = (0, 0), normalizer: str = "spherical",
              key_scale: torch.Tensor | None = None, kv_splits: int | None = None,
              partial: torch.Tensor | None = None, partial_only: bool = False,
              dev_scales: torch.Tensor | None = None, split_tail: bool = False):
    """Launch FlashSign and return ``(o, bad_key)`` without synchronising.

    ``bad_key`` is a 1-element int64 CUDA tensor holding the packed first bad
    row (see ``decode_bad_key``); it may be passed in to avoid an allocation.
    ``key_scale`` (optional): float32 CUDA tensor ``[B, Nkv]`` (or ``[Nkv]`` when
    B == 1) of per-key multiplicities, finite and >= 0 -- not validated here
    (``fwd(check=True)`` does, like attention.py:386-387).
    ``kv_splits``: K/V ranges per (b, h) (None: automatic, see ``plan`` -- every work tile when the
    (b, h, 512-row) tiles cannot fill the GPU, or only the last partial wave's tiles); ranges merge
    by plain addition of (numerator, z) (streaming.py:122-128), in a second small kernel.
    ``split_tail`` (with an explicit ``kv_splits``): split only the last partial wave's work tiles.
    With ``partial_only`` the call returns ``(partial, n_parts)`` instead (see ``fwd_partial``).
    ``dev_scales``: float32 CUDA tensor of 4 elements {q, k, v descale, p_scale} read by the kernel
    instead of the host values (written on the device, e.g. by ``prepare``; no host round trip).
    """
    if normalizer not in NORMALIZERS:
        raise ConfigError(f"flashsign: normalizer must be one of {sorted(NORMALIZERS)} (exp-free), got {normalizer!r}")
    if kv_splits is not None and kv_splits < 0:
        raise ConfigError(f"kv_splits must be >= 0, got {kv_splits}")
    # validation, allocation, the split choice and fs_fwd run in the C++ extension (csrc/fs_torch.cpp)
    args = (q, k, v, out, out_dtype, bad_key, float(scale), float(eps), float(p_scale), float(q_descale),
            float(k_descale), float(v_descale), NORMALIZERS[normalizer], key_scale,
            -1 if kv_splits is None else int(kv_splits), partial, bool(partial_only), dev_scales,
            int(tile_hint[0]), int(tile_hint[1]), bool(split_tail))
    global _ext
    ext = _ext or _lib.load_torch_ext()
    _ext = ext
    if stream is None:
        st, msg, o, bad, part, n_parts = ext.fwd(*args)
    else:
        with torch.cuda.stream(stream):  # buffers the call allocates come from `stream` itself
            st, msg, o, bad, part, n_parts = ext.fwd(*args)
    if st:
        raise _STATUS_EXC.get(st, RuntimeError)(f"flashsign: {msg}")
    if partial_only:
        return part, n_parts
    return o, bad


def plan(b: int, h: int, nq: int, nkv: int, device, d: int = 128, dtype: torch.dtype = torch.bfloat16,
         kv_splits: int | None = None, clusters: int = 0, split_tail: bool = False):
    """The split plan ``fwd_async`` would use (C-ABI ``fs_plan``): ``kv_splits=None`` is the automatic
    choice -- the library's wave model of the persistent grid splits the K/V stream of every work tile
    when the (b, h, 512-row) tiles cannot fill the GPU (small batch, long sequence), or only the tiles
    of the last, partial wave (``split_tail``) when a split there shortens the launch.  Returns the
    ``fs_plan_info`` (splits, split_tail, efficiency, ...).  ``clusters`` > 0 plans for that many
    co-resident 2-CTA clusters without touching a device."""
    p = _lib.FsFwdParams()
    p.batch, p.heads_q, p.heads_kv, p.seqlen_q, p.seqlen_kv, p.head_dim = b, h, h, nq, nkv, d
    p.in_dtype = _IN_CODES[dtype]
    p.kv_splits = _lib.FS_SPLITS_AUTO if kv_splits is None else int(kv_splits)
    p.split_tail = int(bool(split_tail))
    if clusters > 0:
        return _lib.plan(p, clusters)
    with torch.cuda.device(torch.device(device)):
        return _lib.plan(p, 0)


def auto_splits(b: int, h: int, nq: int, nkv: int, device, d: int = 128) -> int:
    """K/V splits of the automatic plan (see ``plan``)."""
    return plan(b, h, nq, nkv, device, d).splits


def fwd_partial(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, **kw):
    """Partial FlashSign over this K/V (shard): returns ``(partial, n_parts)`` -- the fp32
    numerators and z of every query row (``include/flashsign.h``: ``partial_only``), to be
    summed across K/V shards (e.g. ``all_reduce``) and normalised by ``combine``."""
    kw.setdefault("kv_splits", 1)
    return fwd_async(q, k, v, partial_only=True, **kw)


def combine(partial: torch.Tensor, n_parts: int, like_q: torch.Tensor, *, out: torch.Tensor | None = None,
            out_dtype: torch.dtype | None = None, eps: float = 0.0, normalizer: str = "spherical",
            bad_key: torch.Tensor | None = None, stream: torch.cuda.Stream | None = None, check: bool = True):
    """O = sum_s num_s / b(sum_s z_s + eps) from (summed) partials of ``fwd_partial``; ``like_q``
    gives the query shape/dtype.  Raises DegenerateDenominatorError when ``check``."""
    if normalizer not in NORMALIZERS:
        raise ConfigError(f"flashsign: normalizer must be one of {sorted(NORMALIZERS)}, got {normalizer!r}")
    b, nq, h, d = like_q.shape
    if out_dtype is None:
        out_dtype = out.dtype if out is not None else (like_q.dtype if like_q.dtype in (torch.bfloat16, torch.float16)
                                                       else torch.bfloat16)
    if out_dtype not in _OUT_CODES or like_q.dtype not in _IN_CODES:
        raise ShapeMismatchError(f"flashsign: unsupported dtypes {like_q.dtype} -> {out_dtype}")
    if out is None:
        out = torch.empty((b, nq, h, d), dtype=out_dtype, device=like_q.device)
    elif (tuple(out.shape) != (b, nq, h, d) or out.dtype != out_dtype or out.stride(-1) != 1
          or out.device != like_q.device):
        raise ShapeMismatchError(f"flashsign: bad out tensor {tuple(out.shape)} {out.dtype}")
    dk = 128 if (like_q.dtype not in (torch.bfloat16, torch.float16) or d > 64) else 64
    need = int(n_parts) * b * h * nq * (dk + 1)
    if (n_parts < 1 or partial.dtype != torch.float32 or not partial.is_contiguous()
            or partial.numel() < need or partial.device != like_q.device):
        raise ShapeMismatchError(f"flashsign: combine needs a contiguous float32 partial of >= {need} elements "
                                 f"({n_parts} parts) on {like_q.device}")
    if bad_key is None:
        bad_key = torch.empty(1, dtype=torch.int64, device=like_q.device)
    prm = _lib.FsFwdParams()
    prm.o = out.data_ptr()
    prm.o_stride[0], prm.o_stride[1], prm.o_stride[2] = out.stride(0), out.stride(1), out.stride(2)
    prm.batch, prm.heads_q, prm.seqlen_q, prm.head_dim = b, h, nq, d
    prm.in_dtype, prm.out_dtype = _IN_CODES[like_q.dtype], _OUT_CODES[out.dtype]
    prm.eps, prm.normalizer = float(eps), NORMALIZERS[normalizer]
    prm.partial, prm.bad_key = partial.data_ptr(), bad_key.data_ptr()
    if stream is None:
        with torch.cuda.device(like_q.device):
            stream = torch.cuda.current_stream()
    with torch.cuda.device(like_q.device):
        st = _lib.load().fs_combine(ctypes.byref(prm), int(n_parts), ctypes.c_void_p(stream.cuda_stream))
    if st != _lib.FS_OK:
        raise _STATUS_EXC.get(st, RuntimeError)(f"flashsign: {_lib.last_error()}")
    if check:
        raise_if_bad(bad_key, h, nq)
    return out


def _padded_rows(ks: torch.Tensor) -> torch.Tensor:
    """Copy ``ks`` into 16-byte-aligned rows (TMA needs 16-byte row strides)."""
    b, n = ks.shape
    buf = torch.zeros((b, max(4, -(-n // 4) * 4)), dtype=torch.float32, device=ks.device)
    buf[:, :n] = ks
    return buf[:, :n]


def check_key_scale(key_scale: torch.Tensor) -> None:
    """attention.py:386-387: multiplicities must be finite and nonnegative (synchronises)."""
    if key_scale.numel() and bool((~torch.isfinite(key_scale) | (key_scale < 0)).any()):
        raise ValueError("multiplicities must be finite and nonnegative")


def decode_bad_key(key: int, heads_q: int, seqlen_q: int):
    """``None`` or ``(batch, head, row, z)`` for a packed bad-row key."""
    key &= 0xFFFFFFFFFFFFFFFF
    if key == BAD_NONE:
        return None
    lin = key >> 32
    z = ctypes.c_float.from_buffer_copy(ctypes.c_uint32(key & 0xFFFFFFFF)).value
    row = lin % seqlen_q
    bh = lin // seqlen_q
    return bh // heads_q, bh % heads_q, row, z


def raise_if_bad(bad_key: torch.Tensor, heads_q: int, seqlen_q: int):
    """Synchronise on ``bad_key`` and raise the reference's error for the first bad row."""
    info = decode_bad_key(int(bad_key.item()), heads_q, seqlen_q)
    if info is not None:
        _, _, row, z = info
        raise DegenerateDenominatorError(float(z), f"row {row}")


def fwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *, scale: float = 1.0, eps: float = 0.0,
        out: torch.Tensor | None = None, out_dtype: torch.dtype | None = None, p_scale: float = 1.0,
        q_descale: float = 1.0, k_descale: float = 1.0, v_descale: float = 1.0, check: bool = True,
        normalizer: str = "spherical", key_scale: torch.Tensor | None = None,
        kv_splits: int | None = None, split_tail: bool = False) -> torch.Tensor:
    """FlashSign forward ``O = c*sum_j s_ij v_j / sqrt(c^2 sum_j s_ij^2 + eps)`` on BSHD CUDA tensors
    (``normalizer="signed_l1"``: ``/ (|c| sum_j |s_ij| + eps)``)."""
    if check and key_scale is not None:
        check_key_scale(key_scale)
    o, bad = fwd_async(q, k, v, scale=scale, eps=eps, out=out, out_dtype=out_dtype, p_scale=p_scale,
                       q_descale=q_descale, k_descale=k_descale, v_descale=v_descale, normalizer=normalizer,
                       key_scale=key_scale, kv_splits=kv_splits, split_tail=split_tail)
    if check:
        raise_if_bad(bad, q.shape[2], q.shape[1])
    return o


def flops(batch: int, heads: int, n_q: int, n_kv: int, d: int) -> int:
    """Algorithmic FLOPs of one forward, 4*B*H*Nq*Nkv*d (costmodel.py:129)."""
    return 4 * batch * heads * n_q * n_kv * d


class CapturedFwd:
    """A FlashSign forward captured once into a CUDA graph and replayed.

    For repeated calls on fixed shapes (e.g. every layer of a GRN forward), the host work of
    ``fwd_async`` -- validation, three TMA descriptor encodes, the bad-row reset and the launch --
    is paid once at capture; ``replay()`` is one graph launch.  Inputs are read from the
    tensors given at construction (copy new data into them); ``out`` / ``bad_key`` are the
    graph's outputs.
    """

    def __init__(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, **kw):
        self.q, self.k, self.v = q, k, v
        side = torch.cuda.Stream(q.device)
        side.wait_stream(torch.cuda.current_stream(q.device))
        with torch.cuda.stream(side):  # warm-up launch outside the capture (loads the module)
            fwd_async(q, k, v, **kw)
        torch.cuda.current_stream(q.device).wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.out, self.bad_key = fwd_async(q, k, v, **kw)

    def replay(self) -> torch.Tensor:
        self.graph.replay()
        return self.out


_SRC_CODES = {torch.float32: _lib.FS_F32, torch.float64: _lib.FS_F64, torch.float16: _lib.FS_F16,
              torch.bfloat16: _lib.FS_BF16}


def prepare(srcs, dsts, *, stats: torch.Tensor, scales: torch.Tensor, scale: float = 1.0, eps: float = 0.0,
            normalizer: str = "spherical", exact: bool = False, stream: torch.cuda.Stream | None = None) -> None:
    """Convert caller tensors to kernel operands with device-chosen power-of-two scales (C-ABI
    ``fs_prepare``, include/flashsign.h).  ``srcs`` / ``dsts``: three entries (q, k, v), each a 2-D
    CUDA tensor ``[rows, d]`` / ``[rows, d_pad]`` with unit column stride, or ``None`` to reuse that
    slot's stats from an earlier call on the same ``stats`` workspace (float64, 6 elements).
    ``scales`` (float32, 4 elements) receives {q, k, v descale, p_scale} for ``fwd_async(dev_scales=)``.
    Async on ``stream`` (default: current)."""
    prm = _lib.FsPrepParams()
    dst_dtype = d_pad = dev = None
    for i, (x, y) in enumerate(zip(srcs, dsts)):
        if x is None:
            continue
        if x.dim() != 2 or y is None or y.dim() != 2 or x.stride(1) != 1 or y.stride(1) != 1:
            raise ShapeMismatchError("flashsign.prepare: 2-D tensors with unit column stride expected")
        if x.dtype not in _SRC_CODES or y.dtype not in _IN_CODES or x.shape[0] != y.shape[0]:
            raise ShapeMismatchError(f"flashsign.prepare: bad dtypes/rows {x.dtype} {tuple(x.shape)} -> "
                                     f"{y.dtype} {tuple(y.shape)}")
        if dst_dtype is not None and (y.dtype != dst_dtype or y.shape[1] != d_pad):
            raise ShapeMismatchError("flashsign.prepare: every operand must share dtype and padded width")
        dst_dtype, d_pad, dev = y.dtype, y.shape[1], x.device
        t = prm.t[i]
        t.src, t.src_dtype, t.d, t.rows = x.data_ptr(), _SRC_CODES[x.dtype], x.shape[1], x.shape[0]
        t.src_row_stride, t.dst, t.dst_row_stride = x.stride(0), y.data_ptr(), y.stride(0)
    if dst_dtype is None:
        raise ShapeMismatchError("flashsign.prepare: no tensor given")
    if stats.dtype != torch.float64 or stats.numel() < 6 or scales.dtype != torch.float32 or scales.numel() < 4:
        raise ShapeMismatchError("flashsign.prepare: stats float64[6] and scales float32[4] workspaces expected")
    prm.dst_dtype, prm.d_pad = _IN_CODES[dst_dtype], d_pad
    prm.mode = _lib.FS_PREP_EXACT if exact else _lib.FS_PREP_SCALE
    prm.normalizer = NORMALIZERS[normalizer]
    prm.scale, prm.eps = float(scale), float(eps)
    prm.stats, prm.scales = stats.data_ptr(), scales.data_ptr()
    with torch.cuda.device(dev):
        s = stream if stream is not None else torch.cuda.current_stream()
        st = _lib.load().fs_prepare(ctypes.byref(prm), ctypes.c_void_p(s.cuda_stream))
    if st != _lib.FS_OK:
        raise _STATUS_EXC.get(st, RuntimeError)(f"flashsign: {_lib.last_error()}")


def kernel_score_tile(head_dim: int, dtype: torch.dtype = torch.bfloat16) -> int:
    """Scores the kernel holds on chip per Q tile (128 rows x 128 / 192 keys, in TMEM)."""
    bm, bn = _lib.query_tile(min(max(head_dim, 1), 128), _IN_CODES[dtype])
    return bm * bn


def _params_of(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out: torch.Tensor, scale: float, eps: float):
    p = _lib.FsFwdParams()
    p.q, p.k, p.v, p.o = q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr()
    for dst, t in ((p.q_stride, q), (p.k_stride, k), (p.v_stride, v), (p.o_stride, out)):
        dst[0], dst[1], dst[2] = t.stride(0), t.stride(1), t.stride(2)
    p.batch, p.heads_q, p.heads_kv = q.shape[0], q.shape[2], k.shape[2]
    p.seqlen_q, p.seqlen_kv, p.head_dim = q.shape[1], k.shape[1], q.shape[3]
    p.in_dtype, p.out_dtype = _IN_CODES[q.dtype], _OUT_CODES[out.dtype]
    p.scale, p.eps, p.p_scale, p.q_descale, p.k_descale, p.v_descale = float(scale), float(eps), 1.0, 1.0, 1.0, 1.0
    return p


def scale_keys(k: torch.Tensor, key_scale: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """K' = m K (attention.py:381-388, grn.py:150) for 16-bit BSHD keys in one HBM pass (C-ABI
    ``fs_scale_keys``): ``key_scale`` float32 ``[B, Nkv]``; fp32 product, then round to nearest even."""
    if k.dtype not in (torch.bfloat16, torch.float16) or not k.is_cuda or k.dim() != 4 or k.stride(-1) != 1:
        raise ShapeMismatchError("scale_keys: 16-bit BSHD CUDA keys with a contiguous head dim expected")
    ks = key_scale.reshape(k.shape[0], -1) if key_scale.dim() == 1 else key_scale
    if (ks.dtype != torch.float32 or tuple(ks.shape) != (k.shape[0], k.shape[1]) or ks.device != k.device
            or (k.shape[1] > 0 and ks.stride(1) != 1)):
        raise ShapeMismatchError("scale_keys: key_scale must be float32 [B, Nkv] on k's device")
    if out is None:
        out = torch.empty(k.shape, dtype=k.dtype, device=k.device)
    p = _params_of(k, k, k, k, 1.0, 0.0)
    p.key_scale, p.key_scale_stride = ks.data_ptr(), ks.stride(0)
    ost = (ctypes.c_int64 * 3)(out.stride(0), out.stride(1), out.stride(2))
    with torch.cuda.device(k.device):
        st = _lib.load().fs_scale_keys(ctypes.byref(p), ctypes.c_void_p(out.data_ptr()), ost,
                                       ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    if st != _lib.FS_OK:
        raise _STATUS_EXC.get(st, RuntimeError)(f"flashsign: {_lib.last_error()}")
    return out


def gram_fwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *, scale: float = 1.0, eps: float = 0.0,
             out: torch.Tensor | None = None, out_dtype: torch.dtype | None = None,
             key_scale: torch.Tensor | None = None, check: bool = True,
             bad_key: torch.Tensor | None = None) -> torch.Tensor:
    """Spherical attention through its Gram (moment) form, C-ABI ``fs_gram_fwd`` (SURVEY.md section 0
    fact 4): ``O_i = c q_i^T W / sqrt(c^2 q_i^T G q_i + eps)`` with ``G = K^T K``, ``W = K^T V`` per
    (b, h_kv) -- the FlashSign contract (normalizers.py:94-100) at O(N d^2), three tensor-core
    launches, HBM-bound.  16-bit BSHD inputs, spherical normaliser; ``key_scale`` multiplicities are
    applied as K' = m K first (``scale_keys``).  ``check`` raises DegenerateDenominatorError for the
    first bad row like ``fwd``."""
    _check_inputs(q, k, v)
    if q.dtype not in (torch.bfloat16, torch.float16):
        raise ShapeMismatchError(f"gram_fwd: 16-bit inputs only, got {q.dtype}")
    if q.shape[2] % k.shape[2]:
        raise ConfigError(f"query heads must be a multiple of kv heads, got h={q.shape[2]}, h_kv={k.shape[2]}")
    if key_scale is not None:
        if check:
            check_key_scale(key_scale)
        k = scale_keys(k, key_scale)
    if out_dtype is None:
        out_dtype = out.dtype if out is not None else q.dtype
    if out is None:
        out = torch.empty(q.shape, dtype=out_dtype, device=q.device)
    elif tuple(out.shape) != tuple(q.shape) or out.dtype != out_dtype or out.stride(-1) != 1:
        raise ShapeMismatchError(f"gram_fwd: bad out tensor {tuple(out.shape)} {out.dtype}")
    if bad_key is None:
        bad_key = torch.empty(1, dtype=torch.int64, device=q.device)
    p = _params_of(q, k, v, out, scale, eps)
    p.bad_key = bad_key.data_ptr()
    lib = _lib.load()
    with torch.cuda.device(q.device):
        nbytes = int(lib.fs_gram_workspace_bytes(ctypes.byref(p)))
        ws = torch.empty(max(nbytes, 256) + 256, dtype=torch.uint8, device=q.device)
        base = (ws.data_ptr() + 255) & ~255
        st = lib.fs_gram_fwd(ctypes.byref(p), ctypes.c_void_p(base), ctypes.c_int64(nbytes),
                             ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    if st != _lib.FS_OK:
        raise _STATUS_EXC.get(st, RuntimeError)(f"flashsign: {_lib.last_error()}")
    if check:
        raise_if_bad(bad_key, q.shape[2], q.shape[1])
    return out
