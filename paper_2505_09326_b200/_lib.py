"""ctypes binding of the FlashSign C-ABI (``include/flashsign.h``).

The shared library ``_lib/libflashsign.so`` is built in-tree by
``paper_2505_09326_b200/build.py`` (nvcc, sm_100a).  There is no fallback:
if the library is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libflashsign.so")

FS_OK, FS_ERR_SHAPE, FS_ERR_CONFIG, FS_ERR_DTYPE, FS_ERR_UNSUPPORTED, FS_ERR_CUDA = range(6)
FS_F16, FS_BF16, FS_E4M3, FS_F32, FS_F64 = range(5)
FS_PREP_SCALE, FS_PREP_EXACT = range(2)
FS_NORM_SPHERICAL, FS_NORM_SIGNED_L1 = range(2)
FS_BAD_NONE = 0xFFFFFFFFFFFFFFFF

# every symbol include/flashsign.h declares
EXPORTED_SYMBOLS = ("fs_fwd", "fs_last_error", "fs_query_tile", "fs_version", "fs_kv_splits", "fs_partial_floats",
                    "fs_combine", "fs_peer_floats", "fs_fwd_peer", "fs_combine_peer", "fs_ipc_malloc", "fs_ipc_open",
                    "fs_ipc_close", "fs_ipc_free", "fs_prepare", "fs_plan", "fs_scale_keys",
                    "fs_gram_workspace_bytes", "fs_gram_fwd", "fs_exact_fwd", "fs_host_copy")
FS_SPLITS_AUTO = -1


class FsFwdParams(ctypes.Structure):
    """Mirror of ``fs_fwd_params`` (include/flashsign.h)."""

    _fields_ = [
        ("q", ctypes.c_void_p),
        ("k", ctypes.c_void_p),
        ("v", ctypes.c_void_p),
        ("o", ctypes.c_void_p),
        ("q_stride", ctypes.c_int64 * 3),
        ("k_stride", ctypes.c_int64 * 3),
        ("v_stride", ctypes.c_int64 * 3),
        ("o_stride", ctypes.c_int64 * 3),
        ("batch", ctypes.c_int32),
        ("heads_q", ctypes.c_int32),
        ("heads_kv", ctypes.c_int32),
        ("seqlen_q", ctypes.c_int32),
        ("seqlen_kv", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("in_dtype", ctypes.c_int32),
        ("out_dtype", ctypes.c_int32),
        ("scale", ctypes.c_float),
        ("eps", ctypes.c_float),
        ("p_scale", ctypes.c_float),
        ("q_descale", ctypes.c_float),
        ("k_descale", ctypes.c_float),
        ("v_descale", ctypes.c_float),
        ("bad_key", ctypes.c_void_p),
        ("tile_m_hint", ctypes.c_int32),
        ("tile_n_hint", ctypes.c_int32),
        ("normalizer", ctypes.c_int32),
        ("kv_splits", ctypes.c_int32),
        ("key_scale", ctypes.c_void_p),
        ("key_scale_stride", ctypes.c_int64),
        ("partial", ctypes.c_void_p),
        ("partial_only", ctypes.c_int32),
        ("split_tail", ctypes.c_int32),
        ("dev_scales", ctypes.c_void_p),
    ]


class FsPlanInfo(ctypes.Structure):
    """Mirror of ``fs_plan_info`` (include/flashsign.h)."""

    _fields_ = [
        ("splits", ctypes.c_int32),
        ("split_tail", ctypes.c_int32),
        ("clusters", ctypes.c_int32),
        ("n_whole", ctypes.c_int32),
        ("tail_tiles", ctypes.c_int32),
        ("n_kv_tiles", ctypes.c_int32),
        ("work_tiles", ctypes.c_int64),
        ("items", ctypes.c_int64),
        ("partial_floats", ctypes.c_int64),
        ("busiest_steps", ctypes.c_double),
        ("efficiency", ctypes.c_double),
    ]


class FsExactParams(ctypes.Structure):
    """Mirror of ``fs_exact_params`` (include/flashsign.h)."""

    _fields_ = [
        ("q", ctypes.c_void_p),
        ("k", ctypes.c_void_p),
        ("v", ctypes.c_void_p),
        ("o", ctypes.c_void_p),
        ("q_stride", ctypes.c_int64 * 3),
        ("k_stride", ctypes.c_int64 * 3),
        ("v_stride", ctypes.c_int64 * 3),
        ("o_stride", ctypes.c_int64 * 3),
        ("batch", ctypes.c_int32),
        ("heads_q", ctypes.c_int32),
        ("heads_kv", ctypes.c_int32),
        ("seqlen_q", ctypes.c_int32),
        ("seqlen_kv", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("scale", ctypes.c_double),
        ("eps", ctypes.c_double),
        ("normalizer", ctypes.c_int32),
        ("f32_grid", ctypes.c_int32),
        ("bad_key", ctypes.c_void_p),
        ("z_out", ctypes.c_void_p),
    ]


class FsPeerParams(ctypes.Structure):
    """Mirror of ``fs_peer_params`` (include/flashsign.h)."""

    _fields_ = [
        ("world", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("rows_per_rank", ctypes.c_int32),
        ("reserved0", ctypes.c_int32),
        ("peer_partial", ctypes.c_void_p),
        ("local_partial", ctypes.c_void_p),
    ]


class FsPrepTensor(ctypes.Structure):
    """Mirror of ``fs_prep_tensor`` (include/flashsign.h)."""

    _fields_ = [
        ("src", ctypes.c_void_p),
        ("src_dtype", ctypes.c_int32),
        ("d", ctypes.c_int32),
        ("rows", ctypes.c_int64),
        ("src_row_stride", ctypes.c_int64),
        ("dst", ctypes.c_void_p),
        ("dst_row_stride", ctypes.c_int64),
    ]


class FsPrepParams(ctypes.Structure):
    """Mirror of ``fs_prep_params`` (include/flashsign.h)."""

    _fields_ = [
        ("t", FsPrepTensor * 3),
        ("dst_dtype", ctypes.c_int32),
        ("d_pad", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("normalizer", ctypes.c_int32),
        ("scale", ctypes.c_float),
        ("eps", ctypes.c_float),
        ("stats", ctypes.c_void_p),
        ("scales", ctypes.c_void_p),
    ]


IPC_HANDLE_BYTES = 64

_lock = threading.RLock()  # load_torch_ext() calls load() while holding it
_lib = None


def load() -> ctypes.CDLL:
    """Load (once) and return the FlashSign library; raise loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"FlashSign CUDA library not built: {LIB_PATH} is missing. "
                    "Run `python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)."
                )
            lib = ctypes.CDLL(LIB_PATH)
            lib.fs_fwd.argtypes = [ctypes.POINTER(FsFwdParams), ctypes.c_void_p]
            lib.fs_fwd.restype = ctypes.c_int
            lib.fs_last_error.argtypes = []
            lib.fs_last_error.restype = ctypes.c_char_p
            lib.fs_query_tile.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                          ctypes.POINTER(ctypes.c_int)]
            lib.fs_query_tile.restype = ctypes.c_int
            lib.fs_version.argtypes = []
            lib.fs_version.restype = ctypes.c_int
            lib.fs_kv_splits.argtypes = [ctypes.POINTER(FsFwdParams)]
            lib.fs_kv_splits.restype = ctypes.c_int32
            lib.fs_partial_floats.argtypes = [ctypes.POINTER(FsFwdParams)]
            lib.fs_partial_floats.restype = ctypes.c_int64
            lib.fs_combine.argtypes = [ctypes.POINTER(FsFwdParams), ctypes.c_int32, ctypes.c_void_p]
            lib.fs_combine.restype = ctypes.c_int
            pp, fp = ctypes.POINTER(FsPeerParams), ctypes.POINTER(FsFwdParams)
            lib.fs_peer_floats.argtypes = [fp, pp]
            lib.fs_peer_floats.restype = ctypes.c_int64
            lib.fs_fwd_peer.argtypes = [fp, pp, ctypes.c_void_p]
            lib.fs_fwd_peer.restype = ctypes.c_int
            lib.fs_combine_peer.argtypes = [fp, pp, ctypes.c_void_p]
            lib.fs_combine_peer.restype = ctypes.c_int
            lib.fs_ipc_malloc.argtypes = [ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p), ctypes.c_void_p]
            lib.fs_ipc_malloc.restype = ctypes.c_int
            lib.fs_ipc_open.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
            lib.fs_ipc_open.restype = ctypes.c_int
            lib.fs_ipc_close.argtypes = [ctypes.c_void_p]
            lib.fs_ipc_close.restype = ctypes.c_int
            lib.fs_ipc_free.argtypes = [ctypes.c_void_p]
            lib.fs_ipc_free.restype = ctypes.c_int
            lib.fs_prepare.argtypes = [ctypes.POINTER(FsPrepParams), ctypes.c_void_p]
            lib.fs_prepare.restype = ctypes.c_int
            lib.fs_plan.argtypes = [ctypes.POINTER(FsFwdParams), ctypes.c_int32, ctypes.POINTER(FsPlanInfo)]
            lib.fs_plan.restype = ctypes.c_int
            lib.fs_scale_keys.argtypes = [ctypes.POINTER(FsFwdParams), ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64),
                                          ctypes.c_void_p]
            lib.fs_scale_keys.restype = ctypes.c_int
            lib.fs_gram_workspace_bytes.argtypes = [ctypes.POINTER(FsFwdParams)]
            lib.fs_gram_workspace_bytes.restype = ctypes.c_int64
            lib.fs_gram_fwd.argtypes = [ctypes.POINTER(FsFwdParams), ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
            lib.fs_gram_fwd.restype = ctypes.c_int
            lib.fs_exact_fwd.argtypes = [ctypes.POINTER(FsExactParams), ctypes.c_void_p]
            lib.fs_exact_fwd.restype = ctypes.c_int
            _lib = lib
    return _lib


TORCH_EXT_PATH = os.path.join(_HERE, "_lib", "fs_torch.so")
_ext = None


def load_torch_ext():
    """The PyTorch C++ extension over the C-ABI (csrc/fs_torch.cpp, built in-tree by build.py);
    raises loudly if it is missing -- there is no fallback."""
    global _ext
    if _ext is not None:
        return _ext
    with _lock:
        if _ext is None:
            if not os.path.exists(TORCH_EXT_PATH):
                raise RuntimeError(f"FlashSign torch extension not built: {TORCH_EXT_PATH} is missing. "
                                   "Run `python -c 'import __graft_entry__ as g; g.build()'`.")
            import importlib.machinery
            import importlib.util

            import torch  # noqa: F401  (libtorch / libc10 symbols first)

            load()  # libflashsign.so (the extension's $ORIGIN dependency) through the same path
            loader = importlib.machinery.ExtensionFileLoader("fs_torch", TORCH_EXT_PATH)
            spec = importlib.util.spec_from_loader("fs_torch", loader)
            mod = importlib.util.module_from_spec(spec)
            loader.exec_module(mod)
            _ext = mod
    return _ext


def last_error() -> str:
    return load().fs_last_error().decode("utf-8", "replace")


def plan(p: FsFwdParams, clusters: int = 0) -> FsPlanInfo:
    """``fs_plan``: the split plan and wave-model efficiency of a launch (clusters > 0: host only)."""
    info = FsPlanInfo()
    if load().fs_plan(ctypes.byref(p), int(clusters), ctypes.byref(info)) != FS_OK:
        raise ValueError(f"fs_plan: {last_error()}")
    return info


def query_tile(head_dim: int, dtype_code: int) -> tuple[int, int]:
    bm, bn = ctypes.c_int(0), ctypes.c_int(0)
    if load().fs_query_tile(head_dim, dtype_code, ctypes.byref(bm), ctypes.byref(bn)) != 0:
        raise ValueError(f"no FlashSign tile for head_dim={head_dim} dtype={dtype_code}")
    return bm.value, bn.value
