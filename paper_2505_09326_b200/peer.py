"""Context parallelism over peer memory: the FlashSign partials go straight to their owner.

Spherical (and signed-L1) partials over disjoint key ranges merge by plain addition
(streaming.py:122-128; Lemma 1).  ``partition.context_parallel_fwd``
all-reduces the whole (numerator, z) workspace with NCCL; here instead every rank owns the
query positions ``[rank*R, rank*R + R)`` (``R = ceil(Nq / world)``) and the kernel's epilogue
stores each row's partial directly into the owner's workspace (``fs_fwd_peer``: NVLink P2P
stores into CUDA-IPC-mapped peer memory, one slot per source rank).  After one host barrier
the owner adds the ``world`` slots of its rows and normalises them (``fs_combine_peer``).
Per rank, (world-1)/world of the partials cross the link once -- a reduce-scatter fused into
the producing kernel -- and no collective library call sits on the data path.

The result is sequence-sharded like the input keys: rank r's ``out[:, lo:hi]`` (positions
``peer_rows(Nq, world, r)``); ``gather=True`` all-gathers O onto every rank afterwards.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._errors import ConfigError
from .tensor import ShapeMismatchError


def peer_rows(nq: int, world: int, rank: int) -> tuple[int, int]:
    """Query positions [lo, hi) owned by ``rank``: contiguous ranges of ceil(nq / world)."""
    r = max(1, -(-nq // world))
    lo = min(nq, rank * r)
    return lo, min(nq, lo + r)


class PeerWorkspace:
    """An fp32 workspace per rank, mapped into every rank of ``group`` through CUDA IPC.

    ``table`` is the device array of the ``world`` workspace pointers the kernel stores into;
    ``local`` is this rank's own.  Collective to create and to ``close``."""

    def __init__(self, nfloats: int, group=None, device: torch.device | None = None):
        import torch.distributed as dist

        self.lib = _lib.load()
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.nfloats = int(nfloats)
        handle = (ctypes.c_char * _lib.IPC_HANDLE_BYTES)()
        ptr = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            self._check(self.lib.fs_ipc_malloc(4 * self.nfloats, ctypes.byref(ptr), handle))
            self.local = ptr.value
            handles = [bytes(handle)]
            if self.world > 1:
                handles = [None] * self.world
                dist.all_gather_object(handles, bytes(handle), group=group)
            self.opened = []
            ptrs = []
            for r, h in enumerate(handles):
                if r == self.rank:
                    ptrs.append(self.local)
                    continue
                buf = (ctypes.c_char * _lib.IPC_HANDLE_BYTES).from_buffer_copy(h)
                p = ctypes.c_void_p()
                self._check(self.lib.fs_ipc_open(buf, ctypes.byref(p)))
                self.opened.append(p.value)
                ptrs.append(p.value)
            self.table = torch.tensor(ptrs, dtype=torch.int64, device=self.device)

    def _check(self, st):
        if st != _lib.FS_OK:
            raise RuntimeError(f"flashsign peer workspace: {_lib.last_error()}")

    def close(self):
        """Unmap the peers' workspaces, wait for every rank, free this one (collective)."""
        import torch.distributed as dist

        if self.local is None:
            return
        with torch.cuda.device(self.device):
            torch.cuda.synchronize()
            for p in self.opened:
                self._check(self.lib.fs_ipc_close(ctypes.c_void_p(p)))
            self.opened = []
            if self.world > 1:
                dist.barrier(group=self.group)
            self._check(self.lib.fs_ipc_free(ctypes.c_void_p(self.local)))
        self.local = None


_workspaces: dict = {}


def _params(q, k, v, out, scale, eps, normalizer, bad_key):
    from . import flashsign

    prm = _lib.FsFwdParams()
    prm.q, prm.k, prm.v, prm.o = q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr()
    for dst, t in ((prm.q_stride, q), (prm.k_stride, k), (prm.v_stride, v), (prm.o_stride, out)):
        dst[0], dst[1], dst[2] = t.stride(0), t.stride(1), t.stride(2)
    b, nq, h, d = q.shape
    prm.batch, prm.heads_q, prm.heads_kv = b, h, k.shape[2]
    prm.seqlen_q, prm.seqlen_kv, prm.head_dim = nq, k.shape[1], d
    prm.in_dtype, prm.out_dtype = flashsign._IN_CODES[q.dtype], flashsign._OUT_CODES[out.dtype]
    prm.scale, prm.eps, prm.p_scale = float(scale), float(eps), 1.0
    prm.q_descale = prm.k_descale = prm.v_descale = 1.0
    prm.bad_key = bad_key.data_ptr()
    prm.normalizer = flashsign.NORMALIZERS[normalizer]
    prm.kv_splits = 1
    return prm


def context_parallel_fwd_peer(q: torch.Tensor, k_shard: torch.Tensor, v_shard: torch.Tensor, group=None, *,
                              scale: float = 1.0, eps: float = 0.0, normalizer: str = "spherical",
                              out: torch.Tensor | None = None, out_dtype: torch.dtype | None = None,
                              check: bool = True, gather: bool = False) -> tuple[torch.Tensor, tuple[int, int]]:
    """Sequence-parallel FlashSign with the partial reduction done by peer stores.

    Every rank passes all of ``q`` and its contiguous K/V shard (``partition.kv_shard_range``).
    Returns ``(out, (lo, hi))``: ``out[:, lo:hi]`` holds this rank's query positions (the rest
    of ``out`` is untouched unless ``gather``).  Raises ``DegenerateDenominatorError`` for the
    first bad row among this rank's positions when ``check``."""
    import torch.distributed as dist

    from . import flashsign

    flashsign._check_inputs(q, k_shard, v_shard)
    if normalizer not in flashsign.NORMALIZERS:
        raise ConfigError(f"flashsign: normalizer must be one of {sorted(flashsign.NORMALIZERS)}, got {normalizer!r}")
    b, nq, h, d = q.shape
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if out_dtype is None:
        out_dtype = out.dtype if out is not None else (q.dtype if q.dtype in (torch.bfloat16, torch.float16)
                                                       else torch.bfloat16)
    if out is None:
        out = torch.empty((b, nq, h, d), dtype=out_dtype, device=q.device)
    elif tuple(out.shape) != (b, nq, h, d) or out.dtype != out_dtype or out.stride(-1) != 1:
        raise ShapeMismatchError(f"flashsign: bad out tensor {tuple(out.shape)} {out.dtype}")
    bad = torch.empty(1, dtype=torch.int64, device=q.device)
    prm = _params(q, k_shard, v_shard, out, scale, eps, normalizer, bad)
    pp = _lib.FsPeerParams()
    pp.world, pp.rank, pp.rows_per_rank = world, rank, max(1, -(-nq // world))
    lib = _lib.load()
    nfloats = int(lib.fs_peer_floats(ctypes.byref(prm), ctypes.byref(pp)))
    # two workspaces used alternately: a rank may store call i+1's partials into a peer while
    # that peer still reads call i's -- each call's single barrier then suffices
    key = (q.device, id(group), nfloats)
    ent = _workspaces.get(key)
    if ent is None:
        ent = _workspaces[key] = [[PeerWorkspace(nfloats, group, q.device), PeerWorkspace(nfloats, group, q.device)],
                                  0]
    ws = ent[0][ent[1]]
    ent[1] ^= 1
    pp.peer_partial, pp.local_partial = ws.table.data_ptr(), ws.local
    with torch.cuda.device(q.device):
        stream = torch.cuda.current_stream()
        st = lib.fs_fwd_peer(ctypes.byref(prm), ctypes.byref(pp), ctypes.c_void_p(stream.cuda_stream))
        if st != _lib.FS_OK:
            raise flashsign._STATUS_EXC.get(st, RuntimeError)(f"flashsign: {_lib.last_error()}")
        stream.synchronize()  # this rank's stores into the owners' workspaces are complete
        if world > 1:
            dist.barrier(group=group)  # ... and every other rank's into this one
        st = lib.fs_combine_peer(ctypes.byref(prm), ctypes.byref(pp), ctypes.c_void_p(stream.cuda_stream))
        if st != _lib.FS_OK:
            raise flashsign._STATUS_EXC.get(st, RuntimeError)(f"flashsign: {_lib.last_error()}")
    lo, hi = peer_rows(nq, world, rank)
    # collectives first, on every rank, before anything may raise (no rank can leave the others
    # blocked in all_gather / all_reduce)
    if gather and world > 1:
        r = pp.rows_per_rank
        mine = torch.zeros((b, r, h, d), dtype=out.dtype, device=out.device)
        mine[:, :hi - lo] = out[:, lo:hi]
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine, group=group)
        for src, part in enumerate(parts):
            plo, phi = peer_rows(nq, world, src)
            out[:, plo:phi] = part[:, :phi - plo]
    if check:
        key = bad
        if world > 1:
            # every rank raises for the same, globally first bad row: MIN over the packed keys,
            # compared unsigned (xor of the sign bit maps unsigned order onto signed order)
            flip = torch.iinfo(torch.int64).min
            key = torch.bitwise_xor(bad, flip)
            dist.all_reduce(key, op=dist.ReduceOp.MIN, group=group)
            key = torch.bitwise_xor(key, flip)
        info = flashsign.decode_bad_key(int(key.item()), h, nq)
        if info is not None:
            from .normalizers import DegenerateDenominatorError
            raise DegenerateDenominatorError(float(info[3]), f"row {info[2]}")
    return out, (lo, hi)


def release_workspaces():
    """Free the cached peer workspaces (collective over the groups they were made for)."""
    for ent in list(_workspaces.values()):
        for ws in ent[0]:
            ws.close()
    _workspaces.clear()
