"""FlashSign on host-resident inputs: chunked H2D -> kernel -> D2H with overlap.

``fwd_host(q, k, v, out)`` takes pinned CPU tensors in BSHD layout (the
compute dtype, e.g. bf16) and streams them through the GPU on three CUDA
streams -- copy-in, compute, copy-out -- so PCIe transfers overlap the kernel.
The unit of the pipeline is a query slice of one batch chunk (``chunk`` batch rows, by
default one row of >= 64 MB of K/V, else >= 2 rows and >= 32 MB): K/V of the batch
chunk go over first, then its queries in ``q_split`` row slices, each launched
as soon as it lands, so the pipeline fills after ~1/(chunks * q_split) of the
data instead of a whole batch row and drains after one slice.  Device staging
buffers are double-buffered and reused across calls (``HostPipeline``).

This is the end-to-end path a caller with host data uses (what the reference's
numpy API amounts to); the bench reports it as ``e2e``.
"""

from __future__ import annotations

import torch

from . import flashsign


class HostPipeline:
    """Reusable device staging for ``fwd_host`` (two slots per tensor)."""

    # batch rows per chunk when not given: one row when its K/V copies are >= 64 MB, else at least
    # two rows and >= 32 MB (short copies leave the link idle between them; measured C2 +7 %,
    # C5 +4 % with two rows per chunk, C3 best with one)
    KV_CHUNK_BYTES = 32 << 20
    KV_ROW_ALONE_BYTES = 64 << 20

    def __init__(self, device: torch.device | int | None = None, chunk: int | None = None,
                 q_split: int | None = None):
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else
                                   (device if isinstance(device, int) else device.index))
        self.chunk = chunk
        self.q_split = q_split
        self._sms = None
        self._shape_key = None
        self.s_in = torch.cuda.Stream(self.device)
        self.s_cmp = torch.cuda.Stream(self.device)
        self.s_out = torch.cuda.Stream(self.device)

    def _slices(self, nq: int, heads: int = 1, last: bool = False) -> list[tuple[int, int]]:
        # Query slices: as many as keep >= 3 full waves of work tiles per launch (at most 4), so
        # slicing shortens the pipeline's fill/drain without leaving SMs idle in a launch's tail.
        # The last batch chunk is cut finer (8 slices): once the final input bytes have crossed
        # the link, only its last slice's kernel and output copy remain (the drain).
        if self.q_split is not None:
            qs = self.q_split
        elif last:
            qs = 8
        else:
            if self._sms is None:
                self._sms = torch.cuda.get_device_properties(self.device).multi_processor_count
            tiles = self._c * heads * -(-nq // 256)
            qs = max(1, min(4, tiles // (3 * self._sms)))
        step = -(-nq // qs)
        step = -(-step // 256) * 256  # whole 256-row work tiles
        return [(n0, min(nq, n0 + step)) for n0 in range(0, nq, step)] or [(0, 0)]

    def _alloc(self, q, k, out, key_scale=None):
        sl = self._slices(q.shape[1], q.shape[2])
        qmax = max(b - a for a, b in sl)
        key = (tuple(q.shape[1:]), tuple(k.shape[1:]), q.dtype, out.dtype, self._c, qmax,
               None if key_scale is None else tuple(key_scale.shape[1:]))
        if key == self._shape_key:
            return
        c = self._c
        dev = self.device
        qs = (c, qmax) + tuple(q.shape[2:])
        self.dq = [torch.empty(qs, dtype=q.dtype, device=dev) for _ in range(2)]
        self.dk = [torch.empty((c,) + tuple(k.shape[1:]), dtype=k.dtype, device=dev) for _ in range(2)]
        self.dv = [torch.empty((c,) + tuple(k.shape[1:]), dtype=k.dtype, device=dev) for _ in range(2)]
        self.do = [torch.empty(qs, dtype=out.dtype, device=dev) for _ in range(2)]
        self.dm = None if key_scale is None else [
            torch.empty((c,) + tuple(key_scale.shape[1:]), dtype=torch.float32, device=dev) for _ in range(2)]
        self._shape_key = key

    def run(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out: torch.Tensor, *, scale: float = 1.0,
            eps: float = 0.0, check: bool = True, key_scale: torch.Tensor | None = None, **kw) -> torch.Tensor:
        """O = FlashSign(q, k, v) for host tensors; returns ``out`` (host) after synchronising.
        ``key_scale``: optional host float32 [B, Nkv] key multiplicities (validated when ``check``)."""
        if q.is_cuda or k.is_cuda or v.is_cuda or out.is_cuda or (key_scale is not None and key_scale.is_cuda):
            raise ValueError("fwd_host expects host (CPU) tensors; use flashsign.fwd for device tensors")
        if check and key_scale is not None:
            flashsign.check_key_scale(key_scale)
        row_kv = 2 * k[0].numel() * k.element_size()
        auto = 1 if row_kv >= self.KV_ROW_ALONE_BYTES else max(2, -(-self.KV_CHUNK_BYTES // max(row_kv, 1)))
        self._c = self.chunk or max(1, min(q.shape[0], auto))
        self._alloc(q, k, out, key_scale)
        c = self._c
        nb, nq, h = q.shape[0], q.shape[1], q.shape[2]
        slices = self._slices(nq, h)
        tail = self._slices(nq, h, last=True)
        ev_q_free = [None, None]     # compute done with Q slot / O slot producer side
        ev_o_free = [None, None]     # D2H of O slot done
        ev_kv_free = [None, None]    # last compute of a batch chunk done with its K/V slot
        bad_hits = []
        g = 0                        # global slice counter -> Q / O slot
        with torch.cuda.device(self.device):
            for ci, b0 in enumerate(range(0, nb, c)):
                kvs = ci & 1
                b1 = min(b0 + c, nb)
                n = b1 - b0
                ev_kv = torch.cuda.Event()
                with torch.cuda.stream(self.s_in):
                    if ev_kv_free[kvs] is not None:
                        self.s_in.wait_event(ev_kv_free[kvs])
                    self.dk[kvs][:n].copy_(k[b0:b1], non_blocking=True)
                    self.dv[kvs][:n].copy_(v[b0:b1], non_blocking=True)
                    if key_scale is not None:
                        self.dm[kvs][:n].copy_(key_scale[b0:b1], non_blocking=True)
                    ev_kv.record(self.s_in)
                for (n0, n1) in (tail if b1 >= nb and nb > c else slices):
                    s = g & 1
                    g += 1
                    nn = n1 - n0
                    ev_in = torch.cuda.Event()
                    with torch.cuda.stream(self.s_in):
                        if ev_q_free[s] is not None:
                            self.s_in.wait_event(ev_q_free[s])
                        # per batch row: a query slice of several rows is not contiguous on the
                        # host, and a strided pinned copy is neither asynchronous nor fast
                        for i in range(n):
                            self.dq[s][i, :nn].copy_(q[b0 + i, n0:n1], non_blocking=True)
                        ev_in.record(self.s_in)
                    ev_cmp = torch.cuda.Event()
                    with torch.cuda.stream(self.s_cmp):
                        self.s_cmp.wait_event(ev_kv)
                        self.s_cmp.wait_event(ev_in)
                        if ev_o_free[s] is not None:  # slot s's previous output has left the device
                            self.s_cmp.wait_event(ev_o_free[s])
                        _, bad = flashsign.fwd_async(self.dq[s][:n, :nn], self.dk[kvs][:n], self.dv[kvs][:n],
                                                     scale=scale, eps=eps, out=self.do[s][:n, :nn],
                                                     stream=self.s_cmp,
                                                     key_scale=None if key_scale is None else self.dm[kvs][:n],
                                                     **kw)
                        if check:
                            bad_hits.append((b0, n0, nn, bad))
                        ev_cmp.record(self.s_cmp)
                    ev_q_free[s] = ev_cmp
                    with torch.cuda.stream(self.s_out):
                        self.s_out.wait_event(ev_cmp)
                        for i in range(n):
                            out[b0 + i, n0:n1].copy_(self.do[s][i, :nn], non_blocking=True)
                        e = torch.cuda.Event()
                        e.record(self.s_out)
                        ev_o_free[s] = e
                ev_kv_free[kvs] = ev_cmp
            self.s_out.synchronize()
            self.s_cmp.synchronize()
        first = None  # the reference's loop order: batch, head, row
        for b0, n0, nn, bad in bad_hits:
            info = flashsign.decode_bad_key(int(bad.item()), h, nn)
            if info is not None:
                b, hh, row, z = info
                key = ((b0 + b) * h + hh, n0 + row)
                if first is None or key < first[0]:
                    first = (key, z)
        if first is not None:
            from .normalizers import DegenerateDenominatorError
            raise DegenerateDenominatorError(float(first[1]), f"row {first[0][1]}")
        return out


_default: dict = {}


def fwd_host(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out: torch.Tensor | None = None, **kw) -> torch.Tensor:
    """Host-tensor FlashSign with a cached per-device ``HostPipeline``."""
    dev = torch.cuda.current_device()
    if out is None:
        od = kw.get("out_dtype") or (q.dtype if q.dtype in (torch.bfloat16, torch.float16) else torch.bfloat16)
        out = torch.empty(q.shape, dtype=od, pin_memory=True)
    kw.pop("out_dtype", None)
    pipe = _default.get(dev)
    if pipe is None:
        pipe = _default[dev] = HostPipeline(dev)
    return pipe.run(q, k, v, out, **kw)
