"""FlashSign on host-resident inputs: chunked H2D -> kernel -> D2H with overlap.

``fwd_host(q, k, v, out)`` takes pinned CPU tensors in BSHD layout (the
compute dtype, e.g. bf16) and streams them through the GPU one batch chunk at
a time on three CUDA streams -- copy-in, compute, copy-out -- so PCIe
transfers of chunk i+1 and i-1 overlap the kernel on chunk i.  Device staging
buffers are double-buffered and reused across calls (``HostPipeline``).

This is the end-to-end path a caller with host data uses (what the reference's
numpy API amounts to); the bench reports it as ``e2e``.
"""

from __future__ import annotations

import torch

from . import flashsign


class HostPipeline:
    """Reusable device staging for ``fwd_host`` (two slots per tensor)."""

    def __init__(self, device: torch.device | int | None = None, chunk: int = 1):
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else
                                   (device if isinstance(device, int) else device.index))
        self.chunk = chunk
        self._shape_key = None
        self.s_in = torch.cuda.Stream(self.device)
        self.s_cmp = torch.cuda.Stream(self.device)
        self.s_out = torch.cuda.Stream(self.device)

    def _alloc(self, q, k, out, key_scale=None):
        key = (tuple(q.shape[1:]), tuple(k.shape[1:]), q.dtype, out.dtype, self.chunk,
               None if key_scale is None else tuple(key_scale.shape[1:]))
        if key == self._shape_key:
            return
        c = self.chunk
        dev = self.device
        self.dq = [torch.empty((c,) + tuple(q.shape[1:]), dtype=q.dtype, device=dev) for _ in range(2)]
        self.dk = [torch.empty((c,) + tuple(k.shape[1:]), dtype=k.dtype, device=dev) for _ in range(2)]
        self.dv = [torch.empty((c,) + tuple(k.shape[1:]), dtype=k.dtype, device=dev) for _ in range(2)]
        self.do = [torch.empty((c,) + tuple(out.shape[1:]), dtype=out.dtype, device=dev) for _ in range(2)]
        self.bad = [torch.empty(1, dtype=torch.int64, device=dev) for _ in range(2)]
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
        self._alloc(q, k, out, key_scale)
        c = self.chunk
        nb = q.shape[0]
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_cmp = [torch.cuda.Event() for _ in range(2)]
        ev_out = [None, None]
        bad_hits = []
        with torch.cuda.device(self.device):
            for i, b0 in enumerate(range(0, nb, c)):
                s = i & 1
                b1 = min(b0 + c, nb)
                n = b1 - b0
                with torch.cuda.stream(self.s_in):
                    if ev_out[s] is not None:  # slot s's previous output has left the device
                        self.s_in.wait_event(ev_out[s])
                    self.dq[s][:n].copy_(q[b0:b1], non_blocking=True)
                    self.dk[s][:n].copy_(k[b0:b1], non_blocking=True)
                    self.dv[s][:n].copy_(v[b0:b1], non_blocking=True)
                    if key_scale is not None:
                        self.dm[s][:n].copy_(key_scale[b0:b1], non_blocking=True)
                    ev_in[s].record(self.s_in)
                with torch.cuda.stream(self.s_cmp):
                    self.s_cmp.wait_event(ev_in[s])
                    _, bad = flashsign.fwd_async(self.dq[s][:n], self.dk[s][:n], self.dv[s][:n], scale=scale,
                                                 eps=eps, out=self.do[s][:n], bad_key=self.bad[s],
                                                 stream=self.s_cmp,
                                                 key_scale=None if key_scale is None else self.dm[s][:n], **kw)
                    if check:
                        bad_hits.append((b0, bad.clone()))
                    ev_cmp[s].record(self.s_cmp)
                with torch.cuda.stream(self.s_out):
                    self.s_out.wait_event(ev_cmp[s])
                    out[b0:b1].copy_(self.do[s][:n], non_blocking=True)
                    e = torch.cuda.Event()
                    e.record(self.s_out)
                    ev_out[s] = e
            self.s_out.synchronize()
            self.s_cmp.synchronize()
        for b0, bad in bad_hits:
            info = flashsign.decode_bad_key(int(bad.item()), q.shape[2], q.shape[1])
            if info is not None:
                _, _, row, z = info
                from .normalizers import DegenerateDenominatorError
                raise DegenerateDenominatorError(float(z), f"row {row}")
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
