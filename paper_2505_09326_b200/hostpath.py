"""Host-array execution of the drop-in API: numpy Q/K/V in, numpy O out.

This is the data path behind ``attention.streamed_attention_array`` /
``multi_head_attention_array`` (reference attention.py:252-279, 318-361), whose callers
hand over float32 / float64 (or float16) numpy arrays and expect the reference's
result dtype back.  Per call, on three CUDA streams of the current device:

  copy-in   K and V, then Q in row chunks, cross the host link in the caller's own dtype
            (no host-side conversion pass); arrays of >= 8 MB go through a pinned ring that host
            threads fill with non-temporal stores (``fs_host_copy``) while the DMA engine drains
            the previous slot (pinned DMA runs ~5x the pageable rate; staged copy-in 36-38 GB/s
            against 11 GB/s pageable and 20-25 GB/s with a numpy fill), smaller ones
            are copied from pageable memory directly (``FLASHSIGN_H2D=auto``, default;
            ``pageable`` / ``staged`` force one)
  compute   ``fs_prepare`` converts each tensor on the device to the kernel's operand
            dtype with one power-of-two scale per tensor and a Cauchy-Schwarz P scale
            (include/flashsign.h), so no finite input the reference accepts can overflow
            the 16-bit operands; then one FlashSign launch per Q chunk covering every head,
            with ``dev_scales`` folding the scales back out exactly
  copy-out  each chunk's O goes by DMA straight into a pinned host array, which is the
            returned result (no host copy on the way out)

Calls with at most 12 MB of input in one chunk (the GRN per-cell shapes, the reference's own
tests) skip the three-stream pipeline: Q|K|V packed into one pinned buffer, one copy, one
``fs_prepare``, one launch and one synchronisation on the current stream (``_run_small``).

The first degenerate row in the reference's loop order (head, then row; attention.py:196-199,
351-360) is found from one bad-row key per chunk after the final synchronisation.
"""

from __future__ import annotations

import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

from . import flashsign

_SRC_TORCH = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
              np.dtype(np.float16): torch.float16}
_CHUNK_BYTES = int(os.environ.get("FLASHSIGN_CHUNK_MB", "32")) << 20
_STAGE_MIN_BYTES = 8 << 20  # auto mode: pinned staging from this size on
# Q + K + V up to this size: one packed copy, one stream (``_run_small``); measured faster than the
# pipeline up to ~4 MB per array (tests/size_sweep.py: 2 MB arrays 639 vs 816 us, 4 MB equal)
_SMALL_BYTES = 12 << 20
# pinned ring slot: 64 MB measured best for the host-thread fill (C3 drop-in 95 -> 116 TFLOP/s vs 32 MB)
_STAGE_BYTES = int(os.environ.get("FLASHSIGN_STAGE_MB", "64")) << 20


class _Engine:
    """Streams and small device workspaces of one device (created on first use)."""

    def __init__(self, dev: torch.device):
        self.dev = dev
        with torch.cuda.device(dev):
            self.s_h2d = torch.cuda.Stream(dev)
            self.s_cmp = torch.cuda.Stream(dev)
            self.s_d2h = torch.cuda.Stream(dev)
            self.stats = torch.zeros(6, dtype=torch.float64, device=dev)
            self.scales = torch.ones(4, dtype=torch.float32, device=dev)
        self.lock = threading.Lock()  # one call at a time per device (shared workspaces)
        self.mode = os.environ.get("FLASHSIGN_H2D", "auto")
        self.pool = None
        self.ring = []
        self.small_host = self.small_dev = None  # packed Q|K|V of small calls (grown on demand)
        self.copy = None  # staging fill: fs_host_copy (FLASHSIGN_STAGE_COPY=numpy: np.copyto)
        if os.environ.get("FLASHSIGN_STAGE_COPY", "nt") != "numpy":
            import ctypes

            from . import _lib
            fn = _lib.load().fs_host_copy
            fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]
            fn.restype = ctypes.c_int
            self.copy = fn
        self.small_bad = torch.empty(1, dtype=torch.int64, pin_memory=True)

    # ------------------------------------------------------------------ host -> device
    def _h2d(self, dst: torch.Tensor, src: np.ndarray) -> None:
        """Copy the contiguous host array ``src`` into ``dst`` on the copy-in stream."""
        if src.size == 0:
            return
        if self.mode == "pageable" or (self.mode == "auto" and src.nbytes < _STAGE_MIN_BYTES):
            with torch.cuda.stream(self.s_h2d):
                dst.copy_(torch.from_numpy(src).view(dst.shape), non_blocking=True)
            return
        # staged: host threads fill a pinned ring slot while the DMA engine drains the previous one
        flat_src = src.reshape(-1).view(np.uint8)
        flat_dst = dst.view(-1).view(torch.uint8)
        if not self.ring:
            self.pool = ThreadPoolExecutor(int(os.environ.get("FLASHSIGN_H2D_THREADS", 0))
                                           or max(1, min(8, os.cpu_count() or 1)))
            self.ring = [(torch.empty(_STAGE_BYTES, dtype=torch.uint8, pin_memory=True), torch.cuda.Event())
                         for _ in range(3)]
        nthr = self.pool._max_workers
        src_ptr = flat_src.ctypes.data
        for i, lo in enumerate(range(0, flat_src.size, _STAGE_BYTES)):
            hi = min(lo + _STAGE_BYTES, flat_src.size)
            buf, ev = self.ring[i % len(self.ring)]
            ev.synchronize()  # the DMA that last read this slot is done
            step = -(-(hi - lo) // nthr)
            if self.copy is not None:  # non-temporal stores (csrc/fs_host.cpp; ctypes drops the GIL)
                dst_ptr = buf.data_ptr()
                list(self.pool.map(lambda j: self.copy(dst_ptr + j, src_ptr + lo + j, min(step, hi - lo - j)),
                                   range(0, hi - lo, step)))
            else:
                host = buf.numpy()[:hi - lo]
                list(self.pool.map(lambda j: np.copyto(host[j:j + step], flat_src[lo + j:lo + min(j + step, hi - lo)]),
                                   range(0, hi - lo, step)))
            with torch.cuda.stream(self.s_h2d):
                flat_dst[lo:hi].copy_(buf[:hi - lo], non_blocking=True)
                ev.record(self.s_h2d)

    def _reference_z(self, q_row: np.ndarray, k_dev: torch.Tensor, scale: float, normalizer: str, exact: bool):
        """The z the reference reports for a degenerate row (attention.py:161-199): scores in
        float64, rounded to float32 for float32 callers (163-164), scaled, f16-rounded and summed in
        float32 under the f16 emulation (167-168, 157-158).  Recomputed for that one row from the
        caller's values, so e.g. an inf input reports z = inf exactly as the reference does (the
        kernel's zero-filled padding keys would turn it into NaN)."""
        f32 = q_row.dtype == np.float32
        qv = torch.from_numpy(np.ascontiguousarray(q_row, dtype=np.float64)).to(self.dev)
        kd = k_dev.to(torch.float64)
        if exact:
            qv, kd = qv.half().double(), kd.half().double()
        sc = kd @ qv
        if f32 or exact:
            sc = sc.float()
            if scale != 1.0:
                sc = sc * torch.tensor(scale, dtype=torch.float32, device=self.dev)
            if exact:
                sc = sc.half().float()
        elif scale != 1.0:
            sc = sc * scale
        a2 = sc * sc if normalizer == "spherical" else sc.abs()
        return float(a2.sum(dtype=torch.float32 if exact else torch.float64).item())

    # ------------------------------------------------------------------ small calls
    def _run_small(self, q3, k3, v3, *, scale, eps, compute, normalizer, exact, d_pad, k_out, host_out_t, st):
        """One call of at most ``_SMALL_BYTES`` of input (the GRN per-cell shapes, the reference's
        tests): Q|K|V packed into one reused pinned buffer on the host, one H2D copy, one
        ``fs_prepare`` for all three tensors, one FlashSign launch, all on the current stream, and
        one synchronisation -- the multi-stream chunk pipeline of ``run`` only pays off once the
        copies are long enough to overlap.  The whole sequence is one C++ call (``small_call`` in
        csrc/fs_torch.cpp).  Returns ``(out, bad_key, k_device_source)``."""
        n, h, d = q3.shape
        x, hkv, _ = k3.shape
        dev = self.dev
        parts = [a.reshape(-1).view(np.uint8) for a in (q3, k3, v3)]
        al = lambda b: -(-b // 256) * 256  # noqa: E731  (each tensor starts 256-byte aligned)
        offs = [0, al(parts[0].size), al(parts[0].size) + al(parts[1].size)]
        tot = offs[2] + parts[2].size
        if self.small_host is None or self.small_host.numel() < tot:
            cap = max(tot, 1 << 20)
            self.small_host = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
            self.small_dev = torch.empty(cap, dtype=torch.uint8, device=dev)
        ext = flashsign.torch_ext()
        st_, msg, host_out, bad_key = ext.small_call(
            q3.ctypes.data, k3.ctypes.data, v3.ctypes.data, st, n, h, x, hkv, d, self.small_host, self.small_dev,
            self.stats, self.scales, self.small_bad, compute, d_pad, k_out, host_out_t, float(scale), float(eps),
            flashsign.NORMALIZERS[normalizer], bool(exact))
        if st_ != 0:
            raise flashsign._STATUS_EXC.get(st_, RuntimeError)(f"flashsign: {msg}")
        kr = self.small_dev[offs[1]:offs[1] + parts[1].size].view(st).view(-1, d)  # K as copied (bad-row z)
        return host_out.numpy(), int(bad_key), kr

    # ------------------------------------------------------------------ one call
    def run(self, q3: np.ndarray, k3: np.ndarray, v3: np.ndarray, *, scale: float, eps: float, compute: torch.dtype,
            normalizer: str, exact: bool, out_np_dtype) -> np.ndarray:
        n, h, d = q3.shape
        x, hkv, _ = k3.shape
        dev = self.dev
        align = 16 if compute == getattr(torch, "float8_e4m3fn", None) else 8
        d_pad = max(align, -(-d // align) * align)
        out_np_dtype = np.dtype(out_np_dtype)
        k_out = torch.float16 if out_np_dtype == np.float16 else torch.float32  # kernel output dtype
        host_out_t = {np.dtype(np.float16): torch.float16, np.dtype(np.float32): torch.float32,
                      np.dtype(np.float64): torch.float64}[out_np_dtype]
        q3, k3, v3 = (np.ascontiguousarray(a) for a in (q3, k3, v3))
        st = _SRC_TORCH[q3.dtype]
        # rows of Q per chunk: ~_CHUNK_BYTES of source per chunk, whole query positions
        row_bytes = h * d * q3.itemsize
        cq = max(1, min(n, _CHUNK_BYTES // max(1, row_bytes)))
        chunks = [(lo, min(lo + cq, n)) for lo in range(0, n, cq)]
        nb = min(2, len(chunks))
        if x > 0 and len(chunks) == 1 and q3.nbytes + k3.nbytes + v3.nbytes <= _SMALL_BYTES:
            # one source dtype in the packed buffer: K / V in Q's, the rounding the pipeline's
            # device-side copy_ applies to mixed-dtype callers (the reference accepts those)
            k3, v3 = (a if a.dtype == q3.dtype else a.astype(q3.dtype) for a in (k3, v3))
            out, bad_key, kr = self._run_small(q3, k3, v3, scale=scale, eps=eps, compute=compute,
                                               normalizer=normalizer, exact=exact, d_pad=d_pad, k_out=k_out,
                                               host_out_t=host_out_t, st=st)
            first = None
            info = flashsign.decode_bad_key(bad_key, h, n)
            if info is not None:
                _, hh, row, _ = info
                first = (hh, row, self._reference_z(q3[row, hh], kr.view(x, hkv, d)[:, (hh * hkv) // h],
                                                    scale, normalizer, exact))
            if d_pad != d:
                out = np.ascontiguousarray(out[..., :d])
            return out, first

        with torch.cuda.device(dev):
            kr = torch.empty((max(x, 1) * hkv, d), dtype=st, device=dev)
            vr = torch.empty((max(x, 1) * hkv, d), dtype=st, device=dev)
            kq = torch.empty((1, max(x, 1), hkv, d_pad), dtype=compute, device=dev)
            vq = torch.empty((1, max(x, 1), hkv, d_pad), dtype=compute, device=dev)
            qr = [torch.empty((cq * h, d), dtype=st, device=dev) for _ in range(nb)]
            qq = torch.empty((1, cq, h, d_pad), dtype=compute, device=dev)
            oc = [torch.empty((1, cq, h, d_pad), dtype=k_out, device=dev) for _ in range(nb)]
            o64 = ([torch.empty((1, cq, h, d_pad), dtype=torch.float64, device=dev) for _ in range(nb)]
                   if host_out_t == torch.float64 else None)
            bad = torch.empty(len(chunks), dtype=torch.int64, device=dev)
            host_out = torch.empty((n, h, d_pad), dtype=host_out_t, pin_memory=True)
            bad_host = torch.empty(len(chunks), dtype=torch.int64, pin_memory=True)
            ev_q = [torch.cuda.Event() for _ in range(nb)]     # Q chunk landed
            ev_qf = [torch.cuda.Event() for _ in range(nb)]    # Q chunk consumed by prepare
            ev_o = [torch.cuda.Event() for _ in range(nb)]     # O chunk written
            ev_of = [torch.cuda.Event() for _ in range(nb)]    # O chunk copied out
            s_h2d, s_cmp, s_d2h = self.s_h2d, self.s_cmp, self.s_d2h
            for s_ in (s_h2d, s_cmp, s_d2h):
                s_.wait_stream(torch.cuda.current_stream(dev))  # buffers above came from the current stream

            # K, V
            self._h2d(kr[:x * hkv], k3.reshape(-1, d))
            self._h2d(vr[:x * hkv], v3.reshape(-1, d))
            s_cmp.wait_stream(s_h2d)
            with torch.cuda.stream(s_cmp):
                kq_ = kq[0, :x].reshape(x * hkv, d_pad)
                vq_ = vq[0, :x].reshape(x * hkv, d_pad)
                flashsign.prepare([None, kr[:x * hkv], vr[:x * hkv]], [None, kq_, vq_], stats=self.stats,
                                  scales=self.scales, scale=scale, eps=eps, normalizer=normalizer, exact=exact,
                                  stream=s_cmp)
            kt, vt = (kq, vq) if x > 0 else (kq[:, :0], vq[:, :0])

            for c, (lo, hi) in enumerate(chunks):
                j, rows = c % nb, hi - lo
                # copy-in: reuse Q slot j once prepare has consumed its previous chunk
                s_h2d.wait_event(ev_qf[j])
                self._h2d(qr[j][:rows * h], q3[lo:hi].reshape(-1, d))
                ev_q[j].record(s_h2d)
                with torch.cuda.stream(s_cmp):
                    s_cmp.wait_event(ev_q[j])
                    qv = qq[:, :rows]
                    flashsign.prepare([qr[j][:rows * h], None, None], [qv.reshape(rows * h, d_pad), None, None],
                                      stats=self.stats, scales=self.scales, scale=scale, eps=eps,
                                      normalizer=normalizer, exact=exact, stream=s_cmp)
                    ev_qf[j].record(s_cmp)
                    s_cmp.wait_event(ev_of[j])  # O slot j copied out
                    ov = oc[j][:, :rows]
                    flashsign.fwd_async(qv, kt, vt, scale=float(scale), eps=float(eps), out=ov, normalizer=normalizer,
                                        bad_key=bad[c:c + 1], stream=s_cmp, dev_scales=self.scales)
                    if o64 is not None:
                        o64[j][:, :rows].copy_(ov)
                    ev_o[j].record(s_cmp)
                with torch.cuda.stream(s_d2h):
                    s_d2h.wait_event(ev_o[j])
                    src = (o64[j] if o64 is not None else oc[j])[0, :rows]
                    host_out[lo:hi].copy_(src, non_blocking=True)
                    ev_of[j].record(s_d2h)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_stream(s_cmp)
                bad_host.copy_(bad, non_blocking=True)
            s_d2h.synchronize()
            torch.cuda.current_stream(dev).wait_stream(s_d2h)

        first = None  # (head, row, z) first in the reference's loop order
        for c, key in enumerate(bad_host.tolist()):
            info = flashsign.decode_bad_key(key, h, chunks[c][1] - chunks[c][0])
            if info is not None:
                _, hh, row, z = info
                cand = (hh, chunks[c][0] + row, z)
                if first is None or cand[:2] < first[:2]:
                    first = cand
        if first is not None:
            hh, row, _ = first
            first = (hh, row, self._reference_z(q3[row, hh], kr[:x * hkv].view(x, hkv, d)[:, (hh * hkv) // h],
                                                scale, normalizer, exact))
        out = host_out.numpy()
        if d_pad != d:
            out = np.ascontiguousarray(out[..., :d])
        return out, first


_engines: dict = {}
_engines_lock = threading.Lock()


def engine(dev: torch.device) -> _Engine:
    key = dev.index if dev.index is not None else torch.cuda.current_device()
    with _engines_lock:
        if key not in _engines:
            _engines[key] = _Engine(torch.device("cuda", key))
        return _engines[key]


def run(q3, k3, v3, *, scale, eps, compute, normalizer, exact, out_np_dtype, device=None):
    """Execute one drop-in call; returns ``(out, first_bad)`` with ``first_bad`` = ``(head, row, z)`` or None."""
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    e = engine(dev)
    with e.lock:
        return e.run(q3, k3, v3, scale=scale, eps=eps, compute=compute, normalizer=normalizer, exact=exact,
                     out_np_dtype=out_np_dtype)
