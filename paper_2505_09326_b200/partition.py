"""Batch x head sharding of FlashSign across GPUs (one process per GPU).

The unit of work is one (batch element, kv-head group): u = b * H_kv + g.  A
unit owns query heads [g*r, (g+1)*r) (r = H / H_kv) and kv head g of batch b.
Units are independent -- disjoint (o, z) states, no cross-unit reduction
(attention.py:351-360 runs heads independently) -- so ranks take
contiguous unit ranges and the hot path needs no collective.  NCCL is used at
most to gather O shards onto one rank (``gather_output``), timed separately.

A unit range becomes at most three launches: a partial leading batch row, a
block of whole batch rows (one launch), and a partial trailing row.  Each is a
strided BSHD view of the full tensors, so no data moves.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch


def unit_range(n_units: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) of units for ``rank``: sizes ceil/floor(n_units / world)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    base, extra = divmod(n_units, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


@dataclass(frozen=True)
class Piece:
    """One launch: batch rows [b0, b1) x kv heads [g0, g1) (g-range partial only if b1 == b0 + 1)."""

    b0: int
    b1: int
    g0: int
    g1: int


def pieces(batch: int, heads_kv: int, lo: int, hi: int) -> list[Piece]:
    """Cover unit range [lo, hi) with at most three rectangular pieces."""
    if not 0 <= lo <= hi <= batch * heads_kv:
        raise ValueError(f"unit range [{lo}, {hi}) outside [0, {batch * heads_kv})")
    out: list[Piece] = []
    u = lo
    if u < hi and u % heads_kv:
        b, g = divmod(u, heads_kv)
        g1 = min(heads_kv, g + (hi - u))
        out.append(Piece(b, b + 1, g, g1))
        u += g1 - g
    full = (hi - u) // heads_kv
    if full:
        b = u // heads_kv
        out.append(Piece(b, b + full, 0, heads_kv))
        u += full * heads_kv
    if u < hi:
        b = u // heads_kv
        out.append(Piece(b, b + 1, 0, hi - u))
    return out


def piece_views(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, o: torch.Tensor, pc: Piece):
    """Strided BSHD views (no copies) of one piece: q/o heads [g0*r, g1*r), k/v heads [g0, g1)."""
    r = q.shape[2] // k.shape[2]
    b = slice(pc.b0, pc.b1)
    return (q[b, :, pc.g0 * r: pc.g1 * r], k[b, :, pc.g0: pc.g1], v[b, :, pc.g0: pc.g1],
            o[b, :, pc.g0 * r: pc.g1 * r])


def fwd_shard(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, o: torch.Tensor, lo: int, hi: int, fwd,
              key_scale: torch.Tensor | None = None, **kw):
    """Run ``fwd(q_view, k_view, v_view, out=o_view, **kw)`` over units [lo, hi).

    ``q/k/v/o`` are BSHD tensors on this rank's device (``lo/hi`` are unit
    indices relative to them); ``key_scale`` [B, Nkv] (optional per-key
    multiplicities) is sliced by batch row with each piece.  Returns the
    bad-key tensors ``fwd`` produced (async; nothing synchronises here).
    """
    flags = []
    for pc in pieces(q.shape[0], k.shape[2], lo, hi):
        qv, kv_, vv, ov = piece_views(q, k, v, o, pc)
        if key_scale is not None:
            kw["key_scale"] = key_scale[pc.b0: pc.b1]
        res = fwd(qv, kv_, vv, out=ov, **kw)
        if isinstance(res, tuple):
            flags.append(res[1])
    return flags


def kv_shard_range(n_kv: int, world: int, rank: int, align: int = 128) -> tuple[int, int]:
    """Contiguous key range [lo, hi) of ``rank`` for context parallelism, cut at multiples of
    ``align`` (the kernel's K/V tile) so no rank streams a partial tile it does not own."""
    tiles = -(-n_kv // align)
    lo_t, hi_t = unit_range(tiles, world, rank)
    return min(n_kv, lo_t * align), min(n_kv, hi_t * align)


def context_parallel_fwd(q: torch.Tensor, k_shard: torch.Tensor, v_shard: torch.Tensor, group=None, *,
                         eps: float = 0.0, normalizer: str = "spherical", out_dtype=None, check: bool = True,
                         fwd_partial=None, combine=None, **kw) -> torch.Tensor:
    """Sequence-parallel FlashSign: every rank holds all queries and one
    contiguous shard of the K/V sequence (``kv_shard_range``).

    Spherical (and signed-L1) partials over disjoint key ranges merge by plain addition --
    the numerator sum_j s_ij v_j and z = sum_j a2(s_ij) are both linear in the key set
    (streaming.py:122-128) -- so one ``all_reduce(SUM)`` of the fp32
    (numerator, z) workspace, d+1 floats per query row, replaces softmax ring attention's
    max/rescale exchange.  Each rank then normalises locally; every rank returns the full O.
    ``fwd_partial`` / ``combine`` default to the CUDA kernels (injectable for CPU tests).
    """
    import torch.distributed as dist

    if fwd_partial is None or combine is None:
        from . import flashsign
        fwd_partial = fwd_partial or flashsign.fwd_partial
        combine = combine or flashsign.combine
    partial, n_parts = fwd_partial(q, k_shard, v_shard, eps=eps, normalizer=normalizer, **kw)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)
    return combine(partial, n_parts, q, eps=eps, normalizer=normalizer, out_dtype=out_dtype, check=check)


def gather_output(o_local: torch.Tensor, group=None) -> torch.Tensor:
    """all_gather equal-size shard outputs (along batch) into one tensor on every rank."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    o_local = o_local.contiguous()
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world * o_local.shape[0],) + tuple(o_local.shape[1:]), dtype=o_local.dtype,
                          device=o_local.device)
        dist.all_gather_into_tensor(out, o_local, group=group)
        return out
    parts = [torch.empty_like(o_local) for _ in range(world)]
    dist.all_gather(parts, o_local, group=group)
    return torch.cat(parts, dim=0)
