"""Batch x head partitioner (paper_2505_09326_b200/partition.py), CPU only: unit ranges,
launch pieces, and a world-size-2 gloo run where each rank computes its shard (with the
CPU oracle standing in for the kernel) and the shards are all-gathered."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.spherical import gram_batched
from paper_2505_09326_b200 import partition


@pytest.mark.parametrize("n,world", [(128, 8), (512, 8), (256, 3), (7, 4), (3, 8), (0, 2), (1000, 7)])
def test_unit_ranges_tile_exactly(n, world):
    seen = []
    sizes = []
    for r in range(world):
        lo, hi = partition.unit_range(n, world, r)
        seen.extend(range(lo, hi))
        sizes.append(hi - lo)
    assert seen == list(range(n))
    assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("batch,hkv", [(8, 16), (3, 4), (64, 8), (5, 1), (2, 7)])
def test_pieces_cover_range(batch, hkv):
    n = batch * hkv
    rng = np.random.default_rng(batch * 100 + hkv)
    for _ in range(50):
        lo, hi = sorted(rng.integers(0, n + 1, 2))
        ps = partition.pieces(batch, hkv, int(lo), int(hi))
        assert len(ps) <= 3
        units = []
        for p in ps:
            assert p.b1 > p.b0 and p.g1 > p.g0
            if p.b1 - p.b0 > 1:
                assert (p.g0, p.g1) == (0, hkv)
            units.extend(b * hkv + g for b in range(p.b0, p.b1) for g in range(p.g0, p.g1))
        assert units == list(range(lo, hi))


def test_bench_configs_are_one_launch_per_rank():
    for b, hkv in ((8, 16), (16, 16), (64, 8)):
        for world in (1, 2, 4, 8):
            for r in range(world):
                lo, hi = partition.unit_range(b * hkv, world, r)
                assert len(partition.pieces(b, hkv, lo, hi)) == 1


def test_piece_views_are_views():
    q = torch.randn(3, 10, 8, 16)
    k = torch.randn(3, 12, 4, 16)
    o = torch.empty_like(q)
    qv, kv, vv, ov = partition.piece_views(q, k, k, o, partition.Piece(1, 2, 1, 3))
    assert qv.data_ptr() == q[1:2, :, 2:6].data_ptr() and qv.shape == (1, 10, 4, 16)
    assert kv.shape == (1, 12, 2, 16) and ov.shape == (1, 10, 4, 16)


def _oracle_fwd(qv, kv, vv, out, **kw):
    out.copy_(torch.from_numpy(gram_batched(qv.numpy(), kv.numpy(), vv.numpy())).to(out.dtype))


def _worker(rank, world, port, q, k, v, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    B, HKV = q.shape[0], k.shape[2]
    lo, hi = partition.unit_range(B * HKV, world, rank)
    per_rank = (B * HKV) // world
    assert per_rank % HKV == 0  # whole batch rows per rank -> equal-size batch shards
    b0, b1 = lo // HKV, hi // HKV
    o_local = torch.empty_like(q[b0:b1])
    partition.fwd_shard(q[b0:b1], k[b0:b1], v[b0:b1], o_local, 0, hi - lo, _oracle_fwd)
    full = partition.gather_output(o_local)
    if rank == 0:
        result.copy_(full)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_gloo_world2_shards_gather_to_full_result():
    torch.manual_seed(0)
    B, N, H, HKV, D = 4, 40, 4, 2, 16
    q = torch.randn(B, N, H, D, dtype=torch.float64)
    k = torch.randn(B, N, HKV, D, dtype=torch.float64)
    v = torch.randn(B, N, HKV, D, dtype=torch.float64)
    result = torch.zeros_like(q).share_memory_()
    mp.spawn(_worker, args=(2, _free_port(), q, k, v, result), nprocs=2, join=True)
    want = gram_batched(q.numpy(), k.numpy(), v.numpy())
    np.testing.assert_allclose(result.numpy(), want, rtol=0, atol=0)


# ---------------------------------------------------------------- context parallelism

@pytest.mark.parametrize("n_kv,world", [(1000, 2), (128, 2), (5000, 8), (129, 3), (0, 2)])
def test_kv_shard_ranges_tile_aligned_and_exact(n_kv, world):
    rs = [partition.kv_shard_range(n_kv, world, r) for r in range(world)]
    assert rs[0][0] == 0 and rs[-1][1] == n_kv
    for (a, b), (c, d) in zip(rs, rs[1:]):
        assert b == c
    for a, b in rs:
        assert a <= b and (a == b or a % 128 == 0)


def _cpu_partial(q, k, v, eps=0.0, normalizer="spherical", **kw):
    """CPU stand-in for flashsign.fwd_partial with the C-ABI workspace layout
    (include/flashsign.h: numerators [S=1][B][H][Nq][Dk] then z [S][B][H][Nq], Dk = 64 here)."""
    b, nq, h, d = q.shape
    hkv = k.shape[2]
    dk = 64
    num = torch.zeros((b, h, nq, dk), dtype=torch.float64)
    z = torch.zeros((b, h, nq), dtype=torch.float64)
    for bb in range(b):
        for hh in range(h):
            g = hh * hkv // h
            s = q[bb, :, hh].double() @ k[bb, :, g].double().T
            num[bb, hh, :, :d] = s @ v[bb, :, g].double()
            z[bb, hh] = (s * s).sum(1) if normalizer == "spherical" else s.abs().sum(1)
    return torch.cat([num.flatten(), z.flatten()]), 1


def _cpu_combine(ws, n_parts, like_q, eps=0.0, normalizer="spherical", out_dtype=None, check=True):
    b, nq, h, d = like_q.shape
    rows = b * h * nq
    num = ws[: n_parts * rows * 64].view(n_parts, b, h, nq, 64).sum(0)
    z = ws[n_parts * rows * 64: n_parts * rows * 65].view(n_parts, b, h, nq).sum(0)
    den = (z + eps).sqrt() if normalizer == "spherical" else z + eps
    return (num[..., :d] / den[..., None]).permute(0, 2, 1, 3).contiguous()


def _cp_worker(rank, world, port, q, k, v, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = partition.kv_shard_range(k.shape[1], world, rank)
    o = partition.context_parallel_fwd(q, k[:, lo:hi], v[:, lo:hi], eps=1e-6, fwd_partial=_cpu_partial,
                                       combine=_cpu_combine)
    result[rank].copy_(o)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_context_parallel_matches_full():
    # each rank streams half of the keys; one all_reduce(SUM) of (numerator, z) -> the full result
    torch.manual_seed(1)
    B, N, H, HKV, D = 2, 40, 4, 2, 16
    q = torch.randn(B, N, H, D, dtype=torch.float64)
    k = torch.randn(B, 300, HKV, D, dtype=torch.float64)
    v = torch.randn(B, 300, HKV, D, dtype=torch.float64)
    result = torch.zeros((2,) + tuple(q.shape), dtype=torch.float64).share_memory_()
    mp.spawn(_cp_worker, args=(2, _free_port(), q, k, v, result), nprocs=2, join=True)
    want = gram_batched(q.numpy(), k.numpy(), v.numpy(), 1.0, 1e-6)
    for r in range(2):
        np.testing.assert_allclose(result[r].numpy(), want, rtol=1e-10, atol=1e-12)
