"""Batch x head sharding with the REAL kernel in several processes (one GPU, shared).

Each process is one rank (gloo process group on 127.0.0.1), takes its contiguous unit range
(``partition.unit_range``), runs ``partition.fwd_shard`` with ``flashsign.fwd_async`` on its
shard -- the hot path, no collective -- and ``partition.gather_output`` collects O.  The gathered
output must be bitwise equal to the single-process launch over the whole batch: units are
independent and each runs the same tiles in the same order."""

import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, k, v, m, ref, results):
    import torch.distributed as dist
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2505_09326_b200 import flashsign, partition
        B, _, _, _ = q.shape
        hkv = k.shape[2]
        lo, hi = partition.unit_range(B * hkv, world, rank)
        b_lo, b_hi = lo // hkv, -(-hi // hkv)
        qd, kd, vd = (t[b_lo:b_hi].cuda() for t in (q, k, v))
        md = None if m is None else m[b_lo:b_hi].cuda()
        od = torch.zeros(qd.shape, dtype=torch.float32, device="cuda")
        flags = partition.fwd_shard(qd, kd, vd, od, lo - b_lo * hkv, hi - b_lo * hkv, flashsign.fwd_async,
                                    key_scale=md, eps=1e-6, out_dtype=torch.float32)
        torch.cuda.synchronize()
        assert all(flashsign.decode_bad_key(int(f.item()), q.shape[2], q.shape[1]) is None for f in flags)
        # whole batch rows per rank here (units % hkv == 0): gather along batch
        full = partition.gather_output(od.cpu())
        dist.destroy_process_group()
        # plain Python values through the queue (tensors would be shared with an exiting process)
        results.put((rank, bool(torch.equal(full, ref)), float((full - ref).abs().max()), None))
    except Exception as e:  # noqa: BLE001 -- reported to the parent
        results.put((rank, None, None, repr(e)))


@pytest.mark.parametrize("world,dt,mult", [(2, torch.bfloat16, False), (4, torch.float16, False),
                                           (2, torch.bfloat16, True), (4, torch.float8_e4m3fn, False)])
def test_sharded_ranks_gather_bitwise_equal_single_launch(world, dt, mult):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2505_09326_b200 import flashsign
    g = torch.Generator(device="cuda").manual_seed(300 + world)
    B, N, H, HKV = 8, 700, 4, 2
    d = 128 if dt == torch.float8_e4m3fn else 64
    q = torch.randn((B, N, H, d), generator=g, device="cuda").to(dt)
    k = torch.randn((B, N, HKV, d), generator=g, device="cuda").to(dt)
    v = torch.randn((B, N, HKV, d), generator=g, device="cuda").to(dt)
    m = torch.randint(0, 6, (B, N), generator=g, device="cuda").float() if mult else None
    ref = flashsign.fwd(q, k, v, eps=1e-6, out_dtype=torch.float32, key_scale=m).cpu()
    ctx = torch.multiprocessing.get_context("spawn")
    results = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q.cpu(), k.cpu(), v.cpu(),
                                               None if m is None else m.cpu(), ref, results))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [results.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, equal, maxdiff, exc in out:
        assert exc is None, f"rank {rank}: {exc}"
        assert equal, (rank, maxdiff)  # every rank gathered the whole O, bitwise the 1-process result
