"""Context parallelism over peer memory (``peer.context_parallel_fwd_peer``, ``fs_fwd_peer``).

Several processes share the one GPU of the test box: each maps the others' workspaces through
CUDA IPC exactly as ranks on different GPUs do over NVLink, and the kernel's epilogue stores
its partials into them.  Every rank's positions are compared with the single-pass kernel."""

import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, k, v, ref, qbad, results, norm="spherical"):
    import torch.distributed as dist
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2505_09326_b200 import partition, peer
        from paper_2505_09326_b200.normalizers import DegenerateDenominatorError
        qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
        lo, hi = partition.kv_shard_range(kd.shape[1], world, rank)
        out, (a, b) = peer.context_parallel_fwd_peer(qd, kd[:, lo:hi], vd[:, lo:hi], eps=1e-6,
                                                     out_dtype=torch.float32, normalizer=norm)
        assert (a, b) == peer.peer_rows(q.shape[1], world, rank)
        err = float((out[:, a:b].cpu() - ref[:, a:b]).abs().max()) if b > a else 0.0
        # second call: the other workspace of the pair, and the all-gather of O
        out2, _ = peer.context_parallel_fwd_peer(qd, kd[:, lo:hi], vd[:, lo:hi], eps=1e-6,
                                                 out_dtype=torch.float32, gather=True, normalizer=norm)
        err2 = float((out2.cpu() - ref).abs().max())
        # a degenerate row (q = 0, eps = 0) owned by rank 0: every rank raises for it (the bad-row
        # keys are MIN-reduced), after the all-gather -- no rank is left blocked in a collective
        raised = False
        try:
            peer.context_parallel_fwd_peer(qbad.cuda(), kd[:, lo:hi], vd[:, lo:hi], out_dtype=torch.float32,
                                           normalizer=norm, gather=True)
        except DegenerateDenominatorError as e:
            raised = "row 5" in str(e)
        peer.release_workspaces()
        dist.destroy_process_group()
        results.put((rank, err, err2, raised, None))
    except Exception as e:  # noqa: BLE001 -- reported to the parent
        results.put((rank, None, None, None, repr(e)))


@pytest.mark.parametrize("world,dt,nq,nkv,norm", [(2, torch.bfloat16, 700, 1000, "spherical"),
                                                  (3, torch.float16, 513, 777, "spherical"),
                                                  (2, torch.float8_e4m3fn, 256, 300, "spherical"),
                                                  (2, torch.bfloat16, 300, 500, "signed_l1")])
def test_context_parallel_over_peer_memory(world, dt, nq, nkv, norm):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2505_09326_b200 import flashsign
    g = torch.Generator(device="cuda").manual_seed(200 + world)
    d = 128 if dt == torch.float8_e4m3fn else 64
    q = torch.randn((2, nq, 4, d), generator=g, device="cuda").to(dt)
    k = torch.randn((2, nkv, 2, d), generator=g, device="cuda").to(dt)
    v = torch.randn((2, nkv, 2, d), generator=g, device="cuda").to(dt)
    ref = flashsign.fwd(q, k, v, eps=1e-6, out_dtype=torch.float32, kv_splits=1, normalizer=norm).cpu()
    qbad = q.clone()
    qbad[1, 5, 3] = 0
    ctx = torch.multiprocessing.get_context("spawn")
    results = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q.cpu(), k.cpu(), v.cpu(), ref, qbad.cpu(), results,
                                               norm))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [results.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    tol = 2e-5 * max(1.0, float(ref.abs().max()))
    for rank, err, err2, raised, exc in sorted(out, key=lambda t: t[0]):
        assert exc is None, f"rank {rank}: {exc}"
        assert err <= tol and err2 <= tol, (rank, err, err2)
        assert raised, rank  # position 5 belongs to rank 0; every rank reports it


def test_peer_path_single_process_equals_single_pass():
    # world 1 (no process group): the kernel stores every partial into this rank's own workspace
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2505_09326_b200 import flashsign, peer
    g = torch.Generator(device="cuda").manual_seed(300)
    q = torch.randn((2, 333, 4, 128), generator=g, device="cuda").to(torch.bfloat16)
    k = torch.randn((2, 444, 4, 128), generator=g, device="cuda").to(torch.bfloat16)
    v = torch.randn((2, 444, 4, 128), generator=g, device="cuda").to(torch.bfloat16)
    out, (lo, hi) = peer.context_parallel_fwd_peer(q, k, v, eps=1e-6, out_dtype=torch.float32)
    assert (lo, hi) == (0, 333)
    ref = flashsign.fwd(q, k, v, eps=1e-6, out_dtype=torch.float32, kv_splits=1)
    assert float((out - ref).abs().max()) <= 1e-5 * max(1.0, float(ref.abs().max()))
    with pytest.raises(Exception, match="key_scale|unsupported|not supported"):
        # multiplicities are not part of the peer path
        from paper_2505_09326_b200 import _lib
        import ctypes
        prm = peer._params(q, k, v, out, 1.0, 0.0, "spherical", torch.empty(1, dtype=torch.int64, device="cuda"))
        m = torch.ones((2, 444), device="cuda")
        prm.key_scale, prm.key_scale_stride = m.data_ptr(), m.stride(0)
        ws = peer.PeerWorkspace(1 << 20)
        pp = _lib.FsPeerParams()
        pp.world, pp.rank, pp.rows_per_rank = 1, 0, 333
        pp.peer_partial, pp.local_partial = ws.table.data_ptr(), ws.local
        st = _lib.load().fs_fwd_peer(ctypes.byref(prm), ctypes.byref(pp), None)
        ws.close()
        raise RuntimeError(_lib.last_error() if st != _lib.FS_OK else "accepted")
    peer.release_workspaces()
