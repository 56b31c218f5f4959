"""World-size-2 gloo runs of the multi-GPU plumbing on CPU
(paper_1402_5670_b200/dist.py): shearlet-index shards whose reconstruction
partial sums, reduced across ranks, equal the full reconstruction; the
per-rank local computation is the numpy oracle (no GPU here)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1402_5670_b200.dist import frame_range, shard_range


def test_shard_ranges_partition_and_balance():
    for R in (13, 49, 76, 292):
        for world in (1, 2, 3, 4, 8):
            rs = [shard_range(R, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == R
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [hi - lo for lo, hi in rs]
            assert max(sizes) - min(sizes) <= 1
    assert frame_range(64, 3, 8) == (24, 32)
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, dims, levels, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import shearlet_np as O
    from paper_1402_5670_b200.dist import sharded_denoise
    two_d = len(dims) == 2
    s = O.build_system_2d(*dims, levels) if two_d else O.build_system_3d(dims, levels)
    lo, hi = shard_range(s.R, rank, world)
    x = torch.zeros(dims, dtype=torch.float64)
    if rank == 0:
        x = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, dims))

    def local_partial(xt):
        f = xt.numpy()
        if two_d:
            bands = O.forward_2d(f, s)[lo:hi]
            B = np.fft.fft2(bands, axes=(1, 2))
            acc = np.sum(B * (s.filters[lo:hi] / s.frame_weight[None]), axis=0)
            return torch.from_numpy(np.real(np.fft.ifft2(acc)).copy())
        F = np.fft.fftn(f)
        acc = np.zeros(dims, dtype=np.complex128)
        for i in range(lo, hi):
            band = np.real(np.fft.ifftn(np.conj(s.filter_freq(i)) * F))
            acc += np.fft.fftn(band) * s.filter_freq(i) / s.frame_weight
        return torch.from_numpy(np.real(np.fft.ifftn(acc)).copy())

    out = sharded_denoise(x, local_partial)
    if rank == 0:
        ref = O.inverse_2d(O.forward_2d(x.numpy(), s), s) if two_d else x.numpy()
        q.put(float(np.linalg.norm(out.numpy() - ref) / np.linalg.norm(ref)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("dims,levels", [((32, 32), [0, 1]), ((12, 12, 12), [0])])
def test_gloo_world2_shard_reduce_equals_full(dims, levels):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, dims, levels, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) <= 1e-12


def test_library_partition_matches_shard_range():
    # the C-ABI partition (sl_partition, host code: no GPU needed) is the split
    # the in-library NCCL path uses; it equals dist.shard_range
    import paper_1402_5670_b200 as P
    for R in (17, 49, 99, 292):
        for world in (1, 2, 3, 8):
            for r in range(world):
                assert P.partition(R, world, r) == shard_range(R, r, world)
    with pytest.raises(P.ConfigError):
        P.partition(10, 2, 2)


def _lib_id_worker(rank, world, port, q):
    # the library communicator's unique id travels over torch.distributed (gloo
    # here); creating the NCCL communicator itself needs a GPU per rank
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    box = [b"\x01" * 128 if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    q.put((rank, box[0] == b"\x01" * 128))
    dist.destroy_process_group()


def test_unique_id_broadcast_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_lib_id_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert got == {0: True, 1: True}


def _acc_worker(rank, world, port, dims, levels, q):
    # the library's multi-GPU 3D schedule on CPU: broadcast, per-rank accumulator of
    # its bands (numpy oracle), slab-wise sum-reduce onto the root, root-only finish
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import shearlet_np as O
    from paper_1402_5670_b200.dist import sharded_denoise_accumulator
    s = O.build_system_3d(dims, levels)
    lo, hi = shard_range(s.R, rank, world)
    x = torch.zeros(dims, dtype=torch.float64)
    if rank == 0:
        x = torch.from_numpy(np.random.default_rng(6).uniform(-1, 1, dims))
    K = [3.0] * len(levels)

    def local_acc(xt):
        F = np.fft.fftn(xt.numpy())
        acc = np.zeros(dims, dtype=np.complex128)
        for i in range(lo, hi):
            band = np.real(np.fft.ifftn(np.conj(s.filter_freq(i)) * F))
            r = s.index[i]
            if r[1] >= 0:  # hard threshold of the non-lowpass bands (apps.cpp:57-81)
                band[np.abs(band) < K[r[1]] * 0.3 * s.filter_norms[i]] = 0.0
            acc += np.fft.fftn(band) * s.filter_freq(i)
        return torch.from_numpy(acc)

    out = sharded_denoise_accumulator(x, local_acc, lambda a: np.real(np.fft.ifftn(a.numpy() / s.frame_weight)))
    if rank == 0:
        full = O.inverse_3d(O.hard_threshold(O.forward_3d(x.numpy(), s), s.index, 0, s.filter_norms, K, 0.3), s)
        q.put(float(np.linalg.norm(out - full) / np.linalg.norm(full)))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world3_accumulator_reduce_equals_full_denoise():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_acc_worker, args=(r, 3, port, (12, 12, 12), [0], q)) for r in range(3)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) <= 1e-12
