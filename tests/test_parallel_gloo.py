"""world_size-2 gloo runs (CPU) of the multi-GPU plumbing: line-ID sharding with a
variable-length all-gather, and the interleaved screen-tile gather.  The kernels
cannot run here, so each rank's kernel output is stood in for by the CPU oracle
(voxelization) or a synthetic per-pixel pattern (tiles); what is under test is
the partitioning and collective logic in paper_1801_01155_b200/parallel.py."""
import os
import socket
import sys

import numpy as np
import pytest

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(fn, world, *args):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.spawn(_entry, args=(world, port, fn, args), nprocs=world, join=True)


def _entry(rank, world, port, fn, args):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


def _worker_tiles(rank, world, W, H):
    import torch
    from paper_1801_01155_b200 import parallel
    idx, mask = parallel.tile_pixel_indices(rank, world, W, H)
    # stand-in for the render kernel: pixel value = f(pixel index), zeros outside the image
    tiles = np.where(mask, idx, 0).astype(np.float32)[..., None] * np.array([1, 2, 3, 4], np.float32)
    parts = parallel.gather_tiles(torch.from_numpy(tiles), 0)
    if rank != 0:
        assert parts is None
        return
    img = np.full((H * W, 4), -1.0, np.float32)
    for r, part in enumerate(parts):
        i, m = parallel.tile_pixel_indices(r, world, W, H)
        assert part.shape[0] == i.shape[0]
        img[i[m]] = part.numpy()[m]
    want = np.arange(H * W, dtype=np.float32)[:, None] * np.array([1, 2, 3, 4], np.float32)
    assert np.array_equal(img, want)  # every pixel written exactly once, by the right tile


@pytest.mark.parametrize("size", [(150, 70), (64, 32), (33, 17)])
def test_tile_gather_reassembles_the_frame(size):
    _run(_worker_tiles, 2, *size)


def _worker_voxelize(rank, world):
    import torch
    from oracle import lvx_oracle as orc
    from paper_1801_01155_b200 import parallel, synth
    dims = (6, 5, 4)
    pts, attrs, off = synth.lattice_adversarial(301, 9, dims, seed=5)  # ragged, odd count
    n = off.size - 1
    c0, c1 = parallel.shard_range(n, rank, world)
    p0, p1 = int(off[c0]), int(off[c1])
    vox, p_in, p_out, a_in, a_out, curve, within = orc.clip_batch(pts[p0:p1], attrs[p0:p1], off[c0:c1 + 1] - p0, dims)
    # stand-in raw record: (global curve, chord order) key + the chord itself
    rec = np.concatenate([(curve + c0)[:, None].astype(np.float64), within[:, None].astype(np.float64),
                          vox.astype(np.float64), p_in, p_out, a_in[:, None], a_out[:, None]], axis=1)
    parts = parallel.allgather_varlen(torch.from_numpy(rec))
    assert len(parts) == world and parts[rank].shape[0] == rec.shape[0]
    allrec = torch.cat(parts).numpy()
    # rank-order concatenation == the single-process clip of the whole batch
    full = orc.clip_batch(pts, attrs, off, dims)
    want = np.concatenate([full[5][:, None].astype(np.float64), full[6][:, None].astype(np.float64),
                           full[0].astype(np.float64), full[1], full[2], full[3][:, None], full[4][:, None]], axis=1)
    assert np.array_equal(allrec, want)
    # ... hence a stable sort by voxel reproduces the reference's per-voxel order
    lin = allrec[:, 2] + dims[0] * (allrec[:, 3] + dims[1] * allrec[:, 4])
    order = np.argsort(lin, kind="stable")
    key = allrec[order, 0] * 1e6 + allrec[order, 1]
    same = lin[order][1:] == lin[order][:-1]
    assert np.all(key[1:][same] > key[:-1][same])
    # counts: all_reduce of per-rank histograms == global histogram
    import torch.distributed as dist
    V = dims[0] * dims[1] * dims[2]
    mine = np.bincount((vox[:, 0] + dims[0] * (vox[:, 1] + dims[1] * vox[:, 2])).astype(np.int64), minlength=V)
    t = torch.from_numpy(mine.astype(np.int32))
    dist.all_reduce(t)
    assert np.array_equal(t.numpy(), np.bincount(lin.astype(np.int64), minlength=V))


def test_line_id_sharding_and_varlen_allgather():
    _run(_worker_voxelize, 2)


def test_shard_ranges_partition():
    from paper_1801_01155_b200 import parallel
    for n in (0, 1, 7, 1000, 1000003):
        for world in (1, 2, 3, 8):
            edges = [parallel.shard_range(n, r, world) for r in range(world)]
            assert edges[0][0] == 0 and edges[-1][1] == n
            assert all(edges[i][1] == edges[i + 1][0] for i in range(world - 1))
            assert max(h - l for l, h in edges) - min(h - l for l, h in edges) <= 1


def test_tiles_partition_the_screen():
    from paper_1801_01155_b200 import parallel
    for (W, H) in ((1920, 1080), (3840, 2160), (150, 70), (1, 1)):
        for world in (1, 2, 4, 8):
            seen = np.zeros(W * H, np.int32)
            for r in range(world):
                idx, mask = parallel.tile_pixel_indices(r, world, W, H)
                np.add.at(seen, idx[mask], 1)
            assert seen.min() == 1 and seen.max() == 1
            n = [parallel.my_tiles(r, world, W, H).size for r in range(world)]
            assert max(n) - min(n) <= 1
