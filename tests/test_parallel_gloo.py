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
    # sizes are a pure function of (W, H, world): nobody exchanges them
    counts = parallel.tile_counts(world, W, H)
    assert counts[rank] == idx.shape[0] and counts[0] == max(counts)
    m, body, L = parallel.send_layout(world, W, H)
    send = parallel.new_send_buffer(world, W, H, "cpu")
    assert send.numel() == L and m == counts[0]
    # stand-in for the render kernel: pixel value = f(pixel index), zeros outside the image,
    # written straight into the front of the send buffer
    tiles = np.where(mask, idx, 0).astype(np.float32)[..., None] * np.array([1, 2, 3, 4], np.float32)
    parallel.send_tiles_view(send, idx.shape[0]).copy_(torch.from_numpy(tiles))
    # the rank's three counters ride in the tail of the same buffer (values beyond 2^53: bit patterns)
    mine = torch.tensor([10 + rank, (1 << 60) + 7 * rank, rank], dtype=torch.int64)
    parallel.pack_counters(send, mine)
    recv = parallel.gather_tiles(send, 0)
    again = parallel.gather_tiles(send, 0, recv=recv)  # a preallocated receive buffer is filled in place
    if rank != 0:
        assert recv is None and again is None
        return
    assert again is recv
    assert tuple(recv.shape) == (world, L)
    img = np.full((H * W, 4), -1.0, np.float32)
    for r in range(world):
        i, msk = parallel.tile_pixel_indices(r, world, W, H)
        part = parallel.send_tiles_view(recv[r], i.shape[0]).numpy()
        img[i[msk]] = part[msk]
    want = np.arange(H * W, dtype=np.float32)[:, None] * np.array([1, 2, 3, 4], np.float32)
    assert np.array_equal(img, want)  # every pixel written exactly once, by the right tile
    tot = parallel.unpack_counters(recv).tolist()
    assert tot == [sum(10 + r for r in range(world)), world * (1 << 60) + 7 * sum(range(world)), sum(range(world))]


@pytest.mark.parametrize("size", [(150, 70), (64, 32), (33, 17)])
def test_tile_gather_reassembles_the_frame(size):
    _run(_worker_tiles, 2, *size)


def test_tile_gather_three_ranks_uneven():
    _run(_worker_tiles, 3, 150, 70)  # 5 x 5 tiles over 3 ranks: 9 / 8 / 8


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


def _worker_sharded_build(rank, world, fail_rank):
    """`build_voxel_model_sharded` itself, end to end over gloo, with the two GPU stages stood
    in for: the clip of a shard by the CPU oracle (records in the device pipeline's raw format,
    edge_kept as int16 like the kernel's), the merge by a check against the single-process
    result.  Exercises the shard ranges, the failure agreement, the count all-reduce and the
    single-size-exchange all-gather with a 16-bit tensor that must travel as bytes."""
    import torch
    from oracle import lvx_oracle as orc
    from paper_1801_01155_b200 import _lib, parallel, synth, voxelizer as vz
    import paper_1801_01155_b200 as lv
    dims = (6, 5, 4)
    pts, attrs, off = synth.lattice_adversarial(301, 9, dims, seed=5)
    V = dims[0] * dims[1] * dims[2]

    def raw_of(p, a, o, point_base):
        vox, p_in, p_out, a_in, a_out, curve, within = orc.clip_batch(p, a, o, dims)
        lin = (vox[:, 0] + dims[0] * (vox[:, 1] + dims[1] * vox[:, 2])).astype(np.int64)
        # stand-in key: (global first point of the curve, chord order) -- increasing in curve order
        key = ((o[curve] + point_base) << 16) | within
        q = (p_in * 1e3).astype(np.int64).sum(1) * 7 + (p_out * 1e3).astype(np.int64).sum(1)
        kept = np.zeros(p.shape[0], np.int16)
        np.add.at(kept, o[curve], 1)
        return dict(vox_cnt=torch.from_numpy(np.bincount(lin, minlength=V).astype(np.int32)),
                    raw_key=torch.from_numpy(key.astype(np.int64)), raw_q=torch.from_numpy(q),
                    raw_lin=torch.from_numpy(lin.astype(np.int32)), edge_kept=torch.from_numpy(kept),
                    err=torch.zeros(1, dtype=torch.int32))

    def fake_shard(pts_d, attrs_d, off_d, n_curves, spec, point_base, want_edge_kept=True):
        if rank == fail_rank:
            raise MemoryError("this rank's crossing bound exceeds 2^32")
        return raw_of(pts_d.numpy(), attrs_d.numpy(), off_d.numpy(), point_base)

    seen = {}

    def fake_merge(spec, total, keys, qs, lins, *, caches=True, edge_kept=None, off_d=None, n_curves=0,
                   memory_budget=None):
        want = raw_of(pts, attrs, off, 0)
        assert torch.equal(total, want["vox_cnt"])
        assert torch.equal(keys, want["raw_key"]) and torch.equal(qs, want["raw_q"]) and torch.equal(lins, want["raw_lin"])
        assert edge_kept.dtype == torch.int16 and torch.equal(edge_kept, want["edge_kept"])
        assert n_curves == off.size - 1 and torch.equal(off_d, torch.from_numpy(off))
        seen["merged"] = True
        return {"n_segments": int(keys.shape[0]), "dropped": 0}

    def to_cpu(a, dtype=None):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype))

    orig = (parallel.voxelize_shard, parallel.merge_shards, _lib.to_device, _lib.require_device, vz.model_from_device)
    parallel.voxelize_shard, parallel.merge_shards = fake_shard, fake_merge
    _lib.to_device, _lib.require_device = to_cpu, (lambda: torch)
    vz.model_from_device = lambda out, spec, table: out
    try:
        cs = lv.CurveSet.from_flat(pts, attrs, off)
        if fail_rank is None:
            out = parallel.build_voxel_model_sharded(cs, lv.GridSpec(dims))
            assert seen.get("merged") and int(out["err"].item()) == 0
        else:
            # the failing rank's exception surfaces on EVERY rank, before any data collective
            with pytest.raises(MemoryError):
                parallel.build_voxel_model_sharded(cs, lv.GridSpec(dims))
            assert not seen
    finally:
        (parallel.voxelize_shard, parallel.merge_shards, _lib.to_device, _lib.require_device,
         vz.model_from_device) = orig


def test_sharded_build_end_to_end_over_gloo():
    _run(_worker_sharded_build, 2, None)


def test_sharded_build_failure_is_raised_on_every_rank():
    _run(_worker_sharded_build, 2, 1)


def test_allgather_varlen_multi_mixed_dtypes():
    _run(_worker_varlen_multi, 2)


def _worker_varlen_multi(rank, world):
    import torch
    from paper_1801_01155_b200 import parallel
    n = 3 + 2 * rank
    a = torch.arange(n, dtype=torch.int64) + 100 * rank
    b = (torch.arange(n * 2, dtype=torch.int16) - 5 + rank).reshape(n, 2)   # 16-bit: travels as bytes
    c = torch.zeros(0, dtype=torch.int32) if rank == 0 else torch.ones(4, dtype=torch.int32)  # empty on one rank
    pa, pb, pc = parallel.allgather_varlen_multi([a, b, c])
    for r in range(world):
        m = 3 + 2 * r
        assert torch.equal(pa[r], torch.arange(m, dtype=torch.int64) + 100 * r)
        assert pb[r].dtype == torch.int16 and torch.equal(pb[r], (torch.arange(m * 2, dtype=torch.int16) - 5 + r).reshape(m, 2))
    assert pc[0].numel() == 0 and torch.equal(pc[1], torch.ones(4, dtype=torch.int32))


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
