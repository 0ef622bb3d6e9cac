"""Multi-GPU paths (one process per GPU, torch.distributed over NCCL/NVLink).

The reference has no distributed code; the partitioning follows
BASELINE.json's north_star and SURVEY.md 8e:

* rendering  -- the voxel model, LoD and AO field are replicated; the image is cut
  into interleaved screen tiles (tile k belongs to rank k mod world); every rank
  renders its tiles straight into a compact send buffer and rank 0 gathers the
  buffers with one NCCL gather and scatters them into the frame (`lvx_untile`).
  Pixels are independent, so the result is bit-identical to a single-GPU frame.
* voxelization -- polylines are sharded by contiguous line-ID ranges; every rank
  clips its shard, the per-voxel counts are all-reduced, the raw chord records
  all-gathered, and each rank regroups them by voxel (`lvx_raw_regroup`) and runs
  the ordering/cap/pack pass.  Record keys carry the GLOBAL edge index, so the
  per-voxel order -- and therefore every output byte -- equals the single-GPU
  (and the reference's) result.  Every rank ends with the full replicated model.

The collective plumbing (`shard_range`, `allgather_varlen`, `gather_tiles`,
`tile_pixel_indices`) is device-agnostic so it is covered by world_size-2 gloo
tests on CPU; the kernels themselves only run on the GPU.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib
from .raycast import Camera, Frame, FramePlan, RenderParams, resolve_neighbor
from .scene_io import CurveSet, GridSpec

# screen tile of the multi-GPU partition: 4 x 4 warps of 8x4 pixels
MG_TILE_W, MG_TILE_H = 32, 16


# --- partitioning helpers (pure host logic) --------------------------------------------

def shard_range(n: int, rank: int, world: int):
    """Contiguous [lo, hi) share of n items; concatenating the shares in rank order
    gives 0..n, which is what keeps the per-voxel (curve, chord) order intact."""
    lo = (n * rank) // world
    hi = (n * (rank + 1)) // world
    return lo, hi


def tile_grid(width: int, height: int, tile_w: int = MG_TILE_W, tile_h: int = MG_TILE_H):
    return -(-width // tile_w), -(-height // tile_h)


def my_tiles(rank: int, world: int, width: int, height: int, tile_w: int = MG_TILE_W,
             tile_h: int = MG_TILE_H) -> np.ndarray:
    tx, ty = tile_grid(width, height, tile_w, tile_h)
    return np.arange(rank, tx * ty, world, dtype=np.int64)


def tile_pixel_indices(rank: int, world: int, width: int, height: int, tile_w: int = MG_TILE_W,
                       tile_h: int = MG_TILE_H):
    """For rank's compact tile buffer [n_tiles, tile_h, tile_w]: the flat pixel index
    y*W+x of every slot and a mask of the slots that fall inside the image."""
    tx, _ = tile_grid(width, height, tile_w, tile_h)
    tiles = my_tiles(rank, world, width, height, tile_w, tile_h)
    x0 = (tiles % tx) * tile_w
    y0 = (tiles // tx) * tile_h
    xs = x0[:, None, None] + np.arange(tile_w)[None, None, :]
    ys = y0[:, None, None] + np.arange(tile_h)[None, :, None]
    xs, ys = np.broadcast_arrays(xs, ys)
    mask = (xs < width) & (ys < height)
    return (ys * width + xs).astype(np.int64), mask


def allgather_varlen(t, group=None):
    """all_gather of 1-D/2-D tensors whose first dimension differs per rank.
    Returns the list of per-rank tensors (rank order)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(max(sizes), 1)
    pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[:t.shape[0]] = t
    out = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(out, pad, group=group)
    return [o[:s] for o, s in zip(out, sizes)]


def gather_tiles(tiles, dst: int = 0, group=None):
    """Gather every rank's compact tile buffer on `dst` (list in rank order there,
    None elsewhere).  Buffers differ by at most one tile, so they are padded to
    the largest and sent with ONE collective."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = torch.tensor([tiles.shape[0]], dtype=torch.int64, device=tiles.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(max(sizes), 1)
    if tiles.shape[0] == m:
        send = tiles.contiguous()
    else:
        send = torch.zeros((m,) + tuple(tiles.shape[1:]), dtype=tiles.dtype, device=tiles.device)
        send[:tiles.shape[0]] = tiles
    recv = [torch.empty_like(send) for _ in range(world)] if rank == dst else None
    dist.gather(send, recv, dst=dst, group=group)
    if rank != dst:
        return None
    return [r[:s] for r, s in zip(recv, sizes)]


# --- rendering ---------------------------------------------------------------------------

def render_my_tiles(camera: Camera, model, octree, params: RenderParams, rank: int, world: int,
                    moving: bool = False, tile_w: int = MG_TILE_W, tile_h: int = MG_TILE_H, replines=None):
    """Render rank's interleaved tiles into a compact buffer.
    Returns (tiles f32[n_tiles, tile_h, tile_w, 4], row_stats i64[H,3]) on the device."""
    torch = _lib.require_device()
    plan = FramePlan(camera, model, octree, params, resolve_neighbor(params, moving),
                     tile_first=rank, tile_step=world, compact=True, tile_w=tile_w, tile_h=tile_h,
                     replines=replines)
    n = plan.n_my_tiles()
    tiles = torch.zeros((max(n, 1), tile_h, tile_w, 4), dtype=torch.float32, device="cuda")
    stats = torch.zeros((camera.height, 3), dtype=torch.int64, device="cuda")
    plan.launch(tiles, stats)
    return tiles[:n], stats


def untile_into(tiles, rank: int, world: int, width: int, height: int, img_d,
                tile_w: int = MG_TILE_W, tile_h: int = MG_TILE_H):
    """Scatter one rank's compact tiles into the full (H, W, 4) device image."""
    if tiles.shape[0] == 0:
        return
    t = _lib.Tiling()
    t.tile_w, t.tile_h, t.tile_first, t.tile_step, t.compact = tile_w, tile_h, rank, world, 1
    _lib.check(_lib.lib().lvx_untile(_lib.ptr(tiles), C.byref(t), C.c_int32(width), C.c_int32(height),
                                     _lib.ptr(img_d), _lib.stream_ptr()))


def render_frame_tiled(camera: Camera, model, octree=None, replines=None,
                       params: Optional[RenderParams] = None, moving: bool = False, group=None,
                       to_host: bool = True):
    """`render_frame` over all ranks of `group` (default: the world).  Every rank
    must hold the same model.  Returns a Frame on rank 0 and None elsewhere."""
    import torch
    import torch.distributed as dist
    if params is None:
        params = RenderParams()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tiles, stats = render_my_tiles(camera, model, octree, params, rank, world, moving, replines=replines)
    e1.record()
    tot = stats.sum(dim=0)
    dist.reduce(tot, dst=0, group=group)
    parts = gather_tiles(tiles, 0, group)
    if rank != 0:
        return None
    H, W = camera.height, camera.width
    img_d = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
    for r, part in enumerate(parts):
        untile_into(part, r, world, W, H, img_d)
    if to_host:
        host = torch.empty((H, W, 4), dtype=torch.float32, pin_memory=True)
        host.copy_(img_d, non_blocking=True)
    tot = tot.cpu()
    torch.cuda.current_stream().synchronize()
    stats = {"rays": W * H, "voxel_steps": int(tot[0]), "intersection_tests": int(tot[1]),
             "ms": float(e0.elapsed_time(e1)), "workers": world, "window_overflow": int(tot[2]),
             "neighbor": bool(resolve_neighbor(params, moving))}
    return Frame(image=host.numpy() if to_host else img_d, stats=stats)


# --- voxelization ----------------------------------------------------------------------------

def voxelize_shard(pts_d, attrs_d, off_d, n_curves: int, spec: GridSpec, point_base: int,
                   want_edge_kept: bool = True):
    """One rank's share: clip its polylines and emit raw records whose keys carry the
    GLOBAL edge index (local index + point_base).  Returns a dict of device tensors:
    vox_cnt u32[V] (uncapped), raw_key/raw_q/raw_lin [n_local], edge_kept u16[P_local], err."""
    from . import voxelizer as vz
    vox_cnt, raw_key, raw_q, raw_lin, edge_kept, err = vz.stage_clip(pts_d, attrs_d, off_d, n_curves, spec,
                                                                     want_edge_kept)
    if point_base:
        raw_key = raw_key + (int(point_base) << 16)  # (slots without a chord are skipped downstream)
    return {"vox_cnt": vox_cnt, "raw_key": raw_key, "raw_q": raw_q, "raw_lin": raw_lin,
            "edge_kept": edge_kept, "err": err}


def merge_shards(spec: GridSpec, vox_cnt_total, raw_key, raw_q, raw_lin, *, caches: bool = True,
                 edge_kept=None, off_d=None, n_curves: int = 0, memory_budget=None):
    """Merge the concatenated raw records of all shards into the final model tensors
    (global scan -> regroup by voxel -> order/cap/pack)."""
    import torch
    from . import voxelizer as vz
    cursor, offsets, counts, n_raw, S = vz.stage_scan(vox_cnt_total)
    if n_raw > int(raw_key.shape[0]):
        raise RuntimeError(f"shard slots ({int(raw_key.shape[0])}) cannot hold the summed counts ({n_raw})")
    vz.check_budget(spec, S, memory_budget)
    grouped = vz.stage_regroup(raw_key.contiguous(), raw_q.contiguous(), raw_lin.contiguous(), n_raw, cursor)
    prov = edge_kept is not None
    out = vz.stage_compact(grouped, n_raw, vox_cnt_total, cursor, offsets, counts, spec, S, caches, prov)
    if prov:
        out["seg_curve"], out["seg_order"] = vz.stage_provenance(out.pop("seg_key"), S, edge_kept, off_d,
                                                                 n_curves)
    out["n_segments"] = S
    out["dropped"] = n_raw - S
    return out


def build_voxel_model_sharded(curves: CurveSet, spec: GridSpec, transfer_table=None,
                              memory_budget: Optional[int] = None, group=None):
    """`build_voxel_model` with the clipping sharded by line ID over the ranks of
    `group`; every rank passes the same `curves` and receives the same full model."""
    import torch
    import torch.distributed as dist
    from . import voxelizer as vz
    transfer_table = vz._check_table(transfer_table)
    _lib.require_device()
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    pts, attrs, off = curves.flat()
    n_curves = int(off.size - 1)
    c0, c1 = shard_range(n_curves, rank, world)
    p0, p1 = int(off[c0]), int(off[c1])
    local_off = _lib.to_device(off[c0:c1 + 1] - p0, np.int64)
    sh = voxelize_shard(_lib.to_device(pts[p0:p1], np.float64), _lib.to_device(attrs[p0:p1], np.float64),
                        local_off, c1 - c0, spec, p0)
    total = sh["vox_cnt"].clone()
    dist.all_reduce(total, group=group)  # int32 bit patterns of u32 counts add correctly
    err = sh["err"].clone()
    dist.all_reduce(err, op=dist.ReduceOp.MAX, group=group)
    keys = torch.cat(allgather_varlen(sh["raw_key"], group))
    qs = torch.cat(allgather_varlen(sh["raw_q"], group))
    lins = torch.cat(allgather_varlen(sh["raw_lin"], group))
    edge_kept = torch.cat(allgather_varlen(sh["edge_kept"][:p1 - p0], group))
    out = merge_shards(spec, total, keys, qs, lins, edge_kept=edge_kept,
                       off_d=_lib.to_device(off, np.int64), n_curves=n_curves, memory_budget=memory_budget)
    out["err"] = err
    return vz.model_from_device(out, spec, transfer_table)
