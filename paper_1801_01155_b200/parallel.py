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


def _host_staged(group=None) -> bool:
    """True when the group's backend cannot move CUDA tensors (gloo: used to run the multi-rank
    paths with several ranks sharing ONE GPU in tests): collectives then go through host memory."""
    import torch.distributed as dist
    return dist.get_backend(group) == "gloo"


# dtypes every backend (NCCL included) can move; anything else travels as its bytes
_WIRE_DTYPES = ("torch.uint8", "torch.int8", "torch.int32", "torch.int64", "torch.float16", "torch.bfloat16",
                "torch.float32", "torch.float64")


def _as_wire(t):
    """ProcessGroupNCCL has no mapping for int16 / uint16 / uint32 / uint64 / bool: ship the bytes."""
    import torch
    if str(t.dtype) in _WIRE_DTYPES:
        return t, None
    # (rows stay rows: [n, ...] -> [n, bytes per row], so the first dimension keeps its meaning)
    return t.contiguous().reshape(t.shape[0], -1).view(torch.uint8), (t.dtype, tuple(t.shape[1:]))


def allgather_varlen_multi(tensors, group=None):
    """all_gather of several 1-D/2-D tensors whose first dimension differs per rank, with ONE
    size exchange (and one host read) for all of them and one `all_gather_into_tensor` per
    tensor.  Returns, per input tensor, the list of per-rank tensors in rank order."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = tensors[0].device
    if dev.type == "cuda" and _host_staged(group):
        return [[p.to(dev) for p in parts] for parts in allgather_varlen_multi([t.cpu() for t in tensors], group)]
    mine = torch.tensor([int(t.shape[0]) for t in tensors], dtype=torch.int64, device=dev)
    sizes = torch.empty(world * len(tensors), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(sizes, mine, group=group)  # (flat output: what gloo and NCCL both accept)
    sizes = sizes.view(world, len(tensors)).cpu().tolist()  # the one synchronisation: it sizes the receive buffers
    out = []
    for k, t in enumerate(tensors):
        wire, orig = _as_wire(t)
        m = max(max(sizes[r][k] for r in range(world)), 1)
        if wire.shape[0] == m:
            send = wire.contiguous()
        else:
            send = torch.zeros((m,) + tuple(wire.shape[1:]), dtype=wire.dtype, device=dev)
            send[:wire.shape[0]] = wire
        recv = torch.empty(world * send.numel(), dtype=send.dtype, device=dev)
        dist.all_gather_into_tensor(recv, send.reshape(-1), group=group)
        recv = recv.view((world,) + tuple(send.shape))
        parts = [recv[r, :sizes[r][k]] for r in range(world)]
        if orig is not None:
            parts = [p.contiguous().view(orig[0]).reshape((p.shape[0],) + orig[1]) for p in parts]
        out.append(parts)
    return out


def all_reduce_(t, op=None, group=None):
    """all_reduce in place (through host memory when the backend cannot move CUDA tensors)."""
    import torch.distributed as dist
    op = dist.ReduceOp.SUM if op is None else op
    if t.device.type == "cuda" and _host_staged(group):
        h = t.cpu()
        dist.all_reduce(h, op=op, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op, group=group)
    return t


def allgather_varlen(t, group=None):
    """all_gather of one 1-D/2-D tensor whose first dimension differs per rank.
    Returns the list of per-rank tensors (rank order)."""
    return allgather_varlen_multi([t], group)[0]


# --- frame exchange: ONE collective per frame, no host synchronisation ------------------------
#
# Every rank's send buffer is a flat float32 tensor of the same length on all ranks,
#   [ m * tile_h * tile_w * 4 floats of tiles | 8 floats of tail ]
# with m = the largest tile count of any rank (a pure function of W, H, world: rank 0's) and
# the tail holding the rank's three frame counters (voxel_steps, intersection_tests,
# window_overflow) as int64 bit patterns.  The kernels render straight into the front part.

TAIL_FLOATS = 8  # 3 int64 counters + one spare, keeps the buffer a multiple of 16 bytes


def tile_counts(world: int, width: int, height: int, tile_w: int = MG_TILE_W, tile_h: int = MG_TILE_H):
    """Tiles per rank of the interleaved partition (rank order): no communication needed."""
    tx, ty = tile_grid(width, height, tile_w, tile_h)
    total = tx * ty
    return [max(0, (total - r + world - 1) // world) for r in range(world)]


def send_layout(world: int, width: int, height: int, tile_w: int = MG_TILE_W, tile_h: int = MG_TILE_H):
    """(m, tile floats per rank, send-buffer length in floats)."""
    m = max(tile_counts(world, width, height, tile_w, tile_h)[0], 1)
    body = m * tile_h * tile_w * 4
    return m, body, body + TAIL_FLOATS


def new_send_buffer(world: int, width: int, height: int, device, tile_w: int = MG_TILE_W, tile_h: int = MG_TILE_H):
    import torch
    return torch.zeros(send_layout(world, width, height, tile_w, tile_h)[2], dtype=torch.float32, device=device)


def send_tiles_view(send, n_tiles: int, tile_w: int = MG_TILE_W, tile_h: int = MG_TILE_H):
    """The first n_tiles tiles of a send buffer as [n, tile_h, tile_w, 4]."""
    return send[:n_tiles * tile_h * tile_w * 4].view(n_tiles, tile_h, tile_w, 4)


def pack_counters(send, totals):
    """Write the rank's int64[3] counters into the tail of its send buffer (device-side copy)."""
    import torch
    send[-TAIL_FLOATS:].view(torch.int64)[:3].copy_(totals.to(torch.int64))


def unpack_counters(recv):
    """Sum of the ranks' counters: int64[3] tensor (recv is [world, L])."""
    import torch
    return recv[:, -TAIL_FLOATS:].contiguous().view(torch.int64)[:, :3].sum(dim=0)


def gather_tiles(send, dst: int = 0, group=None, recv=None):
    """Gather every rank's send buffer (same length everywhere, see above) on `dst` with ONE
    collective and no size exchange or host read.  Returns the [world, L] receive tensor on
    `dst` (pass `recv` to reuse a preallocated one) and None elsewhere."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if send.device.type == "cuda" and _host_staged(group):
        got = gather_tiles(send.cpu(), dst, group)
        if got is None:
            return None
        if recv is None:
            return got.to(send.device)
        recv.copy_(got)
        return recv
    if rank != dst:
        dist.gather(send, None, dst=dst, group=group)
        return None
    if recv is None:
        recv = torch.empty((world, send.numel()), dtype=send.dtype, device=send.device)
    dist.gather(send, list(recv.unbind(0)), dst=dst, group=group)
    return recv


# --- rendering ---------------------------------------------------------------------------

def render_my_tiles(camera: Camera, model, octree, params: RenderParams, rank: int, world: int,
                    moving: bool = False, tile_w: int = MG_TILE_W, tile_h: int = MG_TILE_H, replines=None,
                    send=None):
    """Render rank's interleaved tiles straight into (the front of) its send buffer.
    Returns (tiles f32[n_tiles, tile_h, tile_w, 4] -- a view of `send` --, row_stats i64[H,3], send)."""
    torch = _lib.require_device()
    plan = FramePlan(camera, model, octree, params, resolve_neighbor(params, moving),
                     tile_first=rank, tile_step=world, compact=True, tile_w=tile_w, tile_h=tile_h,
                     replines=replines)
    n = plan.n_my_tiles()
    if send is None:
        send = new_send_buffer(world, camera.width, camera.height, "cuda", tile_w, tile_h)
    tiles = send_tiles_view(send, max(n, 1), tile_w, tile_h)
    stats = torch.zeros((camera.height, 3), dtype=torch.int64, device="cuda")
    plan.launch(tiles, stats)
    return tiles[:n], stats, send


def untile_into(tiles, rank: int, world: int, width: int, height: int, img_d,
                tile_w: int = MG_TILE_W, tile_h: int = MG_TILE_H):
    """Scatter one rank's compact tiles into the full (H, W, 4) device image."""
    if tiles.shape[0] == 0:
        return
    t = _lib.Tiling()
    t.tile_w, t.tile_h, t.tile_first, t.tile_step, t.compact = tile_w, tile_h, rank, world, 1
    _lib.check(_lib.lib().lvx_untile(_lib.ptr(tiles), C.byref(t), C.c_int32(width), C.c_int32(height),
                                     _lib.ptr(img_d), _lib.stream_ptr()))


def untile_all(recv, world: int, width: int, height: int, img_d, tile_w: int = MG_TILE_W,
               tile_h: int = MG_TILE_H):
    """Scatter the gathered buffers of ALL ranks ([world, L]) into the image with one launch."""
    _lib.check(_lib.lib().lvx_untile_all(_lib.ptr(recv), C.c_int64(int(recv.stride(0))), C.c_int32(world),
                                         C.c_int32(tile_w), C.c_int32(tile_h), C.c_int32(width),
                                         C.c_int32(height), _lib.ptr(img_d), _lib.stream_ptr()))


def render_frame_tiled(camera: Camera, model, octree=None, replines=None,
                       params: Optional[RenderParams] = None, moving: bool = False, group=None,
                       to_host: bool = True):
    """`render_frame` over all ranks of `group` (default: the world).  Every rank
    must hold the same model.  Returns a Frame on rank 0 and None elsewhere.

    Per frame: render into the send buffer, append the three counters, ONE gather, one
    untile launch on rank 0.  No size exchange, no separate reduce, no host read before the
    final copy."""
    import torch
    import torch.distributed as dist
    if params is None:
        params = RenderParams()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tiles, stats, send = render_my_tiles(camera, model, octree, params, rank, world, moving, replines=replines)
    e1.record()
    pack_counters(send, stats.sum(dim=0))
    recv = gather_tiles(send, 0, group)
    if rank != 0:
        return None
    H, W = camera.height, camera.width
    img_d = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
    untile_all(recv, world, W, H, img_d)
    if to_host:
        host = torch.empty((H, W, 4), dtype=torch.float32, pin_memory=True)
        host.copy_(img_d, non_blocking=True)
    tot = unpack_counters(recv).cpu()
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
    `group`; every rank passes the same `curves` and receives the same full model.

    A failure on one rank (MemoryError of its crossing bound, a CUDA error) is agreed on by
    all ranks BEFORE the data collectives, so nobody is left waiting in NCCL."""
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
    sh, failure = None, None
    try:
        sh = voxelize_shard(_lib.to_device(pts[p0:p1], np.float64), _lib.to_device(attrs[p0:p1], np.float64),
                            local_off, c1 - c0, spec, p0)
    except Exception as e:  # agreed on below; re-raised on every rank
        failure = e
    flag = torch.tensor([0 if failure is None else (2 if isinstance(failure, MemoryError) else 1)],
                        dtype=torch.int32, device=local_off.device)
    flag = all_reduce_(flag, dist.ReduceOp.MAX, group)
    if int(flag.item()) != 0:
        if failure is not None:
            raise failure
        kind = MemoryError if int(flag.item()) == 2 else RuntimeError
        raise kind("sharded voxelization failed on another rank")
    total = all_reduce_(sh["vox_cnt"].clone(), dist.ReduceOp.SUM, group)  # int32 bit patterns of u32 counts add correctly
    err = all_reduce_(sh["err"].clone(), dist.ReduceOp.MAX, group)
    # (edge_kept is u16 in an int16 tensor: it travels as bytes, NCCL has no 16-bit integer type)
    keys, qs, lins, kept = allgather_varlen_multi(
        [sh["raw_key"], sh["raw_q"], sh["raw_lin"], sh["edge_kept"][:p1 - p0]], group)
    out = merge_shards(spec, total, torch.cat(keys), torch.cat(qs), torch.cat(lins), edge_kept=torch.cat(kept),
                       off_d=_lib.to_device(off, np.int64), n_curves=n_curves, memory_budget=memory_budget)
    out["err"] = err
    return vz.model_from_device(out, spec, transfer_table)
