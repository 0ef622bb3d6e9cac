"""The multi-GPU paths executed END TO END with two ranks -- real kernels, real collectives -- on the
ONE GPU a test box has: both ranks share cuda:0 and talk over gloo (collectives staged through host
memory, parallel._host_staged).  What a second GPU would add is NCCL's transport, nothing else:
`render_frame_tiled` must return the single-process frame byte for byte (image and counters),
`build_voxel_model_sharded` the single-process model byte for byte on every rank."""
import os
import socket
import sys

import numpy as np
import pytest

from conftest import MODEL_FIELDS, ROOT

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _entry(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        import paper_1801_01155_b200 as lv
        from paper_1801_01155_b200 import parallel, synth
        dims = (20, 16, 12)
        lines = synth.turbulence(300, 50, dims)
        cs = lv.CurveSet.from_flat(*lines)
        spec = lv.GridSpec(dims, 32)
        # voxelization sharded by line ID over the two ranks
        m = parallel.build_voxel_model_sharded(cs, spec)
        single = lv.build_voxel_model(cs, spec)
        for f in MODEL_FIELDS:
            assert np.array_equal(np.asarray(getattr(m, f)), np.asarray(getattr(single, f))), (rank, f)
        assert m.dropped_overflow == single.dropped_overflow
        # the frame: interleaved tiles, one gather, one untile launch
        oc = lv.build_lod(m)
        m.ao = lv.precompute_voxel_ao(m, oc, lv.AOParams(n_rays=12, radius=3.0, step=1.0))
        cam = lv.default_camera(dims, 150, 70)   # not a multiple of the 32x16 tile
        for kw in (dict(base_opacity=0.3, neighbor_mode="on", ao_mode="precomputed"),
                   dict(base_opacity=0.3, neighbor_mode="off"),
                   dict(neighbor_mode="on", shadow_mode="cone", light_dir=(0.3, 0.2, 1.0))):
            p = lv.RenderParams(**kw)
            fr = parallel.render_frame_tiled(cam, m, oc, None, p)
            if rank == 0:
                ref = lv.render_frame(cam, m, oc, None, p)
                assert np.array_equal(fr.image, ref.image), kw
                for k in ("rays", "voxel_steps", "intersection_tests", "window_overflow", "neighbor"):
                    assert fr.stats[k] == ref.stats[k], (kw, k)
                assert fr.stats["workers"] == world
            else:
                assert fr is None
        with open(os.path.join(out_dir, f"ok{rank}"), "w") as fh:
            fh.write("ok")
    finally:
        dist.destroy_process_group()


def test_two_ranks_share_one_gpu(tmp_path):
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_entry, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    assert all(os.path.exists(tmp_path / f"ok{r}") for r in range(world))
