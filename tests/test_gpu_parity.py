"""CUDA path vs the CPU oracle on seeded inputs the oracle finishes in seconds,
edge cases, error behaviour, and size-independent properties at the full
BASELINE.json sizes."""
import numpy as np
import pytest

from conftest import MODEL_FIELDS, assert_model_equal

pytestmark = pytest.mark.gpu

MAX_ERR = 1.0 / 255.0
MEAN_ERR = 1e-3


@pytest.fixture(scope="module")
def lv():
    import paper_1801_01155_b200 as lv
    return lv


@pytest.fixture(scope="module")
def synth():
    from paper_1801_01155_b200 import synth
    return synth


def both(lv, oracle, gen, dims, n_bins=32, table=None):
    pts, attrs, off = gen
    m = lv.build_voxel_model(lv.CurveSet.from_flat(pts, attrs, off), lv.GridSpec(dims, n_bins), table)
    ref = oracle.build_voxel_model(pts, attrs, off, dims, n_bins, table)
    return m, ref


def as_dict(ref):
    return {f: getattr(ref, f) for f in MODEL_FIELDS}


# --- configs[0]: 1k helices x 100 pts, 64^3, 256x256 opaque -------------------------

@pytest.fixture(scope="module")
def c1(lv, oracle, synth):
    dims = (64, 64, 64)
    m, ref = both(lv, oracle, synth.helices(1000, 100, dims), dims)
    return dims, m, ref


def test_c1_voxel_model(c1):
    dims, m, ref = c1
    assert ref.segment_count == 263432  # SURVEY.md 8c golden count
    assert_model_equal(m, as_dict(ref))


def test_c1_golden_hash(c1):
    import hashlib
    _, m, _ = c1
    # sha256 prefix of `packed` observed on the unmodified reference
    assert hashlib.sha256(m.packed.tobytes()).hexdigest()[:16] == "3587d4ece308025c"


def test_c1_lod_and_ao(lv, oracle, c1):
    dims, m, ref = c1
    oc = lv.build_lod(m)
    levels = oracle.build_octree(oracle.compute_density_level0(ref))
    assert oc.n_levels == len(levels) == 7
    for a, b in zip(oc.levels, levels):
        assert np.array_equal(a, b)
    ao = lv.precompute_voxel_ao(m, oc)
    assert np.array_equal(ao.values, oracle.precompute_voxel_ao(ref, levels, 100, 5.0, 1.0))


@pytest.mark.parametrize("kw", [
    dict(neighbor_mode="on"),
    dict(neighbor_mode="off"),
    dict(neighbor_mode="on", base_opacity=0.25),
    dict(neighbor_mode="off", base_opacity=0.25, joint_spheres=False),
    dict(neighbor_mode="on", base_opacity=0.25, ao_mode="precomputed", shadow_mode="cone",
         light_dir=(0.3, 0.2, 1.0)),
    dict(neighbor_mode="off", base_opacity=0.25, ao_mode="density-rays"),
    dict(neighbor_mode="on", base_opacity=0.05, tau=1.0),
], ids=lambda kw: "-".join(f"{k}={v}" for k, v in kw.items() if k != "light_dir"))
@pytest.mark.parametrize("engine", ["tile", "wavefront"])
def test_c1_frames(lv, oracle, c1, kw, engine, monkeypatch):
    monkeypatch.setenv("LVX_ENGINE", engine)
    dims, m, ref = c1
    oc = lv.build_lod(m)
    levels = oracle.build_octree(oracle.compute_density_level0(ref))
    if kw.get("ao_mode") == "precomputed":
        m.ao = lv.precompute_voxel_ao(m, oc)
        ref.ao = oracle.precompute_voxel_ao(ref, levels, 100, 5.0, 1.0)
    fr = lv.render_frame(lv.default_camera(dims, 256, 256), m, oc, None, lv.RenderParams(**kw))
    okw = dict(kw)
    nb = okw.pop("neighbor_mode") == "on"
    img, st = oracle.render(oracle.default_camera(dims, 256, 256), ref, levels, neighbor=nb, **okw)
    err = np.abs(fr.image.astype(np.float64) - img.astype(np.float64))
    assert err.max() <= MAX_ERR and err.mean() < MEAN_ERR
    for k in ("rays", "voxel_steps", "intersection_tests", "window_overflow", "neighbor"):
        assert fr.stats[k] == st[k], k
    if kw == dict(neighbor_mode="on"):
        # counters of the reference's own run of this config
        assert fr.stats["voxel_steps"] == 2430102 and fr.stats["intersection_tests"] == 9073278


# --- other seeded sets vs the oracle --------------------------------------------------

@pytest.mark.parametrize("case", ["turbulence", "wiggles", "lattice", "cap"])
def test_voxelize_matches_oracle(lv, oracle, synth, case):
    if case == "turbulence":
        dims, gen = (64, 64, 64), synth.turbulence(3000, 100, (64, 64, 64))
    elif case == "wiggles":
        dims, gen = (24, 20, 16), synth.wiggles(400, 60, (24, 20, 16))
    elif case == "lattice":
        dims, gen = (12, 10, 8), synth.lattice_adversarial(4000, 12, (12, 10, 8))
    else:
        dims, gen = (3, 3, 3), synth.helices(900, 30, (3, 3, 3), seed=3)
    m, ref = both(lv, oracle, gen, dims)
    assert_model_equal(m, as_dict(ref))
    assert m.dropped_overflow == ref.dropped_overflow
    if case == "cap":
        assert m.dropped_overflow > 0 and m.counts.max() == 255


@pytest.mark.parametrize("n_bins", [2, 4, 16, 64, 256])
def test_bin_resolutions(lv, oracle, synth, n_bins):
    dims = (16, 12, 10)
    m, ref = both(lv, oracle, synth.turbulence(300, 40, dims), dims, n_bins)
    assert_model_equal(m, as_dict(ref))
    assert m.packed.size == lv.record_width(n_bins) * m.segment_count


def test_ragged_and_degenerate_inputs(lv, oracle):
    dims = (5, 4, 3)
    curves = [
        np.array([[0.5, 0.5, 0.5], [4.5, 3.5, 2.5]]),                       # 2 vertices, long diagonal
        np.array([[1.2, 1.2, 1.2], [1.3, 1.4, 1.5], [1.6, 1.1, 1.9]]),      # never leaves its voxel
        np.array([[-3.0, 1.5, 1.5], [9.0, 1.5, 1.5]]),                      # passes through from outside
        np.array([[2.0, 2.0, 1.0], [2.0, 2.0, 1.0], [3.0, 3.0, 2.0]]),      # repeated vertex, lattice points
        np.array([[0.5, 0.5, 0.5], [1.0, 0.5, 0.5], [0.5, 0.5, 0.5]]),      # reversal exactly on a plane
        np.array([[-1.0, -1.0, -1.0], [-2.0, -0.5, -0.2]]),                 # entirely outside
        np.array([[0.5, 3.999999999, 0.5], [4.9, 0.0000001, 2.99999]]),
    ]
    pts = np.concatenate(curves)
    off = np.concatenate([[0], np.cumsum([len(c) for c in curves])]).astype(np.int64)
    attrs = np.linspace(0.0, 1.0, len(pts))
    m, ref = both(lv, oracle, (pts, attrs, off), dims, 8)
    assert_model_equal(m, as_dict(ref))


@pytest.mark.parametrize("seed", [0, 1])
def test_clip_paths_long_edges_and_block_boundaries(lv, oracle, seed):
    """The clip kernel builds chords from a shared-memory tile of a block's events (128 edges) and
    falls back to the edge-parallel path when a block crosses more than 512 planes: mix curves of
    2-5 vertices spanning the whole grid (hundreds of crossings per edge), dense short-edged curves,
    two-vertex curves and curves without any crossing, at lengths that put curve ends on, next to
    and far from the 128-edge block boundaries; provenance (edge, ordinal) included."""
    rng = np.random.default_rng(100 + seed)
    dims = (48, 40, 56)
    hi = np.array(dims, dtype=np.float64)
    curves = []
    for k in range(220):
        kind = rng.integers(0, 6)
        if kind == 0:      # long edges: a few vertices anywhere in (and slightly outside) the grid
            c = rng.uniform(-2.0, hi + 2.0, (int(rng.integers(2, 6)), 3))
        elif kind == 1:    # short steps: a random walk of 100-300 vertices
            n = int(rng.integers(100, 300))
            c = rng.uniform(2.0, hi - 2.0, (1, 3)) + np.cumsum(rng.normal(0.0, 0.45, (n, 3)), axis=0)
        elif kind == 2:    # exactly one block of edges / one less / one more
            n = int(rng.choice([128, 129, 130, 127, 256, 257]))
            c = rng.uniform(2.0, hi - 2.0, (1, 3)) + np.cumsum(rng.normal(0.0, 0.3, (n, 3)), axis=0)
        elif kind == 3:    # the shortest curve the API accepts: two vertices (one edge, zero to a few crossings)
            c = rng.uniform(0.0, hi, (1, 3)) + rng.normal(0.0, 0.8, (2, 3))
        elif kind == 4:    # many vertices inside one voxel: no crossing at all
            c = np.floor(rng.uniform(1.0, hi - 1.0, (1, 3))) + rng.uniform(0.05, 0.95, (int(rng.integers(2, 200)), 3))
        else:              # lattice-aligned vertices (ties between axes)
            c = np.round(rng.uniform(0.0, hi, (int(rng.integers(2, 40)), 3)) * 2.0) / 2.0
        curves.append(np.ascontiguousarray(c, dtype=np.float64))
    pts = np.concatenate(curves)
    off = np.concatenate([[0], np.cumsum([len(c) for c in curves])]).astype(np.int64)
    attrs = rng.uniform(0.0, 1.0, len(pts))
    m, ref = both(lv, oracle, (pts, attrs, off), dims, 16)
    assert_model_equal(m, as_dict(ref))
    assert m.dropped_overflow == ref.dropped_overflow
    assert m.segment_count > 20000


def test_empty_model(lv, oracle):
    dims = (4, 4, 4)
    pts = np.array([[1.1, 1.1, 1.1], [1.2, 1.3, 1.4]])
    m, ref = both(lv, oracle, (pts, np.array([0.0, 1.0]), np.array([0, 2], dtype=np.int64)), dims)
    assert m.segment_count == 0 and ref.segment_count == 0
    assert m.packed.size == 0 and m.seg_a.shape == (0, 3) and not m.counts.any()
    l0 = lv.compute_density_level0(m)
    assert l0.shape == (4, 4, 4) and not l0.any()
    oc = lv.build_octree(l0)
    assert oc.n_levels == 3
    bg = (0.1, 0.2, 0.3, 1.0)
    fr = lv.render_frame(lv.default_camera(dims, 33, 17), m, None, None, lv.RenderParams(background=bg))
    # reference tests/test_raycast.py:402-408: an empty model renders the background
    assert np.allclose(fr.image, np.asarray(bg, np.float32)[None, None, :])
    assert fr.stats["intersection_tests"] == 0 and fr.stats["voxel_steps"] > 0


def test_odd_image_sizes_and_determinism(lv, oracle, synth):
    dims = (10, 9, 7)
    m, ref = both(lv, oracle, synth.wiggles(120, 30, dims), dims)
    levels = oracle.build_octree(oracle.compute_density_level0(ref))
    for (W, H) in ((1, 1), (7, 5), (37, 21), (130, 3)):
        cam = lv.default_camera(dims, W, H)
        fr = lv.render_frame(cam, m, None, None, lv.RenderParams(base_opacity=0.5, neighbor_mode="on"))
        fr2 = lv.render_frame(cam, m, None, None, lv.RenderParams(base_opacity=0.5, neighbor_mode="on"),
                              workers=8)
        img, st = oracle.render(oracle.default_camera(dims, W, H), ref, levels, base_opacity=0.5)
        assert np.array_equal(fr.image, fr2.image) and fr.stats["intersection_tests"] == fr2.stats["intersection_tests"]
        assert np.abs(fr.image - img).max() <= MAX_ERR
        assert fr.stats["voxel_steps"] == st["voxel_steps"]
        assert fr.stats["intersection_tests"] == st["intersection_tests"]


def test_small_frames_after_a_frame_on_a_larger_grid(lv, oracle, synth):
    """The frame scratch (queues, per-ray state) is reused between frames: a tiny frame on a small grid
    right after a frame on a larger one must not pick up anything of it -- lanes past the end of a queue
    once used a stale item's voxel as an address.  Both record sources, both modes."""
    big = (96, 96, 96)
    mb = lv.build_voxel_model(lv.CurveSet.from_flat(*synth.turbulence(3000, 60, big)), lv.GridSpec(big))
    dims = (10, 9, 7)
    m, ref = both(lv, oracle, synth.wiggles(120, 30, dims), dims)
    enc = lv.VoxelModel(spec=m.spec, counts=m.counts.copy(), offsets=m.offsets.copy(), packed=m.packed.copy(),
                        transfer_table=m.transfer_table)
    levels = oracle.build_octree(oracle.compute_density_level0(ref))
    for nb in (True, False):
        mode = "on" if nb else "off"
        for (W, H) in ((1, 1), (7, 5), (130, 3)):
            lv.render_frame(lv.default_camera(big, 320, 200), mb, None, None, lv.RenderParams(base_opacity=0.3, neighbor_mode=mode))
            img, st = oracle.render(oracle.default_camera(dims, W, H), ref, levels, base_opacity=0.5, neighbor=nb)
            for model in (m, enc):
                fr = lv.render_frame(lv.default_camera(dims, W, H), model, None, None,
                                     lv.RenderParams(base_opacity=0.5, neighbor_mode=mode))
                assert np.abs(fr.image - img).max() <= MAX_ERR
                assert fr.stats["voxel_steps"] == st["voxel_steps"]
                assert fr.stats["intersection_tests"] == st["intersection_tests"]


def test_camera_inside_grid_and_auto_neighbor(lv, oracle, synth):
    dims = (12, 12, 12)
    m, ref = both(lv, oracle, synth.turbulence(200, 60, dims), dims)
    levels = oracle.build_octree(oracle.compute_density_level0(ref))
    cam = lv.Camera(position=(6.2, 5.7, 6.1), target=(11.0, 9.0, 7.0), fov=70.0, width=64, height=40)
    ocam = dict(position=(6.2, 5.7, 6.1), target=(11.0, 9.0, 7.0), up=(0.0, 0.0, 1.0), fov=70.0, width=64, height=40)
    p = lv.RenderParams(base_opacity=0.3)
    still = lv.render_frame(cam, m, None, None, p, moving=False)
    moving = lv.render_frame(cam, m, None, None, p, moving=True)
    assert still.stats["neighbor"] is True and moving.stats["neighbor"] is False  # tests/test_raycast.py:450-458
    for fr, nb in ((still, True), (moving, False)):
        img, st = oracle.render(ocam, ref, levels, base_opacity=0.3, neighbor=nb)
        assert np.abs(fr.image - img).max() <= MAX_ERR
        assert fr.stats["intersection_tests"] == st["intersection_tests"]


def test_model_from_host_arrays_renders_identically(lv, synth):
    """A model rebuilt from plain numpy arrays (e.g. decoded from a .vxl file,
    reference tests/test_model_io.py:105-116) renders bit-identically."""
    dims = (16, 16, 16)
    m = lv.build_voxel_model(lv.CurveSet.from_flat(*synth.helices(50, 40, dims)), lv.GridSpec(dims))
    host = lv.VoxelModel(spec=m.spec, counts=m.counts.copy(), offsets=m.offsets.copy(), packed=m.packed.copy(),
                         transfer_table=m.transfer_table, seg_voxel=m.seg_voxel.copy(), seg_a=m.seg_a.copy(),
                         seg_b=m.seg_b.copy(), seg_attr=m.seg_attr.copy(), seg_lid=m.seg_lid.copy(),
                         seg_face_in=m.seg_face_in.copy(), seg_bin_in=m.seg_bin_in.copy(),
                         seg_face_out=m.seg_face_out.copy(), seg_bin_out=m.seg_bin_out.copy())
    cam = lv.default_camera(dims, 80, 60)
    p = lv.RenderParams(base_opacity=0.4, neighbor_mode="on")
    a, b = lv.render_frame(cam, m, None, None, p), lv.render_frame(cam, host, None, None, p)
    assert np.array_equal(a.image, b.image) and a.stats["intersection_tests"] == b.stats["intersection_tests"]
    assert np.array_equal(lv.compute_density_level0(m), lv.compute_density_level0(host))
    # replacing a cache array through the attribute drops the stale device mirror
    host.seg_attr = np.zeros_like(host.seg_attr)
    c = lv.render_frame(cam, host, None, None, p)
    assert not np.array_equal(c.image, b.image)


def test_frame_engines_agree_and_queue_overflow_is_retried(lv, synth):
    """The tile kernel and the wavefront engine produce the same bytes; a wavefront run whose
    queues are too small reports it (LVX_E_RANGE) and is repeated with larger ones."""
    import torch
    from paper_1801_01155_b200.raycast import FramePlan
    dims = (24, 24, 24)
    m = lv.build_voxel_model(lv.CurveSet.from_flat(*synth.turbulence(1500, 50, dims)), lv.GridSpec(dims))
    oc = lv.build_lod(m)
    cam = lv.default_camera(dims, 200, 120)
    for kw in (dict(base_opacity=0.2, neighbor_mode="on"), dict(base_opacity=0.2, neighbor_mode="off"),
               dict(base_opacity=0.03, tau=1.0, neighbor_mode="on", shadow_mode="cone", light_dir=(0.1, 0.5, 1.0))):
        p = lv.RenderParams(**kw)
        nb = 1 if kw["neighbor_mode"] == "on" else 0
        out = {}
        for engine, scale in (("tile", 1.0), ("wavefront", 1.0), ("wavefront-small", 1.0 / 64.0)):
            plan = FramePlan(cam, m, oc, p, nb, engine=engine.split("-")[0])
            plan._scale = scale
            img = torch.empty((120, 200, 4), dtype=torch.float32, device="cuda")
            st = torch.zeros((120, 3), dtype=torch.int64, device="cuda")
            plan.launch(img, st)
            torch.cuda.synchronize()
            out[engine] = (img.cpu().numpy(), st.cpu().numpy(), plan._scale)
        for engine in ("wavefront", "wavefront-small"):
            assert np.array_equal(out["tile"][0], out[engine][0]), (kw, engine)
            assert np.array_equal(out["tile"][1], out[engine][1]), (kw, engine)
    assert out["wavefront-small"][2] > 1.0 / 64.0  # the low-opacity frame does not fit the tiny queues


def test_frame_written_to_pinned_host_memory_equals_device_frame(lv, synth, monkeypatch):
    """render_frame lets the kernels write the image straight into pinned host memory (the
    default) or into HBM followed by a copy: same bytes, same counters, both engines."""
    dims = (24, 24, 24)
    m = lv.build_voxel_model(lv.CurveSet.from_flat(*synth.turbulence(1500, 50, dims)), lv.GridSpec(dims))
    oc = lv.build_lod(m)
    cam = lv.default_camera(dims, 203, 117)
    for kw in (dict(base_opacity=0.2, neighbor_mode="on"), dict(base_opacity=0.2, neighbor_mode="off")):
        out = {}
        for where in ("host", "device"):
            monkeypatch.setenv("LVX_FRAME_OUT", where)
            fr = lv.render_frame(cam, m, oc, None, lv.RenderParams(**kw))
            out[where] = (fr.image.copy(), {k: v for k, v in fr.stats.items() if k != "ms"})
        assert np.array_equal(out["host"][0], out["device"][0]), kw
        assert out["host"][1] == out["device"][1], kw


def test_shares_of_a_frame_rendered_in_place_into_one_host_image(lv, synth):
    """A host image gets the pixels of the rays that miss the grid from a copy engine -- but only when
    the call renders the WHOLE image: the shares of an in-place tiled frame (tile k of every 3, not
    compact) written one after the other into one pinned image must add up to the full frame, each
    share leaving the others' pixels alone; and a frame larger than the 8 MB pattern the copy engine
    repeats equals the frame rendered into device memory."""
    import torch
    from paper_1801_01155_b200.raycast import FramePlan
    dims = (24, 24, 24)
    m = lv.build_voxel_model(lv.CurveSet.from_flat(*synth.turbulence(1500, 50, dims)), lv.GridSpec(dims))
    oc = lv.build_lod(m)
    p = lv.RenderParams(base_opacity=0.2, neighbor_mode="on", background=(0.2, 0.4, 0.6, 0.5))
    for W, H in ((203, 117), (1100, 700)):   # 0.4 MB; 12.3 MB = one and a half patterns
        cam = lv.default_camera(dims, W, H)
        full_d = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
        st = torch.zeros((H, 3), dtype=torch.int64, device="cuda")
        FramePlan(cam, m, oc, p, 1, engine="wavefront").launch(full_d, st)
        whole = torch.full((H, W, 4), -1.0, dtype=torch.float32).pin_memory()
        st1 = torch.zeros((H, 3), dtype=torch.int64, device="cuda")
        FramePlan(cam, m, oc, p, 1, engine="wavefront").launch(whole, st1)
        torch.cuda.synchronize()
        assert np.array_equal(whole.numpy(), full_d.cpu().numpy()), (W, H)
        assert torch.equal(st, st1)
        img = torch.full((H, W, 4), -1.0, dtype=torch.float32).pin_memory()
        st2 = torch.zeros((H, 3), dtype=torch.int64, device="cuda")
        for k in (2, 0, 1):
            FramePlan(cam, m, oc, p, 1, tile_first=k, tile_step=3, engine="wavefront").launch(img, st2)
        torch.cuda.synchronize()
        assert np.array_equal(img.numpy(), full_d.cpu().numpy()), (W, H)
        assert torch.equal(st, st2)


def test_model_from_encoded_arrays_only(lv, synth):
    """a model that arrives as (counts, offsets, packed) only -- what a .vxl
    file holds -- is decoded on the device (lvx_decode_packed, model_io.py:151-179): caches
    equal the builder's bit for bit and the frame is byte-identical (tests/test_model_io.py:105-116)."""
    for dims, n_bins, lines in (((16, 16, 16), 32, synth.helices(50, 40, (16, 16, 16))),
                                ((10, 12, 9), 128, synth.turbulence(80, 40, (10, 12, 9))),
                                ((8, 8, 8), 4, synth.wiggles(40, 20, (8, 8, 8)))):
        m = lv.build_voxel_model(lv.CurveSet.from_flat(*lines), lv.GridSpec(dims, n_bins))
        enc = lv.VoxelModel(spec=m.spec, counts=m.counts.copy(), offsets=m.offsets.copy(), packed=m.packed.copy(),
                            transfer_table=m.transfer_table)
        cam = lv.default_camera(dims, 72, 54)
        p = lv.RenderParams(base_opacity=0.35, neighbor_mode="on")
        a, b = lv.render_frame(cam, m, None, None, p), lv.render_frame(cam, enc, None, None, p)  # records only
        assert np.array_equal(a.image, b.image) and a.stats["intersection_tests"] == b.stats["intersection_tests"]
        for f in ("seg_a", "seg_b", "seg_attr", "seg_lid", "seg_voxel", "seg_face_in", "seg_bin_in",
                  "seg_face_out", "seg_bin_out"):
            assert np.array_equal(getattr(enc, f), getattr(m, f)), f
        assert np.array_equal(lv.compute_density_level0(enc), lv.compute_density_level0(m))
    bad = m.packed.copy()
    bad[0] |= 7  # face_in = 7
    with pytest.raises(ValueError, match="face ID"):
        lv.VoxelModel(spec=m.spec, counts=m.counts, offsets=m.offsets, packed=bad,
                      transfer_table=m.transfer_table).seg_a


_DENSITY_SNIPPET = """
import sys, hashlib, numpy as np
sys.path.insert(0, {root!r})
import paper_1801_01155_b200 as lv
from paper_1801_01155_b200 import synth
for dims, nb in (((23, 17, 40), 32), ((9, 30, 11), 256), ((16, 16, 16), 4)):
    m = lv.build_voxel_model(lv.CurveSet.from_flat(*synth.turbulence(900, 40, dims)), lv.GridSpec(dims, nb))
    enc = lv.VoxelModel(spec=m.spec, counts=m.counts.copy(), offsets=m.offsets.copy(), packed=m.packed.copy(),
                        transfer_table=m.transfer_table)
    d = lv.compute_density_level0(enc)
    assert not enc.has_render_caches()
    print(hashlib.sha256(np.ascontiguousarray(d).tobytes()).hexdigest())
"""


def test_density_from_encoded_records(lv, synth):
    """An encoded-only model gets its level-0 density from the packed records without any expansion
    (lvx_density_l0_packed): both kernels behind it -- the warp-cooperative one for grids whose
    coordinates are exact in float32, and the voxel-aware general one (forced here through
    LVX_DENSITY_GENERAL) -- give the render-record sums bit for bit (lod.py:82-94)."""
    import hashlib, os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    want = []
    for dims, nb in (((23, 17, 40), 32), ((9, 30, 11), 256), ((16, 16, 16), 4)):
        m = lv.build_voxel_model(lv.CurveSet.from_flat(*synth.turbulence(900, 40, dims)), lv.GridSpec(dims, nb))
        assert m.has_render_caches()
        d = lv.compute_density_level0(m)  # render records
        want.append(hashlib.sha256(np.ascontiguousarray(d).tobytes()).hexdigest())
        enc = lv.VoxelModel(spec=m.spec, counts=m.counts.copy(), offsets=m.offsets.copy(), packed=m.packed.copy(),
                            transfer_table=m.transfer_table)
        assert np.array_equal(lv.compute_density_level0(enc), d)
        assert not enc.has_render_caches()  # nothing was expanded for it
        # caller-supplied segment arrays win over the encoded ones (the reference sums seg_a / seg_b)
        enc.seg_a = m.seg_a * np.float32(0.5)
        enc.seg_b = m.seg_b * np.float32(0.5)
        enc.seg_attr, enc.seg_lid, enc.seg_voxel = m.seg_attr, m.seg_lid, m.seg_voxel
        got = lv.compute_density_level0(enc)
        assert not np.array_equal(got, d) and np.allclose(got, 0.5 * d, rtol=1e-6)
    for env in ({}, {"LVX_DENSITY_GENERAL": "1"}):
        out = subprocess.run([sys.executable, "-c", _DENSITY_SNIPPET.format(root=root)], capture_output=True, text=True,
                             env={**os.environ, **env}, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        assert out.stdout.split() == want, env


@pytest.mark.parametrize("n_bins", [4, 32, 128, 256])
def test_packed_records_render_identically(lv, synth, n_bins):
    """Every record width (4, 5, 6, 7 bytes): wavefront frames decoded from the encoded records in
    the kernels == frames from the 32-byte render records, image and counters, in both modes."""
    import torch
    from paper_1801_01155_b200.raycast import FramePlan
    dims = (14, 11, 9)
    m = lv.build_voxel_model(lv.CurveSet.from_flat(*synth.turbulence(260, 50, dims)), lv.GridSpec(dims, n_bins))
    oc = lv.build_lod(m)
    m.ao = lv.precompute_voxel_ao(m, oc, lv.AOParams(n_rays=12, radius=3.0, step=1.0))
    cam = lv.default_camera(dims, 160, 90)
    for kw in (dict(base_opacity=0.3, neighbor_mode="on", ao_mode="precomputed"),
               dict(base_opacity=0.3, neighbor_mode="off", joint_spheres=False),
               dict(neighbor_mode="on", opacity_mode="distance-scaled", base_opacity=0.4, shadow_mode="cone",
                    light_dir=(0.2, 0.4, 1.0))):
        p = lv.RenderParams(**kw)
        nb = 1 if kw["neighbor_mode"] == "on" else 0
        res = []
        for rec in ("rec", "packed"):
            plan = FramePlan(cam, m, oc, p, nb, engine="wavefront", records=rec)
            assert plan.records == rec
            img = torch.empty((90, 160, 4), dtype=torch.float32, device="cuda")
            st = torch.zeros((90, 3), dtype=torch.int64, device="cuda")
            plan.launch(img, st)
            torch.cuda.synchronize()
            res.append((img.cpu().numpy(), st.cpu().numpy()))
        assert np.array_equal(res[0][0], res[1][0]), kw
        assert np.array_equal(res[0][1], res[1][1]), kw
    # geometry secondary rays walk the render records: the plan falls back to them
    plan = FramePlan(cam, m, oc, lv.RenderParams(shadow_mode="hard", light_dir=(0, 0, 1)), 1, engine="wavefront",
                     records="packed")
    assert plan.records == "rec"


# --- error behaviour ------------------------------------------------------

def test_error_conventions(lv, synth):
    dims = (8, 8, 8)
    cs = lv.CurveSet.from_flat(*synth.helices(20, 30, dims))
    with pytest.raises(ValueError, match="transfer table"):
        lv.build_voxel_model(cs, lv.GridSpec(dims), np.zeros((10, 4), np.float32))
    with pytest.raises(MemoryError, match=r"5\*512"):
        lv.build_voxel_model(cs, lv.GridSpec(dims), memory_budget=1000)
    m = lv.build_voxel_model(cs, lv.GridSpec(dims))
    cam = lv.default_camera(dims, 16, 16)
    with pytest.raises(ValueError, match="octree"):
        lv.render_frame(cam, m, None, None, lv.RenderParams(shadow_mode="cone", light_dir=(0, 0, 1)))
    with pytest.raises(ValueError, match="octree"):
        lv.render_frame(cam, m, None, None, lv.RenderParams(ao_mode="density-rays"))
    with pytest.raises(ValueError, match="precomputed AO"):
        lv.render_frame(cam, m, None, None, lv.RenderParams(ao_mode="precomputed"))
    # replines without a field: render_frame builds what is missing (raycast.py:451-465 ensure_lod is the
    # CLI's job there; the kernel call itself raises, raycast.py:416-417)
    from paper_1801_01155_b200.raycast import FramePlan
    with pytest.raises(ValueError, match="representative-line"):
        FramePlan(cam, m, None, lv.RenderParams(shadow_mode="replines", light_dir=(0, 0, 1)), 1)
    with pytest.raises(ValueError):
        lv.build_octree(np.zeros((0, 2, 2), np.float32))


# --- size-independent properties at the full BASELINE.json sizes ---------------------------

def check_model_properties(lv, m):
    counts, offsets = m.counts.astype(np.int64), m.offsets.astype(np.int64)
    S = m.segment_count
    assert counts.sum() == S
    # headers are the exclusive prefix sums in scan order (tests/test_voxelizer.py:324-333)
    assert offsets[0] == 0 and np.array_equal(offsets[1:], np.cumsum(counts)[:-1])
    dx, dy, _ = m.spec.dims
    v = m.seg_voxel.astype(np.int64)
    lin = v[:, 0] + dx * (v[:, 1] + dy * v[:, 2])
    assert np.all(np.diff(lin) >= 0)  # grouped by voxel in scan order
    assert np.array_equal(np.bincount(lin, minlength=counts.size), counts)
    # unpack(packed) == the cached arrays (tests/test_voxelizer.py:336-351)
    u = lv.unpack_records(m.packed, m.spec.bins_per_axis)
    assert np.array_equal(u["face_in"], m.seg_face_in) and np.array_equal(u["bin_in"], m.seg_bin_in)
    assert np.array_equal(u["face_out"], m.seg_face_out) and np.array_equal(u["bin_out"], m.seg_bin_out)
    assert np.array_equal(u["attr"], m.seg_attr) and np.array_equal(u["lid"], m.seg_lid)
    # lid = rank inside the voxel mod 32 (voxelizer.py:442-449)
    rank = np.arange(S) - offsets[lin]
    assert np.array_equal(m.seg_lid, (rank % 32).astype(np.uint8))
    # endpoints sit on a face of their own voxel, at bin centres (tests/test_voxelizer.py:354-361)
    for pts, face in ((m.seg_a, m.seg_face_in), (m.seg_b, m.seg_face_out)):
        local = pts.astype(np.float64) - v
        assert local.min() >= 0.0 and local.max() <= 1.0
        ax = (face >> 1).astype(np.int64)
        assert np.array_equal(local[np.arange(S), ax], (face & 1).astype(np.float64))
    # (curve, chord order) increases inside every voxel: the stable-sort order
    key = m.seg_curve.astype(np.int64) * (1 << 32) + m.seg_order
    same = lin[1:] == lin[:-1]
    assert np.all(key[1:][same] > key[:-1][same])


def test_c2_properties_and_golden_hash(lv, synth):
    """configs[1]: 10k helices x 100 pts, 128^3.  Too slow for the oracle inside a unit
    test at 1080p, so: structural properties, the reference's golden hash and
    counters, run-to-run determinism."""
    import hashlib
    dims = (128, 128, 128)
    cs = lv.CurveSet.from_flat(*synth.helices(10000, 100, dims))
    m = lv.build_voxel_model(cs, lv.GridSpec(dims))
    assert m.segment_count == 5355984
    assert hashlib.sha256(m.packed.tobytes()).hexdigest()[:16] == "7e7d82534e9a9d10"
    check_model_properties(lv, m)
    m2 = lv.build_voxel_model(cs, lv.GridSpec(dims), workers=8)
    assert np.array_equal(m.packed, m2.packed) and np.array_equal(m.seg_order, m2.seg_order)
    oc = lv.build_lod(m)
    # mass conservation: the mean is preserved level to level on power-of-two grids
    tot = [float(l.astype(np.float64).mean()) for l in oc.levels]
    assert np.allclose(tot, tot[0], rtol=1e-5)
    cam = lv.default_camera(dims, 1920, 1080)
    p = lv.RenderParams(base_opacity=0.25, neighbor_mode="on")
    fr = lv.render_frame(cam, m, None, None, p)
    # counters of the unmodified reference on this exact frame
    assert fr.stats["voxel_steps"] == 82325274 and fr.stats["intersection_tests"] == 884660172
    fr2 = lv.render_frame(cam, m, None, None, p)
    assert np.array_equal(fr.image, fr2.image)
    a = fr.image[..., 3]
    assert a.min() >= 0.0 and a.max() <= 1.0 + 1e-6 and np.isfinite(fr.image).all()


def test_c3_turbulence_golden_hash(lv, synth):
    """configs[2] voxelisation: 100k turbulence lines, 256^3 (hashes from SURVEY.md 8c)."""
    import hashlib
    dims = (256, 256, 256)
    m = lv.build_voxel_model(lv.CurveSet.from_flat(*synth.turbulence(100000, 100, dims)), lv.GridSpec(dims))
    assert m.segment_count == 9683143 and m.dropped_overflow == 0
    assert hashlib.sha256(m.packed.tobytes()).hexdigest()[:16] == "bf0cebfed11c4875"
    assert hashlib.sha256(m.counts.tobytes()).hexdigest()[:16] == "1f3e2873ac51a76a"
    check_model_properties(lv, m)


def test_untile_round_trip(lv, synth):
    """Interleaved-tile rendering (the multi-GPU screen partition) reassembles to
    the single-pass frame bit for bit, counters included."""
    import torch
    from paper_1801_01155_b200 import parallel
    dims = (16, 16, 16)
    m = lv.build_voxel_model(lv.CurveSet.from_flat(*synth.helices(60, 40, dims)), lv.GridSpec(dims))
    cam = lv.default_camera(dims, 150, 70)  # not a multiple of the tile size
    p = lv.RenderParams(base_opacity=0.3, neighbor_mode="on")
    full = lv.render_frame(cam, m, None, None, p)
    for world in (2, 3, 8):
        img = torch.zeros((70, 150, 4), dtype=torch.float32, device="cuda")
        stats = torch.zeros((70, 3), dtype=torch.int64, device="cuda")
        for rank in range(world):
            tiles, st, _ = parallel.render_my_tiles(cam, m, None, p, rank, world)
            parallel.untile_into(tiles, rank, world, cam.width, cam.height, img)
            stats += st
        assert np.array_equal(img.cpu().numpy(), full.image), world
        tot = stats.sum(0).tolist()
        assert tot[0] == full.stats["voxel_steps"] and tot[1] == full.stats["intersection_tests"]
        # the multi-GPU frame exchange as rank 0 sees it after the gather: every rank's send buffer
        # (tiles in front, counters in the tail) side by side, scattered with ONE launch
        recv = torch.empty((world, parallel.send_layout(world, cam.width, cam.height)[2]), dtype=torch.float32,
                           device="cuda")
        for rank in range(world):
            _, st, send = parallel.render_my_tiles(cam, m, None, p, rank, world)
            parallel.pack_counters(send, st.sum(dim=0))
            recv[rank].copy_(send)
        img2 = torch.full((70, 150, 4), -1.0, dtype=torch.float32, device="cuda")
        parallel.untile_all(recv, world, cam.width, cam.height, img2)
        assert np.array_equal(img2.cpu().numpy(), full.image), world
        tot2 = parallel.unpack_counters(recv).tolist()
        assert tot2 == [full.stats["voxel_steps"], full.stats["intersection_tests"], full.stats["window_overflow"]]


def test_sharded_voxelization_merges_to_single_gpu_result(lv, synth):
    """Voxelization sharded by line ID (the multi-GPU path, here with the ranks run one
    after another on one GPU): shard -> sum counts -> concatenate records -> merge gives
    the single-pass model byte for byte, cap-255 voxels included."""
    import torch
    from paper_1801_01155_b200 import _lib, parallel
    for dims, gen, world in (((24, 20, 16), synth.wiggles(500, 40, (24, 20, 16)), 3),
                             ((3, 3, 3), synth.helices(900, 30, (3, 3, 3), seed=3), 4)):
        pts, attrs, off = gen
        spec = lv.GridSpec(dims)
        single = lv.build_voxel_model(lv.CurveSet.from_flat(pts, attrs, off), spec)
        n_curves = off.size - 1
        shards = []
        for r in range(world):
            c0, c1 = parallel.shard_range(n_curves, r, world)
            p0, p1 = int(off[c0]), int(off[c1])
            sh = parallel.voxelize_shard(_lib.to_device(pts[p0:p1]), _lib.to_device(attrs[p0:p1]),
                                         _lib.to_device(off[c0:c1 + 1] - p0), c1 - c0, spec, p0)
            sh["edge_kept"] = sh["edge_kept"][:p1 - p0]
            shards.append(sh)
        total = sum(s["vox_cnt"] for s in shards)
        cat = {k: torch.cat([s[k] for s in shards]) for k in ("raw_key", "raw_q", "raw_lin", "edge_kept")}
        out = parallel.merge_shards(spec, total, cat["raw_key"], cat["raw_q"], cat["raw_lin"],
                                    edge_kept=cat["edge_kept"], off_d=_lib.to_device(off), n_curves=n_curves)
        out["err"] = shards[0]["err"]
        from paper_1801_01155_b200.voxelizer import model_from_device
        merged = model_from_device(out, spec, single.transfer_table)
        assert_model_equal(merged, {f: getattr(single, f) for f in MODEL_FIELDS})
        assert merged.dropped_overflow == single.dropped_overflow
