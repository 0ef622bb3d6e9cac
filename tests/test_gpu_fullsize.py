"""Parity at the sizes bench.py times (BASELINE.json configs[1..4]) -- the frames, LoD and AO
bake of C2 / C3 at 1920x1080, the reference's own 256^3 acceptance scene, and the 1 M-line set.

Three independent checkers:
 * fixtures written by the UNMODIFIED reference at full size (tests/golden/big_*.npz,
   accept_tornado256.npz: every 16th / 4th image row, counters, sha256 of the whole image and of
   the model arrays) -- tests/golden/make_golden.py;
 * the CPU oracle on every 16th row of the same frames, and on whole models / LoD / AO fields;
 * the two frame engines against each other (byte equality of image and per-row counters).
"""
import hashlib

import numpy as np
import pytest

from conftest import MODEL_FIELDS, assert_model_equal, golden

pytestmark = pytest.mark.gpu

MAX_ERR = 1.0 / 255.0   # north_star: max per-channel error
MEAN_ERR = 1e-3         # north_star: mean error


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def lv():
    import paper_1801_01155_b200 as lv
    return lv


@pytest.fixture(scope="module")
def synth():
    from paper_1801_01155_b200 import synth
    return synth


def gpu_frame(lv, cam, model, octree, kw, engine=None):
    """(image (H,W,4) f32, row_stats (H,3) i64, engine used) through the C ABI."""
    import torch
    from paper_1801_01155_b200.raycast import FramePlan, resolve_neighbor
    p = lv.RenderParams(**kw)
    plan = FramePlan(cam, model, octree, p, resolve_neighbor(p, False), engine=engine)
    img = torch.empty((cam.height, cam.width, 4), dtype=torch.float32, device="cuda")
    st = torch.zeros((cam.height, 3), dtype=torch.int64, device="cuda")
    plan.launch(img, st)
    torch.cuda.synchronize()
    return img.cpu().numpy(), st.cpu().numpy(), plan.engine


def check_against_fixture(g, img, row_stats):
    """Rows, counters and (when the frame has no pow-dependent pixel difference) the hash of the
    whole image, as the unmodified reference produced them."""
    step = int(g["row_step"])
    want = g["rows"] if "rows" in g.files else None
    err = np.abs(img[::step].astype(np.float64) - want.astype(np.float64))
    assert err.max() <= MAX_ERR and err.mean() < MEAN_ERR, (err.max(), err.mean())
    assert row_stats.sum(0).tolist() == g["stats"].tolist()
    return bool(sha(img) == str(g["image_sha256"])), float(err.max())


def check_against_oracle_rows(oracle, dims, W, H, ref, levels, kw, img, row_stats, step=16):
    okw = dict(kw)
    nb = okw.pop("neighbor_mode") != "off"
    want, st = oracle.render(oracle.default_camera(dims, W, H), ref, levels, neighbor=nb, rows=(0, H, step), **okw)
    sel = np.arange(0, H, step)
    err = np.abs(img[sel].astype(np.float64) - want[sel].astype(np.float64))
    assert err.max() <= MAX_ERR and err.mean() < MEAN_ERR, (err.max(), err.mean())
    sub = row_stats[sel].sum(0).tolist()
    assert sub == [st["voxel_steps"], st["intersection_tests"], st["window_overflow"]]


# --- C3: 100k turbulence lines, 256^3, 1080p, alpha .25 + precomputed AO (the bench frame) --------

C3_DIMS = (256, 256, 256)
C3_KW = dict(base_opacity=0.25, tau=0.95, neighbor_mode="on", ao_mode="precomputed")


@pytest.fixture(scope="module")
def c3(lv, synth):
    lines = synth.turbulence(100000, 100, C3_DIMS)
    m = lv.build_voxel_model(lv.CurveSet.from_flat(*lines), lv.GridSpec(C3_DIMS))
    oc = lv.build_lod(m)
    m.ao = lv.precompute_voxel_ao(m, oc)
    return lines, m, oc


@pytest.fixture(scope="module")
def c3_oracle(oracle, c3):
    (pts, attrs, off), _, _ = c3
    ref = oracle.build_voxel_model(pts, attrs, off, C3_DIMS, 32)
    levels = oracle.build_octree(oracle.compute_density_level0(ref))
    ref.ao = oracle.precompute_voxel_ao(ref, levels, 100, 5.0, 1.0)
    return ref, levels


def test_c3_model_lod_ao_equal_the_oracle(c3, c3_oracle):
    """Whole-model, every LoD level and the 7.2 M-voxel AO bake, bit for bit."""
    _, m, oc = c3
    ref, levels = c3_oracle
    assert_model_equal(m, {f: getattr(ref, f) for f in MODEL_FIELDS})
    assert oc.n_levels == len(levels) == 9
    for a, b in zip(oc.levels, levels):
        assert np.array_equal(a, b)
    assert np.array_equal(np.asarray(m.ao), np.asarray(ref.ao))


def test_c3_matches_the_reference_fixture(lv, c3):
    """Hashes of the reference's own C3 model / LoD / AO field, rows and counters of its 1080p frame."""
    _, m, oc = c3
    g = golden("big_c3_1080p")
    assert m.segment_count == int(g["segments"])
    assert sha(m.packed) == str(g["packed_sha256"]) and sha(m.counts) == str(g["counts_sha256"])
    assert sha(oc.levels[0]) == str(g["level0_sha256"])
    assert [sha(l) for l in oc.levels] == [str(x) for x in g["levels_sha256"]]
    assert sha(np.asarray(m.ao)) == str(g["ao_sha256"])
    img, rs, _ = gpu_frame(lv, lv.default_camera(C3_DIMS, 1920, 1080), m, oc, C3_KW)
    identical, worst = check_against_fixture(g, img, rs)
    print(f"C3 1080p vs reference: whole-image sha256 equal: {identical}, max err on stored rows {worst:.3e}")


@pytest.mark.parametrize("engine", ["wavefront", "tile"])
def test_c3_1080p_frame_vs_oracle_rows(lv, oracle, c3, c3_oracle, engine):
    _, m, oc = c3
    ref, levels = c3_oracle
    img, rs, used = gpu_frame(lv, lv.default_camera(C3_DIMS, 1920, 1080), m, oc, C3_KW, engine)
    assert used == engine
    check_against_oracle_rows(oracle, C3_DIMS, 1920, 1080, ref, levels, C3_KW, img, rs)


@pytest.mark.parametrize("kw", [C3_KW, dict(C3_KW, neighbor_mode="off"),
                                dict(C3_KW, shadow_mode="cone", light_dir=(0.3, 0.2, 1.0))],
                         ids=["neighbour-on", "own-voxel", "cone-shadows"])
def test_c3_1080p_engines_are_byte_identical(lv, c3, kw):
    """tile engine == wavefront engine on image AND per-row counters at full size (the size-dependent
    paths of the wavefront engine -- tail budget, ray spreading, queue growth -- are live here)."""
    _, m, oc = c3
    cam = lv.default_camera(C3_DIMS, 1920, 1080)
    a, sa, _ = gpu_frame(lv, cam, m, oc, kw, "wavefront")
    b, sb, _ = gpu_frame(lv, cam, m, oc, kw, "tile")
    assert np.array_equal(a, b), int((a != b).any(-1).sum())
    assert np.array_equal(sa, sb)


def test_c3_rendered_straight_from_the_encoded_records(lv, c3):
    """the wavefront engine decoding the 5-byte records in its kernels gives the
    frame of the 32-byte render records, byte for byte (image and per-row counters), at full size;
    and a model that carries only (counts, offsets, packed) renders WITHOUT being expanded."""
    import torch
    from paper_1801_01155_b200.raycast import FramePlan
    _, m, oc = c3
    cam = lv.default_camera(C3_DIMS, 1920, 1080)
    for kw in (C3_KW, dict(C3_KW, shadow_mode="cone", light_dir=(0.3, 0.2, 1.0))):
        p = lv.RenderParams(**kw)
        out = {}
        for rec in ("rec", "packed"):
            plan = FramePlan(cam, m, oc, p, 1, engine="wavefront", records=rec)
            assert plan.records == rec
            img = torch.empty((1080, 1920, 4), dtype=torch.float32, device="cuda")
            st = torch.zeros((1080, 3), dtype=torch.int64, device="cuda")
            plan.launch(img, st)
            torch.cuda.synchronize()
            out[rec] = (img.cpu().numpy(), st.cpu().numpy())
        assert np.array_equal(out["rec"][0], out["packed"][0]) and np.array_equal(out["rec"][1], out["packed"][1])
    enc = lv.VoxelModel(spec=m.spec, counts=m.dev("counts"), offsets=m.dev("offsets"), packed=m.dev("packed"),
                        transfer_table=m.transfer_table)
    enc.ao = m.ao
    fr = lv.render_frame(cam, enc, oc, None, lv.RenderParams(**C3_KW))
    ref = lv.render_frame(cam, m, oc, None, lv.RenderParams(**C3_KW))
    assert np.array_equal(fr.image, ref.image) and fr.stats["intersection_tests"] == ref.stats["intersection_tests"]
    assert "seg_rec" not in enc._derived and not enc._has("seg_a")  # nothing was expanded


def test_c3_own_voxel_vs_oracle_rows(lv, oracle, c3, c3_oracle):
    _, m, oc = c3
    ref, levels = c3_oracle
    kw = dict(C3_KW, neighbor_mode="off")
    img, rs, _ = gpu_frame(lv, lv.default_camera(C3_DIMS, 1920, 1080), m, oc, kw)
    check_against_oracle_rows(oracle, C3_DIMS, 1920, 1080, ref, levels, kw, img, rs)


def test_c3_occupancy_dilated(c3, c3_oracle, oracle):
    _, m, _ = c3
    ref, _ = c3_oracle
    assert np.array_equal(m.occupancy_dilated(), oracle.occupancy_dilated(ref))


# --- C2: 10k helices, 128^3, 1080p, alpha .25 ---------------------------------------------------

C2_DIMS = (128, 128, 128)
C2_KW = dict(base_opacity=0.25, tau=0.95, neighbor_mode="on")


@pytest.fixture(scope="module")
def c2(lv, synth):
    lines = synth.helices(10000, 100, C2_DIMS)
    m = lv.build_voxel_model(lv.CurveSet.from_flat(*lines), lv.GridSpec(C2_DIMS))
    return lines, m


@pytest.mark.parametrize("fixture,kw", [("big_c2_1080p", C2_KW), ("big_c2_1080p_own", dict(C2_KW, neighbor_mode="off"))])
def test_c2_matches_the_reference_fixture(lv, c2, fixture, kw):
    _, m = c2
    g = golden(fixture)
    assert sha(m.packed) == str(g["packed_sha256"]) and sha(m.counts) == str(g["counts_sha256"])
    cam = lv.default_camera(C2_DIMS, 1920, 1080)
    for engine in ("wavefront", "tile"):
        img, rs, _ = gpu_frame(lv, cam, m, None, kw, engine)
        identical, worst = check_against_fixture(g, img, rs)
        print(f"{fixture} [{engine}] vs reference: whole-image sha256 equal: {identical}, max err {worst:.3e}")


def test_c2_1080p_frame_vs_oracle_rows(lv, oracle, c2):
    (pts, attrs, off), m = c2
    ref = oracle.build_voxel_model(pts, attrs, off, C2_DIMS, 32)
    assert_model_equal(m, {f: getattr(ref, f) for f in MODEL_FIELDS})
    cam = lv.default_camera(C2_DIMS, 1920, 1080)
    img, rs, _ = gpu_frame(lv, cam, m, None, C2_KW)
    check_against_oracle_rows(oracle, C2_DIMS, 1920, 1080, ref, None, C2_KW, img, rs)
    b, sb, _ = gpu_frame(lv, cam, m, None, C2_KW, "tile")
    assert np.array_equal(img, b) and np.array_equal(rs, sb)


# --- the reference's acceptance scene (tests/test_acceptance.py:144-169) ----------------------------

def test_acceptance_tornado_256(lv):
    g = golden("accept_tornado256")
    dims = tuple(int(d) for d in g["dims"])
    m = lv.build_voxel_model(lv.CurveSet.from_flat(g["pts"], g["attrs"], g["off"]), lv.GridSpec(dims, 32))
    assert m.segment_count == int(g["segments"]) and m.dropped_overflow == int(g["dropped"])
    assert sha(m.packed) == str(g["packed_sha256"]) and sha(m.counts) == str(g["counts_sha256"])
    cam = lv.default_camera(dims, 640, 360)
    step = int(g["row_step"])
    import ast
    for tag in ("opaque", "alpha25"):
        kw = ast.literal_eval(str(g["params_" + tag]))
        for engine in ("wavefront", "tile"):
            img, rs, _ = gpu_frame(lv, cam, m, None, kw, engine)
            err = np.abs(img[::step].astype(np.float64) - g["rows_" + tag].astype(np.float64))
            # the reference's own gate: >= 99.9 % of pixels within 2/255, max <= 8/255; ours: north_star's
            assert err.max() <= MAX_ERR and err.mean() < MEAN_ERR
            assert rs.sum(0).tolist() == g["stats_" + tag].tolist()
            print(f"tornado256 {tag} [{engine}]: sha256 equal {sha(img) == str(g['sha_' + tag])}, max err {err.max():.3e}")


# --- occupancy map against the reference's (raycast.py:351-366) ------------------------------------

@pytest.mark.parametrize("case", ["helices", "turbulence", "lattice", "cap255", "wiggles"])
def test_occupancy_dilated_golden(lv, case):
    v, g = golden("vox_" + case), golden("occ_" + case)
    dims = tuple(int(d) for d in v["dims"])
    m = lv.build_voxel_model(lv.CurveSet.from_flat(v["pts"], v["attrs"], v["off"]), lv.GridSpec(dims, int(v["n_bins"])))
    occ = m.occupancy_dilated()
    want = np.asarray(g["occ"])
    assert occ.dtype == want.dtype == np.uint8
    assert np.array_equal(occ.reshape(-1), want.reshape(-1))


# --- 1 M lines (BASELINE configs[3] / configs[4]) ---------------------------------------------------

def test_one_million_lines(lv, oracle, synth):
    """The 97 M-segment set: (a) one line-ID shard (1/8 of the lines, what one of 8 ranks clips) against
    the oracle on the same lines, every field; (b) structural properties of the full model; (c) the
    multi-GPU merge at full size: 8 shards clipped one after another, counts summed, records
    concatenated, merged -> byte-identical to the single-pass model."""
    import torch
    from paper_1801_01155_b200 import _lib, parallel
    from paper_1801_01155_b200.voxelizer import model_from_device
    dims = (256, 256, 256)
    pts, attrs, off = synth.turbulence(1000000, 100, dims)
    spec = lv.GridSpec(dims, 32)
    n_curves = off.size - 1
    # (a) shard 3 of 8 as its own line set
    c0, c1 = parallel.shard_range(n_curves, 3, 8)
    p0, p1 = int(off[c0]), int(off[c1])
    sub = (pts[p0:p1], attrs[p0:p1], off[c0:c1 + 1] - p0)
    ms = lv.build_voxel_model(lv.CurveSet.from_flat(*sub), spec)
    ref = oracle.build_voxel_model(*sub, dims, 32)
    assert_model_equal(ms, {f: getattr(ref, f) for f in MODEL_FIELDS})
    del ms, ref
    # (b) the full set in one pass
    full = lv.voxelize_device(_lib.to_device(pts), _lib.to_device(attrs), _lib.to_device(off), n_curves, spec,
                              caches=False, provenance=False)
    S = int(full["n_segments"])
    assert S == 96824127 and int(full["dropped"]) == 0
    counts = full["counts"].cpu().numpy().astype(np.int64)
    offsets = full["offsets"].cpu().numpy().view(np.uint32).astype(np.int64)
    assert counts.sum() == S and offsets[0] == 0 and np.array_equal(offsets[1:], np.cumsum(counts)[:-1])
    packed_full = full["packed"].cpu().numpy()
    del full
    # (c) 8 shards merged
    total, keys, qs, lins = None, [], [], []
    for r in range(8):
        a0, a1 = parallel.shard_range(n_curves, r, 8)
        q0, q1 = int(off[a0]), int(off[a1])
        sh = parallel.voxelize_shard(_lib.to_device(pts[q0:q1]), _lib.to_device(attrs[q0:q1]),
                                     _lib.to_device(off[a0:a1 + 1] - q0), a1 - a0, spec, q0, want_edge_kept=False)
        total = sh["vox_cnt"] if total is None else total + sh["vox_cnt"]
        keys.append(sh["raw_key"]); qs.append(sh["raw_q"]); lins.append(sh["raw_lin"])
    out = parallel.merge_shards(spec, total, torch.cat(keys), torch.cat(qs), torch.cat(lins), caches=False)
    del keys, qs, lins
    assert int(out["n_segments"]) == S
    assert np.array_equal(out["counts"].cpu().numpy().astype(np.int64), counts)
    assert np.array_equal(out["packed"].cpu().numpy(), packed_full)


def test_one_million_lines_frame(lv, oracle, synth):
    """BASELINE configs[3]'s scene on one GPU at 1080p (the north-star "<= 16 ms" frame): model, LoD
    and the 16.7 M-voxel AO bake equal the oracle's, the frame equals the oracle's on every 64th row
    (image within the bar, per-row counters equal), both engines agree byte for byte, and the 4K frame
    with cone shadows agrees between the engines too."""
    dims = (256, 256, 256)
    pts, attrs, off = synth.turbulence(1000000, 100, dims)
    m = lv.build_voxel_model(lv.CurveSet.from_flat(pts, attrs, off), lv.GridSpec(dims))
    oc = lv.build_lod(m)
    m.ao = lv.precompute_voxel_ao(m, oc)
    ref = oracle.build_voxel_model(pts, attrs, off, dims, 32)
    del pts, attrs
    assert m.segment_count == ref.segment_count == 96824127
    assert np.array_equal(m.packed, ref.packed) and np.array_equal(m.counts, ref.counts)
    levels = oracle.build_octree(oracle.compute_density_level0(ref))
    for a, b in zip(oc.levels, levels):
        assert np.array_equal(a, b)
    ref.ao = oracle.precompute_voxel_ao(ref, levels, 100, 5.0, 1.0)
    assert np.array_equal(np.asarray(m.ao), np.asarray(ref.ao))
    kw = dict(base_opacity=0.25, tau=0.95, neighbor_mode="on", ao_mode="precomputed")
    cam = lv.default_camera(dims, 1920, 1080)
    img, rs, _ = gpu_frame(lv, cam, m, oc, kw, "wavefront")
    check_against_oracle_rows(oracle, dims, 1920, 1080, ref, levels, kw, img, rs, step=64)
    del ref, levels
    b, sb, _ = gpu_frame(lv, cam, m, oc, kw, "tile")
    assert np.array_equal(img, b) and np.array_equal(rs, sb)
    kw4 = dict(kw, shadow_mode="cone", light_dir=(0.3, 0.2, 1.0))
    cam4 = lv.default_camera(dims, 3840, 2160)
    a4, sa4, _ = gpu_frame(lv, cam4, m, oc, kw4, "wavefront")
    b4, sb4, _ = gpu_frame(lv, cam4, m, oc, kw4, "tile")
    assert np.array_equal(a4, b4) and np.array_equal(sa4, sb4)


def test_packed_only_model_follows_reassignment(lv, synth):
    """A model that carries only (counts, offsets, packed) renders from records decoded on the device;
    assigning new encoded arrays must drop every stale decoded cache."""
    dims = (16, 16, 16)
    a = lv.build_voxel_model(lv.CurveSet.from_flat(*synth.helices(50, 40, dims)), lv.GridSpec(dims))
    b = lv.build_voxel_model(lv.CurveSet.from_flat(*synth.turbulence(70, 40, dims)), lv.GridSpec(dims))
    cam = lv.default_camera(dims, 72, 54)
    p = lv.RenderParams(base_opacity=0.35, neighbor_mode="on")
    enc = lv.VoxelModel(spec=a.spec, counts=a.counts.copy(), offsets=a.offsets.copy(), packed=a.packed.copy(),
                        transfer_table=a.transfer_table)
    assert np.array_equal(lv.render_frame(cam, enc, None, None, p).image, lv.render_frame(cam, a, None, None, p).image)
    assert np.array_equal(enc.seg_a, a.seg_a)
    enc.counts, enc.offsets, enc.packed = b.counts.copy(), b.offsets.copy(), b.packed.copy()
    assert enc.segment_count == b.segment_count
    assert np.array_equal(enc.seg_a, b.seg_a) and np.array_equal(enc.seg_lid, b.seg_lid)
    assert np.array_equal(lv.render_frame(cam, enc, None, None, p).image, lv.render_frame(cam, b, None, None, p).image)
