"""Pins the CPU oracle (oracle/lvx_oracle.c) against fixtures produced by the
unmodified Python reference (tests/golden/make_golden.py) and against the
known-answer tests the reference's own suite holds for this path."""
import numpy as np
import pytest

from conftest import MODEL_FIELDS, RENDER_CASES, VOX_CASES, assert_model_equal, golden, render_kwargs


def oracle_model(oracle, g, transfer_table=None):
    return oracle.build_voxel_model(g["pts"], g["attrs"], g["off"], tuple(int(x) for x in g["dims"]),
                                    int(g["n_bins"]), transfer_table)


@pytest.mark.parametrize("name", VOX_CASES)
def test_voxel_model_bit_exact(oracle, name):
    g = golden("vox_" + name)
    m = oracle_model(oracle, g)
    assert_model_equal(m, g)
    assert m.dropped_overflow == int(g["dropped"])


def test_clip_batch_bit_exact(oracle):
    g = golden("clip_lattice")
    out = oracle.clip_batch(g["pts"], g["attrs"], g["off"], tuple(int(x) for x in g["dims"]))
    for got, key in zip(out, ("vox", "p_in", "p_out", "a_in", "a_out", "curve", "within")):
        assert np.array_equal(got, g[key]), key


@pytest.mark.parametrize("name", ["helices", "turbulence", "wiggles", "cap255"])
def test_lod_bit_exact(oracle, name):
    m = oracle_model(oracle, golden("vox_" + name))
    g = golden("lod_" + name)
    levels = oracle.build_octree(oracle.compute_density_level0(m))
    assert len(levels) == len(g.files)
    for l, lvl in enumerate(levels):
        assert np.array_equal(lvl, g[f"level{l}"]), f"level {l}"


def test_coarsen_odd_sizes(oracle):
    g = golden("lod_random_7x5x9")
    levels = oracle.build_octree(g["level0"])
    assert len(levels) == len(g.files)
    for l, lvl in enumerate(levels):
        assert np.array_equal(lvl, g[f"level{l}"])


@pytest.mark.parametrize("name", ["helices", "turbulence"])
def test_ao_bake_bit_exact(oracle, name):
    m = oracle_model(oracle, golden("vox_" + name))
    levels = oracle.build_octree(oracle.compute_density_level0(m))
    g = golden("ao_" + name)
    ao = oracle.precompute_voxel_ao(m, levels, int(g["n_rays"]), float(g["radius"]), float(g["step"]))
    assert np.array_equal(ao, g["values"])


def oracle_render(oracle, name):
    g = golden("render_" + name)
    mname = str(g["model"])
    vg = golden("vox_" + mname)
    m = oracle_model(oracle, vg, g["transfer_table"])
    dims = tuple(int(x) for x in vg["dims"])
    levels = oracle.build_octree(oracle.compute_density_level0(
        oracle_model(oracle, vg)))  # LoD fixtures were built with the default table
    if mname in ("helices", "turbulence"):
        m.ao = golden("ao_" + mname)["values"]
    kw = render_kwargs(g)
    W, H = (int(x) for x in g["size"])
    okw = dict(kw)
    nb = okw.pop("neighbor_mode") == "on"
    img, st = oracle.render(oracle.default_camera(dims, W, H), m, levels, neighbor=nb, **okw)
    return g, img, st


@pytest.mark.parametrize("name", RENDER_CASES)
def test_render_matches_reference(oracle, name):
    g, img, st = oracle_render(oracle, name)
    # the frame is float64 arithmetic with libm pow in both: bitwise equal
    assert np.array_equal(img, g["image"]), f"max diff {np.abs(img - g['image']).max()}"
    assert [st["voxel_steps"], st["intersection_tests"], st["window_overflow"]] == list(g["stats"])


@pytest.mark.parametrize("mname", ["helices", "turbulence"])
def test_geometry_secondary_ray_probes(oracle, mname):
    """hard_shadow / ao_hemisphere_geometry (illumination.py:96-112, 158-173) as point probes."""
    g = golden("geom_probe_" + mname)
    m = oracle_model(oracle, golden("vox_" + mname))
    P, N, L = g["P"], g["N"], g["L"]
    hs = [oracle.hard_shadow(P[i], L[i], m, 0.3, N[i] if i % 2 == 0 else None, bool(i % 3)) for i in range(len(P))]
    assert hs == list(g["hard"])
    assert 0 < sum(hs) < len(hs)  # the fixture holds lit and shadowed points
    ao = np.array([oracle.ao_hemisphere_geometry(P[i], N[i], m, 9, 3.5, 0.3) for i in range(len(P))])
    assert np.array_equal(ao, g["ao"])
    aoj = np.array([oracle.ao_hemisphere_geometry(P[i], N[i], m, 6, 2.5, 0.25, jitter=0.37)
                    for i in range(0, len(P), 4)])
    assert np.array_equal(aoj, g["ao_jitter"])
    assert ao.max() > 0.0


@pytest.mark.parametrize("mname", ["helices", "turbulence", "wiggles"])
def test_representative_lines(oracle, mname):
    """build_rep_lines (lod.py:224-284) with and without the adjacency pass, and
    replines_shadow (illumination.py:115-139) as point probes."""
    g = golden("rep_" + mname)
    m = oracle_model(oracle, golden("vox_" + mname))
    n_levels = int(g["n_levels"])
    for adjacency, tag in ((True, ""), (False, "loose_")):
        rl = oracle.build_rep_lines(m, n_levels, adjacency=adjacency)
        assert len(rl) == n_levels and rl[0] is None
        for l in range(1, n_levels):
            assert np.array_equal(rl[l].valid, g[f"{tag}valid{l}"]), (tag, l)
            assert np.array_equal(rl[l].a, g[f"{tag}a{l}"]), (tag, l)
            assert np.array_equal(rl[l].b, g[f"{tag}b{l}"]), (tag, l)
            assert np.array_equal(rl[l].weight, g[f"{tag}w{l}"]), (tag, l)
    rl = oracle.build_rep_lines(m, n_levels)
    P, N, L, lev = g["P"], g["N"], g["L"], g["level"]
    sh = [oracle.replines_shadow(P[i], L[i], rl, m.dims, level=int(lev[i]), tube_radius=0.3,
                                 normal=N[i] if i % 2 else None) for i in range(len(P))]
    assert sh == list(g["shadow"])
    assert 0 < sum(sh) < len(sh)


@pytest.mark.parametrize("name", ["rep_frame_helices", "rep_frame_turbulence"])
def test_render_with_replines_shadows(oracle, name):
    g = golden("render_" + name)
    mname = str(g["model"])
    m = oracle_model(oracle, golden("vox_" + mname), g["transfer_table"])
    levels = oracle.build_octree(oracle.compute_density_level0(oracle_model(oracle, golden("vox_" + mname))))
    rl = oracle.build_rep_lines(m, len(levels))
    W, H = (int(x) for x in g["size"])
    kw = dict(render_kwargs(g))
    nb = kw.pop("neighbor_mode") == "on"
    img, st = oracle.render(oracle.default_camera(m.dims, W, H), m, levels, neighbor=nb, replines=rl, **kw)
    assert np.array_equal(img, g["image"]), f"max diff {np.abs(img - g['image']).max()}"
    assert [st["voxel_steps"], st["intersection_tests"], st["window_overflow"]] == list(g["stats"])


def test_tube_and_sphere_primitives(oracle):
    g = golden("prim_tube_sphere")
    r = float(g["r"])
    for i in range(g["o"].shape[0]):
        t64 = oracle.intersect_tube(g["o"][i], g["d"][i], g["a"][i], g["b"][i], r, f32_axis=False)
        t32 = oracle.intersect_tube(g["o"][i], g["d"][i], g["a"][i], g["b"][i], r, f32_axis=True)
        s = oracle.intersect_sphere(g["o"][i], g["d"][i], g["a"][i], r)
        assert np.array_equal(t64, g["tube64"][i]), i
        assert np.array_equal(t32, g["tube32"][i]), i
        assert np.array_equal(s, g["sphere"][i]), i
    assert g["tube32"][:, 0].sum() > 500  # the fixture really exercises hits


def test_dda_windows(oracle):
    g = golden("prim_dda")
    dims = tuple(int(x) for x in g["dims"])
    k = 0
    pos = 0
    for pad in (0, 1):
        for i in range(g["o"].shape[0]):
            vox, t = oracle.dda_collect(g["o"][i], g["d"][i], dims, pad)
            n = int(g["counts"][k])
            assert vox.shape[0] == n
            assert np.array_equal(vox, g["vox"][pos:pos + n])
            assert np.array_equal(t, g["t"][pos:pos + n])
            pos += n
            k += 1


def test_density_probes(oracle):
    g = golden("prim_density")
    vg = golden("vox_turbulence")
    m = oracle_model(oracle, vg)
    levels = oracle.build_octree(oracle.compute_density_level0(m))
    flat, off, ldims, L = oracle.octree_args(levels)
    P, N = g["P"], g["N"]
    for l in range(L):
        got = [oracle.sample_trilinear(flat, int(off[l]), *(int(x) for x in ldims[l]), float(1 << l), P[i])
               for i in range(P.shape[0])]
        assert np.array_equal(np.asarray(got), g["trilinear"][l]), f"level {l}"
    cone = [oracle.cone_blocking(P[i], g["light"] / np.linalg.norm(g["light"]), levels) for i in range(P.shape[0])]
    assert np.array_equal(np.asarray(cone), g["cone"])
    # ao_density_rays re-normalises the normal (illumination.py:86-91 `_unit`)
    aod = [oracle.ao_density_point(P[i], N[i] / float(np.linalg.norm(N[i])), levels, 25, 6.0, 1.0, hemisphere=1)
           for i in range(P.shape[0])]
    assert np.array_equal(np.asarray(aod), g["ao_density"])
    ao = golden("ao_turbulence")["values"]
    rz, ry, rx = ao.shape
    aos = [min(1.0, max(0.0, oracle.sample_trilinear(ao.reshape(-1), 0, rx, ry, rz, 1.0, P[i])))
           for i in range(P.shape[0])]
    assert np.array_equal(np.asarray(aos), g["ao_sample"])
    fib = np.array([oracle.fibonacci_dir(i, 25, 1) for i in range(25)])
    assert np.array_equal(fib, g["fib25_hemi"])
    fib = np.array([oracle.fibonacci_dir(i, 100, 0) for i in range(100)])
    assert np.array_equal(fib, g["fib100_sphere"])


def test_shade_scalar(oracle):
    g = golden("prim_shade")
    got = [oracle.shade_scalar(g["n"][i], g["l"][i], g["v"][i], 0.2, 0.7, 0.3, 32.0) for i in range(500)]
    assert np.array_equal(np.asarray(got), g["shade"])


# --- known-answer tests restated from the reference's own suite ----------------------

def _one_curve(points, attrs=None):
    pts = np.asarray(points, dtype=np.float64)
    at = np.linspace(0.0, 1.0, len(pts)) if attrs is None else np.asarray(attrs, dtype=np.float64)
    return pts, at, np.asarray([0, len(pts)], dtype=np.int64)


def test_kat_axis_aligned_chord(oracle):
    # reference tests/test_voxelizer.py:209-219
    pts, at, off = _one_curve([(0.5, 0.5, 0.5), (2.5, 0.5, 0.5)], [0.0, 1.0])
    vox, p_in, p_out, a_in, a_out, curve, within = oracle.clip_batch(pts, at, off, (4, 4, 4))
    assert vox.tolist() == [[1, 0, 0]]
    assert p_in.tolist() == [[1.0, 0.5, 0.5]] and p_out.tolist() == [[2.0, 0.5, 0.5]]
    assert a_in[0] == pytest.approx(0.25) and a_out[0] == pytest.approx(0.75)


def test_kat_same_voxel_yields_nothing(oracle):
    # tests/test_voxelizer.py:222-224
    pts, at, off = _one_curve([(0.2, 0.2, 0.2), (0.8, 0.7, 0.6)])
    assert oracle.clip_batch(pts, at, off, (4, 4, 4))[0].shape[0] == 0


def test_kat_interior_vertices_bridged(oracle):
    # tests/test_voxelizer.py:227-235: vertices inside a voxel do not split the chord
    pts, at, off = _one_curve([(0.5, 0.5, 0.5), (1.2, 0.5, 0.5), (1.5, 0.9, 0.5), (1.8, 0.5, 0.5), (2.5, 0.5, 0.5)])
    vox, p_in, p_out, *_ = oracle.clip_batch(pts, at, off, (4, 4, 4))
    assert vox.tolist() == [[1, 0, 0]]
    assert p_in[0, 0] == 1.0 and p_out[0, 0] == 2.0


def test_kat_corner_crossing_and_graze(oracle):
    # SURVEY.md 3.1 (verified against the reference): coincident x/y events drop the
    # zero-length chord; a reversal on a plane is counted twice
    pts, at, off = _one_curve([(0.5, 0.5, 0.5), (1.5, 1.5, 0.5), (2.5, 1.5, 0.5)])
    vox, p_in, *_ = oracle.clip_batch(pts, at, off, (4, 4, 4))
    assert vox.tolist() == [[1, 1, 0]]
    assert p_in.tolist() == [[1.0, 1.0, 0.5]]
    m = oracle.build_voxel_model(pts, at, off, (4, 4, 4), 8)
    assert m.seg_face_in.tolist() == [0] and m.seg_order.tolist() == [0]


def test_kat_attr_index_and_widths(oracle):
    pts, at, off = _one_curve([(0.5, 0.5, 0.5), (3.5, 0.5, 0.5)], [0.0, 1.0])
    m = oracle.build_voxel_model(pts, at, off, (4, 4, 4), 32)
    assert m.seg_attr.tolist() == [85, 170]
    # tests/test_voxelizer.py:106-109, tests/test_model_io.py:68
    assert [oracle.record_width(n) for n in (4, 8, 16, 32, 64, 128, 256)] == [4, 4, 5, 5, 6, 6, 7]


def test_kat_cap_255_keeps_first(oracle):
    # tests/test_voxelizer.py:364-377
    n = 300
    pts = np.zeros((n, 2, 3))
    pts[:, 0] = (-0.5, 0.5, 0.5)
    pts[:, 1] = (1.5, 0.5, 0.5)
    pts[:, :, 1] += np.linspace(0.0, 0.3, n)[:, None]
    at = np.tile([0.0, 1.0], n)
    off = np.arange(n + 1, dtype=np.int64) * 2
    m = oracle.build_voxel_model(pts.reshape(-1, 3), at, off, (1, 1, 1), 32)
    assert m.counts.tolist() == [255] and m.dropped_overflow == 45
    assert m.seg_curve.tolist() == list(range(255))
    assert m.seg_lid.tolist() == [i % 32 for i in range(255)]


def test_kat_dda_unit_windows(oracle):
    # tests/test_raycast.py:52-57
    vox, t = oracle.dda_collect((-1.0, 0.5, 0.5), (1.0, 0.0, 0.0), (3, 3, 3))
    assert vox.tolist() == [[0, 0, 0], [1, 0, 0], [2, 0, 0]]
    assert t.tolist() == [[1.0, 2.0], [2.0, 3.0], [3.0, 4.0]]


def test_kat_tube_and_sphere(oracle):
    # tests/test_raycast.py:96-101, 114-116
    h = oracle.intersect_tube((0.0, 0.0, -5.0), (0.0, 0.0, 1.0), (-1.0, 0.0, 0.0), (1.0, 0.0, 0.0), 0.1,
                              f32_axis=False)
    assert h[0] == 1.0 and h[1] == pytest.approx(4.9) and h[2] == pytest.approx(5.1)
    assert h[3:].tolist() == pytest.approx([0.0, 0.0, -1.0])
    s = oracle.intersect_sphere((0.0, 0.0, -5.0), (0.0, 0.0, 1.0), (0.0, 0.0, 0.0), 1.0)
    assert s[0] == 1.0 and s[1] == pytest.approx(4.0) and s[2] == pytest.approx(6.0)


def test_kat_coarsen_spike(oracle):
    # tests/test_lod.py:128-130
    f = np.zeros((2, 2, 2), np.float32)
    f[0, 0, 0] = 1.0
    assert oracle.coarsen(f).tolist() == [[[0.125]]]


def test_kat_density(oracle):
    # tests/test_lod.py:60-74 style: one straight chord of length 1 with sigma 0.75
    pts, at, off = _one_curve([(0.5, 0.5, 0.5), (2.5, 0.5, 0.5)], [0.5, 0.5])
    table = oracle.default_transfer_table()
    table[:, 3] = 0.75
    m = oracle.build_voxel_model(pts, at, off, (4, 4, 4), 32, table)
    l0 = oracle.compute_density_level0(m)
    assert l0[0, 0, 1] == np.float32(0.75) and l0.sum() == np.float32(0.75)
