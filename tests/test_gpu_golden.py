"""CUDA path vs the committed golden fixtures (outputs of the unmodified Python
reference): voxel models, LoD levels and AO bakes bit-exact; frames within the
north-star tolerance (max per-channel error <= 1/255, mean < 1e-3) with exact
counters; point probes bit-exact except where CUDA libm differs (pow)."""
import numpy as np
import pytest

from conftest import (BRUTE_RENDER_CASES, RENDER_CASES, REP_RENDER_CASES, VOX_CASES, assert_model_equal, golden,
                      render_kwargs)

pytestmark = pytest.mark.gpu

MAX_ERR = 1.0 / 255.0  # north_star: max per-channel error 1/255 ...
MEAN_ERR = 1e-3        # ... and mean error below 1e-3


@pytest.fixture(scope="module")
def lv():
    import paper_1801_01155_b200 as lv
    return lv


def gpu_model(lv, g, table=None):
    cs = lv.CurveSet.from_flat(g["pts"], g["attrs"], g["off"])
    return lv.build_voxel_model(cs, lv.GridSpec(tuple(int(x) for x in g["dims"]), int(g["n_bins"])), table)


@pytest.mark.parametrize("name", VOX_CASES)
def test_voxel_model_bit_exact(lv, name):
    g = golden("vox_" + name)
    m = gpu_model(lv, g)
    assert_model_equal(m, g)
    assert m.dropped_overflow == int(g["dropped"])
    assert m.memory_bytes == 5 * m.voxel_count + m.record_width * m.segment_count


@pytest.mark.parametrize("name", ["helices", "turbulence", "wiggles", "cap255"])
def test_lod_bit_exact(lv, name):
    m = gpu_model(lv, golden("vox_" + name))
    g = golden("lod_" + name)
    # reference-shaped API (host arrays in and out) ...
    l0 = lv.compute_density_level0(m)
    assert l0.dtype == np.float32 and np.array_equal(l0, g["level0"])
    oc = lv.build_octree(l0)
    assert oc.n_levels == len(g.files)
    for l, lvl in enumerate(oc.levels):
        assert np.array_equal(lvl, g[f"level{l}"]), f"level {l}"
    # ... and the device-resident shortcut
    oc2 = lv.build_lod(m)
    for l, lvl in enumerate(oc2.levels):
        assert np.array_equal(lvl, g[f"level{l}"]), f"level {l} (build_lod)"


def test_coarsen_odd_sizes(lv):
    g = golden("lod_random_7x5x9")
    oc = lv.build_octree(g["level0"])
    assert oc.n_levels == len(g.files)
    for l, lvl in enumerate(oc.levels):
        assert np.array_equal(lvl, g[f"level{l}"])


@pytest.mark.parametrize("name", ["helices", "turbulence"])
def test_ao_bake_bit_exact(lv, name):
    m = gpu_model(lv, golden("vox_" + name))
    g = golden("ao_" + name)
    ao = lv.precompute_voxel_ao(m, lv.build_lod(m), lv.AOParams(int(g["n_rays"]), float(g["radius"]), float(g["step"])))
    assert ao.values.dtype == np.float32
    assert np.array_equal(ao.values, g["values"])


def gpu_render(lv, name, **extra):
    g = golden("render_" + name)
    mname = str(g["model"])
    vg = golden("vox_" + mname)
    m = gpu_model(lv, vg, g["transfer_table"])
    oc = lv.build_lod(gpu_model(lv, vg))  # LoD fixtures used the default table
    if mname in ("helices", "turbulence"):
        m.ao = golden("ao_" + mname)["values"]
    W, H = (int(x) for x in g["size"])
    cam = lv.default_camera(m.spec.dims, W, H)
    params = lv.RenderParams(**render_kwargs(g))
    rl = lv.build_rep_lines(m, oc) if params.shadow_mode == "replines" else None
    fr = lv.render_frame(cam, m, oc, rl, params, **extra)
    return g, fr


@pytest.mark.parametrize("engine", ["tile", "wavefront"])
@pytest.mark.parametrize("name", RENDER_CASES + REP_RENDER_CASES)
def test_render_matches_reference(lv, name, engine, monkeypatch):
    # both frame engines (csrc/lvx_render.cu, csrc/lvx_wavefront.cu) against every fixture
    monkeypatch.setenv("LVX_ENGINE", engine)
    g, fr = gpu_render(lv, name)
    assert fr.image.shape == g["image"].shape and fr.image.dtype == np.float32
    err = np.abs(fr.image.astype(np.float64) - g["image"].astype(np.float64))
    assert err.max() <= MAX_ERR, f"max per-channel error {err.max()}"
    assert err.mean() < MEAN_ERR
    st = fr.stats
    assert [st["voxel_steps"], st["intersection_tests"], st["window_overflow"]] == list(g["stats"])
    assert st["rays"] == fr.image.shape[0] * fr.image.shape[1]
    # in practice the frame is bit-identical unless CUDA's pow rounds differently
    assert (err > 1e-6).mean() < 1e-3


@pytest.mark.parametrize("mname", ["helices", "turbulence"])
def test_geometry_secondary_ray_probes(lv, mname):
    """hard_shadow / ao_hemisphere_geometry (geometry_ray_blocked, ao_hemisphere_point) against
    the reference's values: booleans and blocked-ray fractions, bit-exact."""
    g = golden("geom_probe_" + mname)
    m = gpu_model(lv, golden("vox_" + mname))
    P, N, L = g["P"], g["N"], g["L"]
    hs = [lv.hard_shadow(P[i], L[i], m, 0.3, N[i] if i % 2 == 0 else None, bool(i % 3)) for i in range(len(P))]
    assert hs == list(g["hard"])
    ao = lv.ao_hemisphere_geometry(P, N, m, lv.AOParams(n_rays=9, radius=3.5), 0.3)
    assert np.array_equal(ao, g["ao"])
    assert lv.ao_hemisphere_geometry(P[3], N[3], m, lv.AOParams(n_rays=9, radius=3.5), 0.3) == g["ao"][3]
    aoj = np.array([lv.ao_hemisphere_geometry(P[i], N[i], m, lv.AOParams(n_rays=6, radius=2.5), 0.25, jitter=0.37)
                    for i in range(0, len(P), 4)])
    assert np.array_equal(aoj, g["ao_jitter"])


@pytest.mark.parametrize("mname", ["helices", "turbulence", "wiggles"])
def test_representative_lines(lv, mname):
    """build_rep_lines (every level, with and without the adjacency pass) and replines_shadow
    against the reference's values, bit-exact (lod.py:224-284, illumination.py:115-139)."""
    g = golden("rep_" + mname)
    m = gpu_model(lv, golden("vox_" + mname))
    oc = lv.build_lod(m)
    n_levels = int(g["n_levels"])
    assert oc.n_levels == n_levels
    for adjacency, tag in ((True, ""), (False, "loose_")):
        rl = lv.build_rep_lines(m, oc, adjacency=adjacency)
        assert len(rl.levels) == n_levels and rl.levels[0] is None
        for l in range(1, n_levels):
            lvl = rl.levels[l]
            assert np.array_equal(lvl.valid, g[f"{tag}valid{l}"]), (tag, l)
            assert np.array_equal(lvl.a, g[f"{tag}a{l}"]), (tag, l)
            assert np.array_equal(lvl.b, g[f"{tag}b{l}"]), (tag, l)
            assert np.array_equal(lvl.weight, g[f"{tag}w{l}"]), (tag, l)
    rl = lv.build_rep_lines(m, oc)
    P, N, L, lev = g["P"], g["N"], g["L"], g["level"]
    sh = [lv.replines_shadow(P[i], L[i], rl, m.spec.dims, level=int(lev[i]), tube_radius=0.3,
                             normal=N[i] if i % 2 else None) for i in range(len(P))]
    assert sh == list(g["shadow"])
    with pytest.raises(ValueError):
        lv.replines_shadow(P[0], L[0], rl, m.spec.dims, level=0)
    with pytest.raises(ValueError):
        lv.replines_shadow(P[0], L[0], rl, m.spec.dims, level=99)


@pytest.mark.parametrize("name", BRUTE_RENDER_CASES)
def test_brute_force_render(lv, name):
    """The GPU brute-force renderer (every primitive at every pixel, no DDA) against the
    reference's brute_force_render, and against both accelerated engines on the same scene:
    the reference's own cross-check (tests/test_metrics.py:117-125, test_illumination.py:363-387)."""
    g = golden("render_" + name)
    mname = str(g["model"])
    vg = golden("vox_" + mname)
    m = gpu_model(lv, vg, g["transfer_table"])
    oc = lv.build_lod(gpu_model(lv, vg))
    if mname in ("helices", "turbulence"):
        m.ao = golden("ao_" + mname)["values"]
    W, H = (int(x) for x in g["size"])
    cam = lv.default_camera(m.spec.dims, W, H)
    params = lv.RenderParams(**render_kwargs(g))
    fr = lv.brute_force_render(cam, m, oc, None, params)
    err = np.abs(fr.image.astype(np.float64) - g["image"].astype(np.float64))
    assert err.max() <= MAX_ERR and err.mean() < MEAN_ERR
    assert (err > 1e-6).mean() < 1e-3
    st = fr.stats
    assert [st["voxel_steps"], st["intersection_tests"], st["window_overflow"]] == list(g["stats"])
    n_prim = (3 if params.joint_spheres else 1) * m.segment_count
    assert st["intersection_tests"] == W * H * n_prim  # tests/test_metrics.py:128-134
    # the accelerated engines agree with it to the bit (neighbour mode: the brute force has no
    # notion of own-voxel gathering)
    import os
    for engine in ("tile", "wavefront"):
        os.environ["LVX_ENGINE"] = engine
        try:
            acc = lv.render_frame(cam, m, oc, None, lv.RenderParams(**{**render_kwargs(g), "neighbor_mode": "on"}))
        finally:
            os.environ.pop("LVX_ENGINE", None)
        assert np.array_equal(acc.image, fr.image), engine
    cmp_ = lv.image_compare(fr, g["image"])
    assert cmp_["fraction_close"] == 1.0
    assert lv.memory_report(m)["total"] == 5 * m.voxel_count + m.record_width * m.segment_count


def test_tube_and_sphere_probes(lv):
    from paper_1801_01155_b200 import raycast
    g = golden("prim_tube_sphere")
    rays = np.concatenate([g["o"], g["d"]], axis=1)
    r = float(g["r"])
    t64 = raycast.probe_tubes(rays, g["a"], g["b"], r, f32_axis=False)
    t32 = raycast.probe_tubes(rays, g["a"], g["b"], r, f32_axis=True)
    sp = raycast.probe_spheres(rays, g["a"], r)
    assert np.array_equal(t64, g["tube64"])
    assert np.array_equal(t32, g["tube32"])
    assert np.array_equal(sp, g["sphere"])


def test_dda_windows(lv):
    from paper_1801_01155_b200 import raycast
    g = golden("prim_dda")
    dims = tuple(int(x) for x in g["dims"])
    k = pos = 0
    for pad in (0, 1):
        for i in range(0, g["o"].shape[0]):
            n = int(g["counts"][k])
            if i % 5 == 0 or i < 25:  # one launch per ray: probe a subset
                w = raycast.probe_dda(g["o"][i], g["d"][i], dims, pad)  # d as stored: no re-normalisation
                assert len(w) == n
                assert np.array_equal(np.asarray([v for v, _, _ in w]).reshape(-1, 3), g["vox"][pos:pos + n])
                assert np.array_equal(np.asarray([(a, b) for _, a, b in w]).reshape(-1, 2), g["t"][pos:pos + n])
            pos += n
            k += 1
    # reference KAT, tests/test_raycast.py:52-57, through the public op
    w = lv.traverse_voxels(((-1.0, 0.5, 0.5), (2.0, 0.0, 0.0)), lv.GridSpec((3, 3, 3)))
    assert w == [((0, 0, 0), 1.0, 2.0), ((1, 0, 0), 2.0, 3.0), ((2, 0, 0), 3.0, 4.0)]


def test_density_probes(lv):
    g = golden("prim_density")
    m = gpu_model(lv, golden("vox_turbulence"))
    oc = lv.build_lod(m)
    P, N = g["P"], g["N"]
    from paper_1801_01155_b200.illumination import _probe_trilinear
    for l in range(oc.n_levels):
        got = _probe_trilinear(oc.flat_device(), int(oc._off[l]), oc.dims(l), float(1 << l), P)
        assert np.array_equal(got, g["trilinear"][l]), f"level {l}"
    assert np.array_equal(lv.cone_soft_shadow(P, g["light"], oc), g["cone"])
    aod = lv.ao_density_rays(P, N, oc, lv.AOParams(n_rays=25, radius=6.0, step=1.0))
    assert np.array_equal(aod, g["ao_density"])
    field = lv.AOField(golden("ao_turbulence")["values"])
    assert np.array_equal(lv.sample_ao(field, P), g["ao_sample"])
    assert lv.sample_ao(field, P[0]) == g["ao_sample"][0]
    from paper_1801_01155_b200 import _lib
    assert np.array_equal(_lib.fibonacci_dirs(25, 1), g["fib25_hemi"])
    assert np.array_equal(_lib.fibonacci_dirs(100, 0), g["fib100_sphere"])


# --- the reference's small operations over the device probes (round 2) -------------------------------

def test_clip_batch_device_matches_reference():
    """_clip_batch (voxelizer.py:213-263) on the device, float64 outputs and all: the adversarial
    lattice fixture (exact plane hits, reversals, corner crossings, out-of-grid excursions)."""
    from paper_1801_01155_b200.voxelizer import clip_batch_device
    g = golden("clip_lattice")
    vox, p_in, p_out, a_in, a_out, key = clip_batch_device(g["pts"], g["attrs"], g["off"], tuple(int(d) for d in g["dims"]))
    assert np.array_equal(vox, g["vox"]) and np.array_equal(p_in, g["p_in"]) and np.array_equal(p_out, g["p_out"])
    assert np.array_equal(a_in, g["a_in"]) and np.array_equal(a_out, g["a_out"])
    assert np.all(np.diff(key.astype(np.int64)) > 0)  # (edge, ordinal) keys strictly increase in reference order


def test_clip_curve_to_voxels_kats():
    """reference tests/test_voxelizer.py:209-235: axis-aligned chord, same-voxel curve, bridged vertices."""
    import paper_1801_01155_b200 as lv
    spec = lv.GridSpec((4, 4, 4), 8)
    segs = lv.clip_curve_to_voxels(lv.Curve(points=np.array([[0.5, 0.5, 0.5], [2.5, 0.5, 0.5]]), attrs=np.array([0.0, 1.0])), spec)
    assert len(segs) == 1 and segs[0].voxel == (1, 0, 0)
    assert np.array_equal(segs[0].entry, [1.0, 0.5, 0.5]) and np.array_equal(segs[0].exit, [2.0, 0.5, 0.5])
    assert segs[0].attr_entry == 0.25 and segs[0].attr_exit == 0.75
    assert lv.clip_curve_to_voxels(lv.Curve(points=np.array([[1.2, 1.2, 1.2], [1.7, 1.4, 1.9]]), attrs=np.array([0.0, 1.0])), spec) == []
    segs = lv.clip_curve_to_voxels(lv.Curve(points=np.array([[0.5, 0.5, 0.5], [1.3, 0.6, 0.5], [1.6, 0.4, 0.5], [2.5, 0.5, 0.5]]),
                                            attrs=np.linspace(0, 1, 4)), spec)
    assert len(segs) == 1 and segs[0].voxel == (1, 0, 0)  # interior vertices inside one voxel are bridged


def test_shade_local_matches_reference():
    """shade_scalar (_kernels.py:316-329): CUDA's pow is within 2 ulp of glibc's."""
    from paper_1801_01155_b200.raycast import probe_shade
    import paper_1801_01155_b200 as lv
    g = golden("prim_shade")
    got = probe_shade(np.concatenate([g["n"], g["l"], g["v"]], axis=1), 0.2, 0.7, 0.3, 32.0)
    assert np.allclose(got, g["shade"], rtol=1e-14, atol=0.0)
    assert (got != g["shade"]).mean() < 0.2
    assert lv.shade_local(g["n"][0], g["l"][0], g["v"][0]) == got[0]


def test_composite_and_gather_reference_ops():
    """reference tests/test_raycast.py:283-288, 324-388: white/black at alpha .5; hits of a voxel in order."""
    import paper_1801_01155_b200 as lv
    p = lv.RenderParams(base_opacity=0.5, tau=1.0, ambient=1.0, diffuse=0.0, specular=0.0, background=(0, 0, 0, 1))
    table = np.ones((256, 4), np.float32)
    table[0, :3] = 0.0
    hits = [lv.HitRecord(t_in=1.0, t_out=2.0, normal=np.array([0.0, 0.0, -1.0]), attr_index=255),
            lv.HitRecord(t_in=3.0, t_out=4.0, normal=np.array([0.0, 0.0, -1.0]), attr_index=0)]
    assert np.allclose(lv.composite(hits, p, table), [0.5, 0.5, 0.5, 1.0])
    dims = (4, 4, 4)
    cs = lv.CurveSet.from_curves([lv.Curve(points=np.array([[0.2, 1.5, 1.5], [3.8, 1.5, 1.5]]), attrs=np.array([0.0, 1.0]))])
    m = lv.build_voxel_model(cs, lv.GridSpec(dims, 32))
    ray = (np.array([1.5, 1.5, -2.0]), np.array([0.0, 0.0, 1.0]))
    got = lv.gather_voxel_hits(ray, (1, 1, 1), m, lv.RenderParams(neighbor_mode="on"))
    assert [h.kind for h in got] == ["tube"] and got[0].voxel == (1, 1, 1) and abs(got[0].t_in - 3.2) < 0.03  # (endpoints are bin centres)
    assert lv.gather_voxel_hits(ray, (1, 1, 1), m, lv.RenderParams(neighbor_mode="on"), seen={21: 1}) == []


def test_representative_line_probe_equals_level_kernel():
    """representative_line (lod.py:141-169) through its probe == what the level kernel computed for
    the same members (children in z,y,x order, each child's segments in stored order)."""
    import paper_1801_01155_b200 as lv
    v = golden("vox_turbulence")
    dims = tuple(int(d) for d in v["dims"])
    m = lv.build_voxel_model(lv.CurveSet.from_flat(v["pts"], v["attrs"], v["off"]), lv.GridSpec(dims, int(v["n_bins"])))
    rep = lv.build_rep_lines(m, lv.build_lod(m), adjacency=False)
    lvl = rep.levels[1]
    pdx, pdy, pdz = lvl.dims
    checked = 0
    for plin in np.nonzero(lvl.valid)[0][:12]:
        px, py, pz = plin % pdx, (plin // pdx) % pdy, plin // (pdx * pdy)
        a, b = [], []
        for dz in range(2):
            for dy in range(2):
                for dx in range(2):
                    x, y, z = 2 * px + dx, 2 * py + dy, 2 * pz + dz
                    if x >= dims[0] or y >= dims[1] or z >= dims[2]:
                        continue
                    lin = x + dims[0] * (y + dims[1] * z)
                    o, c = int(m.offsets[lin]), int(m.counts[lin])
                    a += [m.seg_a[o:o + c]]
                    b += [m.seg_b[o:o + c]]
        qa, qb, w = lv.representative_line(np.concatenate(a), np.concatenate(b), (2.0 * px, 2.0 * py, 2.0 * pz), 2.0,
                                           int(v["n_bins"]))
        assert np.array_equal(qa.astype(np.float32), lvl.a[plin]) and np.array_equal(qb.astype(np.float32), lvl.b[plin])
        assert np.float32(w) == lvl.weight[plin]
        checked += 1
    assert checked > 0
