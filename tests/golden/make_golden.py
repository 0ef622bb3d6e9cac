"""Generates the golden fixtures under tests/golden/ by importing the UNMODIFIED
Python reference from /root/reference/pkg/src (numpy + numba, CPU).

Run in the build container only (the reference does not exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Every fixture stores the inputs (so nothing depends on a generator staying
stable) and the reference's outputs.  The oracle (oracle/lvx_oracle.c) is
pinned against these files by tests/test_oracle_golden.py; the CUDA path is
checked against the same files by tests/test_gpu_golden.py.
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("NUMBA_NUM_THREADS", "8")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import linevox  # noqa: E402  (the reference)
from linevox import _kernels as K  # noqa: E402
from linevox import voxelizer as RV  # noqa: E402
from linevox import raycast as RR  # noqa: E402
from linevox.illumination import (AOParams, ao_density_rays, cone_soft_shadow,  # noqa: E402
                                  precompute_voxel_ao, sample_ao)
from linevox.lod import build_octree, compute_density_level0  # noqa: E402
from linevox.scene_io import Curve, CurveSet, GridSpec  # noqa: E402

from paper_1801_01155_b200 import synth  # noqa: E402  (pure-numpy generators)

MODEL_FIELDS = ["counts", "offsets", "packed", "seg_voxel", "seg_a", "seg_b", "seg_attr", "seg_lid",
                "seg_face_in", "seg_bin_in", "seg_face_out", "seg_bin_out", "seg_curve", "seg_order"]


def curveset(pts, attrs, off):
    return CurveSet.from_curves([Curve(points=pts[off[i]:off[i + 1]], attrs=attrs[off[i]:off[i + 1]])
                                 for i in range(len(off) - 1)])


def ref_model(pts, attrs, off, dims, n_bins):
    return RV.build_voxel_model(curveset(pts, attrs, off), GridSpec(dims, n_bins))


ONLY = None  # `--only <prefix>`: write just the fixtures whose name starts with the prefix


def save(name, **arrays):
    if ONLY is not None and not name.startswith(ONLY):
        return
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"{name}.npz  {os.path.getsize(path) / 1024:.1f} KiB")


VOX_CASES = [
    # name, generator, args, dims, n_bins
    ("helices", synth.helices, (60, 40), (16, 16, 16), 32),
    ("turbulence", synth.turbulence, (150, 50), (20, 16, 12), 32),
    ("wiggles", synth.wiggles, (80, 30), (12, 10, 8), 16),
    ("lattice", synth.lattice_adversarial, (400, 10), (6, 5, 4), 8),
    ("cap255", synth.helices, (700, 24), (4, 4, 4), 32),
    ("bins4", synth.turbulence, (60, 40), (10, 10, 10), 4),
    ("bins128", synth.turbulence, (60, 40), (10, 10, 10), 128),
    ("bins256", synth.wiggles, (40, 20), (8, 8, 8), 256),
]


def make_voxelize():
    models = {}
    for name, gen, args, dims, n_bins in VOX_CASES:
        pts, attrs, off = gen(*args, dims)
        m = ref_model(pts, attrs, off, dims, n_bins)
        out = {f: getattr(m, f) for f in MODEL_FIELDS}
        save("vox_" + name, pts=pts, attrs=attrs, off=off, dims=np.asarray(dims), n_bins=np.int64(n_bins),
             dropped=np.int64(m.dropped_overflow), **out)
        models[name] = (m, dims)
    # raw clip output of one adversarial batch (the seven arrays of _clip_batch)
    pts, attrs, off = synth.lattice_adversarial(200, 9, (5, 4, 3), seed=11)
    pc = np.repeat(np.arange(len(off) - 1), np.diff(off))
    vox, p_in, p_out, a_in, a_out, curve, within = RV._clip_batch(pts, attrs, pc, (5, 4, 3))
    save("clip_lattice", pts=pts, attrs=attrs, off=off, dims=np.asarray((5, 4, 3)), vox=vox, p_in=p_in,
         p_out=p_out, a_in=a_in, a_out=a_out, curve=curve, within=within)
    return models


def make_lod(models):
    out = {}
    for name in ("helices", "turbulence", "wiggles", "cap255"):
        m, dims = models[name]
        oc = build_octree(compute_density_level0(m))
        save("lod_" + name, **{f"level{l}": lvl for l, lvl in enumerate(oc.levels)})
        out[name] = oc
    # odd-sized random fields through _coarsen (edge parents have < 8 children)
    rng = np.random.default_rng(5)
    f = rng.random((7, 5, 9)).astype(np.float32)
    oc = build_octree(f)
    save("lod_random_7x5x9", **{f"level{l}": lvl for l, lvl in enumerate(oc.levels)})
    return out


def make_ao(models, octrees):
    fields = {}
    for name, n_rays, radius in (("helices", 24, 4.0), ("turbulence", 100, 5.0)):
        m, dims = models[name]
        ao = precompute_voxel_ao(m, octrees[name], AOParams(n_rays=n_rays, radius=radius, step=1.0), workers=4)
        save("ao_" + name, values=ao.values, n_rays=np.int64(n_rays), radius=np.float64(radius),
             step=np.float64(1.0))
        fields[name] = ao
    return fields


RENDER_CASES = [
    # name, model, (W,H), RenderParams kwargs
    ("opaque_nb", "helices", (64, 48), dict(neighbor_mode="on")),
    ("opaque_own", "helices", (64, 48), dict(neighbor_mode="off")),
    ("alpha25_nb", "helices", (64, 48), dict(neighbor_mode="on", base_opacity=0.25)),
    ("alpha25_own_nojoints", "helices", (64, 48), dict(neighbor_mode="off", base_opacity=0.25,
                                                         joint_spheres=False)),
    ("alpha25_nb_ao_cone", "helices", (64, 48), dict(neighbor_mode="on", base_opacity=0.25,
                                                       ao_mode="precomputed", shadow_mode="cone",
                                                       light_dir=(0.3, 0.2, 1.0))),
    ("alpha25_own_densao", "turbulence", (48, 36), dict(neighbor_mode="off", base_opacity=0.25,
                                                         ao_mode="density-rays", ao_rays=9, ao_radius=6.0)),
    ("alpha05_tau1_nb", "turbulence", (48, 36), dict(neighbor_mode="on", base_opacity=0.05, tau=1.0)),
    ("distance_scaled", "wiggles", (48, 36), dict(neighbor_mode="on", base_opacity=0.3,
                                                   opacity_mode="distance-scaled",
                                                   background=(0.2, 0.3, 0.4, 0.5))),
    ("transfer_light", "wiggles", (48, 36), dict(neighbor_mode="on", opacity_mode="transfer",
                                                  light_dir=(1.0, -0.5, 0.25), shininess=7.5)),
    ("cap255_overflow", "cap255", (40, 30), dict(neighbor_mode="on", base_opacity=0.02, tau=1.0)),
    # geometry secondary rays: hard shadows, hemisphere-geometry AO
    ("geom_hard_nb", "helices", (48, 36), dict(neighbor_mode="on", base_opacity=0.4, shadow_mode="hard",
                                                light_dir=(0.3, 0.2, 1.0))),
    ("geom_hard_own_nojoints", "turbulence", (40, 30), dict(neighbor_mode="off", base_opacity=0.5,
                                                             shadow_mode="hard", light_dir=(-0.4, 0.7, 0.5),
                                                             joint_spheres=False)),
    ("geom_hemi_nb", "wiggles", (40, 30), dict(neighbor_mode="on", base_opacity=0.5,
                                                ao_mode="hemisphere-geometry", ao_rays=7, ao_radius=3.0)),
    ("geom_hard_hemi", "turbulence", (32, 24), dict(neighbor_mode="on", base_opacity=0.6, shadow_mode="hard",
                                                     light_dir=(0.2, -0.3, 1.0), ao_mode="hemisphere-geometry",
                                                     ao_rays=5, ao_radius=4.0)),
]


def make_render(models, octrees, ao_fields):
    for name, mname, (W, H), kw in RENDER_CASES:
        if ONLY is not None and not ("render_" + name).startswith(ONLY):
            continue
        m, dims = models[mname]
        m.ao = ao_fields[mname].values if mname in ao_fields else None
        if kw.get("opacity_mode") == "transfer":
            # a transfer table with varying opacity
            t = RV.default_transfer_table()
            t[:, 3] = np.linspace(0.1, 0.9, 256).astype(np.float32)
            m.transfer_table = t
        cam = RR.default_camera(dims, W, H)
        fr = RR.render_frame(cam, m, octrees.get(mname), None, RR.RenderParams(**kw), workers=4)
        st = fr.stats
        save("render_" + name, image=fr.image, model=np.array(mname),
             stats=np.asarray([st["voxel_steps"], st["intersection_tests"], st["window_overflow"]], np.int64),
             transfer_table=np.asarray(m.transfer_table, np.float32),
             size=np.asarray([W, H]), params=np.array(repr(kw)))


def make_primitives(models, octrees, ao_fields):
    rng = np.random.default_rng(77)
    n = 3000
    # rays around a small box, segments inside it
    o = rng.uniform(-3, 11, (n, 3))
    tgt = rng.uniform(0, 8, (n, 3))
    d = tgt - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    a = rng.uniform(0, 8, (n, 3))
    b = a + rng.normal(0, 0.8, (n, 3))
    # make a share of them nearly hit: aim rays at a point of the segment
    aim = rng.random(n) < 0.6
    mid = a + (b - a) * rng.random((n, 1)) + rng.normal(0, 0.15, (n, 3))
    d2 = mid - o
    d2 /= np.linalg.norm(d2, axis=1, keepdims=True)
    d[aim] = d2[aim]
    # special cases: parallel to axis, degenerate, origin inside
    d[:20] = (b[:20] - a[:20]) / np.linalg.norm(b[:20] - a[:20], axis=1, keepdims=True)
    b[20:30] = a[20:30]
    o[30:60] = a[30:60] + 0.05
    a32, b32 = a.astype(np.float32), b.astype(np.float32)
    r = 0.3
    tube64 = np.zeros((n, 6))
    tube32 = np.zeros((n, 6))
    sph = np.zeros((n, 6))
    for i in range(n):
        tube64[i] = K.intersect_tube_raw(*o[i], *d[i], *a[i], *b[i], r)
        # float32 scalars select the specialisation the frame kernels compile to
        tube32[i] = K.intersect_tube_raw(*o[i], *d[i], *a32[i], *b32[i], r)
        sph[i] = K.intersect_sphere_raw(*o[i], *d[i], *a[i], r)
    save("prim_tube_sphere", o=o, d=d, a=a, b=b, r=np.float64(r), tube64=tube64, tube32=tube32, sphere=sph)

    # DDA windows
    dims = (7, 5, 6)
    rays_o = rng.uniform(-4, 10, (300, 3))
    rays_t = rng.uniform(0, 6, (300, 3))
    rays_d = rays_t - rays_o
    rays_d /= np.linalg.norm(rays_d, axis=1, keepdims=True)
    rays_d[:10, 0] = 0.0  # axis-parallel components
    rays_d[:10] /= np.linalg.norm(rays_d[:10], axis=1, keepdims=True)
    rays_o[10:20] = np.round(rays_o[10:20])  # lattice origins: ties
    rays_d[10:20] = np.sign(rays_d[10:20]) / np.sqrt(3.0)
    counts, vox_all, t_all = [], [], []
    for pad in (0, 1):
        for i in range(rays_o.shape[0]):
            cap = sum(dims) + 6 * (pad + 2)
            ov = np.empty((cap, 3), np.int64)
            ot = np.empty((cap, 2))
            k = K.dda_collect(*rays_o[i], *rays_d[i], *dims, pad, ov, ot)
            counts.append(k)
            vox_all.append(ov[:k].copy())
            t_all.append(ot[:k].copy())
    save("prim_dda", o=rays_o, d=rays_d, dims=np.asarray(dims), counts=np.asarray(counts),
         vox=np.concatenate(vox_all), t=np.concatenate(t_all))

    # density-grid probes on the turbulence octree
    m, mdims = models["turbulence"]
    oc = octrees["turbulence"]
    P = rng.uniform(-1.0, np.asarray(mdims) + 1.0, (400, 3))
    flat, off, ldims, L = RR._octree_args(oc)
    tri = np.zeros((L, P.shape[0]))
    for l in range(L):
        for i in range(P.shape[0]):
            tri[l, i] = K.sample_field_trilinear(flat, off[l], ldims[l, 0], ldims[l, 1], ldims[l, 2],
                                                 float(1 << l), *P[i])
    light = np.array([0.3, 0.2, 1.0])
    cone = np.array([cone_soft_shadow(P[i], light, oc) for i in range(P.shape[0])])
    N = rng.normal(size=(400, 3))
    N /= np.linalg.norm(N, axis=1, keepdims=True)
    N[:5] = [[1, 0, 0], [-1, 0, 0], [0, 0, 1], [0.95, 0.1, 0], [0, 1, 0]]
    N /= np.linalg.norm(N, axis=1, keepdims=True)
    aod = np.array([ao_density_rays(P[i], N[i], oc, AOParams(n_rays=25, radius=6.0, step=1.0))
                    for i in range(P.shape[0])])
    aos = np.array([sample_ao(ao_fields["turbulence"], P[i]) for i in range(P.shape[0])])
    fib = np.array([[K.fibonacci_dir(i, nn, h, 0.0) for i in range(nn)] for nn, h in ((25, 1),)][0])
    fib100 = np.array([K.fibonacci_dir(i, 100, 0, 0.0) for i in range(100)])
    save("prim_density", P=P, N=N, light=light, trilinear=tri, cone=cone, ao_density=aod, ao_sample=aos,
         fib25_hemi=fib, fib100_sphere=fib100)

    # shading
    nn_ = rng.normal(size=(500, 3))
    nn_ /= np.linalg.norm(nn_, axis=1, keepdims=True)
    ll = rng.normal(size=(500, 3))
    ll /= np.linalg.norm(ll, axis=1, keepdims=True)
    vv = rng.normal(size=(500, 3))
    vv /= np.linalg.norm(vv, axis=1, keepdims=True)
    sh = np.array([K.shade_scalar(*nn_[i], *ll[i], *vv[i], 0.2, 0.7, 0.3, 32.0) for i in range(500)])
    save("prim_shade", n=nn_, l=ll, v=vv, shade=sh)


def make_geometry_probes(models):
    """Point probes of the geometry secondary rays: hard_shadow / ao_hemisphere_geometry."""
    from linevox.illumination import ao_hemisphere_geometry, hard_shadow
    rng = np.random.default_rng(123)
    for mname in ("helices", "turbulence"):
        m, dims = models[mname]
        d = np.asarray(dims, dtype=np.float64)
        n = 160
        P = rng.uniform(0.5, 1.0, (n, 3)) * 0 + rng.uniform(0.2, 0.8, (n, 3)) * d
        # half of the points sit on a segment's surface (the interesting case)
        seg = rng.integers(0, m.seg_a.shape[0], n // 2)
        mid = 0.5 * (m.seg_a[seg].astype(np.float64) + m.seg_b[seg].astype(np.float64))
        off = rng.normal(size=(n // 2, 3))
        off /= np.linalg.norm(off, axis=1, keepdims=True)
        P[: n // 2] = mid + 0.3 * off
        N = rng.normal(size=(n, 3))
        N[: n // 2] = off
        N /= np.linalg.norm(N, axis=1, keepdims=True)
        L = rng.uniform(-0.5, 1.5, (n, 3)) * d
        L[::7] = P[::7] + 0.05 * N[::7]  # a few very close lights
        hs = np.array([hard_shadow(P[i], L[i], m, 0.3, N[i] if i % 2 == 0 else None, bool(i % 3))
                       for i in range(n)], dtype=np.int64)
        ao = np.array([ao_hemisphere_geometry(P[i], N[i], m, AOParams(n_rays=9, radius=3.5), 0.3)
                       for i in range(n)])
        aoj = np.array([ao_hemisphere_geometry(P[i], N[i], m, AOParams(n_rays=6, radius=2.5), 0.25, jitter=0.37)
                        for i in range(0, n, 4)])
        save("geom_probe_" + mname, P=P, N=N, L=L, hard=hs, ao=ao, ao_jitter=aoj)


def make_replines(models, octrees):
    """Representative lines (lod.py:224-284), their shadow probes (illumination.py:115-139)
    and frames with shadow_mode="replines"."""
    from linevox.illumination import replines_shadow
    from linevox.lod import build_rep_lines
    rng = np.random.default_rng(321)
    fields = {}
    for mname in ("helices", "turbulence", "wiggles"):
        m, dims = models[mname]
        oc = octrees[mname]
        rl = build_rep_lines(m, oc)
        loose = build_rep_lines(m, oc, adjacency=False)
        fields[mname] = rl
        out = {"n_levels": np.int64(len(rl.levels))}
        for l in range(1, len(rl.levels)):
            for tag, f in (("", rl), ("loose_", loose)):
                lv_ = f.levels[l]
                out[f"{tag}valid{l}"] = lv_.valid
                out[f"{tag}a{l}"] = lv_.a
                out[f"{tag}b{l}"] = lv_.b
                out[f"{tag}w{l}"] = lv_.weight
        d = np.asarray(dims, dtype=np.float64)
        n = 120
        P = rng.uniform(0.1, 0.9, (n, 3)) * d
        N = rng.normal(size=(n, 3))
        N /= np.linalg.norm(N, axis=1, keepdims=True)
        Lp = rng.uniform(-0.5, 1.5, (n, 3)) * d
        lev = np.array([1 + (i % (len(rl.levels) - 1)) for i in range(n)], dtype=np.int64)
        sh = np.array([replines_shadow(P[i], Lp[i], rl, dims, level=int(lev[i]), tube_radius=0.3,
                                       normal=N[i] if i % 2 else None) for i in range(n)], dtype=np.int64)
        save("rep_" + mname, P=P, N=N, L=Lp, level=lev, shadow=sh, **out)
    cases = [("rep_frame_helices", "helices", (48, 36), dict(neighbor_mode="on", base_opacity=0.4, shadow_mode="replines",
                                                             light_dir=(0.3, 0.2, 1.0), shadow_rep_level=1)),
             ("rep_frame_turbulence", "turbulence", (40, 30), dict(neighbor_mode="off", base_opacity=0.5,
                                                                   shadow_mode="replines", light_dir=(-0.4, 0.7, 0.5)))]
    for name, mname, (W, H), kw in cases:
        if ONLY is not None and not ("render_" + name).startswith(ONLY):
            continue
        m, dims = models[mname]
        m.ao = None
        fr = RR.render_frame(RR.default_camera(dims, W, H), m, octrees.get(mname), fields[mname], RR.RenderParams(**kw),
                             workers=4)
        st = fr.stats
        save("render_" + name, image=fr.image, model=np.array(mname),
             stats=np.asarray([st["voxel_steps"], st["intersection_tests"], st["window_overflow"]], np.int64),
             transfer_table=np.asarray(m.transfer_table, np.float32), size=np.asarray([W, H]), params=np.array(repr(kw)))


def make_brute(models, octrees, ao_fields):
    """The reference's brute-force renderer (metrics.brute_force_render) on small scenes."""
    from linevox.metrics import brute_force_render
    cases = [("brute_opaque", "helices", (40, 30), dict(neighbor_mode="on")),
             ("brute_alpha_cone_ao", "helices", (40, 30), dict(base_opacity=0.3, ao_mode="precomputed", shadow_mode="cone",
                                                               light_dir=(0.3, 0.2, 1.0))),
             ("brute_alpha_nojoints", "turbulence", (36, 28), dict(base_opacity=0.2, joint_spheres=False, tau=1.0)),
             ("brute_hard", "wiggles", (32, 24), dict(base_opacity=0.5, shadow_mode="hard", light_dir=(0.2, -0.3, 1.0)))]
    for name, mname, (W, H), kw in cases:
        m, dims = models[mname]
        m.ao = ao_fields[mname].values if mname in ao_fields else None
        m.transfer_table = RV.default_transfer_table()
        fr = brute_force_render(RR.default_camera(dims, W, H), m, octrees.get(mname), None, RR.RenderParams(**kw), workers=4)
        st = fr.stats
        save("render_" + name, image=fr.image, model=np.array(mname),
             stats=np.asarray([st["voxel_steps"], st["intersection_tests"], st["window_overflow"]], np.int64),
             transfer_table=np.asarray(m.transfer_table, np.float32), size=np.asarray([W, H]), params=np.array(repr(kw)))


def make_occupancy(models):
    """_occupancy_dilated (raycast.py:351-366): u8 map over the grid padded by one voxel."""
    for name in ("helices", "turbulence", "lattice", "cap255", "wiggles"):
        m, dims = models[name]
        m.__dict__.pop("_occ_dilated", None)
        save("occ_" + name, occ=np.ascontiguousarray(RR._occupancy_dilated(m)), dims=np.asarray(dims))


def _sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


ROW_STEP = 16  # big frames: every 16th row of the reference's image is stored (plus the hash of all of it)


def _save_big_frame(name, fr, m, kw, W, H, extra=None):
    st = fr.stats
    save(name, rows=np.ascontiguousarray(fr.image[::ROW_STEP]), row_step=np.int64(ROW_STEP),
         image_sha256=np.array(_sha(fr.image)), size=np.asarray([W, H]), params=np.array(repr(kw)),
         stats=np.asarray([st["voxel_steps"], st["intersection_tests"], st["window_overflow"]], np.int64),
         packed_sha256=np.array(_sha(m.packed)), counts_sha256=np.array(_sha(m.counts)),
         segments=np.int64(m.segment_count), **(extra or {}))


def make_big():
    """The frames bench.py times, rendered by the unmodified reference at full size:
    BASELINE configs[1] (C2) and configs[2] (C3) at 1920x1080 (SURVEY.md 8d generators)."""
    import time
    if ONLY is None or "big_c2_1080p".startswith(ONLY):
        dims = (128, 128, 128)
        t0 = time.time()
        m = ref_model(*synth.helices(10000, 100, dims), dims, 32)
        kw = dict(base_opacity=0.25, tau=0.95, neighbor_mode="on")
        fr = RR.render_frame(RR.default_camera(dims, 1920, 1080), m, None, None, RR.RenderParams(**kw), workers=8)
        print(f"C2: {time.time() - t0:.0f} s, stats {fr.stats}")
        _save_big_frame("big_c2_1080p", fr, m, kw, 1920, 1080)
        # own-voxel mode of the same frame
        kw2 = dict(kw, neighbor_mode="off")
        fr = RR.render_frame(RR.default_camera(dims, 1920, 1080), m, None, None, RR.RenderParams(**kw2), workers=8)
        _save_big_frame("big_c2_1080p_own", fr, m, kw2, 1920, 1080)
    if ONLY is None or "big_c3_1080p".startswith(ONLY):
        dims = (256, 256, 256)
        t0 = time.time()
        m = ref_model(*synth.turbulence(100000, 100, dims), dims, 32)
        print(f"C3 voxelized: {time.time() - t0:.0f} s")
        l0 = compute_density_level0(m)
        oc = build_octree(l0)
        ao = precompute_voxel_ao(m, oc, AOParams(n_rays=100, radius=5.0, step=1.0), workers=8)
        m.ao = ao.values
        print(f"C3 LoD + AO: {time.time() - t0:.0f} s")
        kw = dict(base_opacity=0.25, tau=0.95, neighbor_mode="on", ao_mode="precomputed")
        fr = RR.render_frame(RR.default_camera(dims, 1920, 1080), m, oc, None, RR.RenderParams(**kw), workers=8)
        print(f"C3: {time.time() - t0:.0f} s, stats {fr.stats}")
        _save_big_frame("big_c3_1080p", fr, m, kw, 1920, 1080,
                        extra=dict(level0_sha256=np.array(_sha(l0)), ao_sha256=np.array(_sha(ao.values)),
                                   levels_sha256=np.array([_sha(l) for l in oc.levels])))


def make_acceptance():
    """The reference's own acceptance scene (tests/test_acceptance.py:144-169): tornado(1000, 250, 42)
    normalised into a 256^3 grid, N = 32, 640x360, opaque and alpha = 0.25, neighbour mode on."""
    if ONLY is not None and not "accept_tornado256".startswith(ONLY):
        return
    from linevox.scene_io import generate_tornado, normalize_to_grid
    spec = GridSpec((256, 256, 256), 32)
    cs = normalize_to_grid(generate_tornado(1000, 250, 42), spec)
    m = RV.build_voxel_model(cs, spec)
    pts = np.concatenate([c.points for c in cs.curves])
    attrs = np.concatenate([c.attrs for c in cs.curves])
    off = np.zeros(len(cs.curves) + 1, np.int64)
    np.cumsum([len(c.points) for c in cs.curves], out=off[1:])
    cam = RR.default_camera(spec.dims, 640, 360)
    out = {}
    for tag, kw in (("opaque", dict(neighbor_mode="on")), ("alpha25", dict(neighbor_mode="on", base_opacity=0.25))):
        fr = RR.render_frame(cam, m, None, None, RR.RenderParams(**kw), workers=8)
        st = fr.stats
        out["rows_" + tag] = np.ascontiguousarray(fr.image[::4])
        out["sha_" + tag] = np.array(_sha(fr.image))
        out["stats_" + tag] = np.asarray([st["voxel_steps"], st["intersection_tests"], st["window_overflow"]], np.int64)
        out["params_" + tag] = np.array(repr(kw))
    save("accept_tornado256", pts=pts, attrs=attrs, off=off, dims=np.asarray(spec.dims), row_step=np.int64(4),
         packed_sha256=np.array(_sha(m.packed)), counts_sha256=np.array(_sha(m.counts)),
         segments=np.int64(m.segment_count), dropped=np.int64(m.dropped_overflow), **out)


def main():
    global ONLY
    if "--only" in sys.argv:
        ONLY = sys.argv[sys.argv.index("--only") + 1]
    models = make_voxelize()
    octrees = make_lod(models)
    ao_fields = make_ao(models, octrees)
    make_render(models, octrees, ao_fields)
    make_primitives(models, octrees, ao_fields)
    make_geometry_probes(models)
    make_replines(models, octrees)
    make_brute(models, octrees, ao_fields)
    make_occupancy(models)
    make_acceptance()
    make_big()


if __name__ == "__main__":
    main()
