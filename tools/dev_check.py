"""Developer sweep on a GPU box: every stage against the oracle, with diagnostics
instead of hard stops.  Not part of the test suite."""
import os, sys, time, traceback
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_1801_01155_b200 as lv
from paper_1801_01155_b200 import synth
from oracle import lvx_oracle as orc

FIELDS = ["counts", "offsets", "packed", "seg_voxel", "seg_a", "seg_b", "seg_attr", "seg_lid",
          "seg_face_in", "seg_bin_in", "seg_face_out", "seg_bin_out", "seg_curve", "seg_order"]


def vox_case(name, gen, dims, n_bins=32):
    pts, attrs, off = gen
    t0 = time.time()
    ref = orc.build_voxel_model(pts, attrs, off, dims, n_bins)
    t1 = time.time()
    model = lv.build_voxel_model(lv.CurveSet.from_flat(pts, attrs, off), lv.GridSpec(dims, n_bins))
    torch.cuda.synchronize()
    t2 = time.time()
    bad = []
    for f in FIELDS:
        a, b = getattr(model, f), getattr(ref, f)
        if a.shape != b.shape or not np.array_equal(a, b):
            nbad = -1 if a.shape != b.shape else int((a != b).sum())
            bad.append((f, a.shape, b.shape, nbad))
    print(f"[vox {name}] S={ref.segment_count} dropped={ref.dropped_overflow}/{model.dropped_overflow} "
          f"oracle {t1-t0:.2f}s gpu(e2e) {t2-t1:.3f}s  {'OK' if not bad else 'MISMATCH ' + str(bad)}", flush=True)
    return model, ref


def lod_case(name, model, ref):
    oc = lv.build_lod(model)
    ref_levels = orc.build_octree(orc.compute_density_level0(ref))
    ok = all(np.array_equal(a, b) for a, b in zip(oc.levels, ref_levels)) and len(oc.levels) == len(ref_levels)
    print(f"[lod {name}] levels={len(ref_levels)} {'OK' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        for l, (a, b) in enumerate(zip(oc.levels, ref_levels)):
            print("   level", l, int((a != b).sum()), "of", a.size)
    return oc, ref_levels


def render_case(name, dims, W, H, model, ref, oc, ref_levels, **kw):
    cam = lv.default_camera(dims, W, H)
    p = dict(kw)
    neighbor = p.pop("neighbor", True)
    params = lv.RenderParams(neighbor_mode="on" if neighbor else "off", **p)
    fr = lv.render_frame(cam, model, oc, None, params)
    fr = lv.render_frame(cam, model, oc, None, params)
    t0 = time.time()
    okw = dict(kw)
    okw.pop("neighbor", None)
    if "ao_rays" in okw:
        pass
    img, st = orc.render(orc.default_camera(dims, W, H), ref, ref_levels, neighbor=neighbor, **okw)
    t1 = time.time()
    err = np.abs(fr.image.astype(np.float64) - img.astype(np.float64))
    same = np.array_equal(fr.image, img)
    cnt_ok = all(fr.stats[k] == st[k] for k in ("voxel_steps", "intersection_tests", "window_overflow"))
    print(f"[render {name}] {W}x{H} gpu {fr.stats['ms']:.3f} ms oracle {1e3*(t1-t0):.0f} ms "
          f"max_err {err.max():.3e} mean {err.mean():.3e} bitwise={same} nbad={(err>0).sum()} "
          f"stats {'OK' if cnt_ok else 'MISMATCH %s vs %s' % (fr.stats, st)}", flush=True)


def main():
    print(torch.cuda.get_device_name(0), "oracle threads", orc.num_threads(), flush=True)
    cases = [
        ("helices1k@64", synth.helices(1000, 100, (64, 64, 64)), (64, 64, 64)),
        ("turb2k@64", synth.turbulence(2000, 100, (64, 64, 64)), (64, 64, 64)),
        ("wiggle@24x20x16", synth.wiggles(300, 40, (24, 20, 16)), (24, 20, 16)),
        ("lattice@12x10x8", synth.lattice_adversarial(3000, 12, (12, 10, 8)), (12, 10, 8)),
        ("cap255@4", synth.helices(600, 30, (4, 4, 4), seed=3), (4, 4, 4)),
    ]
    built = {}
    for name, gen, dims in cases:
        try:
            built[name] = vox_case(name, gen, dims) + (dims,)
        except Exception:
            traceback.print_exc()
    for nb in (4, 8, 64, 128, 256):
        try:
            vox_case(f"turb500@32 N={nb}", synth.turbulence(500, 60, (32, 32, 32)), (32, 32, 32), nb)
        except Exception:
            traceback.print_exc()
    lods = {}
    for name, (model, ref, dims) in built.items():
        try:
            lods[name] = lod_case(name, model, ref)
        except Exception:
            traceback.print_exc()
    # AO bake
    for name in ("helices1k@64", "wiggle@24x20x16"):
        try:
            model, ref, dims = built[name]
            oc, ref_levels = lods[name]
            ao = lv.precompute_voxel_ao(model, oc)
            torch.cuda.synchronize()
            t0 = time.time()
            ref_ao = orc.precompute_voxel_ao(ref, ref_levels, 100, 5.0, 1.0)
            t1 = time.time()
            d = np.abs(ao.values.astype(np.float64) - ref_ao)
            print(f"[ao {name}] oracle {t1-t0:.2f}s bitwise={np.array_equal(ao.values, ref_ao)} max {d.max():.3e}", flush=True)
            model.ao = ao
            ref.ao = ref_ao
        except Exception:
            traceback.print_exc()
    name = "helices1k@64"
    model, ref, dims = built[name]
    oc, ref_levels = lods[name]
    rc = [
        ("opaque nb", dict()),
        ("opaque own", dict(neighbor=False)),
        ("a.25 nb", dict(base_opacity=0.25)),
        ("a.25 own nojoint", dict(base_opacity=0.25, neighbor=False, joint_spheres=False)),
        ("a.25 nb pre-AO cone", dict(base_opacity=0.25, ao_mode="precomputed", shadow_mode="cone", light_dir=(0.3, 0.2, 1.0))),
        ("a.25 own densAO", dict(base_opacity=0.25, neighbor=False, ao_mode="density-rays")),
        ("a.05 tau1 nb", dict(base_opacity=0.05, tau=1.0)),
        ("dist-scaled", dict(base_opacity=0.3, opacity_mode="distance-scaled")),
    ]
    for nm, kw in rc:
        try:
            render_case(nm, dims, 256, 256, model, ref, oc, ref_levels, **kw)
        except Exception:
            traceback.print_exc()
    try:
        m2, r2, d2 = built["wiggle@24x20x16"]
        o2, l2 = lods["wiggle@24x20x16"]
        render_case("wiggle a.3 nb AO", d2, 160, 120, m2, r2, o2, l2, base_opacity=0.3, ao_mode="precomputed")
        m3, r3, d3 = built["cap255@4"]
        o3, l3 = lods["cap255@4"]
        render_case("cap255 a.1 tau1 nb (overflow)", d3, 96, 64, m3, r3, o3, l3, base_opacity=0.02, tau=1.0)
    except Exception:
        traceback.print_exc()


if __name__ == "__main__":
    main()
