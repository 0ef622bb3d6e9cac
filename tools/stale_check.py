"""A frame on a large grid followed by tiny frames on a small one, in one process (developer tool; run under
compute-sanitizer): stale queue / scratch contents of the first must not be used as addresses by the second."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_1801_01155_b200 as lv
from paper_1801_01155_b200 import synth
big = (96, 96, 96)
mb = lv.build_voxel_model(lv.CurveSet.from_flat(*synth.turbulence(3000, 60, big)), lv.GridSpec(big))
for nb in ("on", "off"):
    lv.render_frame(lv.default_camera(big, 320, 200), mb, None, None, lv.RenderParams(base_opacity=0.3, neighbor_mode=nb))
small = (10, 9, 7)
ms = lv.build_voxel_model(lv.CurveSet.from_flat(*synth.wiggles(120, 30, small)), lv.GridSpec(small))
for (W, H) in ((1, 1), (7, 5), (37, 21), (130, 3)):
    for nb in ("on", "off"):
        fr = lv.render_frame(lv.default_camera(small, W, H), ms, None, None, lv.RenderParams(base_opacity=0.5, neighbor_mode=nb))
        assert np.isfinite(fr.image).all()
print("OK")
