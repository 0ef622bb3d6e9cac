import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box with -m gpu)")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


MODEL_FIELDS = ["counts", "offsets", "packed", "seg_voxel", "seg_a", "seg_b", "seg_attr", "seg_lid",
                "seg_face_in", "seg_bin_in", "seg_face_out", "seg_bin_out", "seg_curve", "seg_order"]

VOX_CASES = ["helices", "turbulence", "wiggles", "lattice", "cap255", "bins4", "bins128", "bins256"]

RENDER_CASES = ["opaque_nb", "opaque_own", "alpha25_nb", "alpha25_own_nojoints", "alpha25_nb_ao_cone",
                "alpha25_own_densao", "alpha05_tau1_nb", "distance_scaled", "transfer_light",
                "cap255_overflow",
                # geometry secondary rays: hard shadows, hemisphere-geometry AO
                "geom_hard_nb", "geom_hard_own_nojoints", "geom_hemi_nb", "geom_hard_hemi"]

# frames with shadow_mode="replines" (they also need the representative-line field)
REP_RENDER_CASES = ["rep_frame_helices", "rep_frame_turbulence"]

# frames of the reference's brute-force renderer (metrics.brute_force_render)
BRUTE_RENDER_CASES = ["brute_opaque", "brute_alpha_cone_ao", "brute_alpha_nojoints", "brute_hard"]


def render_kwargs(g):
    """The RenderParams kwargs a render fixture was made with."""
    import ast
    return ast.literal_eval(str(g["params"]))


@pytest.fixture(scope="session")
def oracle():
    from oracle import lvx_oracle
    lvx_oracle.build()
    return lvx_oracle


def assert_model_equal(got, want, fields=MODEL_FIELDS):
    for f in fields:
        a, b = np.asarray(getattr(got, f) if not isinstance(got, dict) else got[f]), np.asarray(want[f])
        assert a.shape == b.shape, f"{f}: shape {a.shape} vs {b.shape}"
        assert a.dtype == b.dtype, f"{f}: dtype {a.dtype} vs {b.dtype}"
        assert np.array_equal(a, b), f"{f}: {int((a != b).sum())} of {a.size} entries differ"
