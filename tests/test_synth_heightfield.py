"""The heightfield fixture (synth.generate / oracle_render)
against its own known answers, and its exact depth against the rays the
oracle's pinned ray_from_pixel (camera.cpp:105-124) produces for the fitted
cameras."""
import numpy as np

from paper_2507_01631_b200 import synth
from paper_2507_01631_b200.abi import Roi


def test_flat_scene_nadir_constant_depth():
    roi = Roi(0, 128, 0, 128, 0, 40)
    cam = synth.make_camera(roi, 0.5, 0.0, 0.0, nonlinear=0.0)
    d, *_ = synth.trace(cam, 0.5, roi, [])
    assert np.all(d == 40.0)  # z_max plane to the ground, nadir


def test_box_nadir_rectangle_10m_shallower():
    roi = Roi(0, 128, 0, 128, 0, 40)
    cam = synth.make_camera(roi, 0.5, 0.0, 0.0, nonlinear=0.0)
    d, px, py, z, face = synth.trace(cam, 0.5, roi, [(32.0, 32.0, 64.0, 48.0, 10.0)])
    assert set(np.unique(d).tolist()) == {30.0, 40.0}
    top = d == 30.0
    # footprint = the box footprint in pixels (closed box: both edges included)
    assert np.all((px[top] >= 32) & (px[top] <= 64) & (py[top] >= 32) & (py[top] <= 48))
    assert top.sum() == 65 * 33 and np.all(face[top] == 1)


def test_depth_is_first_hit_along_the_camera_ray(oracle):
    scene = synth.make_heightfield_scene(2, 2, tile_side=64.0, n_views=3, gsd=1.0, seed=5)
    rng = np.random.default_rng(0)
    hits = 0
    for v, cam in enumerate(scene.cams):
        for _ in range(200):
            r, c = int(rng.integers(0, cam.image_rows)), int(rng.integers(0, cam.image_cols))
            ray = oracle.ray_from_pixel(cam, r, c, scene.roi.z_min, scene.roi.z_max)
            assert ray is not None
            o, d = ray
            dep = float(scene.depths[v][r, c])
            p = o + dep * d
            # the hit point lies on the ground or on a box face
            on_ground = abs(p[2] - scene.roi.z_min) < 1e-6
            on_box = any(b[0] - 1e-6 <= p[0] <= b[2] + 1e-6 and b[1] - 1e-6 <= p[1] <= b[3] + 1e-6
                         and p[2] <= b[4] + 1e-6 for b in scene.boxes)
            assert on_ground or on_box, (v, r, c, p)
            hits += on_box
            # nothing is hit earlier: points before the hit are above every box
            for s in np.linspace(0.0, dep, 25)[:-1]:
                q = o + s * d
                assert not any(b[0] < q[0] < b[2] and b[1] < q[1] < b[3] and q[2] < b[4] - 1e-6
                               for b in scene.boxes)
    assert hits > 20
