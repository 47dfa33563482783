"""The oracle's batch cmd_render (tfo_render_pixels, the CPU reference of the
render path and of bench.py's render baseline) is exactly the per-ray
composition of its pinned primitives: ray_from_pixel -> segments ->
sample_segments (midpoints) -> field point -> render."""
import numpy as np

from paper_2507_01631_b200.abi import FieldConfig, Roi
from paper_2507_01631_b200.synth import make_camera


def test_render_pixels_equals_per_ray_composition(oracle):
    o = oracle
    fc = FieldConfig.defaults()
    roi = Roi(0.0, 256.0, 0.0, 256.0, 0.0, 40.0)
    cam = make_camera(roi, 1.0, 21.0, 140.0)
    e, n = o.grid_edges(roi, 2, 2)
    tiles = [(r, c) for r in range(2) for c in range(2)]
    boxes = np.array([[e[c], n[r], 0, e[c + 1], n[r + 1], 40] for r, c in tiles])
    frames = np.array([[b[0], b[1], b[2], 1 / (b[3] - b[0]), 1 / (b[4] - b[1]), 1 / (b[5] - b[2])] for b in boxes])
    rng = np.random.default_rng(3)
    states = []
    for r, c in tiles:
        enc, dnet, occ = o.tile_create(fc, r, c, 4)
        enc = (enc + rng.normal(0, 0.4, enc.shape)).astype(np.float32)
        occ = np.where(rng.random(occ.shape) < 0.3, 0.0, 1.0).astype(np.float32)
        states.append(dict(enc=enc, dnet=dnet, occupancy=occ))
    color = o.color_create(fc, 4)
    px = np.stack([rng.integers(0, cam.image_rows, 64), rng.integers(0, cam.image_cols, 64)], 1).astype(np.int32)
    rgb, dep, op = o.render_pixels(fc, cam, roi, boxes, states, color, px, workers=3)
    for i, (row, col) in enumerate(px):
        ray = o.ray_from_pixel(cam, int(row), int(col), 0.0, 40.0)
        if ray is None:
            assert not np.any(rgb[i]) and dep[i] == 0 and op[i] == 0
            continue
        org, d = ray
        segs = o.segments(org, d, boxes)
        s = o.sample_ray(org, d, segs, frames, spm=63.0 / 40.0, occupancy=[st["occupancy"] for st in states])
        m = len(s["t"])
        sig, col_ = np.zeros(m, np.float32), np.zeros((m, 3), np.float32)
        for k in range(m):
            st = states[s["slot"][k]]
            sig[k], col_[k] = o.query_field(fc, st["enc"], st["dnet"], color, s["local"][k], d.astype(np.float32))
        r_rgb, r_dep, r_op, _, _ = o.render_ray(sig, col_, s["t"], s["delta"])
        assert rgb[i].tobytes() == r_rgb.tobytes()
        assert np.float32(dep[i]) == np.float32(r_dep) and np.float32(op[i]) == np.float32(r_op)
