"""Render end-to-end gap probe: wall of render_pixels on the config-4 view,
first call vs a second call (same process), and the device phase sum."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_01631_b200.abi import FieldConfig, Roi, TrainConfig  # noqa: E402
from paper_2507_01631_b200.synth import Scene, make_camera  # noqa: E402
from paper_2507_01631_b200.tilefield import Context, tile_init  # noqa: E402

roi = Roi(0.0, 512.0, 0.0, 512.0, 0.0, 40.0)
cam = make_camera(roi, 0.125, 12.0, 40.0)
img = np.zeros((cam.image_rows, cam.image_cols, 3), np.uint8)
scene = Scene(roi, 4, 4, [cam], [img], 0.125)
fc = FieldConfig.defaults()
chunk = 1 << 20
ctx = Context(scene, fc, TrainConfig.defaults(batch_rays=chunk), max_rays=chunk)
tiles = [(r, c) for r in range(4) for c in range(4)]
ctx.render_setup(tiles, [tile_init(fc, 1, r, c) for r, c in tiles], ctx.color()[0])
R, W = cam.image_rows, cam.image_cols
rr, cc = np.meshgrid(np.arange(R), np.arange(W), indexing="ij")
px = np.stack([rr.ravel(), cc.ravel()], axis=1).astype(np.int32)
ctx.render_pixels(cam, px[:chunk])
for k in range(3):
    ctx.profile_enable(True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.render_pixels(cam, px)
    wall = time.perf_counter() - t0
    prof = ctx.profile_read()
    dev = sum(prof[p][0] for p in ("sampler", "field_fwd", "composite"))
    print(f"call {k}: wall {wall * 1e3:.1f} ms, device phases {dev:.1f} ms, gap {wall * 1e3 - dev:.1f} ms")

# the same call into pre-touched output arrays (no page faults on the host side)
import ctypes as C  # noqa: E402

from paper_2507_01631_b200.tilefield import lib, ptr  # noqa: E402

n = px.shape[0]
rgb, dep, op = np.ones(3 * n, np.float32), np.ones(n, np.float32), np.ones(n, np.float32)
for k in range(2):
    ctx.profile_enable(True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc = lib().tfg_render_pixels(ctx.h, C.byref(cam), ptr(px), n, ptr(rgb), ptr(dep), ptr(op))
    wall = time.perf_counter() - t0
    prof = ctx.profile_read()
    dev = sum(prof[p][0] for p in ("sampler", "field_fwd", "composite"))
    print(f"pre-touched outputs {k}: rc {rc}, wall {wall * 1e3:.1f} ms, device phases {dev:.1f} ms, gap {wall * 1e3 - dev:.1f} ms")
