"""Synthetic overhead scenes (host-side fixture generator).

The reference's synth module is absent upstream and out of
scope as a product; this is the minimal stand-in the parity tests and the
benchmark need: an ROI tiled H x W, N views with rational (RPC00B-style)
cameras of a given off-nadir angle / azimuth, and 8-bit RGB views.

Camera: a parallel projection along the view direction (off-nadir theta,
azimuth phi) of the ground point at z = 0, written in RPC normalised
coordinates (camera.hpp:11-21) with small cubic and denominator terms so the
rational path of project()/localize() is exercised.  Images: a procedural
albedo of the z = 0 intersection (flat textured ground) - cheap enough to
generate 16 x 1536^2 views for the benchmark.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

from .abi import Roi, Rpc


@dataclasses.dataclass
class Scene:
    roi: Roi
    grid_rows: int
    grid_cols: int
    cams: list
    images: list  # uint8 (rows, cols, 3), row-major from the top row
    gsd: float
    depths: list | None = None  # heightfield scenes: exact depth along each pixel's ray (m from z_max)
    boxes: list | None = None   # heightfield scenes: (x0, y0, x1, y1, height) buildings

    @property
    def n_views(self) -> int:
        return len(self.cams)


def make_camera(
    roi: Roi, gsd: float, off_nadir_deg: float, azimuth_deg: float, nonlinear: float = 2e-4,
    pad_px: int = 8,
) -> Rpc:
    th = math.radians(off_nadir_deg)
    ph = math.radians(azimuth_deg)
    tx, ty = math.tan(th) * math.cos(ph), math.tan(th) * math.sin(ph)
    cam = Rpc()
    cam.long_off = 0.5 * (roi.easting_min + roi.easting_max)
    cam.lat_off = 0.5 * (roi.northing_min + roi.northing_max)
    cam.height_off = 0.5 * (roi.z_min + roi.z_max)
    cam.long_scale = 0.55 * (roi.easting_max - roi.easting_min)
    cam.lat_scale = 0.55 * (roi.northing_max - roi.northing_min)
    cam.height_scale = 0.6 * (roi.z_max - roi.z_min)
    # ground footprint of the ROI box in the z=0 plane, projected along the view
    xs, ys = [], []
    for x in (roi.easting_min, roi.easting_max):
        for y in (roi.northing_min, roi.northing_max):
            for z in (roi.z_min, roi.z_max):
                xs.append(x + z * tx)
                ys.append(y + z * ty)
    x0 = min(xs) - pad_px * gsd
    y0 = max(ys) + pad_px * gsd  # image top = north
    cols = int(math.ceil((max(xs) - min(xs)) / gsd)) + 2 * pad_px
    rows = int(math.ceil((max(ys) - min(ys)) / gsd)) + 2 * pad_px
    cam.samp_scale = cam.long_scale / gsd
    cam.samp_off = (cam.long_off + cam.height_off * tx - x0) / gsd
    cam.line_scale = cam.lat_scale / gsd
    cam.line_off = (y0 - cam.lat_off - cam.height_off * ty) / gsd
    # col = samp_off + samp_scale * (L + kx H + ...), row = line_off + line_scale * (-P - ky H + ...)
    cam.samp_num[1] = 1.0
    cam.samp_num[3] = cam.height_scale * tx / cam.long_scale
    cam.line_num[2] = -1.0
    cam.line_num[3] = -cam.height_scale * ty / cam.lat_scale
    cam.samp_den[0] = 1.0
    cam.line_den[0] = 1.0
    if nonlinear:
        cam.samp_num[4] = nonlinear  # L*P
        cam.samp_num[11] = 0.5 * nonlinear  # L^3
        cam.line_num[7] = -nonlinear  # L^2
        cam.line_num[18] = 0.5 * nonlinear  # P^2 H
        cam.samp_den[2] = 0.25 * nonlinear  # P
        cam.line_den[1] = -0.25 * nonlinear  # L
    cam.image_rows = rows
    cam.image_cols = cols
    cam._x0, cam._y0, cam._tx, cam._ty = x0, y0, tx, ty  # analytic model (fixture only)
    return cam


def procedural_image(cam: Rpc, gsd: float, seed: int) -> np.ndarray:
    rows, cols = cam.image_rows, cam.image_cols
    r = np.arange(rows, dtype=np.float64)[:, None]
    c = np.arange(cols, dtype=np.float64)[None, :]
    x = cam._x0 + c * gsd
    y = cam._y0 - r * gsd
    rng = np.random.default_rng(seed)
    ph = rng.uniform(0, 2 * math.pi, size=6)
    red = 0.5 + 0.3 * np.sin(x / 9.0 + ph[0]) * np.cos(y / 13.0 + ph[1])
    grn = 0.5 + 0.3 * np.sin((x + y) / 17.0 + ph[2]) + 0.1 * np.cos(x / 3.1 + ph[3])
    blu = 0.45 + 0.25 * np.cos(y / 7.0 + ph[4]) * np.sin(x / 23.0 + ph[5])
    checker = ((np.floor(x / 16.0) + np.floor(y / 16.0)) % 2) * 0.15
    img = np.stack([red + checker, grn - checker, blu + 0.5 * checker], axis=-1)
    img = np.broadcast_to(img, (rows, cols, 3))
    return np.ascontiguousarray(np.clip(img * 255.0 + 0.5, 0, 255).astype(np.uint8))


def make_scene(
    grid_rows: int, grid_cols: int, tile_side: float = 128.0, z_extent: float = 40.0,
    n_views: int = 8, gsd: float = 0.5, seed: int = 0, max_off_nadir: float = 30.0,
) -> Scene:
    roi = Roi(0.0, grid_cols * tile_side, 0.0, grid_rows * tile_side, 0.0, z_extent)
    rng = np.random.default_rng(seed)
    cams, images = [], []
    for v in range(n_views):
        off = float(rng.uniform(0.0, max_off_nadir))
        az = float(rng.uniform(0.0, 360.0))
        cam = make_camera(roi, gsd, off, az)
        cams.append(cam)
        images.append(procedural_image(cam, gsd, seed * 1000 + v))
    return Scene(roi, grid_rows, grid_cols, cams, images, gsd)


# ---------------------------------------------------------------- heightfield
# SPEC.md:533-556 (synth.generate / oracle_render): flat ground plus box
# "buildings" with heights in (z_min, z_max], per-face procedural Lambertian
# albedo, a fixed sun, and exact ray-traced depth.  The cameras are the
# parallel projections of make_camera with no nonlinear terms, so a pixel's
# ray is known in closed form: p(z) = (X - z tx, Y - z ty, z) with
# X = x0 + col gsd, Y = y0 - row gsd (the RPC localises exactly onto it).
SUN = np.array([0.35, -0.25, 0.90]) / np.linalg.norm([0.35, -0.25, 0.90])


def make_boxes(roi: Roi, n_boxes: int, seed: int, min_side: float = 8.0, max_side: float = 40.0):
    rng = np.random.default_rng(seed + 7919)
    zt = roi.z_max - roi.z_min
    out = []
    for _ in range(n_boxes):
        w, h = rng.uniform(min_side, max_side, 2)
        x0 = rng.uniform(roi.easting_min, roi.easting_max - w)
        y0 = rng.uniform(roi.northing_min, roi.northing_max - h)
        out.append((x0, y0, x0 + w, y0 + h, roi.z_min + rng.uniform(0.15, 0.85) * zt))
    return out


def trace(cam: Rpc, gsd: float, roi: Roi, boxes, rows=None, cols=None):
    """Exact first hit of each pixel ray with the heightfield: returns depth
    (m along the ray from the z_max plane), hit point (x, y, z) and the hit
    face (0 ground, 1 box top, 2 box side along x, 3 box side along y)."""
    R, W = cam.image_rows, cam.image_cols
    r = np.arange(R, dtype=np.float64)[:, None] if rows is None else rows
    c = np.arange(W, dtype=np.float64)[None, :] if cols is None else cols
    X = cam._x0 + c * gsd + 0.0 * r
    Y = cam._y0 - r * gsd + 0.0 * c
    tx, ty = cam._tx, cam._ty
    zt, zb = roi.z_max, roi.z_min
    # ray parameter = height drop s = zt - z (>= 0); ground hit at s = zt - zb
    best = np.full(X.shape, zt - zb)
    face = np.zeros(X.shape, np.int8)
    ox, oy = X - zt * tx, Y - zt * ty  # ray point at z = zt; p(s) = (ox + s tx, oy + s ty, zt - s)
    for (bx0, by0, bx1, by1, hb) in boxes:
        top = np.full(X.shape, zt - hb)  # s where the ray enters the box's height range
        hi = np.full(X.shape, zt - zb)
        ent = []
        for o, d, a, b in ((ox, tx, bx0, bx1), (oy, ty, by0, by1)):
            if abs(d) < 1e-15:
                inside = (o >= a) & (o <= b)
                ent.append(np.where(inside, -np.inf, np.inf))
                continue
            s0, s1 = (a - o) / d, (b - o) / d
            ent.append(np.minimum(s0, s1))
            hi = np.minimum(hi, np.maximum(s0, s1))
        lo = np.maximum(top, np.maximum(ent[0], ent[1]))
        hit = (lo <= hi) & (lo < best)
        side = np.where(lo == top, 1, np.where(ent[0] >= ent[1], 2, 3))
        face = np.where(hit, side, face)
        best = np.where(hit, lo, best)
    z = zt - best
    px, py = ox + best * tx, oy + best * ty
    depth = best * np.sqrt(tx * tx + ty * ty + 1.0)
    return depth, px, py, z, face


def shade(px, py, z, face, seed: int, tx: float = 0.0, ty: float = 0.0):
    """Per-face procedural albedo x Lambertian sun (+ ambient), [0,1] RGB."""
    rng = np.random.default_rng(seed)
    ph = rng.uniform(0, 2 * math.pi, size=8)
    g = np.stack([0.45 + 0.2 * np.sin(px / 7.0 + ph[0]) * np.cos(py / 11.0 + ph[1]),
                  0.50 + 0.2 * np.sin((px + py) / 13.0 + ph[2]),
                  0.40 + 0.15 * np.cos(py / 5.0 + ph[3])], axis=-1)
    roof = np.stack([0.70 + 0.15 * np.sin(px / 3.0 + ph[4]), 0.35 + 0.1 * np.cos(py / 4.0 + ph[5]),
                     0.30 + 0.1 * np.sin((px - py) / 5.0)], axis=-1)
    wall = np.stack([0.55 + 0.2 * np.sin(z / 2.0 + ph[6]), 0.55 + 0.1 * np.cos(z / 3.0 + ph[7]),
                     0.60 + 0.0 * z], axis=-1)
    alb = np.where((face == 0)[..., None], g, np.where((face == 1)[..., None], roof, wall))
    n = np.zeros(px.shape + (3,))
    n[..., 2] = np.where((face == 0) | (face == 1), 1.0, 0.0)
    n[..., 0] = np.where(face == 2, -np.sign(tx), 0.0)  # the x face the ray enters
    n[..., 1] = np.where(face == 3, -np.sign(ty), 0.0)
    lam = np.clip((n * SUN).sum(-1), 0.0, 1.0)
    return np.clip(alb * (0.35 + 0.65 * lam)[..., None], 0.0, 1.0)


def make_heightfield_scene(grid_rows: int, grid_cols: int, tile_side: float = 128.0, z_extent: float = 40.0,
                           n_views: int = 4, gsd: float = 0.5, seed: int = 0, max_off_nadir: float = 30.0,
                           n_boxes: int | None = None) -> Scene:
    """SPEC.md:533-556 fixture: ground + boxes, exact ray-traced images and
    depth maps (Scene.depths), cameras with exact (affine) RPCs."""
    roi = Roi(0.0, grid_cols * tile_side, 0.0, grid_rows * tile_side, 0.0, z_extent)
    nb = n_boxes if n_boxes is not None else 6 * grid_rows * grid_cols
    boxes = make_boxes(roi, nb, seed)
    rng = np.random.default_rng(seed)
    cams, images, depths = [], [], []
    for v in range(n_views):
        off = float(rng.uniform(0.0, max_off_nadir))
        az = float(rng.uniform(0.0, 360.0))
        cam = make_camera(roi, gsd, off, az, nonlinear=0.0)
        depth, px, py, z, face = trace(cam, gsd, roi, boxes)
        img = shade(px, py, z, face, seed, cam._tx, cam._ty)
        cams.append(cam)
        images.append(np.ascontiguousarray(np.clip(img * 255.0 + 0.5, 0, 255).astype(np.uint8)))
        depths.append(depth.astype(np.float32))
    return Scene(roi, grid_rows, grid_cols, cams, images, gsd, depths=depths, boxes=boxes)


# Benchmark / parity configurations (BASELINE.json configs).
CONFIGS = {
    1: dict(grid=(1, 1), tile_side=128.0, views=4, gsd=0.5, batch=4096),
    2: dict(grid=(3, 3), tile_side=128.0, views=8, gsd=0.5, batch=16384),
    3: dict(grid=(8, 8), tile_side=128.0, views=16, gsd=0.5, batch=16384),
    4: dict(grid=(4, 4), tile_side=128.0, views=1, gsd=0.125, batch=1 << 20),
    5: dict(grid=(6, 6), tile_side=128.0, views=16, gsd=0.5, batch=65536),
}


def config_scene(cfg: int, seed: int = 0) -> Scene:
    c = CONFIGS[cfg]
    return make_scene(c["grid"][0], c["grid"][1], c["tile_side"], 40.0, c["views"], c["gsd"], seed)
