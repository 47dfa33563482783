"""CPU restatement of the evaluation metrics (evalio module).

TEST INFRASTRUCTURE ONLY: imported by tests/ as the checker of the CUDA
metrics (csrc/k_eval.cu, tfg_psnr / tfg_ssim / tfg_depth_mae /
tfg_edge_band_mask).  The reference ships no evalio implementation (SPEC
module only), so this follows the SPEC text, pinned where it is silent:

- psnr: 10 log10(1 / MSE) over all channels, capped at 99 dB.
- ssim: grey = channel mean, 11x11 Gaussian window sigma 1.5
  (normalised weights), K1 0.01, K2 0.03, L 1; mean of the local SSIM over
  the 'valid' windows (windows fully inside the image, as in Wang et al.
  2004's reference implementation).  Parity of this restatement is checked
  against an independent scipy.ndimage formulation in tests/test_eval.py.
- depth_mae: mean |d1 - d2| over the mask; empty mask is an
  error.
- edge_band_mask ("±B px of projected tile edges"): the grid's
  boundary lines (x = east[k] for every k, y = north[k] for every k), at
  z_min and at z_max, sampled every `step` metres from the ROI's low corner;
  each sample projected with the RPC model and a (2B+1)^2 square around
  floor(row), floor(col) set.  step = max(gsd / 8, extent / 1e6), gsd =
  |long_scale| / max(1, |samp_scale|).
"""
from __future__ import annotations

import numpy as np


def psnr(a: np.ndarray, b: np.ndarray) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape or a.size == 0:
        raise ValueError("psnr: shape mismatch or empty")
    mse = float(np.mean((a - b) ** 2))
    return 99.0 if mse == 0.0 else min(99.0, 10.0 * np.log10(1.0 / mse))


def gaussian11() -> np.ndarray:
    x = np.arange(11, dtype=np.float64) - 5.0
    g = np.exp(-(x * x) / (2.0 * 1.5 * 1.5))
    return g / g.sum()


def _valid_sep(img: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Separable 'valid' correlation with an 11-tap kernel (rows, then columns)."""
    H, W = img.shape
    h = sum(w[k] * img[:, k:W - 10 + k] for k in range(11))
    return sum(w[k] * h[k:H - 10 + k, :] for k in range(11))


def ssim(a: np.ndarray, b: np.ndarray) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape or a.ndim != 3 or a.shape[0] < 11 or a.shape[1] < 11:
        raise ValueError("ssim: images smaller than the 11x11 window or shape mismatch")
    x = a.mean(axis=2)
    y = b.mean(axis=2)
    w = gaussian11()
    mx, my = _valid_sep(x, w), _valid_sep(y, w)
    xx, yy, xy = _valid_sep(x * x, w), _valid_sep(y * y, w), _valid_sep(x * y, w)
    sx, sy, sxy = xx - mx * mx, yy - my * my, xy - mx * my
    C1, C2 = 0.01 ** 2, 0.03 ** 2
    m = ((2 * mx * my + C1) * (2 * sxy + C2)) / ((mx * mx + my * my + C1) * (sx + sy + C2))
    return float(m.mean())


def depth_mae(d1: np.ndarray, d2: np.ndarray, mask: np.ndarray | None = None) -> float:
    d1 = np.asarray(d1, np.float64)
    d2 = np.asarray(d2, np.float64)
    if d1.shape != d2.shape:
        raise ValueError("depth_mae: shape mismatch")
    m = np.ones(d1.shape, bool) if mask is None else np.asarray(mask).astype(bool)
    if not m.any():
        raise ValueError("depth_mae: empty mask")
    return float(np.abs(d1 - d2)[m].mean())


def edge_band_mask(oracle, cam, roi, east: np.ndarray, north: np.ndarray, band: int) -> np.ndarray:
    """`oracle` is oracle.pyoracle.Oracle (its FP64 RPC projection)."""
    ext = max(roi.easting_max - roi.easting_min, roi.northing_max - roi.northing_min)
    gsd = abs(cam.long_scale) / max(1.0, abs(cam.samp_scale))
    step = max(gsd / 8.0, ext / 1.0e6)
    per_line = int(ext / step) + 2
    k = np.arange(per_line, dtype=np.float64)
    pts = []
    for z in (roi.z_min, roi.z_max):
        for xe in east:
            y = north[0] + k * step
            y = y[y <= north[-1]]
            pts.append(np.stack([np.full_like(y, xe), y, np.full_like(y, z)], 1))
        for yn in north:
            x = east[0] + k * step
            x = x[x <= east[-1]]
            pts.append(np.stack([x, np.full_like(x, yn), np.full_like(x, z)], 1))
    pts = np.concatenate(pts)
    mask = np.zeros((cam.image_rows, cam.image_cols), np.uint8)
    for p in pts:
        rc = oracle.project(cam, p)
        if rc is None:
            continue
        r, c = int(np.floor(rc[0])), int(np.floor(rc[1]))
        r0, r1 = max(0, r - band), min(cam.image_rows, r + band + 1)
        c0, c1 = max(0, c - band), min(cam.image_cols, c + band + 1)
        if r0 < r1 and c0 < c1:
            mask[r0:r1, c0:c1] = 1
    return mask
