"""Crop cache (build_crop_cache):
per-(view, tile) crops from crop_for_tile (camera.cpp:126-146) + an index, in
the format documented in include/tilefield_gpu.h.  The rects are checked
against the oracle's crop_for_tile (itself pinned to the reference sources),
the file is parsed independently, and a context fed ONLY from the cache trains
on bit-identical accepted lists and batches."""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2507_01631_b200 import synth
from paper_2507_01631_b200.abi import FieldConfig, TrainConfig


def _need_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _parse(path):
    raw = open(path, "rb").read()
    assert raw[:8] == b"TFCROP01"
    ver, nv, gr, gc, margin, _ = np.frombuffer(raw, np.uint32, 6, 8)
    n, data_off = np.frombuffer(raw, np.uint64, 2, 32)
    ent = np.frombuffer(raw, np.int32, int(n) * 12, 48).reshape(int(n), 12)
    offs = ent[:, 8:12].copy().view(np.uint64).reshape(int(n), 2)
    return dict(version=int(ver), n_views=int(nv), rows=int(gr), cols=int(gc), margin=int(margin),
                entries=ent[:, :7], offsets=offs, data=raw[int(data_off):])


def test_crop_cache_format_and_rects(tmp_path):
    _need_gpu()
    from oracle.pyoracle import Oracle
    from paper_2507_01631_b200.tilefield import Context

    scene = synth.make_scene(3, 3, tile_side=96.0, n_views=3, gsd=1.0, seed=31, max_off_nadir=30.0)
    tc = TrainConfig.defaults(batch_rays=1024, seed=2)
    ctx = Context(scene, FieldConfig.defaults(), tc, max_rays=1024)
    path = str(tmp_path / "crops.bin")
    total = ctx.build_crop_cache(path)
    h = _parse(path)
    assert (h["version"], h["n_views"], h["rows"], h["cols"], h["margin"]) == (1, 3, 3, 3, tc.margin_px)
    o = Oracle()
    e, n = o.grid_edges(scene.roi, 3, 3)
    k = 0
    covered = 0
    for v in range(3):
        img = scene.images[v]
        for r in range(3):
            for c in range(3):
                box = [e[c], n[r], scene.roi.z_min, e[c + 1], n[r + 1], scene.roi.z_max]
                ref = o.crop_for_tile(scene.cams[v], box, tc.margin_px)
                ent = h["entries"][k]
                assert tuple(ent[:3]) == (v, r, c)
                if ref is None or ref[0] >= ref[1] or ref[2] >= ref[3]:
                    assert tuple(ent[3:7]) == (0, 0, 0, 0) and h["offsets"][k][1] == 0
                else:
                    assert tuple(int(x) for x in ent[3:7]) == ref
                    assert ctx.crop_rect(v, r, c) == ref
                    off, nb = (int(x) for x in h["offsets"][k])
                    r0, r1, c0, c1 = ref
                    crop = np.frombuffer(h["data"], np.uint8, nb, off).reshape(r1 - r0, c1 - c0, 3)
                    np.testing.assert_array_equal(crop, img[r0:r1, c0:c1])
                    covered += nb
                k += 1
    assert total == covered == len(h["data"])


def test_training_from_crop_cache_is_bit_identical(tmp_path):
    """Downstream training reads only crops: a context built
    without images + load_crop_cache gives the same accepted lists, targets
    and batches along the snake; every accepted pixel lies in a crop of its
    window."""
    _need_gpu()
    from paper_2507_01631_b200.synth import Scene
    from paper_2507_01631_b200.tilefield import Context, TileFieldError, snake_path

    scene = synth.make_scene(3, 3, tile_side=96.0, n_views=3, gsd=1.0, seed=32, max_off_nadir=30.0)
    fc, tc = FieldConfig.defaults(), TrainConfig.defaults(batch_rays=2048, seed=3)
    full = Context(scene, fc, tc, max_rays=2048)
    path = str(tmp_path / "crops.bin")
    full.build_crop_cache(path)
    bare = Scene(scene.roi, scene.grid_rows, scene.grid_cols, scene.cams, None, scene.gsd)
    cached = Context(bare, fc, tc, max_rays=2048)
    cached.load_crop_cache(path)
    for it, pos in enumerate(snake_path(3, 3)):
        full.set_window(*pos)
        cached.set_window(*pos)
        acc = full.accept_list()
        np.testing.assert_array_equal(acc, cached.accept_list())
        # every accepted pixel is inside a crop of one of its window's tiles
        v = (acc >> 40).astype(int)
        row = ((acc >> 20) & 0xFFFFF).astype(int)
        col = (acc & 0xFFFFF).astype(int)
        inside = np.zeros(acc.size, bool)
        for (tr, tcol) in full.window_tiles():
            for view in range(scene.n_views):
                rc = full.crop_rect(view, tr, tcol)
                if rc is None:
                    continue
                r0, r1, c0, c1 = rc
                inside |= (v == view) & (row >= r0) & (row < r1) & (col >= c0) & (col < c1)
        assert inside.all()
        full.sample(it, 0, 2048, True)
        cached.sample(it, 0, 2048, True)
        a, b = full.batch(), cached.batch()
        for f in ("target", "origin", "direction"):
            np.testing.assert_array_equal(a["rays"][f], b["rays"][f])
        np.testing.assert_array_equal(a["t"], b["t"])
    # a cache of another grid is rejected
    other = synth.make_scene(2, 2, tile_side=96.0, n_views=3, gsd=1.0, seed=32, max_off_nadir=30.0)
    ctx2 = Context(Scene(other.roi, 2, 2, other.cams, None, other.gsd), fc, tc, max_rays=256)
    with pytest.raises(TileFieldError, match="differ"):
        ctx2.load_crop_cache(path)


def test_crop_overlap_matches_parallax_band(tmp_path):
    """4x4 grid, oblique views: adjacent tiles' crops overlap by about
    2 x margin + the parallax band (z_max - z_min) tan(off-nadir) / GSD
    (SPEC.md:615), within a few pixels."""
    _need_gpu()
    from paper_2507_01631_b200.tilefield import Context

    scene = synth.make_scene(4, 4, tile_side=64.0, n_views=4, gsd=0.5, seed=33, max_off_nadir=30.0)
    tc = TrainConfig.defaults(batch_rays=256, seed=1)
    ctx = Context(scene, FieldConfig.defaults(), tc, max_rays=256)
    checked = 0
    for v in range(scene.n_views):
        a = ctx.crop_rect(v, 1, 1)
        b = ctx.crop_rect(v, 1, 2)  # east neighbour
        if a is None or b is None:
            continue
        overlap_cols = min(a[3], b[3]) - max(a[2], b[2])
        assert overlap_cols >= 2 * tc.margin_px  # at least the two margins
        assert overlap_cols <= 2 * tc.margin_px + (scene.roi.z_max - scene.roi.z_min) / scene.gsd + 4
        checked += 1
    assert checked >= 2
