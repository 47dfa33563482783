"""O(1) HBM (PAPER.md:65 condition 2): the device
footprint of a context is set by the window (4 tiles, their crops and the
per-window pixel memo), not by the ROI.  memory_report().total_device is the
live sum of every device allocation of the context (dalloc/dfree)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2507_01631_b200 import synth
from paper_2507_01631_b200.abi import FieldConfig, TrainConfig


def _need_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_memory_independent_of_grid_size():
    """memory_report within 10% across 2x2, 3x3 and 4x4 grids
    (same tile side, views and GSD), measured after a full snake."""
    _need_gpu()
    from paper_2507_01631_b200.tilefield import Context, snake_path

    totals = {}
    for g in (2, 3, 4):
        scene = synth.make_scene(g, g, tile_side=128.0, n_views=4, gsd=0.5, seed=7)
        ctx = Context(scene, FieldConfig.defaults(), TrainConfig.defaults(batch_rays=4096, seed=2), max_rays=4096)
        seen = []
        for it, pos in enumerate(snake_path(g, g)):
            ctx.set_window(*pos)
            ctx.train_step(it, 0, 4096)
            seen.append(ctx.memory_report()["total_device"])
        # constant along the snake, and every byte is accounted for
        assert len(set(seen)) == 1, seen
        rep = ctx.memory_report()
        parts = sum(v for k, v in rep.items() if k != "total_device")
        assert rep["total_device"] >= parts
        totals[g] = rep["total_device"]
        ctx.close()
    lo, hi = min(totals.values()), max(totals.values())
    assert (hi - lo) / lo < 0.10, totals


def test_set_scene_twice_does_not_inflate_report():
    """Re-running set_scene frees and re-allocates the scene buffers; the
    report tracks the live allocations (bytes_total was never
    reduced on free)."""
    _need_gpu()
    from paper_2507_01631_b200.tilefield import Context

    scene = synth.make_scene(3, 3, tile_side=128.0, n_views=2, gsd=1.0, seed=3)
    ctx = Context(scene, FieldConfig.defaults(), TrainConfig.defaults(batch_rays=1024), max_rays=1024)
    m0 = ctx.memory_report()["total_device"]
    for _ in range(3):
        ctx._set_scene(scene)
    assert ctx.memory_report()["total_device"] == m0
    ctx.set_window(0, 0)
    ctx.train_step(0, 0, 1024)
