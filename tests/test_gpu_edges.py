"""Edge cases on B200 (SURVEY.md §4's strategy: empty and ragged inputs,
capacity limits, failures reported by name, recovery after an error)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2507_01631_b200 import synth
from paper_2507_01631_b200.abi import FieldConfig, TrainConfig


def _need_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _cmp(ga, gb):
    for f in ("origin", "direction", "target"):
        np.testing.assert_array_equal(ga["rays"][f], gb["rays"][f], err_msg=f)
    for f in ("offsets", "t", "delta", "local", "slot", "endpoint"):
        np.testing.assert_array_equal(ga[f], gb[f], err_msg=f)


def test_ragged_batch_sizes_bit_exact():
    """Batches of 1, 31, 33, 127, 129 and 1000 rays (not multiples of a warp
    or a 128-row tile) sample bit-exactly and train with a matching loss."""
    _need_gpu()
    from oracle.pyoracle import Oracle, Session
    from paper_2507_01631_b200.tilefield import Context

    scene = synth.make_scene(2, 2, tile_side=96.0, n_views=2, gsd=1.0, seed=41)
    fc, tc = FieldConfig.defaults(), TrainConfig.defaults(batch_rays=1000, seed=3)
    ctx = Context(scene, fc, tc, max_rays=1000)
    ses = Session(Oracle(), scene, fc, tc, workers=8)
    ctx.set_window(0, 0)
    ses.set_window(0, 0)
    ses.build_accept()
    for k, n in enumerate((1, 31, 33, 127, 129, 1000)):
        assert ctx.sample(k, 7 * k, n, True) == ses.sample(k, 7 * k, n, True)
        _cmp(ctx.batch(), ses.batch())
    lg, lr = ctx.train_step(9, 0, 129), ses.train_step(9, 0, 129)
    assert abs(lg - lr) <= 1e-2 * lr


def test_sample_capacity_overflow_is_reported_and_recoverable():
    """A batch whose samples exceed the context's capacity (128 x max_rays)
    raises by name; the context keeps working for a batch that fits."""
    _need_gpu()
    from paper_2507_01631_b200.tilefield import Context, TileFieldError

    scene = synth.make_scene(2, 2, tile_side=96.0, n_views=2, gsd=1.0, seed=42)
    tc = TrainConfig.defaults(batch_rays=256, seed=1)
    tc.samples_per_meter = 8.0  # ~320+ samples per ray > 128 per ray of capacity
    ctx = Context(scene, FieldConfig.defaults(), tc, max_rays=256)
    ctx.set_window(0, 0)
    with pytest.raises(TileFieldError, match="sample capacity"):
        ctx.train_step(0, 0, 256)
    # 64 rays x ~330 samples fit into 256 x 128
    loss = ctx.train_step(1, 0, 64)
    assert np.isfinite(loss) and loss > 0


def test_window_without_accepted_rays_is_reported():
    """A view that never sees the window gives an empty accepted list; the
    ray draw reports it instead of sampling garbage."""
    _need_gpu()
    from paper_2507_01631_b200.abi import Roi
    from paper_2507_01631_b200.synth import Scene, make_camera
    from paper_2507_01631_b200.tilefield import Context, TileFieldError

    roi = Roi(0.0, 256.0, 0.0, 256.0, 0.0, 40.0)
    far = Roi(2000.0, 2256.0, 2000.0, 2256.0, 0.0, 40.0)  # camera looking elsewhere
    cam = make_camera(far, 1.0, 5.0, 40.0)
    img = np.zeros((cam.image_rows, cam.image_cols, 3), np.uint8)
    ctx = Context(Scene(roi, 2, 2, [cam], [img], 1.0), FieldConfig.defaults(),
                  TrainConfig.defaults(batch_rays=128), max_rays=128)
    ctx.set_window(0, 0)
    assert ctx.accept_list().size == 0
    with pytest.raises(TileFieldError, match="accepted-ray list is empty|ray generation failed"):
        ctx.train_step(0, 0, 128)


def test_invalid_arguments_raise():
    _need_gpu()
    from paper_2507_01631_b200.tilefield import Context, TileFieldError

    scene = synth.make_scene(2, 2, tile_side=96.0, n_views=1, gsd=2.0, seed=43)
    ctx = Context(scene, FieldConfig.defaults(), TrainConfig.defaults(batch_rays=64), max_rays=64)
    with pytest.raises(TileFieldError, match="set_window"):
        ctx.train_step(0, 0, 64)  # no window yet
    ctx.set_window(0, 0)
    with pytest.raises(TileFieldError):
        ctx.sample(0, 0, 65, True)  # more rays than the context holds
    with pytest.raises(TileFieldError):
        ctx.set_window(5, 5)  # outside the grid
    assert np.isfinite(ctx.train_step(0, 0, 64))


def test_sample_cap_and_delta_cap_bit_exact():
    """A small per-ray sample cap (plan_intervals rescales every segment's
    interval count) and a short last-delta cap sample
    bit-exactly against the oracle, with and without jitter."""
    _need_gpu()
    from oracle.pyoracle import Oracle, Session
    from paper_2507_01631_b200.tilefield import Context

    scene = synth.make_scene(2, 2, tile_side=96.0, n_views=2, gsd=1.0, seed=44, max_off_nadir=30.0)
    fc, tc = FieldConfig.defaults(), TrainConfig.defaults(batch_rays=2048, seed=9)
    tc.max_samples_per_ray = 24
    tc.delta_cap = 0.75
    ctx = Context(scene, fc, tc, max_rays=2048)
    ses = Session(Oracle(), scene, fc, tc, workers=8)
    ctx.set_window(0, 0)
    ses.set_window(0, 0)
    ses.build_accept()
    for it, jitter in ((0, True), (1, False)):
        n = ctx.sample(it, 0, 2048, jitter)
        assert n == ses.sample(it, 0, 2048, jitter)
        b = ctx.batch()
        _cmp(b, ses.batch())
        per_ray = np.diff(b["offsets"])
        assert per_ray.max() <= 24
