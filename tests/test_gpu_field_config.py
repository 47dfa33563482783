"""Non-default hash-grid geometry (FieldConfig n_min / n_max / table_size,
nn.hpp:14-45) on B200.

The default level layout is folded into the hash kernels as constants; any
other layout runs their runtime-layout instantiations (HashLayout::generic,
csrc/tf_hash.cuh hash_level_rt).  Two checks:
  * on the default config the runtime-layout kernels (forced with
    TFG_GENERIC_HASH=1) reproduce the folded ones: the gather bit for bit,
    the gradients up to fp32 atomic order (the runtime scatter has no lane
    butterfly, so its sums associate differently);
  * on other geometries (a smaller and a larger table, other resolutions)
    the GPU matches the oracle, which follows nn.hpp for any FieldConfig,
    within the same stated tolerances as the default (test_gpu_parity.py),
    and trains: three steps' losses agree.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2507_01631_b200 import synth
from paper_2507_01631_b200.abi import FieldConfig, TrainConfig, field_sizes

from tests.test_gpu_parity import (TOL_DEPTH_ATOL, TOL_GRAD_REL, TOL_LOSS_RTOL, TOL_RAY_RGB_ATOL, TOL_RGB_ATOL,
                             TOL_SIGMA_RTOL)

N_RAYS = 2048


def _scene():
    return synth.make_scene(3, 3, tile_side=128.0, n_views=4, gsd=1.0, seed=21)


def _perturbed(state, rng):
    st = dict(state)
    st["enc"] = (st["enc"] + rng.normal(0, 0.5, st["enc"].shape)).astype(np.float32)
    st["dnet"] = (st["dnet"] * 1.5).astype(np.float32)
    return st


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _context(scene, fc, tc, generic=False):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_01631_b200.tilefield import Context

    if generic:
        os.environ["TFG_GENERIC_HASH"] = "1"
    try:
        return Context(scene, fc, tc, max_rays=N_RAYS)
    finally:
        os.environ.pop("TFG_GENERIC_HASH", None)


def test_runtime_layout_matches_folded_on_default():
    scene = _scene()
    fc, tc = FieldConfig.defaults(), TrainConfig.defaults(batch_rays=N_RAYS, seed=5)
    a = _context(scene, fc, tc)
    b = _context(scene, fc, tc, generic=True)
    rng = np.random.default_rng(1)
    for ctx in (a, b):
        ctx.set_window(1, 1)
    for k in range(4):
        st = _perturbed(a.tile_state(k), rng)
        a.set_tile_state(k, st)
        b.set_tile_state(k, st)
    for ctx in (a, b):
        ctx.sample(2, 0, N_RAYS, True)
    sa, ra = a.field_forward()
    sb, rb = b.field_forward()
    np.testing.assert_array_equal(sa, sb)
    np.testing.assert_array_equal(ra, rb)
    ca, cb = a.composite(), b.composite()
    np.testing.assert_array_equal(ca["d_sigma"], cb["d_sigma"])
    a.field_backward()
    b.field_backward()
    for k in range(4):
        for name, x, y in zip(("enc", "dnet", "color"), a.grads(k), b.grads(k)):
            assert _rel(x, y) < 1e-5, (k, name, _rel(x, y))
    # and the occupancy probes (K6, CUDA cores) gather the same way
    a.update_occupancy()
    b.update_occupancy()
    for k in range(4):
        np.testing.assert_array_equal(a.tile_state(k)["occupancy"], b.tile_state(k)["occupancy"])


GEOMETRIES = {
    "T2^14_n8-512": dict(table_size=1 << 14, n_min=8, n_max=512),
    "T2^17_n16-1024": dict(table_size=1 << 17, n_min=16, n_max=1024),
}


@pytest.mark.parametrize("geom", sorted(GEOMETRIES))
def test_geometry_vs_oracle(geom):
    from oracle.pyoracle import Oracle, Session

    fc = FieldConfig.defaults()
    for k, v in GEOMETRIES[geom].items():
        setattr(fc, k, v)
    assert field_sizes(fc)[0] != field_sizes(FieldConfig.defaults())[0]
    scene = _scene()
    tc = TrainConfig.defaults(batch_rays=N_RAYS, seed=5)
    ctx = _context(scene, fc, tc)
    ses = Session(Oracle(), scene, fc, tc, workers=8)
    ctx.set_window(1, 1)
    ses.set_window(1, 1)
    ses.build_accept()
    # fresh tiles are the reference's own init for this geometry
    for k in range(4):
        ga, gb = ctx.tile_state(k), ses.tile_state(k)
        np.testing.assert_array_equal(ga["enc"], gb["enc"])
        np.testing.assert_array_equal(ga["dnet"], gb["dnet"])
    rng = np.random.default_rng(1)
    for k in range(4):
        st = _perturbed(ses.tile_state(k), rng)
        ses.set_tile_state(k, st)
        ctx.set_tile_state(k, st)
    p, m, v, s = ses.color()
    ctx.set_color(p, m, v, s)
    assert ctx.sample(2, 0, N_RAYS, True) == ses.sample(2, 0, N_RAYS, True)
    sg, rgb = ctx.field_forward()
    sr, rr = ses.forward()
    np.testing.assert_allclose(sg, sr, rtol=TOL_SIGMA_RTOL, atol=1e-6)
    np.testing.assert_allclose(rgb, rr, atol=TOL_RGB_ATOL)
    cg, cr = ctx.composite(), ses.composite()
    np.testing.assert_allclose(cg["rgb"], cr["rgb"], atol=TOL_RAY_RGB_ATOL)
    np.testing.assert_allclose(cg["depth"], cr["depth"], atol=TOL_DEPTH_ATOL)
    assert abs(cg["loss"] - cr["loss"]) <= TOL_LOSS_RTOL * abs(cr["loss"])
    ctx.field_backward()
    ses.backward()
    for k in range(4):
        for name, x, y in zip(("enc", "dnet", "color"), ctx.grads(k), ses.grads(k)):
            assert _rel(x, y) < TOL_GRAD_REL[name], (geom, k, name, _rel(x, y))
    for it in range(3):
        lg = ctx.train_step(100 + it, 0, N_RAYS)
        lr = ses.train_step(100 + it, 0, N_RAYS)
        assert abs(lg - lr) <= 1e-2 * abs(lr), (geom, it, lg, lr)
    # the render path (its own slots and fp16 shadows) on the oracle's tiles
    acc = ses.build_accept()
    sel = acc[:: max(1, acc.size // 1500)][:1500]
    px = np.stack([(sel >> 40).astype(np.int32), ((sel >> 20) & 0xFFFFF).astype(np.int32),
                   (sel & 0xFFFFF).astype(np.int32)], axis=1)
    v0 = px[px[:, 0] == 0]
    ses.sample_pixels(v0)
    ses.forward()
    ref = ses.composite()
    ctx.render_setup(ses.window_tiles(), [ses.tile_state(k) for k in range(4)], ses.color()[0])
    rgb, _, op = ctx.render_pixels(ctx.scene.cams[0], v0[:, 1:])
    np.testing.assert_allclose(rgb, ref["rgb"], atol=TOL_RAY_RGB_ATOL)
    np.testing.assert_allclose(op, ref["opacity"], atol=TOL_RAY_RGB_ATOL)


def test_geometry_operator_path():
    """The operator-level entry points (forward_batch / backward_batch over a
    caller-built batch: tfg_batch_import, tfg_field_backward_from) on a padded
    geometry: the oracle's own batch imports bit for bit, and the field
    backward fed the oracle's d_sigma / d_rgb matches the oracle's gradients
    within the default tolerances."""
    from oracle.pyoracle import Oracle, Session

    fc = FieldConfig.defaults()
    for k, v in GEOMETRIES["T2^17_n16-1024"].items():
        setattr(fc, k, v)
    scene = _scene()
    tc = TrainConfig.defaults(batch_rays=N_RAYS, seed=5)
    ctx = _context(scene, fc, tc)
    ses = Session(Oracle(), scene, fc, tc, workers=8)
    ctx.set_window(0, 1)
    ses.set_window(0, 1)
    ses.build_accept()
    rng = np.random.default_rng(3)
    for k in range(4):
        st = _perturbed(ses.tile_state(k), rng)
        ses.set_tile_state(k, st)
        ctx.set_tile_state(k, st)
    p, m, v, s = ses.color()
    ctx.set_color(p, m, v, s)
    ses.sample(7, 0, N_RAYS, True)
    b = ses.batch()
    assert ctx.batch_import(b) == b["offsets"][-1]
    got = ctx.batch()
    for f in ("offsets", "t", "delta", "local", "slot", "endpoint"):
        np.testing.assert_array_equal(got[f], b[f], err_msg=f)
    sr, rr = ses.forward()
    ref = ses.composite()
    sg, rgb = ctx.field_forward()
    np.testing.assert_allclose(sg, sr, rtol=TOL_SIGMA_RTOL, atol=1e-6)
    np.testing.assert_allclose(rgb, rr, atol=TOL_RGB_ATOL)
    ses.backward()
    ctx.field_backward_from(ref["d_sigma"], ref["d_rgb"])
    for k in range(4):
        for name, x, y in zip(("enc", "dnet", "color"), ctx.grads(k), ses.grads(k)):
            assert _rel(x, y) < TOL_GRAD_REL[name], (k, name, _rel(x, y))
