"""CUDA path (libtilefield_gpu.so through its C-ABI) vs the CPU oracle on the
same synthetic scene and seeds.

Contract:
  * bit-exact: accepted-ray list, ray origin/direction/target, per-ray sample
    counts/offsets, t, delta, local, slot, endpoint (K1); Adam on identical
    gradients (K5); window-slide state round trips (K7).
  * toleranced (stated here): field outputs (K2), compositing + loss + its
    backward (K3), parameter gradients (K4), occupancy EMA (K6).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2507_01631_b200 import synth
from paper_2507_01631_b200.abi import FieldConfig, TrainConfig

# ---- stated tolerances of the field/compositor path vs the FP32 oracle.
# The field MLPs run on tcgen05 with bf16 operands and fp32 accumulation
# (measured on B200: sigma rel <= 0.7%, rgb <= 2e-3, gradients norm-relative
# colour 0.4%, density MLP ~2%, hash tables ~7%); compositing is fp32.
TOL_SIGMA_RTOL = 2e-2      # sigma = exp(raw): relative
TOL_RGB_ATOL = 5e-3        # sigmoid outputs
TOL_RAY_RGB_ATOL = 5e-3
TOL_DEPTH_ATOL = 5e-2      # meters
TOL_GRAD_REL = {"enc": 0.12, "dnet": 0.05, "color": 0.02}  # ||g - g_ref|| / ||g_ref||
TOL_LOSS_RTOL = 5e-3

N_RAYS = 2048


@pytest.fixture(scope="module")
def setup():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle.pyoracle import Oracle, Session
    from paper_2507_01631_b200.tilefield import Context

    scene = synth.make_scene(3, 3, tile_side=128.0, n_views=4, gsd=1.0, seed=21)
    fc = FieldConfig.defaults()
    tc = TrainConfig.defaults(batch_rays=N_RAYS, seed=5)
    ctx = Context(scene, fc, tc, max_rays=N_RAYS)
    ses = Session(Oracle(), scene, fc, tc, workers=8)
    return ctx, ses


def _same_window(ctx, ses, r, c):
    ctx.set_window(r, c)
    ses.set_window(r, c)
    assert ctx.window_tiles() == ses.window_tiles()


def test_accept_list_bit_exact(setup):
    ctx, ses = setup
    for pos in [(0, 0), (1, 1), (0, 1)]:
        _same_window(ctx, ses, *pos)
        a = ctx.accept_list()
        b = ses.build_accept()
        assert a.size > 1000
        np.testing.assert_array_equal(a, b)


def _cmp_batch(ga, gb):
    ra, rb = ga["rays"], gb["rays"]
    for f in ("origin", "direction", "target", "image_id", "row", "col"):
        np.testing.assert_array_equal(ra[f], rb[f], err_msg=f)
    np.testing.assert_array_equal(ga["offsets"], gb["offsets"])
    for f in ("t", "delta", "local", "slot", "endpoint"):
        np.testing.assert_array_equal(ga[f], gb[f], err_msg=f)


def test_sampler_bit_exact(setup):
    ctx, ses = setup
    _same_window(ctx, ses, 1, 0)
    ses.build_accept()
    for it, jitter in [(0, True), (7, True), (3, False)]:
        n_gpu = ctx.sample(it, 1000, N_RAYS, jitter)
        n_ref = ses.sample(it, 1000, N_RAYS, jitter)
        assert n_gpu == n_ref
        _cmp_batch(ctx.batch(), ses.batch())


def test_sampler_occupancy_bit_exact(setup):
    ctx, ses = setup
    _same_window(ctx, ses, 0, 0)
    ses.build_accept()
    rng = np.random.default_rng(0)
    for k in range(4):
        st = ctx.tile_state(k)
        st["occupancy"] = np.where(rng.random(32 ** 3) < 0.4, 0.0, 1.0).astype(np.float32)
        ctx.set_tile_state(k, st)
        ses.set_tile_state(k, st)
    n_gpu = ctx.sample(11, 0, N_RAYS, True)
    n_ref = ses.sample(11, 0, N_RAYS, True)
    assert n_gpu == n_ref
    _cmp_batch(ctx.batch(), ses.batch())
    b = ctx.batch()
    counts = np.diff(b["offsets"].astype(np.int64))
    assert counts.mean() < 60  # culling happened


def test_field_composite_backward(setup):
    ctx, ses = setup
    _same_window(ctx, ses, 1, 1)
    ses.build_accept()
    # perturb the fields away from their init so every path carries signal
    rng = np.random.default_rng(1)
    for k in range(4):
        st = ses.tile_state(k)
        st["enc"] = (st["enc"] + rng.normal(0, 0.5, st["enc"].shape)).astype(np.float32)
        st["dnet"] = (st["dnet"] * 1.5).astype(np.float32)
        ses.set_tile_state(k, st)
        ctx.set_tile_state(k, st)
    p, m, v, s = ses.color()
    ctx.set_color(p, m, v, s)
    ctx.sample(2, 0, N_RAYS, True)
    ses.sample(2, 0, N_RAYS, True)
    sg, rgb = ctx.field_forward()
    sr, rr = ses.forward()
    np.testing.assert_allclose(sg, sr, rtol=TOL_SIGMA_RTOL, atol=1e-6)
    np.testing.assert_allclose(rgb, rr, atol=TOL_RGB_ATOL)
    cg = ctx.composite()
    cr = ses.composite()
    np.testing.assert_allclose(cg["rgb"], cr["rgb"], atol=TOL_RAY_RGB_ATOL)
    np.testing.assert_allclose(cg["opacity"], cr["opacity"], atol=TOL_RAY_RGB_ATOL)
    np.testing.assert_allclose(cg["depth"], cr["depth"], atol=TOL_DEPTH_ATOL)
    assert abs(cg["loss"] - cr["loss"]) <= TOL_LOSS_RTOL * abs(cr["loss"])
    scale = np.abs(cr["d_sigma"]).max()
    np.testing.assert_allclose(cg["d_sigma"], cr["d_sigma"], atol=3e-2 * scale)
    np.testing.assert_allclose(cg["d_rgb"], cr["d_rgb"], atol=1e-2 * np.abs(cr["d_rgb"]).max())
    ctx.field_backward()
    ses.backward()
    for k in range(4):
        ge, gd, gc = ctx.grads(k)
        re, rd, rc = ses.grads(k)
        for name, a, b in (("enc", ge, re), ("dnet", gd, rd), ("color", gc, rc)):
            den = np.linalg.norm(b)
            assert den > 0, name
            rel = np.linalg.norm(a - b) / den
            assert rel < TOL_GRAD_REL[name], (k, name, rel)


def test_train_steps_and_adam(setup):
    """Three full iterations on both sides from identical state: the loss
    trajectories agree and parameters stay within tolerance."""
    ctx, ses = setup
    _same_window(ctx, ses, 0, 1)
    ses.build_accept()
    for k in range(4):
        st = ses.tile_state(k)
        ctx.set_tile_state(k, st)
    p, m, v, s = ses.color()
    ctx.set_color(p, m, v, s)
    for it in range(3):
        lg = ctx.train_step(100 + it, 0, N_RAYS)
        lr = ses.train_step(100 + it, 0, N_RAYS)
        assert abs(lg - lr) <= 1e-2 * abs(lr), (it, lg, lr)
    for k in range(4):
        a, b = ctx.tile_state(k), ses.tile_state(k)
        assert a["enc_step"] == b["enc_step"] and a["dnet_step"] == b["dnet_step"]
    # Adam maps every gradient to a ~lr step, so weights whose gradient sums
    # cancel to ~0 may step in opposite directions on the two sides; the
    # contract is on what the field renders (K5 itself is bit-exact below).
    ctx.sample(200, 0, N_RAYS, False)
    ses.sample(200, 0, N_RAYS, False)
    ctx.field_forward()
    ses.forward()
    cg, cr = ctx.composite(), ses.composite()
    # Adam's normalised step amplifies gradient differences on near-zero
    # gradients into +-lr parameter differences, so after three steps the
    # contract is statistical: 99.9% of the rendered values within 5e-3 and
    # none beyond 2e-2
    for f in ("rgb", "opacity"):
        d = np.abs(cg[f] - cr[f]).ravel()
        assert np.quantile(d, 0.999) <= 5e-3 and d.max() <= 2e-2, (f, np.quantile(d, 0.999), d.max())


def test_adam_bit_exact_on_identical_grads(setup):
    """K5 alone: feed the oracle's own gradients through the GPU Adam."""
    ctx, ses = setup
    from oracle.pyoracle import Oracle

    o = Oracle()
    rng = np.random.default_rng(3)
    p = rng.normal(size=6915).astype(np.float32)
    g = rng.normal(size=6915).astype(np.float32) * 1e-3
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    # GPU: load params + grads via the colour group of a fresh window
    _same_window(ctx, ses, 1, 1)
    pc, mc, vc = p.copy(), m.copy(), v.copy()
    step = o.adam_step(pc, g, mc, vc, 0, lr=1e-3)
    ctx.set_color(p, m, v, 0)
    # zero all other grads, colour grads = g, by running a zero-ray-effect trick:
    import torch

    gt = ctx.grad_tensor()
    gt.zero_()
    gt[-6915:] = torch.from_numpy(g).cuda()
    torch.cuda.synchronize()
    ctx.optimizer_step(12345)
    pg, mg, vg, sg = ctx.color()
    assert sg == step
    np.testing.assert_array_equal(mg, mc)
    np.testing.assert_array_equal(vg, vc)
    np.testing.assert_array_equal(pg, pc)


def test_occupancy_update(setup):
    ctx, ses = setup
    _same_window(ctx, ses, 1, 1)
    for k in range(4):
        ctx.set_tile_state(k, ses.tile_state(k))
    ctx.update_occupancy()
    ses.update_occupancy()
    for k in range(4):
        a, b = ctx.tile_state(k)["occupancy"], ses.tile_state(k)["occupancy"]
        np.testing.assert_allclose(a, b, rtol=2e-3, atol=1e-6)  # K6 runs on CUDA cores (fp32)


def test_window_slide_roundtrip_and_constant_memory(setup):
    ctx, ses = setup
    _same_window(ctx, ses, 0, 0)
    before = {t: ctx.tile_state(k) for k, t in enumerate(ctx.window_tiles())}
    mem0 = ctx.memory_report()["total_device"]
    ctx.train_step(500, 0, N_RAYS)
    after_train = {t: ctx.tile_state(k) for k, t in enumerate(ctx.window_tiles())}
    for pos in [(0, 1), (1, 1), (1, 0), (0, 0)]:
        ctx.set_window(*pos)
        assert ctx.memory_report()["total_device"] == mem0
    back = {t: ctx.tile_state(k) for k, t in enumerate(ctx.window_tiles())}
    for t in after_train:
        for f in ("enc", "dnet", "enc_m", "enc_v", "dnet_m", "dnet_v", "occupancy"):
            np.testing.assert_array_equal(back[t][f], after_train[t][f], err_msg=f"{t}.{f}")
        assert back[t]["enc_step"] == after_train[t]["enc_step"] == before[t]["enc_step"] + 1


def test_render_path(setup):
    ctx, ses = setup
    _same_window(ctx, ses, 0, 0)
    acc = ses.build_accept()
    sel = acc[:: max(1, acc.size // 1500)][:1500]
    px = np.stack([(sel >> 40).astype(np.int32), ((sel >> 20) & 0xFFFFF).astype(np.int32),
                   (sel & 0xFFFFF).astype(np.int32)], axis=1)
    v0 = px[px[:, 0] == 0]
    ses.sample_pixels(v0)
    ses.forward()
    ref = ses.composite()
    states = [ses.tile_state(k) for k in range(4)]
    p, _, _, _ = ses.color()
    ctx.render_setup(ses.window_tiles(), states, p)
    rgb, dep, op = ctx.render_pixels(ctx.scene.cams[0], v0[:, 1:])
    np.testing.assert_allclose(rgb, ref["rgb"], atol=TOL_RAY_RGB_ATOL)
    np.testing.assert_allclose(op, ref["opacity"], atol=TOL_RAY_RGB_ATOL)


def test_loss_decreases(setup):
    ctx, ses = setup
    _same_window(ctx, ses, 1, 0)
    losses = [ctx.train_step(1000 + i, 0, N_RAYS) for i in range(40)]
    assert np.mean(losses[-5:]) < 0.7 * np.mean(losses[:5]), losses
