"""Each stage of the CUDA path alone against the CPU oracle, on identical
inputs (VERDICT r1 "pin and isolate the backward"):

  * batch import: a caller-built RaySegmentBatch (here the oracle's) becomes
    the device batch bit-exactly (the forward_batch / backward_batch drop-in);
  * K3 alone: compositing + loss + render backward on the oracle's own
    sigma / rgb, fp32 vs fp32 (tolerance 1e-5);
  * K4 alone: the field backward fed the oracle's d_sigma / d_rgb, so only the
    tcgen05 backward (bf16 operands, fp32 accumulate) differs;
  * K5 over caller spans: adam_step on host arrays and on device tensors,
    bit-exact, with the non-finite error contract.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2507_01631_b200 import synth
from paper_2507_01631_b200.abi import FieldConfig, TrainConfig

N_RAYS = 2048
# K3 in fp32 on both sides: only summation order (warp scans vs sequential)
# and expf differ
TOL_K3 = 1e-5
# K4 alone vs the fp32 oracle: the field's tensor-core operands are bf16
# (fp32 accumulate).  Measured on B200 (r02): enc 6.6%, dnet 1.6%, colour
# 0.4% norm-relative; the CPU numerics model (oracle/bf16_model.py) predicts
# the same 6.6%, and attributes it to ReLU masks of the bf16 forward
# recompute flipping near zero (the backward GEMMs alone cost 0.5%;
# tools/emulate_bwd.py).
TOL_K4_GRAD_REL = {"enc": 0.09, "dnet": 0.03, "color": 0.01}
# GPU vs the bf16 numerics model (same roundings): what is left is fp32
# accumulation order inside the MMAs / atomics, FMA contraction, expf
# (measured r02: enc 5.6e-5, dnet 1.0e-5, colour 3.1e-6)
TOL_MODEL_GRAD_REL = {"enc": 1e-3, "dnet": 1e-3, "color": 1e-4}


@pytest.fixture(scope="module")
def pair():
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
    ctx.set_window(1, 1)
    ses.set_window(1, 1)
    ses.build_accept()
    rng = np.random.default_rng(1)
    for k in range(4):
        st = ses.tile_state(k)
        st["enc"] = (st["enc"] + rng.normal(0, 0.5, st["enc"].shape)).astype(np.float32)
        st["dnet"] = (st["dnet"] * 1.5).astype(np.float32)
        ses.set_tile_state(k, st)
        ctx.set_tile_state(k, st)
    p, m, v, s = ses.color()
    ctx.set_color(p, m, v, s)
    return ctx, ses


def _same_batch(a, b):
    for f in ("origin", "direction", "target", "image_id", "row", "col"):
        np.testing.assert_array_equal(a["rays"][f], b["rays"][f], err_msg=f)
    for f in ("offsets", "t", "delta", "local", "slot", "endpoint"):
        np.testing.assert_array_equal(a[f], b[f], err_msg=f)


def test_batch_import_round_trip(pair):
    ctx, ses = pair
    ctx.sample(3, 0, N_RAYS, True)
    own = ctx.batch()
    assert ctx.batch_import(own) == own["offsets"][-1]
    _same_batch(ctx.batch(), own)
    ses.sample(4, 100, N_RAYS, True)
    ref = ses.batch()
    ctx.batch_import(ref)
    _same_batch(ctx.batch(), ref)


def test_batch_import_rejects_bad_batches(pair):
    from paper_2507_01631_b200.tilefield import TileFieldError

    ctx, ses = pair
    ses.sample(4, 0, 64, True)
    b = ses.batch()
    bad = dict(b)
    bad["slot"] = b["slot"].copy()
    bad["slot"][int(b["offsets"][1]) - 1] = 7  # slot outside the window
    with pytest.raises(TileFieldError, match="one run per loaded slot"):
        ctx.batch_import(bad)
    bad = dict(b)
    bad["offsets"] = b["offsets"].copy()
    bad["offsets"][5] = bad["offsets"][6] + 1
    with pytest.raises(TileFieldError, match="ascend"):
        ctx.batch_import(bad)


def test_composite_alone_matches_oracle(pair):
    """K3 on the oracle's sigma / rgb: ray rgb, depth, opacity, loss and the
    render backward (d_sigma, d_rgb) within 1e-5."""
    ctx, ses = pair
    ses.sample(6, 0, N_RAYS, True)
    sg, rgb = ses.forward()
    ref = ses.composite()
    ctx.batch_import(ses.batch())
    ctx.set_field_outputs(sg, rgb)
    got = ctx.composite()
    np.testing.assert_allclose(got["rgb"], ref["rgb"], rtol=0, atol=TOL_K3)
    np.testing.assert_allclose(got["opacity"], ref["opacity"], rtol=0, atol=TOL_K3)
    np.testing.assert_allclose(got["depth"], ref["depth"], rtol=TOL_K3, atol=TOL_K3)
    assert abs(got["loss"] - ref["loss"]) <= TOL_K3 * abs(ref["loss"])
    np.testing.assert_allclose(got["d_rgb"], ref["d_rgb"], rtol=0, atol=TOL_K3 * np.abs(ref["d_rgb"]).max())
    # d_sigma_k = delta_k sum_c g_c (T_{k+1} c_k - R_k) is a difference of terms
    # bounded by delta_k |g| (|T c|, |R| <= 1): the tolerance scales with that
    b = ses.batch()
    g = 2.0 * (ref["rgb"] - b["rays"]["target"]) / (3.0 * N_RAYS)
    ray_of = np.repeat(np.arange(N_RAYS), np.diff(b["offsets"].astype(np.int64)))
    scale = b["delta"] * np.abs(g[ray_of]).sum(axis=1) * 2.0
    assert np.all(np.abs(got["d_sigma"] - ref["d_sigma"]) <= TOL_K3 * scale + 1e-12)


def test_composite_weight_normalisation(pair):
    """sum_k T_k alpha_k + T_final = 1 within 1e-5 in fp32: with
    black samples the ray colour is T_final * bg, so opacity + rgb / bg = 1."""
    ctx, ses = pair
    ses.sample(7, 0, N_RAYS, True)
    sg, _ = ses.forward()
    ctx.batch_import(ses.batch())
    ctx.set_field_outputs(sg * 3.0, np.zeros((sg.size, 3), np.float32))
    got = ctx.composite()
    tot = got["opacity"] + got["rgb"][:, 0] / 0.5
    np.testing.assert_allclose(tot, 1.0, atol=1e-5)
    assert got["opacity"].min() >= 0.0 and got["opacity"].max() <= 1.0 + 1e-6


def test_field_backward_alone(pair):
    """K4 fed the oracle's d_sigma / d_rgb: the parameter gradients differ
    from the oracle's only by the tcgen05 backward's bf16 operands."""
    ctx, ses = pair
    ses.sample(8, 0, N_RAYS, True)
    ses.forward()
    ref = ses.composite()
    ses.backward()
    ctx.batch_import(ses.batch())
    ctx.field_forward()
    ctx.field_backward_from(ref["d_sigma"], ref["d_rgb"])
    worst = {}
    for k in range(4):
        ge, gd, gc = ctx.grads(k)
        re, rd, rc = ses.grads(k)
        for name, a, b in (("enc", ge, re), ("dnet", gd, rd), ("color", gc, rc)):
            den = np.linalg.norm(b)
            assert den > 0, name
            rel = float(np.linalg.norm(a - b) / den)
            worst[name] = max(worst.get(name, 0.0), rel)
    print("K4-alone norm-relative gradient error:", worst)
    for name, rel in worst.items():
        assert rel < TOL_K4_GRAD_REL[name], (name, rel)


def test_field_matches_bf16_numerics_model(pair):
    """The GPU computes the bf16-operand math it claims: K2's sigma / rgb and
    K4's gradients (fed the oracle's d_sigma / d_rgb) against
    oracle/bf16_model.py with the kernels' roundings."""
    from oracle import bf16_model as M

    ctx, ses = pair
    ses.sample(10, 0, N_RAYS, True)
    ses.forward()
    ref = ses.composite()
    b = ses.batch()
    tiles = [(ses.tile_state(k)["enc"], ses.tile_state(k)["dnet"]) for k in range(4)]
    model = M.batch(tiles, ses.color()[0], b, M.KERNEL, ref["d_sigma"], ref["d_rgb"])
    ctx.batch_import(b)
    sg, rgb = ctx.field_forward()
    rel_s = np.abs(sg - model["sigma"]) / np.maximum(model["sigma"], 1e-6)
    d_rgb = np.abs(rgb - model["rgb"])
    print("K2 vs model: sigma rel p99 %.2e max %.2e, rgb p99 %.2e max %.2e" %
          (np.quantile(rel_s, 0.99), rel_s.max(), np.quantile(d_rgb, 0.99), d_rgb.max()))
    assert np.quantile(rel_s, 0.99) < 1e-4 and np.quantile(d_rgb, 0.99) < 1e-5
    assert rel_s.max() < 2e-2 and d_rgb.max() < 5e-3  # isolated mask flips
    ctx.field_backward_from(ref["d_sigma"], ref["d_rgb"])
    worst = {}
    for k in range(4):
        ge, gd, gc = ctx.grads(k)
        for name, a, m in (("enc", ge, model["grads"][k][0]), ("dnet", gd, model["grads"][k][1]),
                           ("color", gc, model["g_color"])):
            worst[name] = max(worst.get(name, 0.0), float(np.linalg.norm(a - m) / np.linalg.norm(m)))
    print("K4 vs bf16 model, norm-relative:", worst)
    for name, rel in worst.items():
        assert rel < TOL_MODEL_GRAD_REL[name], (name, rel)


def test_field_forward_deterministic(pair):
    """The forward is a pure function of the batch and the parameters: the
    same batch repeated in one context and once in a fresh context give the
    same bits.  (Races that need drifting warps can slip past this; the
    run save/resume test, two contexts training in step, is the stricter
    check: it caught a staging race of colour layer 1's bias columns.)"""
    from paper_2507_01631_b200.tilefield import Context

    ctx, ses = pair
    ses.sample(12, 0, N_RAYS, True)
    b = ses.batch()
    ctx.batch_import(b)
    s1, r1 = ctx.field_forward()
    for _ in range(16):  # a race shows only when warps drift apart: repeat
        ctx.batch_import(b)
        s2, r2 = ctx.field_forward()
        np.testing.assert_array_equal(s1, s2)
        np.testing.assert_array_equal(r1, r2)
    other = Context(ctx.scene, FieldConfig.defaults(), TrainConfig.defaults(batch_rays=N_RAYS, seed=5),
                    max_rays=N_RAYS)
    other.set_window(1, 1)
    for k in range(4):
        other.set_tile_state(k, ctx.tile_state(k))
    p, m, v, st = ctx.color()
    other.set_color(p, m, v, st)
    other.batch_import(b)
    s3, r3 = other.field_forward()
    np.testing.assert_array_equal(s1, s3)
    np.testing.assert_array_equal(r1, r3)


def test_field_backward_zero_in_zero_out(pair):
    """zero loss gradient in -> zero gradients out."""
    ctx, ses = pair
    ses.sample(9, 0, 512, True)
    ctx.batch_import(ses.batch())
    ctx.field_forward()
    S = ctx.n_samples
    ctx.field_backward_from(np.zeros(S, np.float32), np.zeros((S, 3), np.float32))
    for k in range(4):
        for g in ctx.grads(k):
            assert not np.any(g), k


def test_adam_over_caller_spans_bit_exact(pair):
    import torch

    from oracle.pyoracle import Oracle
    from paper_2507_01631_b200.tilefield import NonFiniteGradient

    ctx, _ = pair
    o = Oracle()
    rng = np.random.default_rng(11)
    n = 100_003  # not a multiple of 4
    p = rng.normal(size=n).astype(np.float32)
    g = (rng.normal(size=n) * 1e-2).astype(np.float32)
    m = (rng.normal(size=n) * 1e-3).astype(np.float32)
    v = (rng.random(n) * 1e-4).astype(np.float32)
    for step0, rate in ((0, 1.0), (41, 0.5)):
        pr, mr, vr = p.copy(), m.copy(), v.copy()
        s_ref = o.adam_step(pr, g, mr, vr, step0, lr=3e-3, rate=rate, dsteps=100)
        ph, mh, vh = p.copy(), m.copy(), v.copy()  # host spans
        s_h = ctx.adam_step(ph, g, mh, vh, step0, lr=3e-3, decay_rate=rate, decay_steps=100, group="g")
        assert s_h == s_ref == step0 + 1
        for a, b in ((ph, pr), (mh, mr), (vh, vr)):
            assert a.tobytes() == b.tobytes()
        pd, gd, md, vd = (torch.from_numpy(x.copy()).cuda() for x in (p, g, m, v))  # device spans
        s_d = ctx.adam_step(pd, gd, md, vd, step0, lr=3e-3, decay_rate=rate, decay_steps=100, group="g")
        assert s_d == s_ref
        for a, b in ((pd, pr), (md, mr), (vd, vr)):
            assert a.cpu().numpy().tobytes() == b.tobytes()
    gbad = g.copy()
    gbad[77] = np.inf
    ph = p.copy()
    with pytest.raises(NonFiniteGradient, match="non-finite gradient in group tile\\(9,9\\).enc"):
        ctx.adam_step(ph, gbad, m.copy(), v.copy(), 5, group="tile(9,9).enc")
    assert ph.tobytes() == p.tobytes()
