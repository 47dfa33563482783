"""The numerics model of the tcgen05 field path (oracle/bf16_model.py) on
CPU: with no operand rounding it reproduces the fp32 oracle (so it models the
same function), and with the kernels' bf16 operands it quantifies what bf16
costs against the fp32 reference.  tests/test_gpu_isolated.py then checks the
GPU against the model tightly."""
import numpy as np
import pytest

from oracle import bf16_model as M
from paper_2507_01631_b200 import synth
from paper_2507_01631_b200.abi import FieldConfig, TrainConfig


@pytest.fixture(scope="module")
def case(oracle):
    from oracle.pyoracle import Session

    scene = synth.make_scene(3, 3, tile_side=128.0, n_views=3, gsd=1.5, seed=21)
    fc = FieldConfig.defaults()
    ses = Session(oracle, scene, fc, TrainConfig.defaults(batch_rays=512, seed=5), workers=4)
    ses.set_window(1, 1)
    ses.build_accept()
    rng = np.random.default_rng(1)
    for k in range(4):
        st = ses.tile_state(k)
        st["enc"] = (st["enc"] + rng.normal(0, 0.5, st["enc"].shape)).astype(np.float32)
        st["dnet"] = (st["dnet"] * 1.5).astype(np.float32)
        ses.set_tile_state(k, st)
    ses.sample(8, 0, 512, True)
    sg, rgb = ses.forward()
    comp = ses.composite()
    ses.backward()
    tiles = [(ses.tile_state(k)["enc"], ses.tile_state(k)["dnet"]) for k in range(4)]
    return ses, tiles, ses.color()[0], ses.batch(), sg, rgb, comp


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_model_without_rounding_is_the_oracle(case):
    ses, tiles, color, b, sg, rgb, comp = case
    out = M.batch(tiles, color, b, set(), comp["d_sigma"], comp["d_rgb"])
    np.testing.assert_allclose(out["sigma"], sg, rtol=1e-5, atol=1e-7)
    np.testing.assert_allclose(out["rgb"], rgb, rtol=0, atol=1e-6)
    for k in range(4):
        re, rd, rc = ses.grads(k)
        assert _rel(out["grads"][k][0], re) < 1e-5
        assert _rel(out["grads"][k][1], rd) < 1e-5
    assert _rel(out["g_color"], ses.grads(0)[2]) < 1e-5


def test_model_quantifies_bf16(case):
    """What the kernels' bf16 operands cost against fp32 (the stated
    tolerances of the GPU parity tests rest on this)."""
    ses, tiles, color, b, sg, rgb, comp = case
    out = M.batch(tiles, color, b, M.KERNEL, comp["d_sigma"], comp["d_rgb"])
    assert np.max(np.abs(out["sigma"] - sg) / np.maximum(sg, 1e-6)) < 2e-2
    assert np.max(np.abs(out["rgb"] - rgb)) < 5e-3
    enc = max(_rel(out["grads"][k][0], ses.grads(k)[0]) for k in range(4))
    dn = max(_rel(out["grads"][k][1], ses.grads(k)[1]) for k in range(4))
    assert enc < 0.10 and dn < 0.05, (enc, dn)
    # the backward GEMMs alone (forward recompute in fp32) cost little: the
    # error is the bf16 forward's ReLU masks (tools/emulate_bwd.py)
    bw = M.batch(tiles, color, b, set(M.BWD_OPS), comp["d_sigma"], comp["d_rgb"])
    enc_bw = max(_rel(bw["grads"][k][0], ses.grads(k)[0]) for k in range(4))
    assert enc_bw < 0.02 and enc_bw < enc / 3, (enc_bw, enc)
