"""Finite-difference oracle of the reverse mode (
field.hpp:127-128 templates the batch operators on the scalar "so the
finite-difference oracle can run the identical math in float64").

On a 4-ray micro-batch of a real window (rays crossing tile seams), the
oracle's float64 shadow (tfo_shadow_loss_grad: the hash grid, both MLPs,
the density / sigmoid activations, compositing and the colour loss in
double) gives the loss and its analytic gradient.  Per parameter group
(every slot's hash tables and density MLP, the colour MLP):

  * central differences with step 1e-3 on the float64 shadow agree with the
    analytic gradient within 1e-3 relative (norm over the probed entries).
    An entry whose +-1e-3 stencil straddles a ReLU kink of some sample (the
    loss is only piecewise smooth there: the step-1e-3 and step-1e-4
    differences disagree) is re-measured with step 1e-5; such entries must
    stay a minority;
  * the fp32 oracle's gradient (tfo_backward, the parity reference of the GPU
    path) agrees with the float64 analytic gradient within 1e-3 relative.
"""
import numpy as np
import pytest

from paper_2507_01631_b200 import synth
from paper_2507_01631_b200.abi import FieldConfig, TrainConfig

H = 1e-3
TOL = 1e-3


@pytest.fixture(scope="module")
def micro(oracle):
    from oracle.pyoracle import Session

    scene = synth.make_scene(2, 2, tile_side=64.0, z_extent=20.0, n_views=2, gsd=1.0, seed=13)
    fc = FieldConfig.defaults()
    tc = TrainConfig.defaults(batch_rays=4, seed=3)
    ses = Session(oracle, scene, fc, tc, workers=2)
    ses.set_window(0, 0)
    ses.build_accept()
    rng = np.random.default_rng(4)
    for k in range(4):
        st = ses.tile_state(k)
        st["enc"] = (st["enc"] + rng.normal(0, 0.5, st["enc"].shape)).astype(np.float32)
        st["dnet"] = (st["dnet"] * 1.5 + rng.normal(0, 0.02, st["dnet"].shape)).astype(np.float32)
        ses.set_tile_state(k, st)
    p, m, v, s = ses.color()
    ses.set_color((p + rng.normal(0, 0.02, p.shape)).astype(np.float32), m, v, s)
    # 4 rays, chosen to include rays that cross a tile seam
    ses.sample(1, 0, 4, True)
    for it in range(2, 200):
        if len(set(ses.batch()["slot"].tolist())) >= 2:
            break
        ses.sample(it, 0, 4, True)
    b = ses.batch()
    assert len(set(b["slot"].tolist())) >= 2 and b["offsets"][-1] > 50
    enc = [ses.tile_state(k)["enc"].astype(np.float64) for k in range(4)]
    dnet = [ses.tile_state(k)["dnet"].astype(np.float64) for k in range(4)]
    color = ses.color()[0].astype(np.float64)
    return ses, enc, dnet, color


def _probe(g, k=16, seed=0):
    """Entries to probe: the largest gradients plus random non-zero ones."""
    nz = np.flatnonzero(g)
    top = np.argsort(-np.abs(g))[:k]
    rng = np.random.default_rng(seed)
    extra = rng.choice(nz, size=min(k, nz.size), replace=False) if nz.size else np.zeros(0, np.int64)
    return np.unique(np.concatenate([top, extra]))


def test_fd_matches_analytic_float64(micro):
    ses, enc, dnet, color = micro
    L0, (ge, gd, gc) = ses.shadow_loss_grad(enc, dnet, color)
    assert L0 > 0
    groups = [("color", None, color, gc)]
    for k in range(4):
        groups += [(f"slot{k}.enc", k, enc[k], ge[k]), (f"slot{k}.dnet", k, dnet[k], gd[k])]
    checked = kinks = probes = 0
    for name, _, arr, g in groups:
        if not np.any(g):
            continue  # a slot no sample of the micro-batch reached: zero gradient
        idx = _probe(g, seed=checked)
        fd = np.zeros(idx.size)

        def central(i, h):
            keep = arr[i]
            arr[i] = keep + h
            lp, _ = ses.shadow_loss_grad(enc, dnet, color, grad=False)
            arr[i] = keep - h
            lm, _ = ses.shadow_loss_grad(enc, dnet, color, grad=False)
            arr[i] = keep
            return (lp - lm) / (2 * h)

        for j, i in enumerate(idx):
            fd[j] = central(i, H)
            fine = central(i, H / 10)
            if abs(fd[j] - fine) > TOL * abs(fine):
                kinks += 1
                fd[j] = central(i, H / 100)
        probes += idx.size
        an = g[idx]
        rel = np.linalg.norm(fd - an) / np.linalg.norm(an)
        assert rel < TOL, (name, rel)
        checked += 1
    assert checked >= 5
    assert kinks <= probes // 4, (kinks, probes)


def test_fp32_oracle_gradient_matches_float64(micro):
    ses, enc, dnet, color = micro
    L0, (ge, gd, gc) = ses.shadow_loss_grad(enc, dnet, color)
    ses.forward()
    comp = ses.composite()
    assert abs(comp["loss"] - L0) <= 1e-5 * L0
    ses.backward()
    for k in range(4):
        e32, d32, c32 = ses.grads(k)
        for name, a, b in (("enc", e32, ge[k]), ("dnet", d32, gd[k]), ("color", c32, gc)):
            n = np.linalg.norm(b)
            if n == 0:
                assert not np.any(a), (k, name)
                continue
            assert np.linalg.norm(a - b) / n < TOL, (k, name)
