"""Prints the deviation of the CUDA field path from the oracle (diagnostic)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.pyoracle import Oracle, Session
from paper_2507_01631_b200 import synth
from paper_2507_01631_b200.abi import FieldConfig, TrainConfig
from paper_2507_01631_b200.tilefield import Context

N = 2048
scene = synth.make_scene(3, 3, tile_side=128.0, n_views=4, gsd=1.0, seed=21)
fc, tc = FieldConfig.defaults(), TrainConfig.defaults(batch_rays=N, seed=5)
ctx = Context(scene, fc, tc, max_rays=N)
ses = Session(Oracle(), scene, fc, tc, workers=16)
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
ctx.sample(2, 0, N, True)
ses.sample(2, 0, N, True)
sg, rgb = ctx.field_forward()
sr, rr = ses.forward()
rel = np.abs(sg - sr) / np.maximum(np.abs(sr), 1e-6)
print("sigma rel err: max %.3g p99 %.3g median %.3g" % (rel.max(), np.quantile(rel, 0.99), np.median(rel)))
print("rgb abs err: max %.3g p99 %.3g" % (np.abs(rgb - rr).max(), np.quantile(np.abs(rgb - rr), 0.99)))
cg, cr = ctx.composite(), ses.composite()
for k in ("rgb", "opacity", "depth"):
    d = np.abs(cg[k] - cr[k])
    print(f"ray {k}: max {d.max():.3g} p99 {np.quantile(d, 0.99):.3g}")
print("loss gpu %.6g ref %.6g" % (cg["loss"], cr["loss"]))
ds = np.abs(cg["d_sigma"] - cr["d_sigma"]).max() / np.abs(cr["d_sigma"]).max()
print("d_sigma max err / max |ref|: %.3g" % ds)
ctx.field_backward()
ses.backward()
for k in range(4):
    ge, gd, gc = ctx.grads(k)
    re, rd, rc = ses.grads(k)
    out = []
    for name, a, b in (("enc", ge, re), ("dnet", gd, rd), ("color", gc, rc)):
        out.append(f"{name} {np.linalg.norm(a - b) / np.linalg.norm(b):.3g}")
    print(f"slot {k} grad rel err:", ", ".join(out))
gd0, rd0 = ctx.grads(0)[1], ses.grads(0)[1]
print("dnet slot0 W1 gpu/ref sample:", gd0[:4], rd0[:4])
print("dnet slot0 b1 gpu/ref sample:", gd0[1024:1028], rd0[1024:1028])
print("dnet slot0 W2 gpu/ref:", gd0[1088:1092], rd0[1088:1092], " b2:", gd0[2112:2116], rd0[2112:2116])
gc0, rc0 = ctx.grads(0)[2], ses.grads(0)[2]
for nm, o in (("Wc1", 0), ("bc1", 2496), ("Wc2", 2560), ("bc2", 6656), ("Wc3", 6720), ("bc3", 6912)):
    print(nm, gc0[o:o + 3], rc0[o:o + 3])
