#!/usr/bin/env python
"""Attribution of the field path's bf16 gradient error (diagnostic tool).

Runs the numerics model oracle/bf16_model.py (the K2/K4 math with switchable
operand roundings) on the inputs of tests/test_gpu_isolated.py::
test_field_backward_alone (the oracle's batch, parameters and d_sigma /
d_rgb) and prints the norm-relative hash-table gradient error against the
fp32 oracle for each rounding variant.

  python tools/emulate_bwd.py

Result on the test's inputs (r02): all operands bf16 (the kernels) 6.6%, the
same as the B200 measures; forward recompute in fp32 with the backward GEMMs
in bf16 0.5%; forward bf16 with the backward in fp32 6.6%; forward TF32 2.3%;
forward as bf16 hi+lo pairs 0.5%.  The error is the ReLU masks of the bf16
forward recompute flipping for pre-activations near zero (a flipped mask
switches a whole gradient path of that sample), not the backward GEMMs.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import bf16_model as M  # noqa: E402
from oracle.pyoracle import Oracle, Session  # noqa: E402
from paper_2507_01631_b200 import synth  # noqa: E402
from paper_2507_01631_b200.abi import FieldConfig, TrainConfig  # noqa: E402


def main():
    scene = synth.make_scene(3, 3, tile_side=128.0, n_views=4, gsd=1.0, seed=21)
    fc = FieldConfig.defaults()
    tc = TrainConfig.defaults(batch_rays=2048, seed=5)
    ses = Session(Oracle(), scene, fc, tc, workers=os.cpu_count() or 8)
    ses.set_window(1, 1)
    ses.build_accept()
    rng = np.random.default_rng(1)
    for k in range(4):
        st = ses.tile_state(k)
        st["enc"] = (st["enc"] + rng.normal(0, 0.5, st["enc"].shape)).astype(np.float32)
        st["dnet"] = (st["dnet"] * 1.5).astype(np.float32)
        ses.set_tile_state(k, st)
    ses.sample(8, 0, 2048, True)
    ses.forward()
    comp = ses.composite()
    ses.backward()
    b = ses.batch()
    color = ses.color()[0]
    tiles = [(ses.tile_state(k)["enc"], ses.tile_state(k)["dnet"]) for k in range(4)]
    ref = [ses.grads(k)[0] for k in range(4)]
    allr, fwd = set(M.KERNEL), set(M.FWD_OPS)
    variants = {"fp32 (model check)": set(), "all bf16 (the kernels)": allr,
                "forward fp32, backward bf16": allr - fwd, "forward bf16, backward fp32": fwd}
    for one in M.FWD_OPS:
        variants[f"only {one} bf16"] = {one}
    for mode in ("tf32", "split"):
        variants[f"forward {mode}, backward bf16"] = {**{k: "bf16" for k in allr - fwd}, **{k: mode for k in fwd}}
    for name, rq in variants.items():
        out = M.batch(tiles, color, b, rq, comp["d_sigma"], comp["d_rgb"])
        err = max(np.linalg.norm(out["grads"][k][0] - ref[k]) / np.linalg.norm(ref[k]) for k in range(4))
        print(f"{name:45s} hash-table gradient rel err (max over slots) {err:.4f}")


if __name__ == "__main__":
    main()
