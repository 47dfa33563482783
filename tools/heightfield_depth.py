#!/usr/bin/env python
"""GPU-only training on the heightfield fixture: depth MAE against the exact
ground truth and PSNR over training iterations (the geometry the short
oracle-parity runs cannot reach).

  python tools/heightfield_depth.py [iters] [batch]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2507_01631_b200 import synth  # noqa: E402
from paper_2507_01631_b200.abi import FieldConfig, TrainConfig  # noqa: E402
from paper_2507_01631_b200.tilefield import Context  # noqa: E402


def evaluate(ctx, scene, px):
    ctx.sample_pixels(px)
    ctx.field_forward()
    g = ctx.composite()
    tgt = ctx.batch()["rays"]["target"]
    gt = scene.depths[0][px[:, 1], px[:, 2]]
    op = g["opacity"] > 0.5
    mse = float(np.mean((g["rgb"] - tgt) ** 2))
    return 10 * np.log10(1 / mse), float(np.mean(np.abs(g["depth"][op] - gt[op]))), int(op.sum()), \
        float(np.median(np.abs(g["depth"][op] - gt[op])))


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    for name, scene, win in (("config 1", synth.make_heightfield_scene(1, 1, 128.0, 40.0, 4, 0.5, 3), (0, 0)),
                             ("config 1, 8 views", synth.make_heightfield_scene(1, 1, 128.0, 40.0, 8, 0.5, 3), (0, 0))):
        tc = TrainConfig.defaults(batch_rays=B, seed=11)
        ctx = Context(scene, FieldConfig.defaults(), tc, max_rays=max(B, 8192))
        ctx.set_window(*win)
        acc = ctx.accept_list()
        v0 = acc[(acc >> 40) == 0]
        sel = v0[:: max(1, v0.size // 8192)][:8192]
        px = np.stack([(sel >> 40).astype(np.int32), ((sel >> 20) & 0xFFFFF).astype(np.int32),
                       (sel & 0xFFFFF).astype(np.int32)], axis=1)
        t0 = time.time()
        for it in range(iters + 1):
            if it % 500 == 0:
                p, mae, n, med = evaluate(ctx, scene, px)
                print(f"{name} it {it:5d}: PSNR {p:.2f} dB, depth MAE vs GT {mae:.3f} m (median {med:.3f}) "
                      f"over {n} opaque px ({time.time() - t0:.1f} s)", flush=True)
            ctx.train_step(it, 0, B)
        ctx.close()


if __name__ == "__main__":
    main()
