"""Times the first window's accept pass and window moves on the bench scene
(config 5): wall clock around set_window with a device sync on both sides."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2507_01631_b200 import synth  # noqa: E402
from paper_2507_01631_b200.abi import FieldConfig, TrainConfig  # noqa: E402
from paper_2507_01631_b200.tilefield import Context, snake_path  # noqa: E402

scene = synth.config_scene(5, seed=0)
ctx = Context(scene, FieldConfig.defaults(), TrainConfig.defaults(batch_rays=65536, seed=2), max_rays=65536)
path = snake_path(scene.grid_rows, scene.grid_cols)
ts = []
for pos in path[:9]:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.set_window(*pos)
    torch.cuda.synchronize()
    ts.append(1e3 * (time.perf_counter() - t0))
print("first window ms %.2f, moves:" % ts[0], " ".join(f"{t:.2f}" for t in ts[1:]), "sum %.2f" % sum(ts))

# the same moves after the whole-scene memo fill (tfg_precompute_rays)
ctx2 = Context(scene, FieldConfig.defaults(), TrainConfig.defaults(batch_rays=65536, seed=2), max_rays=65536)
torch.cuda.synchronize()
t0 = time.perf_counter()
ctx2.precompute_rays()
torch.cuda.synchronize()
pre = 1e3 * (time.perf_counter() - t0)
ts = []
for pos in path[:9]:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx2.set_window(*pos)
    torch.cuda.synchronize()
    ts.append(1e3 * (time.perf_counter() - t0))
print("precompute ms %.2f; first window ms %.2f, moves:" % (pre, ts[0]), " ".join(f"{t:.2f}" for t in ts[1:]))
