"""Times the first window's accept pass and window moves on the bench scene
(config 5): wall clock around set_window with a device sync on both sides.
Each move Newton-solves the pixels the previous position did not cover and
copies the rest from its per-window memo."""
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

# prefetched moves (the next position staged on the side stream while the
# current one would train): the move itself
ctx2 = Context(scene, FieldConfig.defaults(), TrainConfig.defaults(batch_rays=65536, seed=2), max_rays=65536)
ctx2.set_window(*path[0])
ctx2.prefetch_window(*path[1])
ts = []
for k, pos in enumerate(path[1:9]):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx2.set_window(*pos)
    torch.cuda.synchronize()
    ts.append(1e3 * (time.perf_counter() - t0))
    ctx2.prefetch_window(*path[k + 2])
    torch.cuda.synchronize()
print("prefetched moves ms:", " ".join(f"{t:.2f}" for t in ts))
