"""Times the render path (config 4 full view) device phases: sampler / field_fwd / composite."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import argparse  # noqa: E402

import bench  # noqa: E402

r = bench.bench_render(argparse.Namespace(no_cpu=True))
print(f"render {r['value'] / 1e6:.2f} M rays/s device, {r['e2e']['value'] / 1e6:.2f} M e2e;",
      {k: round(v, 2) for k, v in r["phases_ms"].items()})
