#!/bin/bash
# tools/ab_sweep.sh variant... : sampler / step time at several per-GPU batches per library variant
for v in "$@"; do
for b in 65536 16384 8192; do
  TFG_LIB=paper_2507_01631_b200/_variants/$v/libtilefield_gpu.so timeout 300 python bench.py --no-render --no-cpu --steps 40 --warmup 5 --global-batch $b 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']
        print('$v', $b, 'ms/step', round(d['ms_per_step'],4), ' '.join(f'{p}={k[p][\"ms_per_step\"]:.4f}' for p in k))
"
done; done
