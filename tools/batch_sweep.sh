#!/bin/bash
# Per-step time against the per-GPU batch (what one rank of an N-GPU strong-
# scaling run sees: 65,536 / N rays).
for b in 65536 32768 16384 8192; do
  timeout 300 python bench.py --no-render --no-cpu --steps 40 --warmup 5 --global-batch $b 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']
        print($b, 'rays: ms/step', round(d['ms_per_step'],4), 'M rays/s', round(d['value']/1e6,2), 'launches/step', d['gpu_launches']/d['steps'], ' '.join(f'{p}={k[p][\"ms_per_step\"]:.4f}' for p in k))
"
done
