#!/bin/bash
# A/B of an environment switch on the bench (device-timed value + phases).
# usage: tools/gpu_ab.sh VAR value_a value_b [reps]
VAR=$1; A=$2; B=$3; N=${4:-2}
for r in $(seq $N); do
  for v in $A $B; do
    env $VAR=$v python bench.py --steps 20 --warmup 5 --no-render --no-cpu 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']
        print('$VAR=$v', round(d['value']/1e6,3), 'M rays/s', ' '.join(f'{p}={k[p][\"ms_per_step\"]:.4f}' for p in k))
"
  done
done
